// K1: the H -> H' rearrangement kernel for sm_100a.
//
// Persistent CTAs walk work units u = blockIdx.x + k * gridDim.x.  One
// elected thread stages unit k + stages - 1 with 1-D bulk TMA
// (cp.async.bulk global -> shared, completion on an mbarrier) while all
// warps consume unit k from a ring of `stages` shared-memory buffers:
// each output row is written with 16-byte st.global.v4 on its aligned body
// and scalar stores on the (<= 3 element) head/tail.  Values are moved as
// uint32/uint64 words, so the copy is bit-exact (-0.0, denormals, NaN
// payloads).  See hprime_plan.h for the index map.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hprime_plan.h"

namespace hp {

template <int E> struct Word;
template <> struct Word<4> { using T = uint32_t; };
template <> struct Word<8> { using T = unsigned long long; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "HP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra HP_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void st_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

__device__ __forceinline__ void st_v2_64(void* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

struct Unit {
  int64_t z, y;
  int32_t t0, jb;        // band start and rows
  int32_t i_lo, i_hi;    // output i range
  int32_t s_lo;          // first staged s
  int64_t run_elems;     // staged run length per x
  int64_t run_off0;      // element offset of the x = 0 run in the source array
};

__device__ __forceinline__ Unit decode_unit(const HpPlan& p, uint32_t u) {
  Unit w;
  uint32_t r = hp_div(p.ny_div, u);
  w.y = u - r * p.ny_div.d;
  uint32_t r2 = hp_div(p.nb_div, r);
  const int32_t band = static_cast<int32_t>(r - r2 * p.nb_div.d);
  uint32_t r3 = hp_div(p.nc_div, r2);
  const int32_t chunk = static_cast<int32_t>(r2 - r3 * p.nc_div.d);
  w.z = p.z_begin + r3;
  w.t0 = band * p.J;
  w.jb = min(p.J, static_cast<int32_t>(p.n_t) - w.t0);
  w.i_lo = chunk * p.C;
  w.i_hi = min(static_cast<int32_t>(p.n_s), w.i_lo + p.C);
  if (p.n_chunks == 1) {
    w.s_lo = 0;
    w.run_elems = static_cast<int64_t>(w.jb) * p.n_s;
  } else {  // J == 1: source s in [2c_s - i_hi + 1, 2c_s - i_lo] clipped to [0, n_s)
    const int32_t two_c = 2 * p.c_s;
    const int32_t s_lo = max(0, two_c - w.i_hi + 1);
    const int32_t s_hi = min(static_cast<int32_t>(p.n_s), two_c - w.i_lo + 1);
    w.s_lo = s_lo;
    w.run_elems = s_hi > s_lo ? (s_hi - s_lo) : 0;
  }
  w.run_off0 = w.s_lo + p.n_s * (w.t0 + p.n_t * (p.n_x * (w.y + p.n_y * w.z)));
  return w;
}

// Producer: stage the n_x source runs of unit `u` into `stage`; arrival on `bar`.
template <int E>
__device__ __forceinline__ void issue_unit(const HpPlan& p, const uint8_t* __restrict__ src, uint32_t u,
                                           uint8_t* stage, uint32_t bar) {
  using T = typename Word<E>::T;
  const Unit w = decode_unit(p, u);
  const int64_t run_bytes = w.run_elems * E;
  const int64_t xstride = p.n_s * p.n_t * E;
  const int64_t lim = p.total_bytes & ~int64_t(15);
  uint32_t tx = 0;
  int64_t b = w.run_off0 * E;
  if (run_bytes > 0) {
    for (int32_t x = 0; x < p.n_x; ++x, b += xstride) {
      const int64_t a_lo = b & ~int64_t(15);
      int64_t a_hi = (b + run_bytes + 15) & ~int64_t(15);
      if (a_hi > lim) a_hi = lim > a_lo ? lim : a_lo;
      uint8_t* dst = stage + static_cast<int64_t>(x) * p.row_pitch;
      if (a_hi > a_lo) {
        const uint32_t n = static_cast<uint32_t>(a_hi - a_lo);
        bulk_g2s(smem_u32(dst), src + a_lo, n, bar);
        tx += n;
      }
      // words past the last aligned 16 B of the allocation: plain loads
      for (int64_t q = (a_hi > b ? a_hi : b); q < b + run_bytes; q += E)
        *reinterpret_cast<T*>(dst + (q - a_lo)) = *reinterpret_cast<const T*>(src + q);
    }
  }
  mbar_arrive_expect_tx(bar, tx);  // tx-count may be transiently negative: legal
}

// Consumers: all warps write the J * n_x output rows of unit `u` from `stage`.
template <int E>
__device__ __forceinline__ void consume_unit(const HpPlan& p, uint8_t* __restrict__ dst, uint32_t u,
                                             const uint8_t* stage) {
  using T = typename Word<E>::T;
  constexpr int VE = 16 / E;
  const Unit w = decode_unit(p, u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int32_t n_x = static_cast<int32_t>(p.n_x);
  const int32_t o0 = static_cast<int32_t>((w.run_off0 * E) & 15);
  const int32_t rows = w.jb * n_x;
  for (int32_t r = warp; r < rows; r += nwarps) {
    const int32_t tl = static_cast<int32_t>(hp_div(p.nx_div, static_cast<uint32_t>(r)));
    const int32_t xp = r - tl * n_x;
    const int32_t t = w.t0 + tl;
    int64_t j, yp;
    const bool zero_row = t >= p.v_t;  // dropped source row t = n_t - 1 (even n_t)
    if (!zero_row) {
      j = 2 * p.c_t - t;
      yp = hp_mod(p.ny_div, static_cast<uint32_t>(w.y + t + p.ny_off));
    } else {  // carries the all-zero output row j = n_t - 1 at y' = y
      j = p.n_t - 1;
      yp = w.y;
    }
    const int64_t O = p.n_s * (j + p.n_t * (xp + p.n_x * (yp + p.n_y * w.z)));
    const int64_t e0 = O + w.i_lo, e1 = O + w.i_hi;
    const int64_t g0 = e0 & ~int64_t(VE - 1);
    const int32_t ng = static_cast<int32_t>((((e1 + VE - 1) & ~int64_t(VE - 1)) - g0) / VE);
    const int32_t sbase = tl * static_cast<int32_t>(p.n_s) - w.s_lo;
    for (int32_t g = lane; g < ng; g += 32) {
      const int64_t ge = g0 + static_cast<int64_t>(g) * VE;
      const int32_t i0 = static_cast<int32_t>(ge - O);
      uint32_t x = hp_mod(p.nx_div, static_cast<uint32_t>(xp + i0 + p.nx_off + 4 * n_x));
      T v[VE];
      bool ok[VE];
      bool full = true;
#pragma unroll
      for (int q = 0; q < VE; ++q) {
        const int32_t i = i0 + q;
        ok[q] = i >= w.i_lo && i < w.i_hi;
        full = full && ok[q];
        T val = 0;
        if (ok[q] && !zero_row && i < p.v_s) {
          const int32_t s = 2 * p.c_s - i;
          const int32_t ox = (o0 + static_cast<int32_t>(x) * p.xs16) & 15;
          const uint8_t* a = stage + static_cast<int32_t>(x) * p.row_pitch + ox + (sbase + s) * E;
          val = *reinterpret_cast<const T*>(a);
        }
        v[q] = val;
        x = (x + 1 == static_cast<uint32_t>(n_x)) ? 0u : x + 1;
      }
      uint8_t* out = dst + ge * E;
      if (full) {
        if constexpr (E == 4)
          st_v4(out, v[0], v[1], v[2], v[3]);
        else
          st_v2_64(out, v[0], v[1]);
      } else {
#pragma unroll
        for (int q = 0; q < VE; ++q)
          if (ok[q]) reinterpret_cast<T*>(out)[q] = v[q];
      }
    }
  }
}

template <int E>
__global__ void __launch_bounds__(512) hprime_kernel(const HpPlan p, const uint8_t* __restrict__ src,
                                                     uint8_t* __restrict__ dst) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* stages = smem + 128;
  const uint32_t first = blockIdx.x, step = gridDim.x;
  if (first >= p.n_units) return;
  const uint32_t n_units = static_cast<uint32_t>(p.n_units);
  const uint32_t mine = (n_units - first + step - 1) / step;
  const int S = p.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_barrier_init();
    const uint32_t pre = mine < static_cast<uint32_t>(S - 1) ? mine : static_cast<uint32_t>(S - 1);
    for (uint32_t k = 0; k < pre; ++k)
      issue_unit<E>(p, src, first + k * step, stages + static_cast<int64_t>(k) * p.stage_bytes,
                    smem_u32(&bars[k]));
  }
  __syncthreads();
  int st = 0;
  uint32_t phase = 0;
  for (uint32_t k = 0; k < mine; ++k) {
    if (threadIdx.x == 0 && k + S - 1 < mine) {
      int s2 = st + S - 1;
      if (s2 >= S) s2 -= S;
      fence_proxy_async_smem();  // order earlier generic reads of this buffer before the async writes
      issue_unit<E>(p, src, first + (k + S - 1) * step, stages + static_cast<int64_t>(s2) * p.stage_bytes,
                    smem_u32(&bars[s2]));
    }
    mbar_wait(smem_u32(&bars[st]), phase);
    consume_unit<E>(p, dst, first + k * step, stages + static_cast<int64_t>(st) * p.stage_bytes);
    __syncthreads();
    if (++st == S) {
      st = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace hp
