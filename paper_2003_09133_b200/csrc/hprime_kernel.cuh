// K1: the H -> H' rearrangement kernel for sm_100a.
//
// Persistent, warp-specialised CTAs.  Producer warp(s) take work units --
// from a per-launch ticket counter (HP_FLAG_DYNAMIC, the tuned plans) or
// round-robin u = blockIdx.x + k * gridDim.x -- and stage each unit's n_x
// source runs with 1-D bulk TMA (cp.async.bulk global -> shared, completion
// on a full mbarrier) into a ring of `stages` shared-memory buffers.  The
// consumer warps gather the mirrored, phase-shifted output rows out of
// shared memory (the row consumer, or the (row, phase-class) task consumer
// with HP_FLAG_TASKS) and write them with 16-byte st.global.v4 on each row's
// aligned body and scalar stores on the (<= 3 element) head/tail, then
// release the stage on an empty mbarrier.  Values are moved as uint32/uint64
// words, so the copy is bit-exact (-0.0, denormals, NaN payloads).  See
// hprime_plan.h for the index map and DESIGN.md section 3 for the design.
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

// HP_CHECKED builds (tools/build_variant.sh CHECKED -DHP_CHECKED): every
// shared-memory load and global store is bounds-checked, and the ring
// protocol is checked (a stage's unit must not change while its consumers
// use it).  compute-sanitizer is unavailable on the GPU pool; this build
// plus the fuzz sweep stands in for memcheck / racecheck.
#if defined(HP_CHECKED)
__shared__ const uint8_t* hp_chk_dst;
__shared__ unsigned long long hp_chk_bytes;
__device__ __forceinline__ uint32_t dyn_smem_size() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
#define HP_CHECK(cond, what)                                                                    \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("HP_CHECKED: %s failed (block %d thread %d)\n", what, blockIdx.x, threadIdx.x);    \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#define HP_CHECK_STORE(ptr, bytes)                                                              \
  HP_CHECK(reinterpret_cast<const uint8_t*>(ptr) >= hp_chk_dst &&                               \
               reinterpret_cast<const uint8_t*>(ptr) + (bytes) <= hp_chk_dst + hp_chk_bytes,    \
           "global store in bounds")
#else
#define HP_CHECK(cond, what) ((void)0)
#define HP_CHECK_STORE(ptr, bytes) ((void)0)
#endif

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

// Decoded unit, written by the producer at the head of its stage so the
// consumer warps read it with a few LDS instead of re-decoding.
struct UnitHdr {
  long long plane_off;  // z * plane_elems
  int32_t y, t0, jb, i_lo, i_hi, s_lo, o0;
  int32_t next_row;     // work counter: consumer warps claim rows with atomicAdd
  int32_t rot;          // HP_FLAG_ROTATE: rows are claimed starting at this one
  int32_t stop;         // HP_FLAG_DYNAMIC: no unit in this stage, the consumers exit
  uint32_t unit;        // the unit index (ring-protocol checks of HP_CHECKED builds)
};
constexpr int kHdrBytes = 64;

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
  int32_t band;
  uint32_t r2;
  if (p.flags & HP_FLAG_DIAGONAL) {
    // blocks of tile_y diagonals y' = (y + t0 - c_t) mod n_y; inside a block
    // the diagonal is fastest, then the band: a window of consecutive units
    // writes runs of adjacent rows of few y' and reads runs of tile_y
    // adjacent rows of each y
    r2 = hp_div(p.zc_div, u);
    const uint32_t r = u - r2 * p.zc_div.d;
    const uint32_t db = hp_div(p.yblk_div, r);
    const uint32_t rem = r - db * p.yblk_div.d;
    const HpFastDiv& tdiv = (static_cast<int32_t>(db) == p.n_yblocks - 1) ? p.tyl_div : p.ty_div;
    const uint32_t b = hp_div(tdiv, rem);
    band = static_cast<int32_t>(b);
    const uint32_t d = db * p.ty_div.d + (rem - b * tdiv.d);
    const uint32_t tm = hp_mod(p.ny_div, static_cast<uint32_t>(band * p.J));
    const uint32_t cm = hp_mod(p.ny_div, static_cast<uint32_t>(p.c_t));
    w.y = hp_mod(p.ny_div, d + cm + p.ny_div.d - tm);
  } else if (p.flags & HP_FLAG_BAND_FASTEST) {  // consecutive units read adjacent t-bands
    const uint32_t r = hp_div(p.nb_div, u);
    band = static_cast<int32_t>(u - r * p.nb_div.d);
    r2 = hp_div(p.ny_div, r);
    w.y = r - r2 * p.ny_div.d;
  } else if (p.n_yblocks == 1) {  // consecutive units: neighbouring y (their output rows interleave in L2)
    const uint32_t r = hp_div(p.ny_div, u);
    w.y = u - r * p.ny_div.d;
    r2 = hp_div(p.nb_div, r);
    band = static_cast<int32_t>(r - r2 * p.nb_div.d);
  } else {  // the same inside y blocks of tile_y (wide shapes)
    r2 = hp_div(p.zc_div, u);
    const uint32_t r = u - r2 * p.zc_div.d;
    const uint32_t yb = hp_div(p.yblk_div, r);
    const uint32_t rem = r - yb * p.yblk_div.d;
    const HpFastDiv& tdiv = (static_cast<int32_t>(yb) == p.n_yblocks - 1) ? p.tyl_div : p.ty_div;
    const uint32_t b = hp_div(tdiv, rem);
    band = static_cast<int32_t>(b);
    w.y = yb * p.ty_div.d + (rem - b * tdiv.d);
  }
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

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Producer warp `pw` of p.producers: stage its share of the n_x source runs
// of unit `u` into `stage`, one run per lane (x = 32 pw + lane, then
// + 32 producers, ...), completion on `bar` (one expect_tx arrive per
// producer warp).  The bulk copies take uniform operands, so ptxas issues a
// warp's runs one lane at a time; several producer warps issue in parallel.
// TASKS: run x's aligned superset starts at stage + 80 + x * row_pitch (row
// pitch a multiple of 16), so element k of run x sits at that address plus
// (run byte offset mod 16) + k * E; the task consumer resolves x per task.
template <int E, bool TASKS>
__device__ __forceinline__ void issue_unit(const HpPlan& p, const uint8_t* __restrict__ src, uint32_t u,
                                           uint8_t* stage, uint32_t bar, int lane, int pw, uint64_t policy) {
  using T = typename Word<E>::T;
  const Unit w = decode_unit(p, u);
  const int64_t run_bytes = w.run_elems * E;
  const int64_t xstride = p.n_s * p.n_t * E;
  const int64_t lim = p.total_bytes & ~int64_t(15);
  const int64_t b0 = w.run_off0 * E;
  uint32_t tx = 0;
  if (run_bytes > 0) {
    const int32_t rot = (p.flags & HP_FLAG_ROTATE) ? static_cast<int32_t>(hp_mod(p.nx_div, u)) : 0;
    for (int32_t xl = 32 * pw + lane; xl < p.n_x; xl += 32 * p.producers) {
      // lanes issue in order; with HP_FLAG_ROTATE unit u starts at run u mod n_x
      const int32_t x = xl + rot < p.n_x ? xl + rot : xl + rot - static_cast<int32_t>(p.n_x);
      const int64_t b = b0 + x * xstride;
      const int64_t a_lo = b & ~int64_t(15);
      int64_t a_hi = (b + run_bytes + 15) & ~int64_t(15);
      if (a_hi > lim) a_hi = lim > a_lo ? lim : a_lo;
      // element k of run x lives at R0 + x*row_pitch + k*E (see hprime_plan.h);
      // its 16-byte aligned superset starts (b & 15) bytes earlier
      uint8_t* dst = TASKS ? stage + kHdrBytes + 16 + static_cast<int64_t>(x) * p.row_pitch
                           : stage + kHdrBytes + 16 + (b0 & 15) + static_cast<int64_t>(x) * p.row_pitch - (b & 15);
#if defined(HP_DBG_NOLOAD)  // pattern probe build: no reads of H
      a_hi = a_lo;
#endif
      if (a_hi > a_lo) {
        const uint32_t n = static_cast<uint32_t>(a_hi - a_lo);
        if (p.flags & HP_FLAG_LOAD_EVICT_FIRST)
          bulk_g2s_hint(smem_u32(dst), src + a_lo, n, bar, policy);
        else
          bulk_g2s(smem_u32(dst), src + a_lo, n, bar);
        tx += n;
      }
      // words past the last aligned 16 B of the allocation: plain loads
      for (int64_t q = (a_hi > b ? a_hi : b); q < b + run_bytes; q += E)
        *reinterpret_cast<T*>(dst + (q - a_lo)) = *reinterpret_cast<const T*>(src + q);
    }
  }
  if (lane == 0 && pw == 0) {
    UnitHdr* h = reinterpret_cast<UnitHdr*>(stage);
    h->plane_off = w.z * (p.n_s * p.n_t * p.n_x * p.n_y);
    h->y = static_cast<int32_t>(w.y);
    h->t0 = w.t0;
    h->jb = w.jb;
    h->i_lo = w.i_lo;
    h->i_hi = w.i_hi;
    h->s_lo = w.s_lo;
    h->o0 = static_cast<int32_t>(b0 & 15);
    h->next_row = 0;
    h->rot = (p.flags & HP_FLAG_ROTATE) ? static_cast<int32_t>(u % static_cast<uint32_t>(w.jb * p.n_x)) : 0;
    h->stop = 0;
    h->unit = u;
  }
  tx = __reduce_add_sync(0xffffffffu, tx);
  __syncwarp();                                    // header and tail stores before the release
  if (lane == 0) mbar_arrive_expect_tx(bar, tx);  // tx-count may be transiently negative: legal
}

template <int E>
__device__ __forceinline__ typename Word<E>::T lds(uint32_t addr) {
#if defined(HP_CHECKED)
  {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t lo = smem_u32(smem) + 128;
    HP_CHECK(addr >= lo && addr + E <= smem_u32(smem) + dyn_smem_size(), "shared load in bounds");
  }
#endif
  if constexpr (E == 4) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  } else {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
  }
}

template <int E>
__device__ __forceinline__ void st_vec(typename Word<E>::T* dst, const typename Word<E>::T* v) {
  HP_CHECK_STORE(dst, 16);
  HP_CHECK((reinterpret_cast<uintptr_t>(dst) & 15) == 0, "16-byte store aligned");
  if constexpr (E == 4)
    st_v4(dst, v[0], v[1], v[2], v[3]);
  else
    st_v2_64(dst, v[0], v[1]);
}

// Values of the VE elements of group g whose first element has source phase
// x0 and smem address a0, for any n_x (general wrap); used for row edges and
// for n_x < VE.
template <int E>
__device__ __forceinline__ void load_group_general(typename Word<E>::T* v, uint32_t a0, uint32_t x0, int32_t n_x,
                                                   int32_t step, int32_t nr) {
  constexpr int VE = 16 / E;
  uint32_t a = a0, x = x0;
#pragma unroll
  for (int q = 0; q < VE; ++q) {
    v[q] = lds<E>(a);
    const bool last = x == static_cast<uint32_t>(n_x - 1);
    a += last ? step - nr : step;
    x = last ? 0u : x + 1;
  }
}

// The VE values of one 16-byte output group whose first element has source
// phase x0 and smem address a0.  WRAP1 (n_x >= VE): x wraps at most once
// inside the group, so each load picks one of two bases.
template <int E, bool WRAP1>
__device__ __forceinline__ void load_group(typename Word<E>::T* v, uint32_t a0, uint32_t x0, int32_t n_x,
                                           int32_t step, int32_t nr) {
  constexpr int VE = 16 / E;
#if defined(HP_DBG_NOLDS)  // pattern probe build: no shared-memory reads
#pragma unroll
  for (int q = 0; q < VE; ++q) v[q] = a0 + q;
  return;
#endif
  if constexpr (WRAP1) {
    const int32_t d = n_x - static_cast<int32_t>(x0);   // elements before the wrap
    const uint32_t aw = a0 - nr;
    v[0] = lds<E>(a0);
#pragma unroll
    for (int q = 1; q < VE; ++q) v[q] = lds<E>((q >= d ? aw : a0) + q * step);
  } else {
    load_group_general<E>(v, a0, x0, n_x, step, nr);
  }
}

// One sub-warp lane's groups g, g+W, ... of a row: a masked leading group
// (only when the row starts inside a 16-byte group), unmasked full groups,
// a masked trailing group.
template <int E, bool WRAP1>
__device__ __forceinline__ void row_groups(typename Word<E>::T* o, int32_t g, int32_t ng, bool last_full, int32_t i0,
                                           int32_t i_lo, int32_t i_end, uint32_t x0, uint32_t a0, int32_t n_x,
                                           int32_t step, int32_t nr, int32_t W, uint32_t inc_x, int32_t inc_a) {
  using T = typename Word<E>::T;
  constexpr int VE = 16 / E;
  const int32_t inc_a_w = inc_a - nr;
  auto advance = [&]() {
    o += W * VE;
    i0 += W * VE;
    x0 += inc_x;
    const bool wr = x0 >= static_cast<uint32_t>(n_x);
    x0 = wr ? x0 - n_x : x0;
    a0 += wr ? inc_a_w : inc_a;
  };
  auto masked = [&]() {
    T v[VE];
    load_group<E, WRAP1>(v, a0, x0, n_x, step, nr);
#pragma unroll
    for (int q = 0; q < VE; ++q)
      if (i0 + q >= i_lo && i0 + q < i_end) {
        HP_CHECK_STORE(o + q, E);
        o[q] = v[q];
      }
  };
  if (i0 < i_lo) {  // leading partial group (g == 0)
    masked();
    advance();
    g += W;
  }
  const int32_t g_hi = last_full ? ng : ng - 1;
  if (g < g_hi) {  // full groups, software-pipelined: load group k+1 before storing group k;
                   // unrolled by two with alternating register sets (no copies between them)
    T va[VE], vb[VE];
    load_group<E, WRAP1>(va, a0, x0, n_x, step, nr);
    for (;;) {
      g += W;
      if (g >= g_hi) {
        st_vec<E>(o, va);
        advance();
        break;
      }
      T* oa = o;
      advance();
      load_group<E, WRAP1>(vb, a0, x0, n_x, step, nr);
      st_vec<E>(oa, va);
      g += W;
      if (g >= g_hi) {
        st_vec<E>(o, vb);
        advance();
        break;
      }
      T* ob = o;
      advance();
      load_group<E, WRAP1>(va, a0, x0, n_x, step, nr);
      st_vec<E>(ob, vb);
    }
  }
  if (g < ng) masked();  // trailing partial group
}

// Consumer warps (cw of nc) write the J * n_x output rows of the unit staged
// at `stage` (smem address `stage_s`).  Each warp is split into 32/W
// sub-warps of W = 2..32 lanes (p.sub_width); a sub-warp owns one output row at a
// time, so the per-row index arithmetic is shared by 32/W rows and every
// store instruction still writes W*16 contiguous bytes per row.  A row is cut
// on the 16-byte grid of H' into groups of VE = 16/E elements; lane l of the
// sub-warp takes groups l, l+W, ...  Full groups are one st.global.v4; the
// (at most two) partial edge groups use predicated scalar stores.  Stepping
// i -> i+1 moves the smem address by rp - E, minus n_x*rp when the source
// phase x wraps (at most once per group when n_x >= VE): no divisions in the
// element loop.
template <int E>
__device__ __forceinline__ void consume_unit(const HpPlan& p, uint8_t* __restrict__ dst, const uint8_t* stage,
                                             uint32_t stage_s, int cw, int nc, int lane) {
  using T = typename Word<E>::T;
  constexpr int VE = 16 / E;
#if defined(HP_DBG_NOSTORE)  // pattern probe build: bulk reads only
  return;
#endif
  const UnitHdr h = *reinterpret_cast<const UnitHdr*>(stage);
  const int32_t n_x = static_cast<int32_t>(p.n_x);
  const int32_t n_s = static_cast<int32_t>(p.n_s);
  const int32_t W = p.sub_width;
  const int32_t lw = W == 2 ? 1 : W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : 5;  // log2(W): no division below
  const int32_t sl = lane & (W - 1);               // lane within the sub-warp
  const int32_t R = 32 >> lw;                      // rows in flight per warp
  const int32_t rp = p.row_pitch;
  const int32_t step = rp - E;                     // x -> x+1, s -> s-1
  const int32_t nr = n_x * rp;                     // ... minus this when x wraps to 0
  const uint32_t base = stage_s + kHdrBytes + 16 + static_cast<uint32_t>(h.o0);
  const int32_t i_lo = h.i_lo;
  const int32_t i_end = min(h.i_hi, p.v_s);        // loaded elements: [i_lo, i_end)
  const int32_t xs = n_s * static_cast<int32_t>(p.n_t);   // in-plane offsets are 32-bit
  const int32_t zmis = static_cast<int32_t>(h.plane_off & (VE - 1));
  const uint32_t inc_x = static_cast<uint32_t>(p.gx_inc);              // (W*VE) mod n_x
  const int32_t inc_a = p.gx_inc * rp - W * VE * E;                    // smem step of W groups
  T* dz = reinterpret_cast<T*>(dst) + h.plane_off;
  int* next_row = &reinterpret_cast<UnitHdr*>(const_cast<uint8_t*>(stage))->next_row;
  const int32_t rows = h.jb * n_x;
  // rows are claimed R at a time (dynamic balance across warps); the next
  // claim is issued before the current rows are written
  int32_t claim = 0;
  if (lane == 0) claim = atomicAdd(next_row, R);
  for (;;) {
    const int32_t r0 = __shfl_sync(0xffffffffu, claim, 0);
    if (r0 >= rows) break;
    if (lane == 0) claim = atomicAdd(next_row, R);
    const int32_t rc = r0 + (lane >> lw);
    do {  // this sub-warp's row (none past the end of the unit)
    if (rc >= rows) break;
    const int32_t r = rc + h.rot < rows ? rc + h.rot : rc + h.rot - rows;
    const int32_t tl = static_cast<int32_t>(hp_div(p.nx_div, static_cast<uint32_t>(r)));
    const int32_t xp = r - tl * n_x;
    const int32_t t = h.t0 + tl;
    const bool zero_row = t >= p.v_t;  // dropped source row t = n_t - 1 (even n_t)
    const int32_t j = zero_row ? static_cast<int32_t>(p.n_t) - 1 : 2 * p.c_t - t;
    const int32_t yp = zero_row ? h.y : static_cast<int32_t>(hp_mod(p.ny_div, static_cast<uint32_t>(h.y + t + p.ny_off)));
    const int32_t o_in = n_s * j + xs * (xp + n_x * yp);
    T* orow = dz + o_in;
    if (zero_row) {
      for (int32_t i = i_lo + sl; i < h.i_hi; i += W) {
        HP_CHECK_STORE(orow + i, E);
        orow[i] = T(0);
      }
    } else {
      if (i_end < h.i_hi && sl == 0) {  // even n_s: row i = n_s - 1 is zero
        HP_CHECK_STORE(orow + n_s - 1, E);
        orow[n_s - 1] = T(0);
      }
      const int32_t gs = i_lo - ((o_in + zmis + i_lo) & (VE - 1));   // first group start (element i)
      const int32_t ng = i_end > i_lo ? (i_end - gs + VE - 1) / VE : 0;
      int32_t g = sl;
      if (g < ng) {
        // smem address of (x, i) = base + x*rp + (tl*n_s - s_lo + 2c_s - i)*E
        const uint32_t x0 = hp_mod(p.nx_div, static_cast<uint32_t>(xp + gs + p.nx_off + VE * n_x + g * VE));
        const uint32_t a0 =
            base + static_cast<uint32_t>((tl * n_s - h.s_lo + 2 * p.c_s - gs - g * VE) * E) + x0 * rp;
        const int32_t i0 = gs + g * VE;
        const bool last_full = ((i_end - gs) & (VE - 1)) == 0;
        if (n_x >= VE)
          row_groups<E, true>(orow + i0, g, ng, last_full, i0, i_lo, i_end, x0, a0, n_x, step, nr, W, inc_x, inc_a);
        else
          row_groups<E, false>(orow + i0, g, ng, last_full, i0, i_lo, i_end, x0, a0, n_x, step, nr, W, inc_x, inc_a);
      }
    }
    } while (0);
  }
}

__device__ __forceinline__ int32_t atom_add_smem(int* p, int32_t v) {
  int32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// HP_FLAG_TASKS consumer.  A task is (output row r, phase class c < n_x):
// the 16-byte groups g = c, c + n_x, c + 2 n_x, ... of row r.  Stepping n_x
// groups moves VE * n_x elements along i, which brings the source phase
// x = (x' + i - c_s) mod n_x back to the same value for every element of the
// group, so the VE shared-memory addresses of a task's groups are VE fixed
// bases minus m * 16 n_x bytes: the steady loop is VE LDS, VE address adds
// and one 16-byte store per group, with no wrap selects.  All per-row and
// per-phase index arithmetic (the mirror, the phase and the row's 16-byte
// alignment) happens once per task.  Lanes take consecutive tasks (32 per
// claim), so the classes of one row go to neighbouring lanes and a warp's
// stores cover ~16 n_x contiguous bytes of a row.
template <int E>
__device__ __forceinline__ void consume_unit_tasks(const HpPlan& p, uint8_t* __restrict__ dst, const uint8_t* stage,
                                                   uint32_t stage_s, int lane) {
  using T = typename Word<E>::T;
  constexpr int VE = 16 / E;
  const UnitHdr h = *reinterpret_cast<const UnitHdr*>(stage);
  const int32_t n_x = static_cast<int32_t>(p.n_x);
  const int32_t n_s = static_cast<int32_t>(p.n_s);
  const int32_t n_t = static_cast<int32_t>(p.n_t);
  const int32_t xs = n_s * n_t;                       // in-plane offsets are 32-bit
  const int32_t ntask = h.jb * n_x * n_x;
  const int32_t i_lo = h.i_lo, i_hi = h.i_hi;
  const int32_t i_end = min(i_hi, p.v_s);              // loaded elements: [i_lo, i_end)
  const int32_t zmis = static_cast<int32_t>(h.plane_off & (VE - 1));
  const int32_t rp = p.row_pitch;
  const int32_t dstep = 16 * n_x;                      // smem bytes per n_x groups
  const int32_t ostep = VE * n_x;                      // H' elements per n_x groups
  const uint32_t sbase = stage_s + kHdrBytes + 16;
  const int32_t kbase = 2 * p.c_s - h.s_lo;            // k = tl * n_s + kbase - i
  T* dz = reinterpret_cast<T*>(dst) + h.plane_off;
  int* counter = &reinterpret_cast<UnitHdr*>(const_cast<uint8_t*>(stage))->next_row;
  int32_t claim = 0;
  if (lane == 0) claim = atom_add_smem(counter, 32);
  for (;;) {
    const int32_t tb = __shfl_sync(0xffffffffu, claim, 0);
    if (tb >= ntask) break;
    if (lane == 0) claim = atom_add_smem(counter, 32);
    const int32_t task = tb + lane;
    if (task >= ntask) continue;
    const int32_t r = static_cast<int32_t>(hp_div(p.nx_div, static_cast<uint32_t>(task)));
    const int32_t c = task - r * n_x;
    const int32_t tl = static_cast<int32_t>(hp_div(p.nx_div, static_cast<uint32_t>(r)));
    const int32_t xp = r - tl * n_x;
    const int32_t t = h.t0 + tl;
    const bool zero_row = t >= p.v_t;  // dropped source row t = n_t - 1 (even n_t)
    const int32_t j = zero_row ? n_t - 1 : 2 * p.c_t - t;
    const int32_t yp = zero_row ? h.y : static_cast<int32_t>(hp_mod(p.ny_div, static_cast<uint32_t>(h.y + t + p.ny_off)));
    const int32_t o_in = n_s * j + xs * (xp + n_x * yp);
    T* orow = dz + o_in;
    if (c == 0 && i_end < i_hi) {  // even n_s: row i = n_s - 1 is zero
      HP_CHECK_STORE(orow + n_s - 1, E);
      orow[n_s - 1] = T(0);
    }
    const int32_t gs = i_lo - ((o_in + zmis + i_lo) & (VE - 1));   // first group start (element i)
    const int32_t ng = i_end > i_lo ? (i_end - gs + VE - 1) / VE : 0;
    if (c >= ng) continue;
    const int32_t cnt = static_cast<int32_t>(hp_div(p.nx_div, static_cast<uint32_t>(ng - c - 1))) + 1;
    const int32_t i0 = gs + VE * c;                    // first element of the task's group m = 0
    T* o = orow + i0;
    const bool head = c == 0 && gs < i_lo;             // group 0 starts before i_lo
    const bool tail = c + (cnt - 1) * n_x == ng - 1 && ((i_end - gs) & (VE - 1)) != 0;
    if (zero_row) {
      for (int32_t m = 0; m < cnt; ++m)
#pragma unroll
        for (int q = 0; q < VE; ++q) {
          const int32_t i = i0 + m * ostep + q;
          if (i >= i_lo && i < i_end) {
            HP_CHECK_STORE(o + m * ostep + q, E);
            o[m * ostep + q] = T(0);
          }
        }
      continue;
    }
    // smem address of element q of group m: A[q] - m * dstep
    uint32_t A[VE];
    const uint32_t x0 = static_cast<uint32_t>(xp + i0 + p.nx_off + VE * n_x);  // >= 0
    const int32_t k0 = tl * n_s + kbase - i0;
#pragma unroll
    for (int q = 0; q < VE; ++q) {
      const uint32_t x = hp_mod(p.nx_div, x0 + q);
      A[q] = sbase + x * rp + ((h.o0 + x * p.xs16) & 15) + static_cast<uint32_t>((k0 - q) * E);
    }
    auto masked = [&](int32_t m) {
      const uint32_t off = static_cast<uint32_t>(m * dstep);
#pragma unroll
      for (int q = 0; q < VE; ++q) {
        const int32_t i = i0 + m * ostep + q;
        if (i >= i_lo && i < i_end) {
          HP_CHECK_STORE(o + m * ostep + q, E);
          o[m * ostep + q] = lds<E>(A[q] - off);
        }
      }
    };
    const int32_t m0 = head ? 1 : 0;
    const int32_t m1 = tail ? cnt - 1 : cnt;
    if (head) masked(0);
    if (m0 < m1) {  // full groups, software-pipelined, two alternating register sets
      T va[VE], vb[VE];
      uint32_t a = A[0] - static_cast<uint32_t>(m0 * dstep);
      const uint32_t d1 = A[1] - A[0], d2 = A[VE > 2 ? 2 : 1] - A[0], d3 = A[VE - 1] - A[0];
      auto load = [&](T* v) {
        v[0] = lds<E>(a);
        if constexpr (VE == 2) {
          v[1] = lds<E>(a + d1);
        } else {
          v[1] = lds<E>(a + d1);
          v[2] = lds<E>(a + d2);
          v[3] = lds<E>(a + d3);
        }
      };
      T* oo = o + m0 * ostep;
      int32_t m = m0;
      load(va);
      for (;;) {
        if (++m >= m1) {
          st_vec<E>(oo, va);
          break;
        }
        a -= dstep;
        T* oa = oo;
        oo += ostep;
        load(vb);
        st_vec<E>(oa, va);
        if (++m >= m1) {
          st_vec<E>(oo, vb);
          break;
        }
        a -= dstep;
        T* ob = oo;
        oo += ostep;
        load(va);
        st_vec<E>(ob, vb);
      }
    }
    if (tail && !(head && cnt == 1)) masked(cnt - 1);
  }
}

// Warps 0..producers-1 produce, the rest consume; full/empty mbarrier ring
// of `stages` buffers, so consumer warps never wait for each other.
template <int E, bool TASKS>
__global__ void __launch_bounds__(544, 1) hprime_kernel(const HpPlan p, const uint8_t* __restrict__ src,
                                                     uint8_t* __restrict__ dst) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  uint8_t* stages = smem + 128;
  const uint32_t first = blockIdx.x, stride = gridDim.x;
  // (the planner keeps grid <= n_units; with HP_FLAG_DYNAMIC every CTA must
  // take part in the ticket slot's reset count)
  if (first >= p.n_units && !(p.flags & HP_FLAG_DYNAMIC)) return;
  const uint32_t n_units = static_cast<uint32_t>(p.n_units);
  const uint32_t mine = (n_units - first + stride - 1) / stride;
  const int S = p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = p.producers;
  const int nc = (blockDim.x >> 5) - np;
#if defined(HP_CHECKED)
  if (threadIdx.x == 0) {
    hp_chk_dst = dst;
    hp_chk_bytes = static_cast<unsigned long long>(p.total_bytes);
  }
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), np);
      mbar_init(smem_u32(&empty[s]), nc);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const bool dynamic = (p.flags & HP_FLAG_DYNAMIC) != 0;  // planner: only with one producer warp
  if (warp < np) {
    const uint64_t policy = policy_evict_first();
    int st = 0;
    uint32_t ph = 0;
    if (dynamic) {
      // units are handed out in global order by one counter per launch, so
      // the units in flight always form one window of ~grid * stages units
      // and no CTA drifts ahead of the others; producer warp 0 fetches the
      // next ticket while the current unit is issued and, with several
      // producer warps, passes it on through the stage header (named
      // barrier 1 over the producer warps)
      unsigned long long* ctr = p.counter;
      uint32_t u = 0, nxt = 0;
      if (warp == 0 && lane == 0) u = static_cast<uint32_t>(atomicAdd(ctr, 1ull));
      for (uint32_t k = 0;; ++k) {
        if (k >= static_cast<uint32_t>(S)) {
          mbar_wait(smem_u32(&empty[st]), ph ^ 1u);
          fence_proxy_async_smem();
        }
        uint8_t* stage = stages + static_cast<int64_t>(st) * p.stage_bytes;
        if (np == 1) {
          u = __shfl_sync(0xffffffffu, u, 0);
        } else {
          if (warp == 0 && lane == 0) reinterpret_cast<volatile UnitHdr*>(stage)->unit = u;
          asm volatile("bar.sync 1, %0;" ::"r"(32 * np) : "memory");
          u = reinterpret_cast<volatile UnitHdr*>(stage)->unit;
          asm volatile("bar.sync 1, %0;" ::"r"(32 * np) : "memory");
        }
        if (u >= n_units) {
          if (warp == 0 && lane == 0) {
            reinterpret_cast<UnitHdr*>(stage)->stop = 1;
            // this CTA takes no more tickets; the last CTA to get here zeroes
            // the slot for its next launch (no memset on the stream)
            if (atomicAdd(ctr + 1, 1ull) == static_cast<unsigned long long>(gridDim.x) - 1) {
              atomicExch(ctr, 0ull);
              atomicExch(ctr + 1, 0ull);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(smem_u32(&full[st]), 0);
          break;
        }
        if (warp == 0 && lane == 0) nxt = static_cast<uint32_t>(atomicAdd(ctr, 1ull));
        issue_unit<E, TASKS>(p, src, u, stage, smem_u32(&full[st]), lane, warp, policy);
        u = nxt;
        if (++st == S) {
          st = 0;
          ph ^= 1u;
        }
      }
      return;
    }
    for (uint32_t k = 0; k < mine; ++k) {
      if (k >= static_cast<uint32_t>(S)) {
        mbar_wait(smem_u32(&empty[st]), ph ^ 1u);
        fence_proxy_async_smem();
      }
      issue_unit<E, TASKS>(p, src, first + k * stride, stages + static_cast<int64_t>(st) * p.stage_bytes,
                           smem_u32(&full[st]), lane, warp, policy);
      if (++st == S) {
        st = 0;
        ph ^= 1u;
      }
    }
    return;
  }
  const uint32_t stage0 = smem_u32(stages);
  int st = 0;
  uint32_t ph = 0;
  for (uint32_t k = 0; dynamic || k < mine; ++k) {
    mbar_wait(smem_u32(&full[st]), ph);
    const uint8_t* stage = stages + static_cast<int64_t>(st) * p.stage_bytes;
    if (dynamic && reinterpret_cast<const volatile UnitHdr*>(stage)->stop) break;
#if defined(HP_CHECKED)
    const uint32_t unit_in = reinterpret_cast<const volatile UnitHdr*>(stage)->unit;
    HP_CHECK(dynamic || unit_in == first + k * stride, "stage holds this warp's next unit");
    HP_CHECK(unit_in < n_units, "unit index in range");
#endif
    if constexpr (TASKS)
      consume_unit_tasks<E>(p, dst, stage, stage0 + static_cast<uint32_t>(st) * p.stage_bytes, lane);
    else
      consume_unit<E>(p, dst, stage, stage0 + static_cast<uint32_t>(st) * p.stage_bytes, warp - np, nc, lane);
    __syncwarp();
    HP_CHECK(reinterpret_cast<const volatile UnitHdr*>(stage)->unit == unit_in, "stage not refilled while in use");
    if (lane == 0) mbar_arrive(smem_u32(&empty[st]));
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  }
}

}  // namespace hp
