// K6: seeded synthetic H planes on the device (bench / test input
// generation, not the hot path).
//
// Produces, bit for bit, paper_2003_09133_b200.synth.baseline_plane: plane z
// draws one numpy Generator.random() stream from PCG64 seeded with
// SeedSequence([seed, z]) (the host passes the generator's initial 128-bit
// state and increment), element e of the plane (F order, s fastest) taking
// draw e; the value is (u * a[s, x]) * b[t, y] (product law) or
// (a[s, x] + b[t, y] <= r2 ? u : 0) (disc law: a, b the squared offsets) in
// float64, then rounded to the element type.  Every operation is a
// correctly rounded IEEE multiply / add / compare, so the device reproduces
// numpy's bits (pinned by the golden input digests).
//
// numpy's PCG64 (pcg64.h): state <- state * M + inc (mod 2^128), output
// XSL-RR: rotr64(hi ^ lo, state >> 122); random() = (out >> 11) * 2^-53.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hp {

typedef unsigned __int128 u128;

struct SynthPlane {
  uint64_t state_lo, state_hi, inc_lo, inc_hi;
};

__device__ __forceinline__ u128 pcg_mult() {
  return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
}

// (A, C) of k LCG steps: s_k = A * s_0 + C
__device__ __forceinline__ void lcg_jump(uint64_t k, u128 inc, u128& A, u128& C) {
  u128 a = pcg_mult(), c = inc;
  A = 1;
  C = 0;
  while (k) {
    if (k & 1) {
      A = a * A;
      C = a * C + c;
    }
    c = a * c + c;
    a = a * a;
    k >>= 1;
  }
}

__device__ __forceinline__ double pcg_double(u128 s) {
  const uint64_t hi = uint64_t(s >> 64), lo = uint64_t(s);
  const uint64_t x = hi ^ lo;
  const unsigned rot = unsigned(s >> 122);
  const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
  return __dmul_rn(double(out >> 11), 1.0 / 9007199254740992.0);
}

// grid (blocks over the plane, planes); each warp fills 32 * kSynthPer
// consecutive elements of one plane, lane l taking elements l, l + 32, ...
constexpr int kSynthPer = 64;

template <typename T>
__global__ void __launch_bounds__(256) synth_kernel(T* __restrict__ dst, int64_t n_s, int64_t n_t, int64_t n_x,
                                                   int64_t n_y, const SynthPlane* __restrict__ planes,
                                                   const double* __restrict__ tab_s,
                                                   const double* __restrict__ tab_t,
                                                   const double* __restrict__ disc_r2) {
  const int64_t P = n_s * n_t * n_x * n_y;
  const int z = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t e0 = warp * 32 * kSynthPer + lane;
  if (e0 >= P) return;
  const SynthPlane pl = planes[z];
  const u128 inc = (u128(pl.inc_hi) << 64) | pl.inc_lo;
  u128 s = (u128(pl.state_hi) << 64) | pl.state_lo;
  u128 A, C;
  lcg_jump(uint64_t(e0) + 1, inc, A, C);  // draw e is taken after e + 1 steps
  s = A * s + C;
  u128 A32, C32;
  lcg_jump(32, inc, A32, C32);
  const double* ts = tab_s + int64_t(z) * n_s * n_x;
  const double* tt = tab_t + int64_t(z) * n_t * n_y;
  const double r2 = disc_r2 ? disc_r2[z] : 0.0;
  T* out = dst + int64_t(z) * P;
  for (int k = 0; k < kSynthPer; ++k) {
    const int64_t e = e0 + int64_t(k) * 32;
    if (e >= P) break;
    const double u = pcg_double(s);
    int64_t r = e;
    const int64_t si = r % n_s;
    r /= n_s;
    const int64_t ti = r % n_t;
    r /= n_t;
    const int64_t xi = r % n_x;
    const int64_t yi = r / n_x;
    const double a = ts[si + n_s * xi], b = tt[ti + n_t * yi];
    double v;
    if (disc_r2)
      v = (__dadd_rn(a, b) <= r2) ? u : 0.0;
    else
      v = __dmul_rn(__dmul_rn(u, a), b);
    if constexpr (sizeof(T) == 4)
      out[e] = __double2float_rn(v);
    else
      out[e] = v;
    s = A32 * s + C32;
  }
}

}  // namespace hp
