// K3: per-(s, t) sorted-order plane sums on the device -- the verification
// reductions of the reference (`_plane_sum`, lfbp/arrays.py:211-221, behind
// `sum_forward_plane` / `sum_backward_plane`, arrays.py:224-239).
//
// The reference sorts the n_x * n_y values of every (s, t) pattern slice of a
// depth plane and sums them in float64 with numpy's pairwise summation, so
// the result depends only on the value multiset: the sums of H and of H' then
// agree bitwise after a 180-degree rotation (acceptance criterion 3).  This
// kernel reproduces that bit for bit: one warp per slice gathers the K values
// into shared memory as order-preserving uint64 keys, bitonic-sorts them, and
// lane 0 adds them in numpy's pairwise order (blocks of <= 128 with eight
// interleaved accumulators, halving splits rounded to multiples of 8).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hp {

// total order on doubles matching numpy's sort: -inf .. -0, +0 .. +inf, NaN
__device__ __forceinline__ unsigned long long sort_key(double v) {
  if (v != v) return ~0ull - 1ull;  // every NaN sorts last (before the padding)
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double key_value(unsigned long long k) {
  if (k == ~0ull - 1ull) return __longlong_as_double(0x7ff8000000000000ll);
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

// numpy's pairwise_sum (umath loops_utils) for n <= 128: eight accumulators
__device__ __forceinline__ double pairwise_leaf(const unsigned long long* a, int n) {
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; ++i) res += key_value(a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = key_value(a[j]);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += key_value(a[i + j]);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += key_value(a[i]);
  return res;
}

// full recursion with an explicit stack (depth <= log2(K / 128) + 1)
__device__ double pairwise_sum(const unsigned long long* a, int n) {
  struct Frame {
    int off, n, stage;
    double left;
  };
  Frame st[24];
  int sp = 0;
  st[0] = {0, n, 0, 0.};
  double ret = 0.;
  for (;;) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(a + f.off, f.n);
      if (sp == 0) return ret;
      --sp;
      continue;  // deliver ret to the parent
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {  // descend left
      f.stage = 1;
      st[++sp] = {f.off, n2, 0, 0.};
    } else if (f.stage == 1) {  // left done, descend right
      f.left = ret;
      f.stage = 2;
      st[++sp] = {f.off + n2, f.n - n2, 0, 0.};
    } else {  // both done
      ret = f.left + ret;
      if (sp == 0) return ret;
      --sp;
    }
  }
}

// out[(z - z_begin) * n_s * n_t + t * n_s + s] = sum of the sorted slice
template <typename T>
__global__ void __launch_bounds__(256) plane_sums_kernel(const T* __restrict__ src, double* __restrict__ out,
                                                         int32_t n_s, int32_t n_t, int32_t K, int32_t P,
                                                         int64_t z_begin, int64_t n_slices) {
  extern __shared__ unsigned long long keys[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  unsigned long long* buf = keys + static_cast<int64_t>(warp) * P;
  const int64_t st_stride = static_cast<int64_t>(n_s) * n_t;
  for (int64_t sl = static_cast<int64_t>(blockIdx.x) * wpc + warp; sl < n_slices;
       sl += static_cast<int64_t>(gridDim.x) * wpc) {
    const int64_t zr = sl / st_stride;
    const int64_t st = sl - zr * st_stride;  // s + n_s * t
    const T* base = src + (z_begin + zr) * st_stride * K + st;
    for (int k = lane; k < P; k += 32)
      buf[k] = k < K ? sort_key(static_cast<double>(base[static_cast<int64_t>(k) * st_stride])) : ~0ull;
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1) {
      for (int half = size >> 1; half > 0; half >>= 1) {
        for (int i = lane; i < (P >> 1); i += 32) {
          const int lo = 2 * i - (i & (half - 1));
          const int hi = lo + half;
          const bool up = (lo & size) == 0;
          const unsigned long long a = buf[lo], b = buf[hi];
          if ((a > b) == up) {
            buf[lo] = b;
            buf[hi] = a;
          }
        }
        __syncwarp();
      }
    }
    // numpy reduces into the identity 0.0 first: 0.0 + (-0.0) = +0.0
    if (lane == 0) out[sl] = 0.0 + pairwise_sum(buf, K);
    __syncwarp();
  }
}

}  // namespace hp
