// TMA piece-pattern probe (not product code): the H -> H' piece pattern of a
// K1 unit moved with bulk TMA only (global -> smem -> global, no shear, no
// consumer warps), to separate the DRAM cost of the access pattern from K1's
// shared-memory gather and store path.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma_pattern_probe tools/tma_pattern_probe.cu
//   tools/tma_pattern_probe n_t n_x n_y piece_bytes planes layout order stages [reps]
//
// Unit (t, y, z) reads pieces (t, x, y, z), x < n_x, and writes them to
// pieces (n_t-1-t, x, (y+t) mod n_y, z) (K1's map at piece granularity).
// layout 0 = H layout (piece (t, x, y) at (t + n_t (x + n_x y)) * P);
// layout 1 = a unit's pieces contiguous; layout 2 = plain copy (unit u's
// pieces at u * n_x * P on both sides).  order 0 = y fastest, 1 = t fastest.
// One thread per CTA issues everything; `stages` units in flight per CTA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

struct Geo {
  int64_t n_t, n_x, n_y, P, planes;
  int layout, order, stages;
};

__device__ __forceinline__ int64_t piece_off(const Geo& g, int64_t t, int64_t x, int64_t y, int64_t z) {
  int64_t idx = g.layout == 0 ? t + g.n_t * (x + g.n_x * y) : x + g.n_x * (t + g.n_t * y);
  return (idx + z * g.n_t * g.n_x * g.n_y) * g.P;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32, 1) probe(Geo g, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint8_t* buf = smem + 128;
  const int64_t unit_bytes = g.n_x * g.P;
  const int64_t n_units = g.n_t * g.n_y * g.planes;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < g.stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase = 0;
  int64_t k = 0;
  auto src_dst = [&](int64_t u, int64_t x, int64_t& so, int64_t& dO) {
    if (g.layout == 2) {
      so = dO = (u * g.n_x + x) * g.P;
      return;
    }
    const int64_t z = u / (g.n_t * g.n_y), r = u - z * g.n_t * g.n_y;
    int64_t t, y;
    if (g.order == 0) { y = r % g.n_y; t = r / g.n_y; } else { t = r % g.n_t; y = r / g.n_t; }
    so = piece_off(g, t, x, y, z);
    dO = piece_off(g, g.n_t - 1 - t, x, (y + t) % g.n_y, z);
  };
  // prologue: fill all stages
  int64_t u_next = blockIdx.x;
  const int S = g.stages;
  for (int s = 0; s < S && u_next < n_units; ++s, u_next += gridDim.x) {
    uint8_t* b = buf + s * unit_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"((uint32_t)unit_bytes) : "memory");
    for (int64_t x = 0; x < g.n_x; ++x) {
      int64_t so, dO;
      src_dst(u_next, x, so, dO);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                       "r"(su32(b + x * g.P)), "l"(src + so), "r"((uint32_t)g.P), "r"(su32(&bar[s])) : "memory");
    }
  }
  int s = 0;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++k) {
    uint8_t* b = buf + s * unit_bytes;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar[s])), "r"(phase) : "memory");
    for (int64_t x = 0; x < g.n_x; ++x) {
      int64_t so, dO;
      src_dst(u, x, so, dO);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + dO), "r"(su32(b + x * g.P)), "r"((uint32_t)g.P) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the oldest store group has read its smem once at most S-1 groups are pending... refill this stage
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (u_next < n_units) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"((uint32_t)unit_bytes) : "memory");
      for (int64_t x = 0; x < g.n_x; ++x) {
        int64_t so, dO;
        src_dst(u_next, x, so, dO);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                         "r"(su32(b + x * g.P)), "l"(src + so), "r"((uint32_t)g.P), "r"(su32(&bar[s])) : "memory");
      }
      u_next += gridDim.x;
    }
    if (++s == S) { s = 0; phase ^= 1; }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  if (argc < 9) {
    fprintf(stderr, "usage: %s n_t n_x n_y piece_bytes planes layout order stages [reps] [ctas_per_sm]\n", argv[0]);
    return 2;
  }
  Geo g;
  g.n_t = atoll(argv[1]); g.n_x = atoll(argv[2]); g.n_y = atoll(argv[3]); g.P = atoll(argv[4]);
  g.planes = atoll(argv[5]); g.layout = atoi(argv[6]); g.order = atoi(argv[7]); g.stages = atoi(argv[8]);
  const int reps = argc > 9 ? atoi(argv[9]) : 20;
  const int cps = argc > 10 ? atoi(argv[10]) : 1;
  const size_t bytes = size_t(g.n_t * g.n_x * g.n_y * g.planes * g.P);
  uint8_t *a, *b;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) { fprintf(stderr, "alloc failed\n"); return 1; }
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 128 + g.stages * int(g.n_x * g.P);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<<<sms * cps, 32, smem>>>(g, a, b);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) probe<<<sms * cps, 32, smem>>>(g, a, b);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  cudaError_t err = cudaGetLastError();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float mc = 0; cudaEventElapsedTime(&mc, e0, e1); mc /= reps;
  printf("{\"probe\": \"tma\", \"n_t\": %lld, \"n_x\": %lld, \"n_y\": %lld, \"P\": %lld, \"planes\": %lld, \"layout\": %d, "
         "\"order\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"memcpy_GBps\": %.1f, \"err\": \"%s\"}\n",
         (long long)g.n_t, (long long)g.n_x, (long long)g.n_y, (long long)g.P, (long long)g.planes, g.layout, g.order,
         g.stages, cps, ms, 2.0 * bytes / ms / 1e6, 2.0 * bytes / mc / 1e6, cudaGetErrorString(err));
  return 0;
}
