// Memory-pattern probe (not product code): copies the H -> H' piece pattern
// of a K1 unit WITHOUT the in-row shear, to separate the DRAM / TLB cost of
// the access pattern from the cost of the kernel's shared-memory gather.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pattern_probe tools/pattern_probe.cu
//   tools/pattern_probe n_t n_x n_y piece_bytes planes [layout] [order]
//
// A "piece" is one staged run / one output row (piece_bytes, a multiple of
// 16).  Unit (t, y, z) reads pieces (t, x, y, z) for x < n_x and writes
// pieces (n_t-1-t, x, (y+t) mod n_y, z).  layout 0 = the H layout (piece
// (t, x, y) at ((t + n_t*(x + n_x*y)) * P): the n_x pieces of a unit are
// n_t*P apart); layout 1 = x fastest (a unit's pieces are contiguous).
// order 0 = y fastest (K1's order), 1 = t fastest.  One warp copies one
// piece with 16-byte loads/stores.  Prints GB/s (read + write).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

struct Geo {
  int64_t n_t, n_x, n_y, P, planes;
  int layout, order;
};

__device__ __forceinline__ int64_t piece_off(const Geo& g, int64_t t, int64_t x, int64_t y, int64_t z) {
  int64_t idx = g.layout == 0 ? t + g.n_t * (x + g.n_x * y) : x + g.n_x * (t + g.n_t * y);
  return (idx + z * g.n_t * g.n_x * g.n_y) * g.P;
}

__global__ void __launch_bounds__(256) probe(Geo g, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t w0 = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t n_units = g.n_t * g.n_y * g.planes;
  const int64_t n_pieces = n_units * g.n_x;
  for (int64_t q = w0; q < n_pieces; q += warps) {
    const int64_t u = q / g.n_x, x = q - u * g.n_x;
    int64_t t, y, z = u / (g.n_t * g.n_y);
    const int64_t r = u - z * g.n_t * g.n_y;
    if (g.order == 0) {
      y = r % g.n_y;
      t = r / g.n_y;
    } else {
      t = r % g.n_t;
      y = r / g.n_t;
    }
    const uint4* s = reinterpret_cast<const uint4*>(src + piece_off(g, t, x, y, z));
    uint4* d = reinterpret_cast<uint4*>(dst + piece_off(g, g.n_t - 1 - t, x, (y + t) % g.n_y, z));
    const int n16 = int(g.P / 16);
    int k = lane;
    for (; k + 96 < n16; k += 128) {
      uint4 a = s[k], b = s[k + 32], c = s[k + 64], e = s[k + 96];
      d[k] = a;
      d[k + 32] = b;
      d[k + 64] = c;
      d[k + 96] = e;
    }
    for (; k < n16; k += 32) d[k] = s[k];
  }
}

int main(int argc, char** argv) {
  if (argc < 6) {
    fprintf(stderr, "usage: %s n_t n_x n_y piece_bytes planes [layout] [order] [reps]\n", argv[0]);
    return 2;
  }
  Geo g;
  g.n_t = atoll(argv[1]);
  g.n_x = atoll(argv[2]);
  g.n_y = atoll(argv[3]);
  g.P = atoll(argv[4]);
  g.planes = atoll(argv[5]);
  g.layout = argc > 6 ? atoi(argv[6]) : 0;
  g.order = argc > 7 ? atoi(argv[7]) : 0;
  const int reps = argc > 8 ? atoi(argv[8]) : 20;
  const size_t bytes = size_t(g.n_t * g.n_x * g.n_y * g.planes * g.P);
  uint8_t *a, *b;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
    fprintf(stderr, "alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bpsm = 4; bpsm <= 8; bpsm *= 2) {
    probe<<<sms * bpsm, 256>>>(g, a, b);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) probe<<<sms * bpsm, 256>>>(g, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("{\"n_t\": %lld, \"n_x\": %lld, \"n_y\": %lld, \"P\": %lld, \"planes\": %lld, \"layout\": %d, \"order\": %d, "
           "\"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
           (long long)g.n_t, (long long)g.n_x, (long long)g.n_y, (long long)g.P, (long long)g.planes, g.layout,
           g.order, bpsm, ms, 2.0 * bytes / ms / 1e6);
  }
  // plain contiguous copy of the same bytes
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("{\"memcpy_d2d_GBps\": %.1f}\n", 2.0 * bytes / ms / 1e6);
  fprintf(stderr, "%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
