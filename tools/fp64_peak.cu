// FP64 throughput probe (not product code): scalar DFMA vs the FP64 MMA
// (mma.sync.m8n8k4.f64) on this GPU -- is a tensor-core formulation of the
// projector worth it?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm = 4; bpsm <= 8; bpsm *= 2) {
      dfma_kernel<<<sms * bpsm, 256>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<<<sms * bpsm, 256>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * double(sms * bpsm * 256);
      printf("{\"op\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"TFLOPs\": %.2f}\n", bpsm, ms, flops / ms / 1e9);
      dmma_kernel<<<sms * bpsm, 256>>>(out, iters);
      cudaEventRecord(e0);
      dmma_kernel<<<sms * bpsm, 256>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      // per warp per mma: 8x8x4 MACs = 256 FMA = 512 flops
      flops = 512.0 * 4 * iters * double(sms * bpsm * 256 / 32);
      printf("{\"op\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"TFLOPs\": %.2f}\n", bpsm, ms, flops / ms / 1e9);
    }
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
