// Dev micro-benchmark: FP64 FMA throughput of this B200 (the FP64 roofline
// denominator for k_elem and the ACCD narrow phase).  Every thread runs 8
// independent DFMA chains; a full wave of CTAs per SM; CUDA events, best of
// 10.  Prints one JSON line: {"fp64_tflops": ..., "dfma_per_s": ...}.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(int iters, double a, double b, double* sink) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b);
      x1 = fma(x1, a, b);
      x2 = fma(x2, a, b);
      x3 = fma(x3, a, b);
      x4 = fma(x4, a, b);
      x5 = fma(x5, a, b);
      x6 = fma(x6, a, b);
      x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1.2345) sink[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink;
  cudaMalloc(&sink, 8);
  const int threads = 256, iters = 4096;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dfma, threads, 0);
  const int grid = sms * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<grid, threads>>>(16, 0.999999, 1e-7, sink);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<grid, threads>>>(iters, 0.999999, 1e-7, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma = (double)grid * threads * iters * 16 * 8;
  printf("{\"fp64_tflops\": %.3f, \"dfma_per_s\": %.4e, \"grid\": %d, \"threads\": %d, \"sms\": %d, \"ms\": %.3f, "
         "\"how\": \"independent DFMA chains, 2 flop per DFMA, full wave, best of 10\"}\n",
         2.0 * fma / (best * 1e-3) / 1e12, fma / (best * 1e-3), grid, threads, sms, best);
  return 0;
}
