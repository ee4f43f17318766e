// Dev micro-benchmark: cost of a grid-wide barrier on B200 for the PCG's
// launch shape (592 CTAs x 224 threads): cooperative_groups grid.sync vs a
// hand-rolled sense-reversing barrier (one atomic per CTA, acquire spin).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x * 1e-9;
    g.sync();
  }
  if (acc < -1) sink[0] = acc;
}

__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks, unsigned& local_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = local_gen + 1;
    __threadfence();
    const unsigned arrived = atomicAdd(count, 1);
    if (arrived == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicExch((unsigned*)gen, target);
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen));
      } while (g != target);
    }
    local_gen = target;
  }
  __syncthreads();
}

__global__ void k_mine(int iters, unsigned* count, unsigned* gen, double* sink) {
  unsigned local_gen = 0;
  if (threadIdx.x == 0) local_gen = *((volatile unsigned*)gen);
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x * 1e-9;
    my_barrier(count, gen, gridDim.x, local_gen);
  }
  if (acc < -1) sink[0] = acc;
}

// barrier + fixed-order grid reduction as k_pcg does it: block tree sum,
// partial to global, grid.sync, warp 0 sums the G partials, broadcast
__device__ double block_total(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double r = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  __syncthreads();
  return r;
}
__global__ void k_reduce(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double sh[33];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    const double v = block_total(threadIdx.x * 1e-9 + i, sh);
    if (threadIdx.x == 0) part[(i & 1) * gridDim.x + blockIdx.x] = v;
    g.sync();
    if (threadIdx.x < 32) {
      double t = 0;
      for (int k = threadIdx.x; k < (int)gridDim.x; k += 32) t += part[(i & 1) * gridDim.x + k];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) sh[32] = t;
    }
    __syncthreads();
    acc += sh[32];
    __syncthreads();
  }
  if (acc < -1) sink[0] = acc;
}

// variant: every thread loads its strided partials (<= 3 at 592 CTAs x 224),
// then one block tree: a single L2 round trip instead of ~19 per lane
__global__ void k_reduce_block(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double sh[33];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    const double v = block_total(threadIdx.x * 1e-9 + i, sh);
    if (threadIdx.x == 0) part[(i & 1) * gridDim.x + blockIdx.x] = v;
    g.sync();
    double t = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) t += part[(i & 1) * gridDim.x + k];
    acc += block_total(t, sh);
  }
  if (acc < -1) sink[0] = acc;
}

int main() {
  int iters = 2000;
  double* sink;
  unsigned *count, *gen;
  cudaMalloc(&sink, 8);
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(count, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148, 296, 444, 592}) {
    for (int threads : {224, 448, 896, 1024}) {
      if (grid > 148 * 2048 / threads) continue;
      void* args[] = {&iters, &sink};
      cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      void* args2[] = {&iters, &count, &gen, &sink};
      cudaLaunchCooperativeKernel((void*)k_mine, grid, threads, args2, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_mine, grid, threads, args2, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms2;
      cudaEventElapsedTime(&ms2, a, b);
      double* part;
      cudaMalloc(&part, 2 * grid * sizeof(double));
      void* args3[] = {&iters, &part, &sink};
      cudaLaunchCooperativeKernel((void*)k_reduce, grid, threads, args3, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_reduce, grid, threads, args3, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms3;
      cudaEventElapsedTime(&ms3, a, b);
      cudaMalloc(&part, 2 * grid * sizeof(double));
      cudaLaunchCooperativeKernel((void*)k_reduce_block, grid, threads, args3, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_reduce_block, grid, threads, args3, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms4;
      cudaEventElapsedTime(&ms4, a, b);
      printf("   block-wide reduce %.2f us\n", 1e3 * ms4 / iters);
      cudaFree(part);
      printf("grid %d threads %d: cg.sync %.2f us, own barrier %.2f us, sync+reduce %.2f us  (%s)\n", grid, threads,
             1e3 * ms / iters, 1e3 * ms2 / iters, 1e3 * ms3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
