// Microbenchmark: cost of cooperative-groups grid.sync() and of __syncthreads() on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void gsync(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void bsync(int iters, int* out) {
  int x = threadIdx.x;
  for (int i = 0; i < iters; ++i) { __syncthreads(); x += i; }
  if (x == -1) out[0] = x;
}
// hand-rolled barrier: one atomic per CTA + spin on a generation counter
__global__ void mysync(int iters, unsigned* bar, int* out) {
  unsigned gen = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++gen;
      __threadfence();
      const unsigned arrived = atomicAdd(&bar[0], 1u) + 1;
      if (arrived == gen * gridDim.x) atomicExch(&bar[1], gen);
      while (atomicAdd(&bar[1], 0u) < gen) __nanosleep(20);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

int main() {
  int* d; unsigned* bar;
  cudaMalloc(&d, 4); cudaMalloc(&bar, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int grid : {8, 72, 148, 296}) {
    int iters = 2000;
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)gsync, grid, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)gsync, grid, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  grid=%4d: %.3f us/sync (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    cudaMemset(bar, 0, 8);
    void* args2[] = {&iters, &bar, &d};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)mysync, grid, 256, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("atomic bar grid=%4d: %.3f us/sync (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  int iters = 100000;
  bsync<<<148, 256>>>(iters, d);
  cudaEventRecord(a);
  bsync<<<148, 256>>>(iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("__syncthreads 256 thr: %.1f ns\n", ms * 1e6 / iters);
  return 0;
}
