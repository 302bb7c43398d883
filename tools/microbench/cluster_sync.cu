// Cost of a thread-block-cluster barrier and of a dependent distributed-shared-memory load,
// for cluster sizes 2..16 (one CTA per SM).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  // dependent remote loads (pointer chase through the next CTA's shared memory)
  const int nb = (cl.block_rank() + 1) % cl.num_blocks();
  double* rs = cl.map_shared_rank(sm, nb);
  int idx = threadIdx.x & 7;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) idx = ((int)rs[idx] + 1) & 1023;
  long long t3 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = idx; }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int p : {2, 4, 8, 16}) {
    for (int nt : {256, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(p); cfg.blockDim = dim3(nt); cfg.dynamicSmemBytes = 100 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = p; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      const int it = 2000;
      cudaLaunchKernelEx(&cfg, k, d, it);
      cudaLaunchKernelEx(&cfg, k, d, it);
      long long h[3];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("cluster %2d threads %4d: cluster.sync %.0f clk, dependent DSMEM load %.0f clk (%s)\n", p, nt,
             (double)h[0] / it, (double)h[1] / it, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
