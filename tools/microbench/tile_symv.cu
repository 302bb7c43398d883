// One warp, one 32x32 tile of a packed column-major lower triangle in shared memory:
// y_row = T v_J (lane = row) and y_col = T^T v_I (lane = column). Variants of how v reaches
// the lanes and how loads are predicated, timed in SM clocks per tile.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 192;
__device__ __forceinline__ int pidx(int i, int j, int m) { return j * m - (j * (j - 1)) / 2 + (i - j); }

template <int VAR>
__global__ void k(double* out, long long* cyc, int reps, int I, int J) {
  extern __shared__ double ps[];
  double* vs = ps + M * (M + 1) / 2;
  for (int i = threadIdx.x; i < M * (M + 1) / 2 + M; i += blockDim.x) ps[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    const int gc0 = 32 * J + (rep & 1);
    const double vI = vs[32 * I + lane], vJ = vs[32 * J + lane];
    double yr0 = 0, yr1 = 0, yc0 = 0, yc1 = 0;
    int pr = pidx(32 * I + lane + 32, gc0, M), step = M - gc0 - 1;
    const int gc = 32 * J + lane;
    const int pc = pidx(gc, gc, M) + (32 * I + 32 - gc);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      double vj;
      if (VAR == 0) vj = __shfl_sync(0xffffffffu, vJ, jj);
      else vj = vs[32 * J + jj];
      const double x = ps[pr];
      pr += step;
      --step;
      if (jj & 1) yr1 += x * vj; else yr0 += x * vj;
    }
#pragma unroll
    for (int ii = 0; ii < 32; ++ii) {
      double vi;
      if (VAR == 0) vi = __shfl_sync(0xffffffffu, vI, ii);
      else vi = vs[32 * I + ii];
      const double x = ps[pc + ii];
      if (ii & 1) yc1 += x * vi; else yc0 += x * vi;
    }
    acc += yr0 + yr1 + yc0 + yc1;
    __syncwarp();
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 8192 * 8); cudaMalloc(&c, 64);
  const int sm = (M * (M + 1) / 2 + M) * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int w : {32, 256}) {
    long long h;
    k<0><<<1, w, sm>>>(d, c, 1000, 3, 1); k<0><<<1, w, sm>>>(d, c, 1000, 3, 1);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %3d  shfl-v      : %.0f clk per tile (all warps run the same tile)\n", w, h / 1000.0);
    k<1><<<1, w, sm>>>(d, c, 1000, 3, 1); k<1><<<1, w, sm>>>(d, c, 1000, 3, 1);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %3d  broadcast-v : %.0f clk per tile\n", w, h / 1000.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
