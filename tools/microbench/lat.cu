// Dependent-chain latencies on this GPU: DFMA, DADD, SHFL (f64 value), LDS.64, and
// FP64 division / sqrt as compiled (software sequences), in SM clocks.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-9 * i;
  __syncthreads();
  double x = 1.0 + threadIdx.x * 1e-12, y = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = x + y;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 0.0;
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) { idx = (int)sm[idx & 1023] + idx + 1; }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 2.0);
  long long t5 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 2.0);
  long long t6 = clock64();
  out[threadIdx.x] = x + idx;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 8192); cudaMalloc(&c, 64);
  const int it = 4096;
  for (int w : {32, 1024}) {
    k<<<1, w>>>(d, c, it); k<<<1, w>>>(d, c, it);
    long long h[6]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%4d  DFMA %.1f  DADD %.1f  SHFL+DADD %.1f  LDS.64+cvt+IADD %.1f  DDIV %.1f  DSQRT %.1f clk/op\n", w,
           (double)h[0] / it, (double)h[1] / it, (double)h[2] / it, (double)h[3] / it, (double)h[4] / it, (double)h[5] / it);
  }
  return 0;
}
