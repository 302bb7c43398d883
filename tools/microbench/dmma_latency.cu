// Microbenchmark: DMMA (mma.sync m8n8k4 f64) dependent-chain latency and throughput vs the
// number of independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chain(double* out, int iters, long long* cyc) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
void run(int warps, double* d, long long* dc) {
  const int iters = 2048;
  chain<CH><<<1, 32 * warps>>>(d, iters, dc);
  chain<CH><<<1, 32 * warps>>>(d, iters, dc);
  long long c;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (iters * CH);
  printf("chains/warp=%d warps=%2d: %.2f clk per DMMA per warp, SM rate %.3f DMMA/clk (peak 0.25)\n", CH, warps,
         per, warps / per);
}

int main() {
  double* d;
  long long* dc;
  cudaMalloc(&d, 8);
  cudaMalloc(&dc, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, d, dc);
    run<2>(w, d, dc);
    run<4>(w, d, dc);
    run<8>(w, d, dc);
  }
  return 0;
}
