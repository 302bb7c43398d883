// Per-phase cycle split of tridiag_tiles_kernel as seen by warp 0 (TT_PROFILE build).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DTT_PROFILE tt_phases.cu -o tt_phases
#include <cstdio>
#include <random>
#include <vector>
#ifndef TT_NOPROF
#define TT_PROFILE 1
#endif
#include "../../paper_0901_2665_b200/csrc/tridiag_tiles.cu"
namespace feastgpu { int64_t g_launches = 0; }
using namespace feastgpu;
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 192;
  std::vector<double> a((size_t)m * m);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(-1, 1);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i <= j; ++i) a[i + (size_t)j * m] = a[j + (size_t)i * m] = u(g);
  double *da, *d, *e, *hv, *tau;
  cudaMalloc(&da, sizeof(double) * m * m); cudaMalloc(&hv, sizeof(double) * m * m);
  cudaMalloc(&d, sizeof(double) * m); cudaMalloc(&e, sizeof(double) * m); cudaMalloc(&tau, sizeof(double) * m);
  cudaMemcpy(da, a.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
  for (int w = 0; w < 3; ++w) tridiag_tiles(m, da, d, e, hv, tau, 0);
  unsigned long long z[16] = {0};
#ifdef TT_PROFILE
  cudaMemcpyToSymbol(tt_prof, z, sizeof(z));
#endif
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  const int reps = 10;
  cudaEventRecord(t0);
  for (int w = 0; w < reps; ++w) tridiag_tiles(m, da, d, e, hv, tau, 0);
  cudaEventRecord(t1); cudaEventSynchronize(t1);
  float ms; cudaEventElapsedTime(&ms, t0, t1);
  unsigned long long p[16] = {0};
#ifdef TT_PROFILE
  cudaMemcpyFromSymbol(p, tt_prof, sizeof(p));
#endif
  const char* nm[] = {"", "(a) tiles, warp 0", "barrier (a)", "(b) v, hv stores", "barrier (b)",
                      "(b) row sums p, p.v", "(b) w, column, xn2", "(b) sqrt, div"};
  printf("m=%d: %.1f us per launch (%s)\n", m, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  for (int i = 1; i <= 7; ++i) printf("  %-28s %8.0f clk per column\n", nm[i], (double)p[i] / reps / m);
  return 0;
}
