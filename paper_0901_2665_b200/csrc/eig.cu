// eig.cu — the reduced generalized eigensolver on device (reduced_gevp, eigh.hpp:178-225).
//
//   (cholesky / trsm_lower / trsm_lower_t live in chol.cu)
//   sym_eig       symmetric eigendecomposition, ascending, orthonormal vectors (the role of
//                 jacobi_eigh, eigh.hpp:84-163): Householder tridiagonalisation + Sturm
//                 multisection + inverse iteration + back-transformation (tridiag*.cu,
//                 tri_back.cu). A different method from the reference's cyclic Jacobi; the
//                 eigenpairs agree to rounding (tests/test_gpu_parity.py).
//   EigWork       its device workspace, cached process-wide per (device, size) so a fresh
//                 context (every end-to-end solve opens one) does not pay cudaMalloc/cudaFree.

#include <algorithm>
#include <cfloat>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

int tri_max_dim();
cudaError_t tri_eig(int m, const double* a, double* evals, double* v, double* ws, int* iws, cudaStream_t st,
                    double vfloor, bool low_smem, cudaEvent_t ev_tridiag);

struct EigWork {
  int mmax = 0;
  int dev = 0;
  double* tws = nullptr;  // tridiagonal route: 6m^2 + 3m
  int* tiws = nullptr;    // m^2
};

static std::mutex g_eig_mu;
static std::vector<EigWork*> g_eig_cache;
constexpr size_t kEigCacheMax = 4;

EigWork* eig_create(int mmax) {
  int cur = 0;
  cudaGetDevice(&cur);
  {
    std::lock_guard<std::mutex> lk(g_eig_mu);
    for (size_t i = 0; i < g_eig_cache.size(); ++i)
      if (g_eig_cache[i]->mmax == mmax && g_eig_cache[i]->dev == cur) {
        EigWork* w = g_eig_cache[i];
        g_eig_cache.erase(g_eig_cache.begin() + i);
        return w;
      }
  }
  EigWork* w = new EigWork();
  w->dev = cur;
  w->mmax = mmax;
  const size_t tm = (size_t)std::min(mmax, tri_max_dim());
  if (cudaMalloc(&w->tws, sizeof(double) * (6 * tm * tm + 3 * tm)) != cudaSuccess ||
      cudaMalloc(&w->tiws, sizeof(int) * tm * tm) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(w->tws);
    delete w;
    return nullptr;
  }
  return w;
}

void eig_destroy(EigWork* w) {
  if (!w) return;
  {
    std::lock_guard<std::mutex> lk(g_eig_mu);  // (the caller has synchronised its stream)
    if (g_eig_cache.size() < kEigCacheMax) {
      g_eig_cache.push_back(w);
      return;
    }
  }
  cudaFree(w->tws);
  cudaFree(w->tiws);
  delete w;
}

cudaError_t sym_eig(EigWork* w, int m, double* a, double* evals, double* v, cudaStream_t st, double vfloor,
                    bool low_smem, cudaEvent_t ev_tridiag) {
  if (!w || m < 1 || m > w->mmax || m > tri_max_dim()) return cudaErrorInvalidValue;
  return tri_eig(m, a, evals, v, w->tws, w->tiws, st, vfloor, low_smem, ev_tridiag);
}

__global__ void transpose_kernel(const double* __restrict__ src, int m, int n, int lds,
                                 double* __restrict__ dst, int ldd) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = bx + threadIdx.x, c = by + j;
    if (r < m && c < n) tile[j][threadIdx.x] = src[r + (int64_t)c * lds];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + threadIdx.x, c = bx + j;  // dst(r, c) = src(c, r)
    if (r < n && c < m) dst[r + (int64_t)c * ldd] = tile[threadIdx.x][j];
  }
}

cudaError_t transpose(const double* src, int m, int n, int lds, double* dst, int ldd, cudaStream_t st) {
  dim3 grid((m + 31) / 32, (n + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, m, n, lds, dst, ldd);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void scale_columns_kernel(const double* v, int m, const int* keep, const double* d, int nk,
                                     double* s) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)m * nk;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    const int kj = keep[j];
    const double inv = 1.0 / sqrt(d[kj]);  // eigh.hpp:216-218
    s[i + (int64_t)j * m] = v[i + (int64_t)kj * m] * inv;
  }
}

cudaError_t scale_columns(const double* v, int m, const int* keep, const double* d, int nk, double* s,
                          cudaStream_t st) {
  const int64_t total = (int64_t)m * nk;
  scale_columns_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 1024), 256, 0, st>>>(
      v, m, keep, d, nk, s);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
