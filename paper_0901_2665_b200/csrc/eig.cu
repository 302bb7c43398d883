// eig.cu — the reduced generalized eigensolver on device (reduced_gevp, eigh.hpp:178-225).
//
//   (cholesky / trsm_lower / trsm_lower_t live in chol.cu)
//   sym_eig       symmetric eigendecomposition, ascending, stable order (jacobi_eigh,
//                 eigh.hpp:84-163). Same method class as the reference (cyclic Jacobi, so
//                 multiplicities and tiny eigenvalues come out as accurately), re-shaped for
//                 148 SMs: BLOCK Jacobi. The m x m matrix is cut into 2k blocks of bs rows;
//                 each round pairs the blocks by the circle method, every pair's 2bs x 2bs
//                 sub-problem is diagonalised in shared memory by parallel (round-robin)
//                 Jacobi, and the pair rotations are applied to W and V as small GEMM tiles
//                 by all CTAs — one cooperative kernel, two grid barriers per round.

#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

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
