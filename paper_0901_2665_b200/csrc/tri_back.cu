// tri_back.cu — back-transformation V = H_0 H_1 ... H_{m-3} Z of the tridiagonal eigenvectors
// (the last step of the reduced eigensolve that replaces jacobi_eigh, eigh.hpp:84-163), blocked:
// NB consecutive reflectors form one block reflector I - Y T Y^T (LAPACK's dlarft, forward,
// columnwise), and each block is applied to a CTA's columns of Z as three small products
//   W = Y^T Z,  W <- T W,  Z <- Z - Y W,
// so a column sees m/NB dependent reductions instead of m - 2 (tri_back_kernel in tridiag.cu
// chains one warp reduction per reflector).
//
//   tri_larft_kernel   one CTA per block: G = Y^T Y, then T column by column
//                      (T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j), T(j, j) = tau_j)
//   tri_back_wy_kernel one CTA per CB columns of Z; blocks applied last to first

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

constexpr int TBK_CB = 8;    // columns of Z per CTA
constexpr int TBK_NT = 256;  // threads

// T for block b (reflectors k0 = NB b .. k0 + NB - 1, those >= nrefl are zero) -> tw + b NB^2
template <int NB>
__global__ void __launch_bounds__(NB * NB) tri_larft_kernel(int m, int nrefl, const double* __restrict__ hv,
                                                           const double* __restrict__ tau, double* __restrict__ tw) {
  extern __shared__ __align__(16) double ysm[];  // Y block, m x NB column-major, ld m | 1 (odd: the
                                                 // G dots read one column per lane, conflict-free)
  __shared__ double G[NB][NB + 1];
  __shared__ double T[NB][NB + 1];
  const int b = blockIdx.x, k0 = b * NB;
  const int i = threadIdx.x % NB, j = threadIdx.x / NB;  // G(i, j)
  const int ly = m | 1;
  for (int e = threadIdx.x; e < m * NB; e += NB * NB) {
    const int r = e % m, jj = e / m, k = k0 + jj;
    const bool ok = k < nrefl && r > k;
    cp_async8z(ysm + r + jj * ly, ok ? hv + r + (size_t)k * m : hv, ok);
  }
  cp_async_wait_all();
  __syncthreads();
  {
    const double* vi = ysm + (size_t)i * ly;
    const double* vj = ysm + (size_t)j * ly;
    double s0 = 0.0, s1 = 0.0;
    int r = k0 + max(i, j) + 1;
    for (; r + 1 < m; r += 2) {
      s0 = fma(vi[r], vj[r], s0);
      s1 = fma(vi[r + 1], vj[r + 1], s1);
    }
    if (r < m) s0 = fma(vi[r], vj[r], s0);
    G[i][j] = s0 + s1;
    T[i][j] = 0.0;
  }
  __syncthreads();
  for (int c = 0; c < NB; ++c) {
    const double tc = k0 + c < nrefl ? tau[k0 + c] : 0.0;
    // row i < c of column c: -tau_c * sum_{l=i}^{c-1} T(i, l) G(l, c)
    if (j == 0 && i <= c) {
      double s = 0.0;
      for (int l = i; l < c; ++l) s = fma(T[i][l], G[l][c], s);
      T[i][c] = i == c ? tc : -tc * s;
    }
    __syncthreads();
  }
  tw[(size_t)b * NB * NB + i + j * NB] = T[i][j];
}

template <int NB>
__global__ void __launch_bounds__(TBK_NT) tri_back_wy_kernel(int m, int nrefl, const double* __restrict__ hv,
                                                            const double* __restrict__ tw,
                                                            const double* __restrict__ z, double* __restrict__ v) {
  extern __shared__ __align__(16) double bsm[];
  double* Zs = bsm;                  // m x CB, column-major (ld m)
  const int ly = m | 1;              // odd: W = Y^T Z reads one Y column per lane
  double* Ys = Zs + m * TBK_CB;      // m x NB, column-major (ld ly)
  double* Ts = Ys + ly * NB;         // NB x NB (ld NB)
  double* Ws = Ts + NB * NB;         // NB x CB
  double* W2 = Ws + NB * TBK_CB;     // NB x CB
  const int tid = threadIdx.x, c0 = blockIdx.x * TBK_CB;
  const int ncols = min(TBK_CB, m - c0);
  for (int e = tid; e < m * TBK_CB; e += TBK_NT) {
    const int r = e % m, c = e / m;
    cp_async8z(Zs + e, z + r + (size_t)(c0 + min(c, ncols - 1)) * m, c < ncols);
  }
  const int nblk = (nrefl + NB - 1) / NB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int k0 = b * NB, rlo = k0 + 1;  // rows below k0 are untouched by this block
    __syncthreads();
    for (int e = tid; e < m * NB; e += TBK_NT) {
      const int r = e % m, jj = e / m, k = k0 + jj;
      const bool ok = k < nrefl && r > k;
      cp_async8z(Ys + r + jj * ly, ok ? hv + r + (size_t)k * m : hv, ok);
    }
    for (int e = tid; e < NB * NB; e += TBK_NT) cp_async8z(Ts + e, tw + (size_t)b * NB * NB + e, true);
    cp_async_wait_all();
    __syncthreads();
    // W = Y^T Z: NB x CB dots over rows >= rlo, four partial sums each
    for (int e = tid; e < NB * TBK_CB; e += TBK_NT) {
      const int jj = e % NB, c = e / NB;
      const double* y = Ys + jj * ly;
      const double* zc = Zs + c * m;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int r = rlo + jj;  // Y(:, jj) is zero above row k0 + jj + 1
      for (; r + 3 < m; r += 4) {
        s0 = fma(y[r], zc[r], s0);
        s1 = fma(y[r + 1], zc[r + 1], s1);
        s2 = fma(y[r + 2], zc[r + 2], s2);
        s3 = fma(y[r + 3], zc[r + 3], s3);
      }
      for (; r < m; ++r) s0 = fma(y[r], zc[r], s0);
      Ws[jj + c * NB] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    // W2 = T W (T upper triangular)
    for (int e = tid; e < NB * TBK_CB; e += TBK_NT) {
      const int jj = e % NB, c = e / NB;
      double s = 0.0;
      for (int l = jj; l < NB; ++l) s = fma(Ts[jj + l * NB], Ws[l + c * NB], s);
      W2[jj + c * NB] = s;
    }
    __syncthreads();
    // Z -= Y W2 on rows >= rlo
    for (int e = tid; e < (m - rlo) * TBK_CB; e += TBK_NT) {
      const int r = rlo + e % (m - rlo), c = e / (m - rlo);
      double s = 0.0;
#pragma unroll 8
      for (int jj = 0; jj < NB; ++jj) s = fma(Ys[r + jj * ly], W2[jj + c * NB], s);
      Zs[r + c * m] -= s;
    }
  }
  __syncthreads();
  for (int e = tid; e < m * ncols; e += TBK_NT) {
    const int r = e % m, c = e / m;
    v[r + (size_t)(c0 + c) * m] = Zs[e];
  }
}

size_t tri_back_wy_ws(int m) { return (size_t)(m / 16 + 1) * 32 * 32; }

template <int NB>
static cudaError_t launch_back_wy(int m, const double* hv, const double* tau, const double* z, double* v,
                                  double* tw, cudaStream_t st) {
  const int nrefl = m - 2, nblk = (nrefl + NB - 1) / NB;
  static bool lattr = false;
  if (!lattr) {
    cudaFuncSetAttribute(tri_larft_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    lattr = true;
  }
  tri_larft_kernel<NB><<<nblk, NB * NB, sizeof(double) * (size_t)(m | 1) * NB, st>>>(m, nrefl, hv, tau, tw);
  ++g_launches;
  const size_t sm = sizeof(double) * ((size_t)m * TBK_CB + (size_t)(m | 1) * NB + NB * NB + 2 * NB * TBK_CB);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tri_back_wy_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  tri_back_wy_kernel<NB><<<(m + TBK_CB - 1) / TBK_CB, TBK_NT, sm, st>>>(m, nrefl, hv, tw, z, v);
  ++g_launches;
  return cudaGetLastError();
}

// m >= 3; tw: tri_back_wy_ws(m) doubles
cudaError_t tri_back_wy(int m, const double* hv, const double* tau, const double* z, double* v, double* tw,
                        cudaStream_t st) {
  if (m < 3 || m > 1024) return cudaErrorInvalidValue;
  return m <= 384 ? launch_back_wy<32>(m, hv, tau, z, v, tw, st) : launch_back_wy<16>(m, hv, tau, z, v, tw, st);
}

}  // namespace feastgpu
