// chol_tiles.cu — Cholesky of the projected mass matrix B_Q (cholesky(), eigh.hpp:20-43) for
// m <= 192 in ONE CTA: blocked left-looking over 16 x 16 tiles held in shared memory, the
// tile products on the FP64 tensor cores (DMMA m8n8k4).
//
// Same contract as chol_kernel (chol.cu): lower factor in place (strict upper triangle zeroed),
// status[0] = 1 when a pivot d <= 0 or d <= rel_tol * max(initial diagonal) (the relative floor
// that sends reduced_gevp to its truncation fallback, eigh.hpp:28-31), and the inverses of the
// 32 x 32 diagonal tiles of L in dinv for the triangular solves.
//
// Per 16-column tile column J (three block barriers):
//   (1) A_IJ -= sum_{K<J} L_IK L_JK^T for I >= J: one warp per tile, DMMA accumulators;
//   (2) warp 0 factors the diagonal tile (16 column steps, column broadcast through shared
//       memory) and inverts it (lane per column, forward substitution);
//   (3) L_IJ = A_IJ L_JJ^{-T} for I > J: one warp per tile, DMMA.
// The critical path is (2): ~16 column steps per tile column, ~250 clk each.

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

constexpr int CT_NW = 16, CT_NT = CT_NW * 32, CT_MAXNB = 12;
constexpr int CT_NTILES = CT_MAXNB * (CT_MAXNB + 1) / 2;

int chol_tiles_max_dim() { return 16 * CT_MAXNB; }

__device__ __forceinline__ int ct_id(int I, int J) { return I * (I + 1) / 2 + J; }
// 16 x 16 tile, row-major with the column index XOR-swizzled by the row's low two bits: the
// DMMA fragment loads X[8i + g][4k + t] (g = lane >> 2, t = lane & 3) hit 16 distinct banks
__device__ __forceinline__ int ct_sw(int r, int c) { return r * 16 + (c ^ ((r & 3) << 2)); }

// acc(16x16 as 2x2 DMMA C fragments) += sign * X Y^T, X, Y 16 x 16 tiles in shared memory
__device__ __forceinline__ void ct_gemm_nt(double (&acc)[2][2][2], const double* X, const double* Y, double sign,
                                           int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    double xa[2], yb[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      xa[i] = sign * X[ct_sw(8 * i + g, 4 * kk + t)];
      yb[i] = Y[ct_sw(8 * i + g, 4 * kk + t)];
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], xa[mi], yb[ni]);
  }
}
__device__ __forceinline__ void ct_load_acc(double (&acc)[2][2][2], const double* X, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[mi][ni][h] = X[ct_sw(8 * mi + g, 8 * ni + 2 * t + h)];
}
__device__ __forceinline__ void ct_store_acc(const double (&acc)[2][2][2], double* X, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) X[ct_sw(8 * mi + g, 8 * ni + 2 * t + h)] = acc[mi][ni][h];
}

__global__ void __launch_bounds__(CT_NT, 1) chol_tiles_kernel(int m, double* __restrict__ a, double rel_tol,
                                                              int* __restrict__ status, double* __restrict__ dinv) {
  extern __shared__ __align__(16) double ctsm[];
  const int nb = (m + 15) >> 4;
  double* L = ctsm;                              // ct_id(I, J) * 256: lower tiles
  double* Li = L + CT_NTILES * 256;              // J * 256: inverses of the diagonal tiles
  double* colj = Li + CT_MAXNB * 256;            // 16: column broadcast of the diagonal factor
  double* scr = colj + 16;                       // (CT_MAXNB / 2) * 256: dinv assembly
  __shared__ double red[CT_NW];
  __shared__ double rsd[16];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // load the lower tiles (identity padding beyond m): one warp per tile, every copy in flight
  for (int I = 0, t = 0; I < nb; ++I)
    for (int J = 0; J <= I; ++J, ++t) {
      if (t % CT_NW != warp) continue;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = lane + 32 * q, r = e & 15, c = e >> 4, gi = 16 * I + r, gj = 16 * J + c;
        const bool ok = gi < m && gj < m;
        double* dst = L + t * 256 + ct_sw(r, c);
        if (ok) cp_async8z(dst, a + gi + (size_t)gj * m, true);
        else *dst = gi == gj ? 1.0 : 0.0;
      }
    }
  cp_async_wait_all();
  __syncthreads();
  double md = 0.0;
  for (int i = tid; i < m; i += CT_NT) md = fmax(md, L[ct_id(i >> 4, i >> 4) * 256 + ct_sw(i & 15, i & 15)]);
  md = warp_max(md);
  if (lane == 0) red[warp] = md;
  if (tid == 0) bad = 0;
  __syncthreads();
  double dmax = 0.0;
#pragma unroll
  for (int w = 0; w < CT_NW; ++w) dmax = fmax(dmax, red[w]);
  const double floor_ = rel_tol * dmax;

  for (int J = 0; J < nb; ++J) {
    // (1) left-looking update of tile column J
    if (J > 0) {
      for (int I = J + warp; I < nb; I += CT_NW) {
        double acc[2][2][2];
        double* X = L + ct_id(I, J) * 256;
        ct_load_acc(acc, X, lane);
        for (int K = 0; K < J; ++K) ct_gemm_nt(acc, L + ct_id(I, K) * 256, L + ct_id(J, K) * 256, -1.0, lane);
        ct_store_acc(acc, X, lane);
      }
      __syncthreads();
    }
    // (2) warp 0: factor the diagonal tile, then invert it
    if (warp == 0) {
      double* T = L + ct_id(J, J) * 256;
      double* Ti = Li + J * 256;
      const int r = lane & 15, h = lane >> 4;
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = T[ct_sw(r, 8 * h + c)];
      bool fail = false;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // lane (j, j >> 3) holds the pivot in x[j & 7]
        const double d = __shfl_sync(0xffffffffu, x[j & 7], j + 16 * (j >> 3));
        if (16 * J + j < m && (d <= 0.0 || d <= floor_)) fail = true;  // uniform
        const double rs = rsqrt(d), ljj = d * rs;
        if (lane == 0) rsd[j] = rs;  // 1 / l_jj for the inverse below
        if (h == (j >> 3)) {  // the lanes holding column j
          const double l = r == j ? ljj : (r > j ? x[j & 7] * rs : 0.0);
          x[j & 7] = l;
          colj[r] = l;
        }
        __syncwarp();
        const double lr = colj[r];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int cc = 8 * h + c;
          if (cc > j && cc <= r) x[c] = fma(-lr, colj[cc], x[c]);
        }
        __syncwarp();
      }
      if (fail) {
        if (lane == 0) bad = 1;
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) T[ct_sw(r, 8 * h + c)] = (8 * h + c <= r) ? x[c] : 0.0;
        __syncwarp();
        // inverse: lane c < 16 solves L y = e_c (forward substitution, 4 partial sums)
        if (lane < 16) {
          const int c = lane;
          double y[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            double s0 = i == c ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int k = 0; k < i; ++k) {
              const double lk = T[ct_sw(i, k)] * y[k];
              if ((k & 3) == 0) s0 -= lk;
              else if ((k & 3) == 1) s1 -= lk;
              else if ((k & 3) == 2) s2 -= lk;
              else s3 -= lk;
            }
            y[i] = ((s0 + s1) + (s2 + s3)) * rsd[i];  // no division on the chain
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) Ti[ct_sw(i, c)] = y[i];
        }
      }
    }
    __syncthreads();
    if (bad) {
      if (tid == 0) status[0] = 1;
      return;
    }
    // (3) L_IJ = A_IJ L_JJ^{-T}
    for (int I = J + 1 + warp; I < nb; I += CT_NW) {
      double acc[2][2][2] = {};
      double* X = L + ct_id(I, J) * 256;
      ct_gemm_nt(acc, X, Li + J * 256, 1.0, lane);
      __syncwarp();
      ct_store_acc(acc, X, lane);
    }
    __syncthreads();
  }

  // outputs: L (lower, zero strict upper) column-major; dinv 32 x 32 tile inverses
  // (column per warp, rows over lanes: a 64-bit idx % m here cost ~20 us of integer division)
  for (int j = warp; j < m; j += CT_NW) {
    double* aj = a + (size_t)j * m;
    for (int i = lane; i < m; i += 32)
      aj[i] = i >= j ? L[ct_id(i >> 4, j >> 4) * 256 + ct_sw(i & 15, j & 15)] : 0.0;
  }
  // [[Li0, 0], [X, Li1]], X = -Li1 (L10 Li0) (16-tiles 2p, 2p+1; identity padding beyond m)
  const int n32 = (m + 31) >> 5;
  for (int p = warp; p < n32; p += CT_NW) {
    double* Di = dinv + (size_t)p * 1024;
    const int t0 = 2 * p, t1 = 2 * p + 1;
    const double* Li0 = Li + t0 * 256;
    double* W = scr + p * 256;  // W = L10 Li0, row-major
    if (t1 < nb) {
      const double* L10 = L + ct_id(t1, t0) * 256;
      for (int e = lane; e < 256; e += 32) {
        const int i = e >> 4, c = e & 15;
        double u = 0.0;
#pragma unroll
        for (int l = 0; l < 16; ++l) u = fma(L10[ct_sw(i, l)], Li0[ct_sw(l, c)], u);
        W[e] = u;
      }
      __syncwarp();
    }
    for (int e = lane; e < 1024; e += 32) {
      const int i = e & 31, c = e >> 5;
      double v;
      if (i < 16 && c < 16) v = Li0[ct_sw(i, c)];
      else if (i < 16) v = 0.0;
      else if (t1 >= nb) v = i == c ? 1.0 : 0.0;
      else if (c >= 16) v = Li[t1 * 256 + ct_sw(i - 16, c - 16)];
      else {
        const double* Li1 = Li + t1 * 256;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) s = fma(Li1[ct_sw(i - 16, k)], W[k * 16 + c], s);
        v = -s;
      }
      Di[i + c * 32] = v;
    }
  }
}

size_t chol_tiles_smem() { return sizeof(double) * ((size_t)(CT_NTILES + CT_MAXNB + CT_MAXNB / 2) * 256 + 16); }

cudaError_t chol_tiles(int m, double* a, double rel_tol, int* status, double* dinv, cudaStream_t st) {
  if (m < 1 || m > chol_tiles_max_dim()) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_tiles_smem());
    attr = true;
  }
  chol_tiles_kernel<<<1, CT_NT, chol_tiles_smem(), st>>>(m, a, rel_tol, status, dinv);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
