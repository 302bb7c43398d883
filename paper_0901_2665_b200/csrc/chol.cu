// chol.cu — tiled Cholesky and triangular solves for the reduced problem (m <= 1024).
//
//   cholesky      lower Cholesky with the relative pivot floor of eigh.hpp:20-43
//                 (kCholeskyRelTol = 1e-13 -> NotPositiveDefinite -> truncation fallback).
//                 Blocked right-looking, 32x32 tiles, one cooperative kernel: per panel the
//                 diagonal tile is factored in shared memory (and inverted for the solves),
//                 the panel below is solved against it, then the trailing tiles are updated
//                 by all CTAs — three grid barriers per 32-column panel.
//   trsm_lower    X <- L^{-1} X      (solve_lower_in_place, eigh.hpp:46-58)
//   trsm_lower_t  X <- L^{-T} X      (solve_lower_adjoint_in_place, eigh.hpp:61-73)
//                 One CTA per 16-column tile of X; the tile stays in shared memory while the
//                 CTA walks the block substitution chain, L tiles streamed from L2, diagonal
//                 tiles applied through their precomputed inverses.

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

constexpr int TB = 32;  // tile
constexpr int TL = TB + 1;

struct CholArgs {
  int m;
  double* a;
  double* dinv;  // nblk * TB*TB, inverse of each diagonal L tile (ld TB)
  double rel_tol;
  int* status;
};

__global__ void __launch_bounds__(256) chol_kernel(CholArgs p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double T[TB * TL], U[TB * TL], Vt[TB * TL];
  __shared__ double red[33];
  __shared__ int bad;
  const int m = p.m, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = (m + TB - 1) / TB;
  double* A = p.a;

  // max initial diagonal (every CTA computes the same value)
  double md = 0.0;
  for (int i = tid; i < m; i += nt) md = fmax(md, A[i + (int64_t)i * m]);
  md = warp_max(md);
  if (lane == 0) red[warp] = md;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < (nt >> 5); ++w) r = fmax(r, red[w]);
    red[32] = r;
    bad = 0;
  }
  __syncthreads();
  const double floor_ = p.rel_tol * red[32];

  for (int pn = 0; pn < nblk; ++pn) {
    const int p0 = pn * TB, pb = min(TB, m - p0);
    // ---- phase 1: diagonal tile (CTA 0, one warp) ----
    if (blockIdx.x == 0) {
      for (int idx = tid; idx < TB * TB; idx += nt) {
        const int i = idx % TB, j = idx / TB;
        if (i < pb && j < pb) cp_async8z(T + i + j * TL, A + (p0 + i) + (int64_t)(p0 + j) * m, true);
        else T[i + j * TL] = i == j ? 1.0 : 0.0;
      }
      cp_async_wait_all();
      __syncthreads();
      // right-looking factor of the tile by all threads (pivot d = a_jj - sum_k l_jk^2
      // after the updates; failure is uniform because every thread reads the same d)
      for (int j = 0; j < pb; ++j) {
        const double d = T[j + j * TL];
        if (d <= 0.0 || d <= floor_) {
          bad = 1;
          break;
        }
        const double ljj = sqrt(d);
        __syncthreads();
        if (tid == 0) T[j + j * TL] = ljj;
        for (int i = j + 1 + tid; i < pb; i += nt) T[i + j * TL] /= ljj;
        __syncthreads();
        const int r = pb - j - 1;
        for (int idx = tid; idx < r * r; idx += nt) {
          const int i = j + 1 + idx % r, k = j + 1 + idx / r;
          if (k <= i) T[i + k * TL] -= T[i + j * TL] * T[k + j * TL];
        }
        __syncthreads();
      }
      __syncthreads();
      if (!bad) {
        // L^{-1} of the tile: forward substitution on all identity columns at once
        for (int idx = tid; idx < TB * TB; idx += nt) {
          const int i = idx % TB, c = idx / TB;
          U[i + c * TL] = i == c ? 1.0 : 0.0;
        }
        __syncthreads();
        for (int k = 0; k < pb; ++k) {
          for (int c = tid; c <= k; c += nt) U[k + c * TL] /= T[k + k * TL];
          __syncthreads();
          const int r = pb - k - 1;
          for (int idx = tid; idx < r * (k + 1); idx += nt) {
            const int i = k + 1 + idx % r, c = idx / r;
            U[i + c * TL] -= T[i + k * TL] * U[k + c * TL];
          }
          __syncthreads();
        }
        double* Di = p.dinv + (int64_t)pn * TB * TB;
        for (int idx = tid; idx < TB * TB; idx += nt) {
          const int i = idx % TB, c = idx / TB;
          Di[i + c * TB] = (i < pb && c < pb) ? U[i + c * TL] : (i == c ? 1.0 : 0.0);
        }
      }
      __syncthreads();
      if (bad) {
        if (tid == 0) p.status[0] = 1;
      } else {
        for (int idx = tid; idx < pb * pb; idx += nt) {
          const int i = idx % pb, j = idx / pb;
          A[(p0 + i) + (int64_t)(p0 + j) * m] = i >= j ? T[i + j * TL] : 0.0;
        }
      }
    }
    grid.sync();
    if (p.status[0]) return;
    // ---- phase 2: L_ip = A_ip * (L_pp^{-1})^T for row tiles below ----
    const int below = nblk - pn - 1;
    for (int task = blockIdx.x; task < below; task += gridDim.x) {
      const int i0 = (pn + 1 + task) * TB, ib = min(TB, m - i0);
      const double* Di = p.dinv + (int64_t)pn * TB * TB;
      for (int idx = tid; idx < TB * TB; idx += nt) {
        const int r = idx % TB, c = idx / TB;
        const bool v = r < ib && c < pb;
        cp_async8z(U + r + c * TL, v ? A + (i0 + r) + (int64_t)(p0 + c) * m : A, v);
        cp_async8z(Vt + r + c * TL, Di + r + c * TB, true);
      }
      cp_async_wait_all();
      __syncthreads();
      for (int idx = tid; idx < ib * pb; idx += nt) {
        const int r = idx % ib, c = idx / ib;
        double s = 0.0;
        for (int k = 0; k < pb; ++k) s += U[r + k * TL] * Vt[c + k * TL];
        A[(i0 + r) + (int64_t)(p0 + c) * m] = s;
      }
      __syncthreads();
    }
    grid.sync();
    // ---- phase 3: A_ij -= L_ip L_jp^T, p < j <= i ----
    const int ntask = below * (below + 1) / 2;
    for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= task) ++ti;
      const int tj = task - ti * (ti + 1) / 2;
      const int i0 = (pn + 1 + ti) * TB, j0 = (pn + 1 + tj) * TB;
      const int ib = min(TB, m - i0), jb = min(TB, m - j0);
      for (int idx = tid; idx < TB * TB; idx += nt) {
        const int r = idx % TB, c = idx / TB;
        const bool vu = r < ib && c < pb, vv = r < jb && c < pb;
        cp_async8z(U + r + c * TL, vu ? A + (i0 + r) + (int64_t)(p0 + c) * m : A, vu);
        cp_async8z(Vt + r + c * TL, vv ? A + (j0 + r) + (int64_t)(p0 + c) * m : A, vv);
      }
      cp_async_wait_all();
      __syncthreads();
      for (int idx = tid; idx < ib * jb; idx += nt) {
        const int r = idx % ib, c = idx / ib;
        double s = 0.0;
        for (int k = 0; k < pb; ++k) s += U[r + k * TL] * Vt[c + k * TL];
        A[(i0 + r) + (int64_t)(j0 + c) * m] -= s;
      }
      __syncthreads();
    }
    grid.sync();
  }
  // strict upper triangle -> 0 (cholesky() returns a lower factor)
  for (int64_t idx = blockIdx.x * (int64_t)nt + tid; idx < (int64_t)m * m; idx += (int64_t)gridDim.x * nt) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    if (i < j) A[idx] = 0.0;
  }
}

cudaError_t cholesky(int m, double* a, double rel_tol, int* status, double* dinv, cudaStream_t st) {
  if (m > 1024 || m < 1) return cudaErrorInvalidValue;
  // m <= 192: one CTA, 16 x 16 tiles in shared memory, DMMA tile products (chol_tiles.cu);
  // beyond: the cooperative kernel above
  if (m <= chol_tiles_max_dim()) return chol_tiles(m, a, rel_tol, status, dinv, st);
  const int nblk = (m + TB - 1) / TB;
  int grid = std::max(1, nblk * (nblk - 1) / 2);
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_kernel, 256, 0);
  grid = std::min(grid, sms * std::max(occ, 1));
  CholArgs p{m, a, dinv, rel_tol, status};
  void* args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)chol_kernel, grid, 256, args, 0, st);
  ++g_launches;
  return e;
}

// ---------------------------------------------------------------------------
// triangular solves on 16-column tiles of X (resident in shared memory)
// ---------------------------------------------------------------------------
constexpr int XC = 16;

template <bool TRANS>
__global__ void __launch_bounds__(256) trsm_tile_kernel(int m, const double* __restrict__ l,
                                                        const double* __restrict__ dinv, double* x,
                                                        int ldx, int ncols) {
  extern __shared__ double xs[];  // m x XC, column-major (ld m)
  __shared__ double Lt[TB * TL];
  __shared__ double acc_s[TB * XC];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int c0 = blockIdx.x * XC, nc = min(XC, ncols - c0);
  const int nblk = (m + TB - 1) / TB;
  for (int idx = tid; idx < m * XC; idx += nt) {
    const int i = idx % m, c = idx / m;
    xs[idx] = c < nc ? x[i + (int64_t)(c0 + c) * ldx] : 0.0;
  }
  __syncthreads();
  // thread -> (row r, columns c, c+8) of a TB x XC tile
  const int r = tid % TB, cA = tid / TB, cB = cA + 8;
  for (int step = 0; step < nblk; ++step) {
    const int bi = TRANS ? nblk - 1 - step : step;
    const int i0 = bi * TB, ib = min(TB, m - i0);
    double accA = (r < ib) ? xs[(i0 + r) + cA * m] : 0.0;
    double accB = (r < ib) ? xs[(i0 + r) + cB * m] : 0.0;
    const int jlo = TRANS ? bi + 1 : 0, jhi = TRANS ? nblk : bi;
    // the L tile feeding update bj: L_ij (lower) or L_ji^T (transposed); the next tile is
    // loaded into registers while the current one is consumed (latency off the chain)
    constexpr int PER = TB * TB / 256;
    double nxt[PER];
    auto fetch = [&](int bj) {
      const int j0 = bj * TB, jb = min(TB, m - j0);
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * 256, rr = idx % TB, cc = idx / TB;
        double v = 0.0;
        if (!TRANS) { if (rr < ib && cc < jb) v = l[(i0 + rr) + (int64_t)(j0 + cc) * m]; }
        else { if (cc < jb && rr < ib) v = l[(j0 + cc) + (int64_t)(i0 + rr) * m]; }
        nxt[q] = v;
      }
    };
    if (jlo < jhi) fetch(jlo);
    for (int bj = jlo; bj < jhi; ++bj) {
      const int j0 = bj * TB, jb = min(TB, m - j0);
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * 256;
        Lt[(idx % TB) + (idx / TB) * TL] = nxt[q];
      }
      __syncthreads();
      if (bj + 1 < jhi) fetch(bj + 1);
      double sA = 0.0, sB = 0.0;
      for (int k = 0; k < jb; ++k) {
        const double lv = Lt[r + k * TL];
        sA += lv * xs[(j0 + k) + cA * m];
        sB += lv * xs[(j0 + k) + cB * m];
      }
      accA -= sA;
      accB -= sB;
      __syncthreads();
    }
    // apply the inverse of the diagonal tile (transposed for L^{-T})
    acc_s[r + cA * TB] = accA;
    acc_s[r + cB * TB] = accB;
    const double* Di = dinv + (int64_t)bi * TB * TB;
    for (int idx = tid; idx < TB * TB; idx += nt) {
      const int rr = idx % TB, cc = idx / TB;
      Lt[rr + cc * TL] = TRANS ? Di[cc + rr * TB] : Di[rr + cc * TB];
    }
    __syncthreads();
    if (r < ib) {
      double sA = 0.0, sB = 0.0;
      for (int k = 0; k < ib; ++k) {
        sA += Lt[r + k * TL] * acc_s[k + cA * TB];
        sB += Lt[r + k * TL] * acc_s[k + cB * TB];
      }
      xs[(i0 + r) + cA * m] = sA;
      xs[(i0 + r) + cB * m] = sB;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < m * XC; idx += nt) {
    const int i = idx % m, c = idx / m;
    if (c < nc) x[i + (int64_t)(c0 + c) * ldx] = xs[idx];
  }
}

// The same solves for m <= 192 with every lower 32 x 32 tile of L resident in shared memory
// (21 tiles + the X tile: ~200 KB): the substitution chain never waits on L2, the diagonal-tile
// inverse of the next step is fetched into registers while the current step runs, and each
// tile product is split over four partial sums.
constexpr int RS_MAXB = 6;  // 32-row blocks: m <= 192
template <bool TRANS>
__global__ void __launch_bounds__(256) trsm_res_kernel(int m, const double* __restrict__ l,
                                                       const double* __restrict__ dinv, double* x, int ldx,
                                                       int ncols) {
  extern __shared__ double rsm[];
  double* xs = rsm;                                 // m x XC, column-major (ld m)
  double* Ls = xs + (size_t)m * XC;                 // lower tiles, id I(I+1)/2 + J, TB x TL col-major
  double* Ds = Ls + (size_t)RS_MAXB * (RS_MAXB + 1) / 2 * TB * TL;  // current diagonal inverse
  double* acc_s = Ds + TB * TL;                     // TB x XC
  const int tid = threadIdx.x, nt = blockDim.x;
  const int c0 = blockIdx.x * XC, nc = min(XC, ncols - c0);
  const int nblk = (m + TB - 1) / TB;
  // every staging copy in flight at once (cp.async, zero fill outside): the tiles are ~170 KB
  for (int idx = tid; idx < m * XC; idx += nt) {
    const int i = idx % m, c = idx / m;
    cp_async8z(xs + idx, x + i + (int64_t)(c0 + min(c, nc - 1)) * ldx, c < nc);
  }
  for (int I = 0; I < nblk; ++I)
    for (int J = 0; J <= I; ++J) {
      double* T = Ls + (size_t)(I * (I + 1) / 2 + J) * TB * TL;
      for (int idx = tid; idx < TB * TB; idx += nt) {
        const int rr = idx % TB, cc = idx / TB, gi = I * TB + rr, gj = J * TB + cc;
        const bool ok = gi < m && gj < m;
        cp_async8z(T + rr + cc * TL, ok ? l + gi + (int64_t)gj * m : l, ok);
      }
    }
  cp_async_wait_all();
  const int r = tid % TB, cA = tid / TB, cB = cA + 8;
  constexpr int PER = TB * TB / 256;
  double dn[PER];
  auto fetch_d = [&](int bi) {
#pragma unroll
    for (int q = 0; q < PER; ++q) dn[q] = dinv[(int64_t)bi * TB * TB + tid + q * 256];
  };
  fetch_d(TRANS ? nblk - 1 : 0);
  __syncthreads();
  for (int step = 0; step < nblk; ++step) {
    const int bi = TRANS ? nblk - 1 - step : step;
    const int i0 = bi * TB, ib = min(TB, m - i0);
#pragma unroll
    for (int q = 0; q < PER; ++q) {  // Di (transposed for L^{-T}) into shared memory
      const int idx = tid + q * 256, rr = idx % TB, cc = idx / TB;
      if (TRANS) Ds[cc + rr * TL] = dn[q];
      else Ds[rr + cc * TL] = dn[q];
    }
    if (step + 1 < nblk) fetch_d(TRANS ? bi - 1 : bi + 1);
    double a0 = (r < ib) ? xs[(i0 + r) + cA * m] : 0.0, a1 = 0.0;
    double b0 = (r < ib) ? xs[(i0 + r) + cB * m] : 0.0, b1 = 0.0;
    const int jlo = TRANS ? bi + 1 : 0, jhi = TRANS ? nblk : bi;
    for (int bj = jlo; bj < jhi; ++bj) {
      const int j0 = bj * TB, jb = min(TB, m - j0);
      // !TRANS: L(bi, bj)[r][k]; TRANS: L(bj, bi)[k][r]
      const double* T = Ls + (size_t)(TRANS ? bj * (bj + 1) / 2 + bi : bi * (bi + 1) / 2 + bj) * TB * TL;
      const double* xa = xs + j0 + cA * m;
      const double* xb = xs + j0 + cB * m;
      int k = 0;
      for (; k + 1 < jb; k += 2) {
        const double l0 = TRANS ? T[k + r * TL] : T[r + k * TL];
        const double l1 = TRANS ? T[k + 1 + r * TL] : T[r + (k + 1) * TL];
        a0 = fma(-l0, xa[k], a0);
        b0 = fma(-l0, xb[k], b0);
        a1 = fma(-l1, xa[k + 1], a1);
        b1 = fma(-l1, xb[k + 1], b1);
      }
      if (k < jb) {
        const double l0 = TRANS ? T[k + r * TL] : T[r + k * TL];
        a0 = fma(-l0, xa[k], a0);
        b0 = fma(-l0, xb[k], b0);
      }
    }
    acc_s[r + cA * TB] = a0 + a1;
    acc_s[r + cB * TB] = b0 + b1;
    __syncthreads();
    if (r < ib) {
      double sA = 0.0, sB = 0.0, tA = 0.0, tB = 0.0;
      int k = 0;
      for (; k + 1 < ib; k += 2) {
        sA = fma(Ds[r + k * TL], acc_s[k + cA * TB], sA);
        sB = fma(Ds[r + k * TL], acc_s[k + cB * TB], sB);
        tA = fma(Ds[r + (k + 1) * TL], acc_s[k + 1 + cA * TB], tA);
        tB = fma(Ds[r + (k + 1) * TL], acc_s[k + 1 + cB * TB], tB);
      }
      if (k < ib) {
        sA = fma(Ds[r + k * TL], acc_s[k + cA * TB], sA);
        sB = fma(Ds[r + k * TL], acc_s[k + cB * TB], sB);
      }
      xs[(i0 + r) + cA * m] = sA + tA;
      xs[(i0 + r) + cB * m] = sB + tB;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < m * XC; idx += nt) {
    const int i = idx % m, c = idx / m;
    if (c < nc) x[i + (int64_t)(c0 + c) * ldx] = xs[idx];
  }
}

template <bool TRANS>
static cudaError_t trsm_tiles(int m, const double* l, const double* dinv, double* x, int ldx, int ncols,
                              cudaStream_t st, bool low_smem) {
  // every lower tile of L resident in shared memory (~200 KB: a whole SM); beyond, or when the
  // solve must share SMs with a concurrent kernel (low_smem), L streamed from L2
  if (m <= RS_MAXB * TB && !low_smem) {
    const size_t rs = sizeof(double) * ((size_t)m * XC + (size_t)(RS_MAXB * (RS_MAXB + 1) / 2 + 1) * TB * TL +
                                        TB * XC);
    static bool rattr = false;
    if (!rattr) {
      cudaFuncSetAttribute(trsm_res_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(trsm_res_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      rattr = true;
    }
    trsm_res_kernel<TRANS><<<(ncols + XC - 1) / XC, 256, rs, st>>>(m, l, dinv, x, ldx, ncols);
    ++g_launches;
    return cudaGetLastError();
  }
  const size_t sm = sizeof(double) * (size_t)m * XC;
  cudaFuncSetAttribute(trsm_tile_kernel<TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  trsm_tile_kernel<TRANS><<<(ncols + XC - 1) / XC, 256, sm, st>>>(m, l, dinv, x, ldx, ncols);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t trsm_lower(int m, const double* l, const double* dinv, double* x, int ldx, int ncols,
                       cudaStream_t st, bool low_smem) {
  return trsm_tiles<false>(m, l, dinv, x, ldx, ncols, st, low_smem);
}
cudaError_t trsm_lower_t(int m, const double* l, const double* dinv, double* x, int ldx, int ncols,
                         cudaStream_t st, bool low_smem) {
  return trsm_tiles<true>(m, l, dinv, x, ldx, ncols, st, low_smem);
}

}  // namespace feastgpu
