// blocktri.cu — block-tridiagonal shifted solves (z_e B - A) X = Y for all contour nodes.
//
// Replaces the reference's BandedLU path for sparse pencils (lu.hpp:104-206 via
// DirectSolver's Auto policy, inner_solver.hpp:79-103) with a block-Thomas recursion:
//   S_0 = M_0,  S_{l+1} = M_{l+1} - C_l S_l^{-1} C_l^T,   C_l = M(l+1, l) = z B_l+1,l - A_l+1,l
//   forward : y_0 = S_0^{-1} Y_0,  y_l = S_l^{-1} (Y_l - C_{l-1} y_{l-1})
//   backward: x_{L-1} = y_{L-1},   x_l = y_l - G_l x_{l+1},   G_l = S_l^{-1} C_l^T
// (zB - A is complex symmetric, so M(l, l+1) = C_l^T.) The factor stage stores the
// explicit block inverses S_l^{-1} and G_l so every sweep step is a pure complex GEMM on
// FP64 DMMA tiles. The quadrature epilogue Re(c_e x) of accumulate_subspace_real
// (core.hpp:174-179) is fused into the backward sweep.
//
// Numerics: the imaginary part of zB - A is Im(z) B (SPD), so every Schur complement S_l
// has a positive-definite imaginary part and is nonsingular; partial pivoting inside each
// S_l handles local growth (Gauss-Jordan below).

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

int64_t g_launches = 0;

// ---------------------------------------------------------------------------
// Factor: one CTA per node walks the L-step chain. v0: any b; [S | I] lives in shared
// memory for b <= 64 and in global scratch otherwise.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bt_factor_kernel(BtFactorArgs a) {
  const int s = blockIdx.x;
  const int L = a.L, b = a.b, tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const double2 z = a.z[s];
  const int ld = b + 1;
  extern __shared__ __align__(16) double2 fsm[];
  double2* f = fsm;                                   // b
  double2* aug = (b <= 64) ? fsm + b : a.scratch + (size_t)s * b * 2 * ld;
  __shared__ int piv_s;
  __shared__ int bad_s;
  const size_t bb = (size_t)b * b;
  double2* sinv = a.sinv + (size_t)s * L * bb;
  double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * bb;
  if (tid == 0) bad_s = 0;

  for (int l = 0; l < L; ++l) {
    // (a) S_l = M_l - C_{l-1} G_{l-1};  right half = I
    const double2* ab = a.abdiag + (size_t)l * bb;
    for (int idx = tid; idx < b * b; idx += nt) {
      const int i = idx % b, j = idx / b;
      const double2 e = ab[idx];
      double2 v = make_double2(z.x * e.y - e.x, z.y * e.y);
      if (l > 0) {
        const double2* cl = a.ablow + (size_t)(l - 1) * bb;
        const double2* gp = gm + (size_t)(l - 1) * bb;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < b; ++k) {
          const double2 ce = cl[i + (size_t)k * b];
          const double2 c = make_double2(z.x * ce.y - ce.x, z.y * ce.y);
          acc = cadd(acc, cmul(c, gp[k + (size_t)j * b]));
        }
        v = csub(v, acc);
      }
      aug[i + (size_t)j * ld] = v;
      aug[i + (size_t)(b + j) * ld] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();

    // (b) Gauss-Jordan with partial pivoting (largest |.|, first index on ties,
    //     the DenseLU / BandedLU rule of lu.hpp:29-38)
    for (int k = 0; k < b; ++k) {
      if (warp == 0) {
        double best = -1.0;
        int bi = b;
        for (int i = k + lane; i < b; i += 32) {
          const double v = cabs_(aug[i + (size_t)k * ld]);
          if (v > best) { best = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) {
          piv_s = bi;
          if (!(best > 0.0)) bad_s = 1;
        }
      }
      __syncthreads();
      if (bad_s) {
        if (tid == 0) atomicExch(a.status, 1);
        return;
      }
      const int p = piv_s;
      if (p != k)
        for (int j = k + tid; j < 2 * b; j += nt) {
          const double2 t0 = aug[k + (size_t)j * ld];
          aug[k + (size_t)j * ld] = aug[p + (size_t)j * ld];
          aug[p + (size_t)j * ld] = t0;
        }
      __syncthreads();
      const double2 pv = aug[k + (size_t)k * ld];
      __syncthreads();
      for (int j = k + 1 + tid; j < 2 * b; j += nt)
        aug[k + (size_t)j * ld] = cdiv(aug[k + (size_t)j * ld], pv);
      for (int i = tid; i < b; i += nt) f[i] = aug[i + (size_t)k * ld];
      __syncthreads();
      const int ncol = 2 * b - k - 1;
      for (int idx = tid; idx < b * ncol; idx += nt) {
        const int i = idx % b, j = k + 1 + idx / b;
        if (i == k) continue;
        aug[i + (size_t)j * ld] = csub(aug[i + (size_t)j * ld], cmul(f[i], aug[k + (size_t)j * ld]));
      }
      __syncthreads();
    }

    // Sinv_l out
    double2* si = sinv + (size_t)l * bb;
    for (int idx = tid; idx < b * b; idx += nt) {
      const int i = idx % b, j = idx / b;
      si[idx] = aug[i + (size_t)(b + j) * ld];
    }
    // (c) G_l = S_l^{-1} C_l^T
    if (l + 1 < L) {
      const double2* cl = a.ablow + (size_t)l * bb;
      double2* gp = gm + (size_t)l * bb;
      for (int idx = tid; idx < b * b; idx += nt) {
        const int i = idx % b, j = idx / b;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < b; ++k) {
          const double2 ce = cl[j + (size_t)k * b];   // C_l(j, k)
          const double2 c = make_double2(z.x * ce.y - ce.x, z.y * ce.y);
          acc = cadd(acc, cmul(aug[i + (size_t)(b + k) * ld], c));
        }
        gp[idx] = acc;
      }
    }
    // (d) H_l = S_l^{-1} C_{l-1}: folds the coupling into one GEMM per forward sweep step
    if (l > 0) {
      const double2* cl = a.ablow + (size_t)(l - 1) * bb;
      double2* hp = a.h + ((size_t)s * (L - 1) + (l - 1)) * bb;
      for (int idx = tid; idx < b * b; idx += nt) {
        const int i = idx % b, j = idx / b;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < b; ++k) {
          const double2 ce = cl[k + (size_t)j * b];   // C_{l-1}(k, j)
          const double2 c = make_double2(z.x * ce.y - ce.x, z.y * ce.y);
          acc = cadd(acc, cmul(aug[i + (size_t)(b + k) * ld], c));
        }
        hp[idx] = acc;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Large blocks (b >= 128): the same recursion, every dense b x b operation batched over the
// nodes and run on the DMMA GEMM / batched-LU kernels (one layer at a time):
//   S_l = M_l - C_{l-1} G_{l-1}  (zgemm) ;  S_l^{-1} by block Gauss-Jordan in place (below;
//   FEAST_BT_FACTOR=lu selects pivoted LU + solve against I instead) ;
//   H_l = S_l^{-1} C_{l-1} ;  G_l = S_l^{-1} C_l^T  (zgemm) ; all three packed into panels
// ---------------------------------------------------------------------------
cudaError_t zgemm_batched(int m, int n, int k, double2 alpha, const double2* a, int lda, int64_t sa,
                          const double2* b, int ldb, int64_t sb, double2 beta, double2* c, int ldc,
                          int64_t sc, int batch, cudaStream_t st);
cudaError_t zgetrf_batched(int n, int nodes, double2* lu, int64_t stride, int* ipiv, int* perm, double2* dinv,
                           int* status, cudaStream_t st);
cudaError_t zgetrs_batched(int n, int nodes, int m, const double2* lu, int64_t stride, const int* perm,
                           const double2* dinv, double2* w, int ldv, double2* scratch, cudaStream_t st);

// out_s = z_s * B - A for a block of (A, B) pairs (optionally transposed), or the identity
__global__ void bt_make_kernel(int b, const double2* __restrict__ ab, const double2* __restrict__ z,
                               double2* __restrict__ out, int mode) {
  const int s = blockIdx.y;
  const double2 zz = z[s];
  double2* o = out + (size_t)s * b * b;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < b * b; idx += gridDim.x * blockDim.x) {
    const int i = idx % b, j = idx / b;
    if (mode == 2) {
      o[idx] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    } else {
      const double2 e = ab[mode == 1 ? j + i * b : idx];
      o[idx] = make_double2(zz.x * e.y - e.x, zz.y * e.y);
    }
  }
}

// col-major b x b (blockIdx.y = node, node stride b*b) -> panel layout (kernels.h)
__global__ void pack_panels_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int64_t dstride,
                                   int b, int rb) {
  const int64_t bb = (int64_t)b * b;
  src += blockIdx.y * bb;
  dst += blockIdx.y * dstride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / b), i = (int)(e - (int64_t)k * b);
    const int p = i / rb, r = i - p * rb;
    dst[(int64_t)p * b * rb + (int64_t)k * rb + (r ^ (2 * (k & 3)))] = src[e];
  }
}

// ---------------------------------------------------------------------------
// In-place inversion of S_l by block Gauss-Jordan (block width GJ_NB, batched over nodes).
// Im(S_l) = Im(z) x (SPD) is positive definite, so elimination without pivoting across
// blocks is stable (growth factor < 3 for complex symmetric matrices with a definite real or
// imaginary part, Higham, Accuracy and Stability, 2nd ed., §10.4); inside a diagonal block
// the same argument holds, so the diagonal-block inverse runs pivot-free with ONE barrier per
// column: every thread keeps its 16 entries of [D | I] in registers and the next pivot row and
// column are published into double-buffered shared staging by their owners.
// Per block column k (rows/cols kb = [k0, k0 + NB)):
//   D = S_kk^{-1};  P = S[:, kb];  R = D S[kb, :] (R[:, kb] := D + I)
//   S -= P R   (rows outside kb get the Gauss-Jordan update; S[:, kb] becomes -P D)
//   S[kb, :] = R with S[kb, kb] = D
// ---------------------------------------------------------------------------
constexpr int GJ_NB = 64;

__global__ void __launch_bounds__(512) gj_diag_kernel(double2* __restrict__ S, int n, int64_t sstride, int k0,
                                                      double2* __restrict__ D, double2* __restrict__ P,
                                                      double2* __restrict__ R, int* status) {
  constexpr int NB = GJ_NB, NQ = 2 * NB / 8;  // thread: row i, columns (t & 7) + 8q of [A | I]
  __shared__ double2 rowst[2][2 * NB];
  __shared__ double2 colst[2][NB];
  __shared__ int bad;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int i = tid >> 3, c8 = tid & 7;
  double2* Sn = S + s * sstride;
  double2* Dn = D + (int64_t)s * NB * NB;
  double2* Pn = P + (int64_t)s * n * NB;
  double2* Rn = R + (int64_t)s * NB * n;
  // panel copy P = S[:, kb] (n x NB, ld n)
  for (int e = tid; e < n * NB; e += 512) {
    const int r = e % n, c = e / n;
    Pn[e] = Sn[r + (int64_t)(k0 + c) * n];
  }
  double2 v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = c8 + 8 * q;
    v[q] = j < NB ? Sn[(k0 + i) + (int64_t)(k0 + j) * n] : make_double2(j - NB == i ? 1.0 : 0.0, 0.0);
  }
  if (tid == 0) bad = 0;
  // publish pivot row/column 0
  if (i == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) rowst[0][c8 + 8 * q] = v[q];
  }
  if (c8 == 0) colst[0][i] = v[0];
  for (int k = 0; k < NB; ++k) {
    __syncthreads();
    const double2* rs = rowst[k & 1];
    const double2 piv = colst[k & 1][k];
    if (!(cabs_(piv) > 0.0) || !isfinite(piv.x) || !isfinite(piv.y)) {
      if (tid == 0) {
        bad = 1;
        atomicExch(status, 1);
      }
    }
    const double2 g = cdiv(colst[k & 1][i], piv);
    const double2 rp = cdiv(make_double2(1.0, 0.0), piv);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = c8 + 8 * q;
      const bool active = (j < NB) ? (j >= k) : (j - NB <= k);
      if (active) {
        if (i == k) v[q] = cmul(v[q], rp);
        else v[q] = csub(v[q], cmul(g, rs[j]));
      }
    }
    if (k + 1 < NB) {
      if (i == k + 1) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) rowst[(k + 1) & 1][c8 + 8 * q] = v[q];
      }
#pragma unroll
      for (int q = 0; q < NQ / 2; ++q)
        if (c8 + 8 * q == k + 1) colst[(k + 1) & 1][i] = v[q];
    }
  }
  __syncthreads();
  if (bad) return;
  // D = right half; R[:, kb] = D + I
#pragma unroll
  for (int q = NQ / 2; q < NQ; ++q) {
    const int j = c8 + 8 * q - NB;
    Dn[i + j * NB] = v[q];
    Rn[i + (int64_t)(k0 + j) * NB] = make_double2(v[q].x + (i == j ? 1.0 : 0.0), v[q].y);
  }
}

// S[kb, :] = R, except S[kb, kb] = D
__global__ void gj_rowput_kernel(double2* __restrict__ S, int n, int64_t sstride, int k0,
                                 const double2* __restrict__ D, const double2* __restrict__ R) {
  constexpr int NB = GJ_NB;
  const int s = blockIdx.y;
  double2* Sn = S + s * sstride;
  const double2* Dn = D + (int64_t)s * NB * NB;
  const double2* Rn = R + (int64_t)s * NB * n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < NB * n; e += gridDim.x * blockDim.x) {
    const int r = e % NB, j = e / NB;
    const bool diag = j >= k0 && j < k0 + NB;
    Sn[(k0 + r) + (int64_t)j * n] = diag ? Dn[r + (j - k0) * NB] : Rn[e];
  }
}

// S_s <- S_s^{-1} for the batch (n % GJ_NB == 0); work: nodes * (2 n NB + NB^2) double2
static cudaError_t gj_invert_batched(double2* S, int n, int64_t sstride, int nodes, double2* work, int* status,
                                     cudaStream_t st) {
  constexpr int NB = GJ_NB;
  double2* P = work;
  double2* R = P + (int64_t)nodes * n * NB;
  double2* D = R + (int64_t)nodes * NB * n;
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0), zero = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < n; k0 += NB) {
    gj_diag_kernel<<<nodes, 512, 0, st>>>(S, n, sstride, k0, D, P, R, status);
    ++g_launches;
    // R[:, j] = D S[kb, j] for j outside kb (two column ranges)
    if (k0 > 0) zgemm_batched(NB, k0, NB, one, D, NB, NB * NB, S + k0, n, sstride, zero, R, NB, (int64_t)NB * n, nodes, st);
    if (k0 + NB < n)
      zgemm_batched(NB, n - k0 - NB, NB, one, D, NB, NB * NB, S + k0 + (int64_t)(k0 + NB) * n, n, sstride, zero,
                    R + (int64_t)(k0 + NB) * NB, NB, (int64_t)NB * n, nodes, st);
    zgemm_batched(n, n, NB, mone, P, n, (int64_t)n * NB, R, NB, (int64_t)NB * n, one, S, n, sstride, nodes, st);
    dim3 g((unsigned)std::min(((int64_t)NB * n + 255) / 256, (int64_t)256), nodes);
    gj_rowput_kernel<<<g, 256, 0, st>>>(S, n, sstride, k0, D, R);
    ++g_launches;
  }
  return cudaGetLastError();
}

static bool factor_use_lu() {
  static const bool lu = [] {
    const char* e = getenv("FEAST_BT_FACTOR");
    return e && e[0] == 'l';
  }();
  return lu;
}

static cudaError_t bt_factor_big(const BtFactorArgs& a, cudaStream_t st) {
  const bool lu = factor_use_lu();  // FEAST_BT_FACTOR=lu: pivoted LU + solve (comparison path)
  const int L = a.L, b = a.b, nodes = a.nodes;
  const int64_t bb = (int64_t)b * b, lnode = (int64_t)L * bb, gnode = (int64_t)(L > 1 ? L - 1 : 0) * bb;
  double2* S = a.work;                 // LU of S_l            (nodes x bb)
  double2* Cp = S + nodes * bb;        // C_{l-1}, then C_l
  double2* CT = Cp + nodes * bb;       // C_l^T
  double2* X = CT + nodes * bb;        // S_l^{-1}
  double2* scr = X + nodes * bb;       // zgetrs scratch
  double2* dinv = scr + nodes * bb;    // diagonal-block inverses
  double2* gjw = dinv + (int64_t)nodes * ((b + kDenseNb - 1) / kDenseNb) * 2 * kDenseNb * kDenseNb;  // GJ work
  int* ipiv = a.iwork;
  int* perm = ipiv + nodes * b;
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0), zero = make_double2(0.0, 0.0);
  dim3 g((unsigned)std::min<int64_t>((bb + 255) / 256, 512), nodes);
  // factors leave in the sweep's panel layout; G_l also stays col-major in scr until the
  // next layer's Schur update has used it (zgetrs reuses scr only after that)
  const int rb = bt_panel_rows(b);
  auto pack = [&](const double2* src, double2* dst, int64_t dstride) {
    pack_panels_kernel<<<g, 256, 0, st>>>(src, dst, dstride, b, rb);
    ++g_launches;
  };
  for (int l = 0; l < L; ++l) {
    bt_make_kernel<<<g, 256, 0, st>>>(b, a.abdiag + l * bb, a.z, S, 0);
    ++g_launches;
    if (l > 0) zgemm_batched(b, b, b, mone, Cp, b, bb, scr, b, bb, one, S, b, bb, nodes, st);
    if (lu) {  // FEAST_BT_FACTOR=lu
      zgetrf_batched(b, nodes, S, bb, ipiv, perm, dinv, a.status, st);
      bt_make_kernel<<<g, 256, 0, st>>>(b, nullptr, a.z, X, 2);
      ++g_launches;
      zgetrs_batched(b, nodes, b, S, bb, perm, dinv, X, b, scr, st);
    }
    if (!lu) {
      // S^{-1} by pivot-free block Gauss-Jordan, then one Newton-Schulz refinement step
      // X' = X + X (I - S X): the near-real-axis nodes lose ~1 digit without pivoting, and
      // the refinement squares that residual (two DMMA GEMMs per layer)
      cudaMemcpyAsync(X, S, sizeof(double2) * nodes * bb, cudaMemcpyDeviceToDevice, st);  // keep S
      gj_invert_batched(S, b, bb, nodes, gjw, a.status, st);  // S <- S^{-1} in place
      bt_make_kernel<<<g, 256, 0, st>>>(b, nullptr, a.z, scr, 2);  // scr = I
      ++g_launches;
      zgemm_batched(b, b, b, mone, X, b, bb, S, b, bb, one, scr, b, bb, nodes, st);  // R = I - S X
      cudaMemcpyAsync(X, S, sizeof(double2) * nodes * bb, cudaMemcpyDeviceToDevice, st);
      zgemm_batched(b, b, b, one, S, b, bb, scr, b, bb, one, X, b, bb, nodes, st);  // X + X R
    }
    const double2* Xi = X;  // S_l^{-1}
    pack(Xi, a.sinv + l * bb, lnode);  // S_l^{-1} (node stride L*bb)
    if (l > 0) {  // H_l = S_l^{-1} C_{l-1}, via CT (C_{l-1}^T is spent)
      zgemm_batched(b, b, b, one, Xi, b, bb, Cp, b, bb, zero, CT, b, bb, nodes, st);
      pack(CT, a.h + (l - 1) * bb, gnode);
    }
    if (l + 1 < L) {
      bt_make_kernel<<<g, 256, 0, st>>>(b, a.ablow + l * bb, a.z, Cp, 0);
      bt_make_kernel<<<g, 256, 0, st>>>(b, a.ablow + l * bb, a.z, CT, 1);
      g_launches += 2;
      zgemm_batched(b, b, b, one, Xi, b, bb, CT, b, bb, zero, scr, b, bb, nodes, st);
      pack(scr, a.g + l * bb, gnode);
    }
  }
  return cudaGetLastError();
}

size_t bt_factor_work_elems(int b, int nodes) {  // double2 elements of BtFactorArgs::work
  const int nblk = (b + kDenseNb - 1) / kDenseNb;
  return (size_t)nodes * (5 * (size_t)b * b + (size_t)nblk * 2 * kDenseNb * kDenseNb + 2 * (size_t)b * GJ_NB +
                          (size_t)GJ_NB * GJ_NB);
}

cudaError_t bt_factor(const BtFactorArgs& a, cudaStream_t st) {
  if (a.b >= 128) return bt_factor_big(a, st);
  size_t sm = sizeof(double2) * (size_t)a.b;
  if (a.b <= 64) sm += sizeof(double2) * (size_t)a.b * 2 * (a.b + 1);
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(bt_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  bt_factor_kernel<<<a.nodes, 256, sm, st>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Q = -sum_s T_s, ascending s from zero (the ordered reduction of core.hpp:181-183)
// ---------------------------------------------------------------------------
__global__ void reduce_terms_kernel(const double* __restrict__ t, int nodes, int64_t slice, int n,
                                    int m, int ld, double* __restrict__ q, int accumulate) {
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const int64_t off = i + j * ld;
    double acc = accumulate ? q[off] : 0.0;  // node batches continue the same ascending sum
    for (int s = 0; s < nodes; ++s) acc -= t[s * slice + off];
    q[off] = acc;
  }
}

cudaError_t reduce_terms(const double* t, int nodes, int64_t slice, int n, int m, int ld, double* q,
                         cudaStream_t st, int accumulate) {
  const int64_t total = (int64_t)n * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  reduce_terms_kernel<<<blocks, 256, 0, st>>>(t, nodes, slice, n, m, ld, q, accumulate);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
