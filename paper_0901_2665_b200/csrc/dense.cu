// dense.cu — batched complex-fp64 LU with partial pivoting and the multi-RHS solve for
// dense pencils (the reference's DenseShiftSystem: assemble_shifted_dense assemble.hpp:12-38,
// DenseLU ctor lu.hpp:24-52, DenseLU::solve_in_place lu.hpp:56-95), all contour nodes of
// this rank batched into every launch (blockIdx.z / blockIdx.x = node slot).
//
// Factor (right-looking, panel width nb = 64, LAPACK getrf structure):
//   panel_kernel    unblocked partial-pivot LU of the n-k0 x nb panel (pivot rule of
//                   lu.hpp:29-38: largest |.|, first index on ties; NumericalError on 0)
//   laswp_kernel    the panel's row interchanges applied to the other columns
//   diag_inv_kernel explicit inverses of the unit-lower L11 and upper U11 blocks
//   zgemm           U12 = L11^{-1} A12 (in place) and A22 -= L21 U12  (DMMA tiles)
// Solve (per pass, multi-RHS, blocked forward/backward substitution):
//   R = P Y; for k: Z_k = L_kk^{-1} R_k; R_{>k} -= L_{>k,k} Z_k;
//            for k desc: X_k = U_kk^{-1} R_k; R_{<k} -= U_{<k,k} X_k;  T = Re(c_e X)

#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

cudaError_t zgemm_batched(int m, int n, int k, double2 alpha, const double2* a, int lda, int64_t sa,
                          const double2* b, int ldb, int64_t sb, double2 beta, double2* c, int ldc,
                          int64_t sc, int batch, cudaStream_t st);

__global__ void assemble_kernel(int n, const double* __restrict__ a, const double* __restrict__ bm,
                                const double2* __restrict__ z, double2* __restrict__ lu) {
  const int s = blockIdx.y;
  const double2 zz = z[s];
  const int64_t nn = (int64_t)n * n;
  double2* out = lu + s * nn;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double bv = bm[idx], av = a[idx];
    out[idx] = make_double2(zz.x * bv - av, zz.y * bv);  // z*B - A (assemble.hpp:33-43)
  }
}

// One CTA per node. Columns [k0, k0+kb), rows [k0, n).
__global__ void __launch_bounds__(1024) panel_kernel(int n, int64_t stride, int k0, int kb, double2* lu,
                                                     int* ipiv, int* status) {
  const int s = blockIdx.x;
  double2* A = lu + (int64_t)s * stride;
  int* piv = ipiv + (int64_t)s * n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int p_s;
  __shared__ double2 rowk[kDenseNb];
  for (int j = 0; j < kb; ++j) {
    const int col = k0 + j;
    double best = -1.0;
    int bi = n;
    for (int i = col + tid; i < n; i += nt) {
      const double v = cabs_(A[i + (int64_t)col * n]);
      if (v > best) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { rv[warp] = best; ri[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < (nt >> 5) ? rv[lane] : -1.0;
      bi = lane < (nt >> 5) ? ri[lane] : n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        p_s = (best > 0.0) ? bi : -1;
        if (!(best > 0.0)) atomicExch(status, 1);
      }
    }
    __syncthreads();
    const int p = p_s;
    if (p < 0) return;  // singular: DenseLU throws NumericalError (lu.hpp:38)
    if (tid == 0) piv[col] = p;
    if (p != col && tid < kb) {
      const int c = k0 + tid;
      const double2 t0 = A[col + (int64_t)c * n];
      A[col + (int64_t)c * n] = A[p + (int64_t)c * n];
      A[p + (int64_t)c * n] = t0;
    }
    __syncthreads();
    const double2 pv = A[col + (int64_t)col * n];
    if (tid < kb) rowk[tid] = A[col + (int64_t)(k0 + tid) * n];
    for (int i = col + 1 + tid; i < n; i += nt) A[i + (int64_t)col * n] = cdiv(A[i + (int64_t)col * n], pv);
    __syncthreads();
    for (int i = col + 1 + tid; i < n; i += nt) {
      const double2 l = A[i + (int64_t)col * n];
      for (int c = j + 1; c < kb; ++c) {
        double2* e = A + i + (int64_t)(k0 + c) * n;
        *e = csub(*e, cmul(l, rowk[c]));
      }
    }
    __syncthreads();
  }
}

// The same unblocked panel on a cluster of kPanelCluster CTAs per node: the panel of a large
// matrix (8192 x 64 complex = 8 MB) streams through L2 once per column step, which one SM's load
// path sustains at ~100 GB/s (6 ms per panel at n = 8192, longer than the whole trailing update
// beside it). Rows are dealt to the cluster in chunks of 1024 (row r belongs to CTA (r / 1024) % CL,
// so a 128-byte line of a column has one owner); per column step
//   (1) every CTA finds its pivot candidate and posts it to all CTAs of the cluster (DSMEM);
//       cluster barrier; every CTA picks the same winner (largest modulus, lowest row on ties);
//   (2) every CTA reads the old pivot row and the old row `col` of the panel (L2 loads: another
//       SM may hold a stale L1 line of a neighbouring former pivot row); cluster barrier;
//   (3) the owners of rows col and p write the exchanged rows, then every thread scales and
//       updates its own rows.
// Same pivots and the same arithmetic per element as panel_kernel: bit-identical factors.
constexpr int kPanelCluster = 8;
__global__ void __cluster_dims__(kPanelCluster, 1, 1) __launch_bounds__(1024)
    panel_cluster_kernel(int n, int64_t stride, int k0, int kb, double2* lu, int* ipiv, int* status) {
  constexpr int CL = kPanelCluster;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int s = blockIdx.x / CL;
  double2* A = lu + (int64_t)s * stride;
  int* piv = ipiv + (int64_t)s * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ double cand_v[2][CL];   // candidates of all CTAs, double-buffered by column parity
  __shared__ int cand_i[2][CL];
  __shared__ double2 rowk[kDenseNb], rowc[kDenseNb];
  auto owner = [&](int r) { return (r >> 10) % CL; };
  for (int j = 0; j < kb; ++j) {
    const int col = k0 + j;
    double best = -1.0;
    int bi = n;
    // my rows: chunks rank, rank + CL, ... of 1024 rows; start at the first row >= col
    for (int base = (rank << 10); base < n; base += CL << 10) {
      const int i = base + tid;
      if (i >= col && i < n) {
        const double v = cabs_(A[i + (int64_t)col * n]);
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { rv[warp] = best; ri[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = rv[lane];
      bi = ri[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane < CL) {  // post to CTA `lane`
        *cluster.map_shared_rank(&cand_v[j & 1][rank], lane) = best;
        *cluster.map_shared_rank(&cand_i[j & 1][rank], lane) = bi;
      }
    }
    cluster.sync();  // (1)
    best = -1.0;
    bi = n;
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      const double ov = cand_v[j & 1][r];
      const int oi = cand_i[j & 1][r];
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int p = (best > 0.0) ? bi : -1;
    if (p < 0) {  // singular: DenseLU throws NumericalError (lu.hpp:38); uniform over the cluster
      if (rank == 0 && tid == 0) atomicExch(status, 1);
      return;
    }
    if (rank == 0 && tid == 0) piv[col] = p;
    if (tid < kb) {
      rowk[tid] = __ldcg(A + p + (int64_t)(k0 + tid) * n);
      rowc[tid] = __ldcg(A + col + (int64_t)(k0 + tid) * n);
    }
    cluster.sync();  // (2) every CTA holds the old rows before their owners overwrite them
    if (p != col && tid < kb) {
      if (owner(col) == rank) A[col + (int64_t)(k0 + tid) * n] = rowk[tid];
      if (owner(p) == rank) A[p + (int64_t)(k0 + tid) * n] = rowc[tid];
    }
    __syncthreads();
    const double2 pv = rowk[j];
    for (int base = (rank << 10); base < n; base += CL << 10) {
      const int i = base + tid;
      if (i > col && i < n) {
        const double2 l = cdiv(A[i + (int64_t)col * n], pv);
        A[i + (int64_t)col * n] = l;
        for (int c = j + 1; c < kb; ++c) {
          double2* e = A + i + (int64_t)(k0 + c) * n;
          *e = csub(*e, cmul(l, rowk[c]));
        }
      }
    }
    __syncthreads();
  }
}

// row interchanges ipiv[r0 .. r0+nr) applied to columns [c0, c0+nc)
__global__ void laswp_kernel(int n, int64_t stride, int r0, int nr, int c0, int nc, double2* lu, const int* ipiv) {
  const int s = blockIdx.y;
  double2* A = lu + (int64_t)s * stride;
  const int* piv = ipiv + (int64_t)s * n;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    double2* col = A + (int64_t)(c0 + c) * n;
    for (int r = r0; r < r0 + nr; ++r) {
      const int p = piv[r];
      if (p != r) {
        const double2 t0 = col[r];
        col[r] = col[p];
        col[p] = t0;
      }
    }
  }
}

// inverses of the diagonal block k: dinv[s][blk][0] = L11^{-1} (unit lower), [1] = U11^{-1}
__global__ void __launch_bounds__(128) diag_inv_kernel(int n, int64_t stride, int blk, int nblk,
                                                       const double2* lu, double2* dinv) {
  constexpr int NB = kDenseNb;
  const int s = blockIdx.x;
  const int k0 = blk * NB, kb = min(NB, n - k0);
  const double2* A = lu + (int64_t)s * stride + k0 + (int64_t)k0 * n;
  double2* Li = dinv + ((int64_t)s * nblk + blk) * 2 * NB * NB;
  double2* Ui = Li + NB * NB;
  extern __shared__ double2 T[];  // NB x (NB+1)
  for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
    const int i = idx % kb, j = idx / kb;
    T[i + j * (NB + 1)] = A[i + (int64_t)j * n];
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < kb) {
    // column j of L^{-1}: x_j = 1, x_i = -sum_{k=j}^{i-1} L_ik x_k
    double2 x[NB];
    for (int i = 0; i < kb; ++i) x[i] = make_double2(0.0, 0.0);
    x[j] = make_double2(1.0, 0.0);
    for (int i = j + 1; i < kb; ++i) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = j; k < i; ++k) acc = cadd(acc, cmul(T[i + k * (NB + 1)], x[k]));
      x[i] = make_double2(-acc.x, -acc.y);
    }
    for (int i = 0; i < kb; ++i) Li[i + j * NB] = x[i];
    // column j of U^{-1}: x_j = 1/U_jj, x_i = -(sum_{k=i+1}^{j} U_ik x_k) / U_ii
    for (int i = 0; i < kb; ++i) x[i] = make_double2(0.0, 0.0);
    x[j] = cdiv(make_double2(1.0, 0.0), T[j + j * (NB + 1)]);
    for (int i = j - 1; i >= 0; --i) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = i + 1; k <= j; ++k) acc = cadd(acc, cmul(T[i + k * (NB + 1)], x[k]));
      x[i] = cdiv(make_double2(-acc.x, -acc.y), T[i + i * (NB + 1)]);
    }
    for (int i = 0; i < kb; ++i) Ui[i + j * NB] = x[i];
  }
}

__global__ void perm_kernel(int n, int nodes, const int* ipiv, int* perm) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nodes) return;
  int* pm = perm + (int64_t)s * n;
  const int* pv = ipiv + (int64_t)s * n;
  for (int i = 0; i < n; ++i) pm[i] = i;
  for (int k = 0; k < n; ++k) {
    const int p = pv[k];
    if (p != k) { const int t = pm[k]; pm[k] = pm[p]; pm[p] = t; }
  }
}

// Batched right-looking LU with partial pivoting of `nodes` complex n x n matrices stored
// `stride` apart (in place), plus the row permutation and the diagonal-block inverses the
// blocked solves use. Shared by the dense path and the SPIKE reduced systems.
//
// Two levels for n >= 2048: super-panels of W = 256 columns are factored with 64-column panels
// whose updates stay inside the super-panel; the columns to its right get the super-panel's row
// interchanges, U12 = L_SS^{-1} A12 block by block, and ONE trailing update with K = 256. (A K = 64
// trailing update moves 32 bytes of C per 512 flops, 16 flop/B against the 5.7 flop/B ridge with
// nothing left for A and B; ncu had it at 0.58 of the DMMA peak, the K = 256 GEMM runs at 0.70.)
//
// Look-ahead (la != nullptr): the unblocked panels run on one CTA (or one cluster) per node, so on
// the main stream they left most SMs idle for about as long as the trailing updates take. The
// columns of the next super-panel are therefore updated first, and the next super-panel is
// factored on the high-priority side stream beside the update of the remaining columns; only its
// row interchanges on the other columns wait for both.
cudaError_t zgetrf_batched(int n, int nodes, double2* lu, int64_t stride, int* ipiv, int* perm, double2* dinv,
                           int* status, cudaStream_t st, const LuLookahead* la) {
  const int nb = kDenseNb;
  const int nblk = (n + nb - 1) / nb;
  const int W = n >= 2048 ? 256 : nb;
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0),
                zero = make_double2(0.0, 0.0);
  const int64_t sd = (int64_t)nblk * 2 * nb * nb;
  {
    const int sm = (int)sizeof(double2) * nb * (nb + 1);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(diag_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      attr = true;
    }
  }
  auto gemm = [&](int m_, int n_, int k_, double2 alpha, const double2* a_, const double2* b_, double2 beta,
                  double2* c_, cudaStream_t s) {
    if (m_ > 0 && n_ > 0 && k_ > 0) zgemm_batched(m_, n_, k_, alpha, a_, n, stride, b_, n, stride, beta, c_, n, stride, nodes, s);
  };
  auto at = [&](int r, int c) { return lu + r + (int64_t)c * n; };
  auto linv = [&](int k0) { return dinv + (int64_t)(k0 / nb) * 2 * nb * nb; };
  auto laswp = [&](int r0, int r1, int c0, int c1, cudaStream_t s) {
    if (c1 - c0 <= 0 || r1 - r0 <= 0) return;
    dim3 grid((c1 - c0 + 255) / 256, nodes);
    laswp_kernel<<<grid, 256, 0, s>>>(n, stride, r0, r1 - r0, c0, c1 - c0, lu, ipiv);
    ++g_launches;
  };
  // columns [K0, K1) from row K0 down: panels of nb columns, interchanges and updates inside [K0, K1)
  auto factor_super = [&](int K0, int K1, cudaStream_t s) {
    for (int k0 = K0; k0 < K1; k0 += nb) {
      const int kb = std::min(nb, K1 - k0), k1 = k0 + kb;
      // tall panels: a cluster of CTAs per node (the rows of one CTA would stream through one SM)
      if (n - k0 >= 4096) panel_cluster_kernel<<<nodes * kPanelCluster, 1024, 0, s>>>(n, stride, k0, kb, lu, ipiv, status);
      else panel_kernel<<<nodes, 1024, 0, s>>>(n, stride, k0, kb, lu, ipiv, status);
      diag_inv_kernel<<<nodes, 128, (int)sizeof(double2) * nb * (nb + 1), s>>>(n, stride, k0 / nb, nblk, lu, dinv);
      g_launches += 2;
      laswp(k0, k1, K0, k0, s);
      laswp(k0, k1, k1, K1, s);
      // U12 = L11^{-1} A12 (in place), A22 -= L21 U12 on the super-panel's remaining columns
      if (K1 - k1 > 0)
        zgemm_batched(kb, K1 - k1, kb, one, linv(k0), nb, sd, at(k0, k1), n, stride, zero, at(k0, k1), n, stride,
                      nodes, s);
      gemm(n - k1, K1 - k1, kb, mone, at(k1, k0), at(k0, k1), one, at(k1, k1), s);
    }
  };
  // columns [c0, c0 + nc) right of the factored super-panel [K0, K1): U12 block by block, then the
  // trailing rows with K = K1 - K0
  auto outer = [&](int K0, int K1, int c0, int nc, cudaStream_t s) {
    if (nc <= 0) return;
    for (int k0 = K0; k0 < K1; k0 += nb) {
      const int kb = std::min(nb, K1 - k0), k1 = k0 + kb;
      zgemm_batched(kb, nc, kb, one, linv(k0), nb, sd, at(k0, c0), n, stride, zero, at(k0, c0), n, stride, nodes, s);
      gemm(K1 - k1, nc, kb, mone, at(k1, k0), at(k0, c0), one, at(k1, c0), s);
    }
    gemm(n - K1, nc, K1 - K0, mone, at(K1, K0), at(K0, c0), one, at(K1, c0), s);
  };
  const bool ahead = la && la->side && n > W;
  factor_super(0, std::min(W, n), st);
  for (int K0 = 0; K0 < n; K0 += W) {
    const int K1 = std::min(K0 + W, n);
    laswp(K0, K1, 0, K0, st);
    laswp(K0, K1, K1, n, st);
    if (K1 >= n) break;
    const int K2 = std::min(K1 + W, n);
    outer(K0, K1, K1, K2 - K1, st);
    if (ahead) {
      cudaEventRecord(la->ev_cols, st);
      cudaStreamWaitEvent(la->side, la->ev_cols, 0);
      factor_super(K1, K2, la->side);
      cudaEventRecord(la->ev_panel, la->side);
      outer(K0, K1, K2, n - K2, st);
      cudaStreamWaitEvent(st, la->ev_panel, 0);
    } else {
      outer(K0, K1, K2, n - K2, st);
      factor_super(K1, K2, st);
    }
  }
  perm_kernel<<<(nodes + 31) / 32, 32, 0, st>>>(n, nodes, ipiv, perm);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t dense_factor(const DenseFactorArgs& a, cudaStream_t st) {
  const int n = a.n, nodes = a.nodes;
  const int64_t nn = (int64_t)n * n;
  dim3 grid((unsigned)std::min<int64_t>((nn + 255) / 256, 1024), nodes);
  assemble_kernel<<<grid, 256, 0, st>>>(n, a.a, a.bm, a.z, a.lu);
  ++g_launches;
  return zgetrf_batched(n, nodes, a.lu, nn, a.ipiv, a.perm, a.dinv, a.status, st, a.la.side ? &a.la : nullptr);
}

// R_s = P_s Y (real -> complex), or P_s W_s (complex, via scratch copy in t-as-double2)
__global__ void permute_rhs_kernel(int n, int m, int ldv, const int* perm, const double* y,
                                   const double2* src, double2* w) {
  const int s = blockIdx.y;
  const int* pm = perm + (int64_t)s * n;
  double2* W = w + (int64_t)s * ldv * m;
  const double2* S = src ? src + (int64_t)s * ldv * m : nullptr;
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n);
    const int64_t j = idx / n;
    const int pi = pm[i];
    W[i + j * ldv] = S ? S[pi + j * ldv] : make_double2(y[pi + j * ldv], 0.0);
  }
}

__global__ void term_kernel(int n, int m, int ldv, const double2* coeff, const double2* w, double* t) {
  const int s = blockIdx.y;
  const double2 c = coeff[s];
  const double2* W = w + (int64_t)s * ldv * m;
  double* T = t + (int64_t)s * ldv * m;
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n);
    const int64_t j = idx / n;
    const double2 x = W[i + j * ldv];
    T[i + j * ldv] = c.x * x.x - c.y * x.y;  // Re(coeff * x) (core.hpp:179)
  }
}

// blocked forward/backward substitution on the factors of zgetrf_batched, in place on the
// (already row-permuted) right-hand sides W (n x m per node, ld ldv, batch stride sv).
// Two levels: inside an outer block of kSolveNbo rows the 64-row blocks are solved with their
// diagonal-block inverses and update only the rest of the outer block; the rows below (above, for
// U) get ONE update per outer block with K = kSolveNbo. With K = 64 every trailing update was a
// short-K GEMM that spent most of each CTA in pipeline fill and the C read-modify-write
// (ncu: DMMA pipe 58 %, long-scoreboard stalls on the epilogue loads); K = 256 amortises both
// (config 4 solve 141 -> 99 ms per pass). The same two-level scheme in zgetrf_batched measured
// slower (1.11 -> 1.53 s at config 4: the panel-restricted inner updates and the outer U12 rows
// cost more than the K = 256 trailing update saves), so the factorisation keeps one level.
constexpr int kSolveNbo = 256;
static void zgetrs_core(int n, int nodes, int m, const double2* lu, int64_t stride, const double2* dinv,
                        double2* w, int ldv, int64_t sv, cudaStream_t st) {
  const int nb = kDenseNb, nblk = (n + nb - 1) / nb;
  const int64_t sd = (int64_t)nblk * 2 * nb * nb;
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0),
                zero = make_double2(0.0, 0.0);
  const int nbo = n >= 2048 ? kSolveNbo : nb;  // (small n: the extra outer step only adds latency)
  for (int K0 = 0; K0 < n; K0 += nbo) {  // L: forward
    const int K1 = std::min(K0 + nbo, n);
    for (int blk = K0 / nb; blk * nb < K1; ++blk) {
      const int k0 = blk * nb, kb = std::min(nb, n - k0);
      double2* rk = w + k0;
      zgemm_batched(kb, m, kb, one, dinv + (int64_t)blk * 2 * nb * nb, nb, sd, rk, ldv, sv, zero, rk, ldv, sv,
                    nodes, st);
      const int rest = K1 - k0 - kb;
      if (rest > 0)
        zgemm_batched(rest, m, kb, mone, lu + (k0 + kb) + (int64_t)k0 * n, n, stride, rk, ldv, sv, one,
                      w + k0 + kb, ldv, sv, nodes, st);
    }
    if (n - K1 > 0)
      zgemm_batched(n - K1, m, K1 - K0, mone, lu + K1 + (int64_t)K0 * n, n, stride, w + K0, ldv, sv, one, w + K1,
                    ldv, sv, nodes, st);
  }
  for (int K1 = n; K1 > 0;) {  // U: backward
    const int K0 = ((K1 - 1) / nbo) * nbo;
    for (int blk = (K1 - 1) / nb; blk * nb >= K0 && blk >= 0; --blk) {
      const int k0 = blk * nb, kb = std::min(nb, n - k0);
      double2* rk = w + k0;
      zgemm_batched(kb, m, kb, one, dinv + (int64_t)blk * 2 * nb * nb + nb * nb, nb, sd, rk, ldv, sv, zero, rk,
                    ldv, sv, nodes, st);
      if (k0 > K0)
        zgemm_batched(k0 - K0, m, kb, mone, lu + K0 + (int64_t)k0 * n, n, stride, rk, ldv, sv, one, w + K0, ldv, sv,
                      nodes, st);
    }
    if (K0 > 0)
      zgemm_batched(K0, m, K1 - K0, mone, lu + (int64_t)K0 * n, n, stride, w + K0, ldv, sv, one, w, ldv, sv, nodes,
                    st);
    K1 = K0;
  }
}

// W <- A^{-1} W for complex right-hand sides (scratch: nodes * ldv * m double2)
cudaError_t zgetrs_batched(int n, int nodes, int m, const double2* lu, int64_t stride, const int* perm,
                           const double2* dinv, double2* w, int ldv, double2* scratch, cudaStream_t st) {
  const int64_t sv = (int64_t)ldv * m, total = (int64_t)n * m;
  dim3 g1((unsigned)std::min<int64_t>((total + 255) / 256, 1024), nodes);
  cudaMemcpyAsync(scratch, w, sizeof(double2) * sv * nodes, cudaMemcpyDeviceToDevice, st);
  permute_rhs_kernel<<<g1, 256, 0, st>>>(n, m, ldv, perm, nullptr, scratch, w);
  ++g_launches;
  zgetrs_core(n, nodes, m, lu, stride, dinv, w, ldv, sv, st);
  return cudaGetLastError();
}

cudaError_t dense_solve(const DenseSolveArgs& a, cudaStream_t st) {
  const int n = a.n, nodes = a.nodes, m = a.m;
  const int64_t nn = (int64_t)n * n, sv = (int64_t)a.ldv * m;
  const int64_t total = (int64_t)n * m;
  dim3 g1((unsigned)std::min<int64_t>((total + 255) / 256, 1024), nodes);
  if (a.complex_mode)  // the t buffer is sized for a complex copy in complex mode
    return zgetrs_batched(n, nodes, m, a.lu, nn, a.perm, a.dinv, a.w, a.ldv, reinterpret_cast<double2*>(a.t), st);
  permute_rhs_kernel<<<g1, 256, 0, st>>>(n, m, a.ldv, a.perm, a.y, nullptr, a.w);
  ++g_launches;
  zgetrs_core(n, nodes, m, a.lu, nn, a.dinv, a.w, a.ldv, sv, st);
  {
    term_kernel<<<g1, 256, 0, st>>>(n, m, a.ldv, a.coeff, a.w, a.t);
    ++g_launches;
  }
  return cudaGetLastError();
}

}  // namespace feastgpu
