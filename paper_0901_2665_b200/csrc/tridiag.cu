// tridiag.cu — symmetric eigendecomposition for the reduced problem when it fits one SM
// (m <= 1024): the dense -> tridiagonal -> eigenpairs route of LAPACK's syevx, re-shaped for
// one B200 CTA plus a grid of warps. Used by sym_eig (eig.cu) for every reduced size; same contract as jacobi_eigh (eigh.hpp:84-163): eigenvalues ascending,
// orthonormal eigenvectors, repeated eigenvalues allowed.
//
//   tridiag_kernel      Householder reduction A = Q T Q^T (dsytd2, lower); the working
//                       matrix lives in packed lower-triangular SHARED memory (m(m+1)/2
//                       doubles, 148 KB at m = 192); one CTA of 1024 threads; reflectors out.
//   tri_eigvals_kernel  a group of 1-4 warps per eigenvalue: (128 x warps)-point multisection
//                       of the Sturm count of T - sigma I (dstebz) down to round-off;
//                       eigenvalue j is the j-th.
//   tri_eigvecs_kernel  one warp per cluster (|lam_i - lam_j| <= 1e-5 ||T||, cf. dstein):
//                       inverse iteration with the partial-pivot tridiagonal LU (dgttrf /
//                       dgtts2), modified Gram-Schmidt against earlier cluster members.
//   tri_back_kernel     V = H_0 H_1 ... H_{m-3} Z, one warp per column.

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

__device__ __forceinline__ int pidx(int i, int j, int m) {  // packed lower, column-major, i >= j
  return j * m - (j * (j - 1)) / 2 + (i - j);
}

__device__ double tri_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  const double out = red[32];
  __syncthreads();
  return out;
}

// ---------------------------------------------------------------------------
// 1. Householder tridiagonalisation
//    out: d[m], e[m-1], hv (m x m: column k holds v_k in rows k+1.., v_k[k+1] = 1), tau[m]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) tridiag_kernel(int m, const double* __restrict__ a, double* d,
                                                       double* e, double* hv, double* tau) {
  extern __shared__ double ps[];      // packed lower triangle
  double* v = ps + m * (m + 1) / 2;   // m
  double* w = v + m;                  // m
  __shared__ double red[2][32];
  __shared__ double red33[33];
  __shared__ double refl[3];  // next reflector's (t, beta, scal): one thread computes them
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  // Householder scalars of the column below row k+1 from alpha = A(k+1, k) and
  // xn2 = ||A(k+2:, k)||^2 (sqrt + two divisions: one thread, not 1024)
  auto reflector = [&](double alpha, double xn2) {
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    refl[0] = t;
    refl[1] = beta;
    refl[2] = scal;
  };
  for (int idx = tid; idx < m * m; idx += nt) {  // all loads in flight at once
    const int i = idx % m, j = idx / m;
    if (i >= j) cp_async8z(ps + pidx(i, j, m), a + idx, true);
  }
  cp_async_wait_all();
  __syncthreads();
  {
    double part = 0.0;  // ||A(2:, 0)||^2 for the first reflector
    for (int i = 2 + tid; i < m; i += nt) part += ps[pidx(i, 0, m)] * ps[pidx(i, 0, m)];
    const double s = tri_block_sum(part, red33);
    if (tid == 0 && m > 2) reflector(ps[pidx(1, 0, m)], s);
    __syncthreads();
  }

  // Three barriers per column: (A) reflector built, (C) p and p.v, (D) rank-2 update + the
  // next column's norm
  for (int k = 0; k + 2 < m; ++k) {
    const int r = m - k - 1;  // rows below the diagonal
    const double t = refl[0], beta = refl[1], scal = refl[2];
    for (int i = tid; i < r; i += nt) {
      const double vi = i == 0 ? 1.0 : (t != 0.0 ? ps[pidx(k + 1 + i, k, m)] * scal : 0.0);
      v[i] = vi;
      hv[(k + 1 + i) + (int64_t)k * m] = vi;
    }
    if (tid == 0) {
      d[k] = ps[pidx(k, k, m)];
      e[k] = beta;
      tau[k] = t;
    }
    __syncthreads();  // (A)
    if (t != 0.0) {
      // p = t * A22 v (symmetric, packed lower), column-oriented: warp w owns columns
      // j = w + 32c; lanes walk the contiguous column j (rows i >= j): the lower part
      // accumulates into per-lane registers pacc[q] (row lane + 32q), the strictly-lower
      // part gives dots[c] = sum_i A(i,j) v_i for p_j; the 7 reductions run interleaved
      // p = t * A22 v (symmetric, packed lower): 4 threads per row i; thread q takes
      // columns j = q, q+4, ...: row part A(i, j<=i) through incrementally advanced packed
      // offsets, column part A(j>i, i) from the contiguous column i. Work per thread tracks
      // the trailing size (no predicated-off iterations).
      double pv = 0.0;
      {
        const int i = tid >> 2, q = tid & 3;
        double s = 0.0;
        if (i < r) {
          const int gi = k + 1 + i, base = k + 1;
          int off = pidx(gi, base + q, m);  // A(gi, base + j) for j = q
          for (int j = q; j <= i; j += 4) {
            s += ps[off] * v[j];
            // advance 4 columns: pidx(gi, c+4) - pidx(gi, c) = 4m - 4c - 10, c = base + j
            off += 4 * m - 4 * (base + j) - 10;
          }
          const double* coli = ps + pidx(gi, gi, m) - i;  // coli[j] = A(base + j, gi), j >= i
          int j0 = i + 1 + ((q - (i + 1)) & 3);           // first j > i with j == q (mod 4)
          for (int j = j0; j < r; j += 4) s += coli[j] * v[j];
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (i < r && q == 0) {
          s *= t;
          w[i] = s;
          pv = s * v[i];
        }
      }
      pv = warp_sum(pv);
      if (lane == 0) red[k & 1][warp] = pv;
      __syncthreads();  // (C)
      double pvt = 0.0;
#pragma unroll 8
      for (int ww = 0; ww < nw; ++ww) pvt += red[k & 1][ww];
      const double c = -0.5 * t * pvt;
      // A22 -= v w^T + w v^T with w = p + c v (lower): warp per column, lanes over rows;
      // warp 0 updates column k+1 and leaves ||A(k+3:, k+1)||^2 for the next reflector
      // v w'^T + w' v^T with w' = p + c v equals v (p + 2c v)^T + p v^T elementwise pair-wise:
      // A(i,j) -= v_i (p_j + 2c v_j) + p_i v_j  (2 FMAs per element)
      for (int j = warp; j < r; j += nw) {
        double* col = ps + pidx(k + 1 + j, k + 1 + j, m) - j;
        const double vj = v[j], wj = w[j] + 2.0 * c * vj;
        if (j == 0) {
          double nrm = 0.0;
          for (int i = lane; i < r; i += 32) {
            const double x = col[i] - (v[i] * wj + w[i] * vj);
            col[i] = x;
            if (i >= 2) nrm += x * x;
          }
          nrm = warp_sum(nrm);
          __syncwarp();
          if (lane == 0 && k + 3 < m) reflector(col[1], nrm);  // A(k+2, k+1) is final here
        } else {
          for (int i = j + lane; i < r; i += 32) col[i] -= v[i] * wj + w[i] * vj;
        }
      }
      __syncthreads();  // (D)
    } else {
      double part = 0.0;  // no reflection: the next column's norm directly
      for (int i = 2 + tid; i < r; i += nt) part += ps[pidx(k + 1 + i, k + 1, m)] * ps[pidx(k + 1 + i, k + 1, m)];
      const double s = tri_block_sum(part, red33);
      if (tid == 0 && k + 3 < m) reflector(ps[pidx(k + 2, k + 1, m)], s);
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (m >= 2) {
      d[m - 2] = ps[pidx(m - 2, m - 2, m)];
      e[m - 2] = ps[pidx(m - 1, m - 2, m)];
      tau[m - 2] = 0.0;
    }
    d[m - 1] = ps[pidx(m - 1, m - 1, m)];
    tau[m - 1] = 0.0;
  }
}


// ---------------------------------------------------------------------------
// 1b. Householder tridiagonalisation for m beyond one SM's shared memory: cooperative grid,
//     packed lower triangle in global memory (L2-resident: 2.4 MB at m = 768). Trailing
//     column j belongs to CTA j mod G (one warp per column, coalesced down the column).
//     Per column, three grid barriers:
//       (1) every CTA: v (from column k), its columns' dots p_j = A(j:, j).v(j:) and its
//           per-warp axpy partials A(i, j) v_j -> part[c][i]        (fixed-order sums)
//       (2) CTA c: p_i = t (dot_i + sum_c part[c][i]) for its row slice, and p.v partials
//       (3) every CTA: w = p - (t/2)(p.v) v, rank-2 update of its columns; the owner of the
//           next column leaves its norm
//     Data written by other CTAs is read with ld.global.cg (L2), never through a stale L1.
// ---------------------------------------------------------------------------
struct TriCoopArgs {
  int m;
  const double* a;  // m x m input
  double *d, *e, *hv, *tau;
  double* gps;      // packed lower triangle, m(m+1)/2
  double* part;     // G x m per-CTA axpy partials
  double* pcol;     // m column dots
  double* pvec;     // m: p = t A v
  double* pvp;      // G: per-CTA p.v partials
  double* xn2;      // 1: ||A(k+3:, k+1)||^2 for the next reflector
};

constexpr int TC_NT = 256, TC_NW = TC_NT / 32;

__global__ void __launch_bounds__(TC_NT) tridiag_coop_kernel(TriCoopArgs p) {
  cg::grid_group grid = cg::this_grid();
  const int m = p.m, G = gridDim.x, c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double csm[];
  double* vsh = csm;          // m
  double* wsh = vsh + m;      // m
  double* qw = wsh + m;       // TC_NW x m per-warp axpy partials
  __shared__ double red33[33];
  __shared__ double bc;
  double* gps = p.gps;
  for (int64_t idx = c * (int64_t)TC_NT + tid; idx < (int64_t)m * m; idx += (int64_t)G * TC_NT) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    if (i >= j) gps[pidx(i, j, m)] = p.a[idx];
  }
  grid.sync();
  if (c == 0) {
    double part = 0.0;
    for (int i = 2 + tid; i < m; i += TC_NT) {
      const double x = __ldcg(gps + pidx(i, 0, m));
      part += x * x;
    }
    const double sm = tri_block_sum(part, red33);
    if (tid == 0) *p.xn2 = sm;
  }
  grid.sync();

  for (int k = 0; k + 2 < m; ++k) {
    const int r = m - k - 1;
    const double* colk = gps + pidx(k + 1, k, m);
    const double xn2 = __ldcg(p.xn2);
    const double alpha = __ldcg(colk);
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = tid; i < r; i += TC_NT) {
      const double vi = i == 0 ? 1.0 : (t != 0.0 ? __ldcg(colk + i) * scal : 0.0);
      vsh[i] = vi;
      if (c == 0) p.hv[(k + 1 + i) + (int64_t)k * m] = vi;
    }
    if (c == 0 && tid == 0) {
      p.d[k] = __ldcg(gps + pidx(k, k, m));
      p.e[k] = beta;
      p.tau[k] = t;
    }
    for (int i = tid; i < TC_NW * r; i += TC_NT) qw[(i / r) * m + (i % r)] = 0.0;
    __syncthreads();
    // ---- (1) column dots and per-warp axpy partials ----
    if (t != 0.0) {
      for (int jj = warp; c + G * jj < r; jj += TC_NW) {
        const int j = c + G * jj;
        const double* colj = gps + pidx(k + 1 + j, k + 1 + j, m) - j;  // colj[i] = A22(i, j)
        const double vj = vsh[j];
        double ds = 0.0;
        double* q = qw + warp * m;
        for (int i0 = j + lane; i0 < r; i0 += 256) {  // 8 L2 loads in flight per lane
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = i0 + 32 * u < r ? __ldcg(colj + i0 + 32 * u) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = i0 + 32 * u;
            if (i < r) {
              if (i == j) {
                ds += x[u] * vj;
              } else {
                ds += x[u] * vsh[i];
                q[i] += x[u] * vj;
              }
            }
          }
        }
        ds = warp_sum(ds);
        if (lane == 0) p.pcol[j] = ds;
      }
    }
    __syncthreads();
    if (t != 0.0)
      for (int i = tid; i < r; i += TC_NT) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < TC_NW; ++w) sacc += qw[w * m + i];
        p.part[(int64_t)c * m + i] = sacc;
      }
    grid.sync();  // (1)
    // ---- (2) p = t A v on this CTA's row slice ----
    if (t != 0.0) {
      // rows [i0, i1) of this CTA (<= 8 when G >= r / 8); thread cc reads partial cc of all of
      // them at once, then a fixed-order reduction over threads
      const int sl = (r + G - 1) / G, i0 = c * sl, i1 = min(r, i0 + sl);
      double pv = 0.0;
      for (int b0 = i0; b0 < i1; b0 += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x[u] = 0.0;
          for (int cc = tid; cc < G; cc += TC_NT)
            if (b0 + u < i1) x[u] += __ldcg(p.part + (int64_t)cc * m + b0 + u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x[u] = warp_sum(x[u]);
          if (lane == 0) qw[u * TC_NW + warp] = x[u];  // qw is free again here
        }
        __syncthreads();
        if (tid < 8 && b0 + tid < i1) {
          const int i = b0 + tid;
          double pf = __ldcg(p.pcol + i);
#pragma unroll
          for (int w = 0; w < TC_NW; ++w) pf += qw[tid * TC_NW + w];
          pf *= t;
          p.pvec[i] = pf;
          pv += pf * vsh[i];
        }
        __syncthreads();
      }
      pv = tri_block_sum(pv, red33);
      if (tid == 0) p.pvp[c] = pv;
    }
    grid.sync();  // (2)
    // ---- (3) w and the rank-2 update of this CTA's columns ----
    if (t != 0.0) {
      if (warp == 0) {
        double s = 0.0;
        for (int cc = lane; cc < G; cc += 32) s += __ldcg(p.pvp + cc);
        s = warp_sum(s);
        if (lane == 0) bc = s;
      }
      __syncthreads();
      const double cf = -0.5 * t * bc;
      for (int i = tid; i < r; i += TC_NT) wsh[i] = __ldcg(p.pvec + i) + cf * vsh[i];
      __syncthreads();
      for (int jj = warp; c + G * jj < r; jj += TC_NW) {
        const int j = c + G * jj;
        double* colj = gps + pidx(k + 1 + j, k + 1 + j, m) - j;
        const double vj = vsh[j], wj = wsh[j];
        double nrm = 0.0;
        for (int i0 = j + lane; i0 < r; i0 += 256) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = i0 + 32 * u < r ? __ldcg(colj + i0 + 32 * u) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = i0 + 32 * u;
            if (i < r) {
              const double y = x[u] - (vsh[i] * wj + wsh[i] * vj);
              __stcg(colj + i, y);
              if (i >= 2) nrm += y * y;
            }
          }
        }
        if (j == 0) {
          nrm = warp_sum(nrm);
          if (lane == 0) *p.xn2 = nrm;
        }
      }
    } else if (c == 0) {  // no reflection: the next column's norm directly
      double part = 0.0;
      const double* coln = gps + pidx(k + 1, k + 1, m);
      for (int i = 2 + tid; i < r; i += TC_NT) {
        const double x = __ldcg(coln + i);
        part += x * x;
      }
      const double sm = tri_block_sum(part, red33);
      if (tid == 0) *p.xn2 = sm;
    }
    grid.sync();  // (3)
  }
  if (c == 0 && tid == 0) {
    if (m >= 2) {
      p.d[m - 2] = __ldcg(gps + pidx(m - 2, m - 2, m));
      p.e[m - 2] = __ldcg(gps + pidx(m - 1, m - 2, m));
      p.tau[m - 2] = 0.0;
    }
    p.d[m - 1] = __ldcg(gps + pidx(m - 1, m - 1, m));
    p.tau[m - 1] = 0.0;
  }
}


// ---------------------------------------------------------------------------
// 1c. Householder tridiagonalisation on a thread-block cluster of TCL_P CTAs: global column g
//     lives (packed, rows g..m-1) in the shared memory of CTA g mod TCL_P, so all matrix
//     traffic stays on-chip; only vectors cross CTAs, through distributed shared memory.
//     Per column k, two cluster barriers:
//       (a) each CTA: dots of its own columns (A(g:, g) . v) and its axpy partial
//           q[i] = sum_{own g < i} A(i, g) v_g, both in its own shared memory
//       (c) every CTA gathers all partials through DSMEM reads into the FULL p (same order in
//           every CTA, so p, p.v and w agree bit for bit), w = p - (t/2)(p.v) v, the rank-2
//           update of its own columns; the owner of column k+1 builds the next reflector
//           and pushes it (and t) into every CTA's other v buffer
//     All sums run in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int TCL_P = 16, TCL_NT = 512, TCL_NW = TCL_NT / 32;

__host__ __device__ inline int tcl_ncols(int m, int q) { return q < m ? (m - q + TCL_P - 1) / TCL_P : 0; }
// offset of the t-th own column (global g = q + t P, rows g..m-1) in CTA q's packed storage
__host__ __device__ inline int tcl_off(int m, int q, int t) { return t * (m - q) - TCL_P * (t * (t - 1) / 2); }
__host__ __device__ inline int tcl_local(int m, int q) { return tcl_off(m, q, tcl_ncols(m, q)); }

__global__ void __launch_bounds__(TCL_NT) tridiag_cluster_kernel(int m, const double* __restrict__ a, double* d,
                                                                 double* e, double* hv, double* tau) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double ksm[];
  const int loc = tcl_local(m, 0);  // same layout size in every CTA (CTA 0 holds the most)
  double* cols = ksm;               // own columns, packed
  double* vb = cols + loc;          // 2 x m: reflector (trailing index), double-buffered by parity
  double* ww = vb + 2 * m;          // m: p, then w (trailing index), full in every CTA
  double* qp = ww + m;              // m: my axpy partial (trailing row index), read by every CTA
  double* dc = qp + m;              // m: dots of my own columns (trailing column index)
  __shared__ double scal_s[2];      // t per parity, pushed by the reflector's owner
  __shared__ double xn2_s;          // owner of the next column: ||A(k+3:, k+1)||^2
  __shared__ double red33[33];
  const int ncol = tcl_ncols(m, q);
  for (int t = 0; t < ncol; ++t) {  // own columns
    const int g = q + t * TCL_P;
    const int off = tcl_off(m, q, t);
    for (int i = g + tid; i < m; i += TCL_NT) cols[off + (i - g)] = a[i + (int64_t)g * m];
  }
  __syncthreads();
  // owner of column k (column k up to date locally): reflector into every CTA's v buffer
  auto build = [&](int k, int par, bool fresh) {
    const int t = (k - q) / TCL_P;
    const double* ck = cols + tcl_off(m, q, t) - k;  // ck[i] = A(i, k), i >= k
    const int r = m - k - 1;
    double xn2;
    if (fresh) {  // first column, or the previous step skipped its update (no norm left)
      double part = 0.0;
      for (int i = k + 2 + tid; i < m; i += TCL_NT) part += ck[i] * ck[i];
      xn2 = tri_block_sum(part, red33);
    } else {
      xn2 = xn2_s;
    }
    const double alpha = ck[k + 1];
    double tt = 0.0, beta = alpha, sc = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      tt = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    for (int i = tid; i < r; i += TCL_NT) {
      const double vi = i == 0 ? 1.0 : (tt != 0.0 ? ck[k + 1 + i] * sc : 0.0);
      hv[(k + 1 + i) + (int64_t)k * m] = vi;
#pragma unroll
      for (int qq = 0; qq < TCL_P; ++qq) cl.map_shared_rank(vb + par * m, qq)[i] = vi;
    }
    if (tid < TCL_P) *cl.map_shared_rank(&scal_s[par], tid) = tt;
    if (tid == 0) {
      d[k] = ck[k];
      e[k] = beta;
      tau[k] = tt;
    }
  };
  // every CTA of the cluster must be running before its shared memory is written remotely (the
  // first reflector below is pushed into all 16 CTAs)
  cl.sync();
  if (m > 2 && q == 0) build(0, 0, true);
  cl.sync();

  for (int k = 0; k + 2 < m; ++k) {
    const int r = m - k - 1, par = k & 1, base = k + 1;  // trailing index = global - base
    const double* v = vb + par * m;
    const double tt = scal_s[par];
    const int t0 = base > q ? (base - q + TCL_P - 1) / TCL_P : 0;  // first own column >= base
    // ---- (a) dots of own columns and axpy partials, pushed to the slice owners ----
    if (tt != 0.0) {
      for (int t = t0 + warp; t < ncol; t += TCL_NW) {
        const int g = q + t * TCL_P;
        const double* cg_ = cols + tcl_off(m, q, t) - g;  // cg_[i] = A(i, g)
        double s = 0.0;
        for (int i = g + lane; i < m; i += 32) s += cg_[i] * v[i - base];
        s = warp_sum(s);
        if (lane == 0) dc[g - base] = s;
      }
      for (int i = base + tid; i < m; i += TCL_NT) {
        const int tend = min(ncol, (i - q + TCL_P - 1) / TCL_P);  // own g in [base, i)
        double s0 = 0.0, s1 = 0.0;
        int t = t0, off = tcl_off(m, q, t0), g = q + t0 * TCL_P;
        for (; t + 1 < tend; t += 2) {
          const int off1 = off + (m - g), g1 = g + TCL_P;
          s0 += cols[off + (i - g)] * v[g - base];
          s1 += cols[off1 + (i - g1)] * v[g1 - base];
          off = off1 + (m - g1);
          g = g1 + TCL_P;
        }
        if (t < tend) s0 += cols[off + (i - g)] * v[g - base];
        qp[i - base] = s0 + s1;
      }
    }
    cl.sync();  // (a)
    // ---- (b) every CTA gathers all partials (DSMEM reads) into the full p, then w ----
    //      (each CTA sums in the same order, so p, p.v and w are identical in all of them)
    if (tt != 0.0) {
      double pv = 0.0;
      for (int ti = tid; ti < r; ti += TCL_NT) {
        double x[TCL_P];
#pragma unroll
        for (int qq = 0; qq < TCL_P; ++qq) x[qq] = *cl.map_shared_rank(qp + ti, qq);  // all in flight
        double pf = *cl.map_shared_rank(dc + ti, (base + ti) % TCL_P);
#pragma unroll
        for (int qq = 0; qq < TCL_P; ++qq) pf += x[qq];
        pf *= tt;
        ww[ti] = pf;
        pv += pf * v[ti];
      }
      pv = tri_block_sum(pv, red33);
      const double cf = -0.5 * tt * pv;
      for (int ti = tid; ti < r; ti += TCL_NT) ww[ti] += cf * v[ti];
      __syncthreads();
      for (int t = t0 + warp; t < ncol; t += TCL_NW) {
        const int g = q + t * TCL_P;
        double* cg_ = cols + tcl_off(m, q, t) - g;
        const double vg = v[g - base], wg = ww[g - base];
        double nrm = 0.0;
        for (int i = g + lane; i < m; i += 32) {
          const double y = cg_[i] - (v[i - base] * wg + ww[i - base] * vg);
          cg_[i] = y;
          if (i >= g + 2) nrm += y * y;
        }
        if (g == base) {  // the next reflector's column: its norm below the subdiagonal
          nrm = warp_sum(nrm);
          if (lane == 0) xn2_s = nrm;
        }
      }
    }
    __syncthreads();
    if (k + 3 < m && q == base % TCL_P) build(base, par ^ 1, tt == 0.0);
    cl.sync();  // (c)
  }
  if (m >= 2 && q == (m - 2) % TCL_P && tid == 0) {
    const int t = (m - 2 - q) / TCL_P;
    const double* ck = cols + tcl_off(m, q, t) - (m - 2);
    d[m - 2] = ck[m - 2];
    e[m - 2] = ck[m - 1];
    tau[m - 2] = 0.0;
  }
  if (q == (m - 1) % TCL_P && tid == 0) {
    const int t = (m - 1 - q) / TCL_P;
    d[m - 1] = cols[tcl_off(m, q, t)];
    tau[m - 1] = 0.0;
  }
}

// largest m whose cluster layout fits the 227 KB opt-in shared memory
static size_t tcl_smem(int m) { return sizeof(double) * ((size_t)tcl_local(m, 0) + 5 * (size_t)m); }

// ---------------------------------------------------------------------------
// 2. eigenvalues: Sturm-count multisection
// ---------------------------------------------------------------------------
// 1/x from the hardware approximation plus two Newton steps (full double precision): the
// recurrences below are chains of dependent divisions, so division latency is the clock
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

__device__ __forceinline__ int sturm(int m, const double* d, const double* e2, double sigma, double pivmin) {
  int cnt = 0;
  double q = d[0] - sigma;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = (d[i] - sigma) - e2[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// reciprocal to ~2^-46 relative (one Newton step on the hardware approximation): the Sturm
// counts only need the sign of each pivot, and a relative error of 1e-14 in q_i is a relative
// perturbation of the same order in e_{i-1}^2, i.e. eigenvalue shifts of O(1e-14 ||T||)
__device__ __forceinline__ double fast_rcp1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}

// NCH Sturm counts at once (independent chains interleaved: the latency of one chain's
// reciprocal and FMAs hides behind the others; the chain step is latency-bound at 4)
template <int NCH>
__device__ __forceinline__ void sturm_n(int m, const double* d, const double* e2, const double (&sg)[NCH],
                                        double pivmin, int (&cnt)[NCH]) {
  double q[NCH];
#pragma unroll
  for (int u = 0; u < NCH; ++u) {
    q[u] = d[0] - sg[u];
    if (fabs(q[u]) < pivmin) q[u] = -pivmin;
    cnt[u] = q[u] < 0.0;
  }
  for (int i = 1; i < m; ++i) {
    const double di = d[i], ei = e2[i - 1];
#pragma unroll
    for (int u = 0; u < NCH; ++u) {
      q[u] = (di - sg[u]) - ei * fast_rcp1(q[u]);
      if (fabs(q[u]) < pivmin) q[u] = -pivmin;
      cnt[u] += q[u] < 0.0;
    }
  }
}

struct TriArgs {
  int m;
  const double* d;
  const double* e;
  double* lam;  // eigenvalues ascending
  double* z;    // m x m eigenvectors of T
  double* lu;   // 4*m per eigenpair (LU bands)
  int* piv;     // m per eigenpair
  double vfloor;  // > 0: vectors only for lam > vfloor * lam_max (others zero)
};

__device__ void tri_bounds(int m, const double* d, const double* e, double& lo, double& hi, double& tnorm,
                           double& pivmin) {
  lo = 1e300, hi = -1e300, tnorm = 0.0;
  double emax2 = 0.0;
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    tnorm = fmax(tnorm, fabs(d[i]) + r);
    if (i + 1 < m) emax2 = fmax(emax2, e[i] * e[i]);
  }
  pivmin = DBL_MIN * fmax(1.0, emax2);
  const double slack = 2.0 * DBL_EPSILON * tnorm + 2.0 * pivmin;
  lo -= slack;
  hi += slack;
}

// WPE warps per eigenvalue (a named barrier per group of WPE warps), EPC = warps / WPE
// eigenvalues per CTA: each step is a (128 WPE)-point multisection, the WPE warps of a group
// sitting on different SM sub-partitions so the wider step costs no more than a one-warp one
template <int WPE, int NCH>
__global__ void tri_eigvals_kernel(TriArgs p) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e2 = d + p.m;
  double* e = e2 + p.m;
  __shared__ int s_nb[2][32];
  const int m = p.m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    d[i] = p.d[i];
    if (i + 1 < m) {
      e[i] = p.e[i];
      e2[i] = p.e[i] * p.e[i];
    }
  }
  __syncthreads();
  double lo, hi, tnorm, pivmin;
  tri_bounds(m, d, e, lo, hi, tnorm, pivmin);  // from shared memory: one pass, no L2 round trips
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / WPE, wg = warp % WPE;
  const int epc = (blockDim.x >> 5) / WPE;
  const int j = blockIdx.x * epc + grp;
  if (j >= m) return;
  constexpr int PT = 32 * NCH * WPE;       // points per step
  constexpr double INV = 1.0 / (PT + 1);   // (exact enough: only the grid's spacing uses it)
  // points a + w (P + 1) / (PT + 1), P = 32 NCH wg + NCH lane + u, computed identically on every
  // lane of the group; invariant count(a) <= j < count(b)
  double a = lo, b = hi;
  for (int it = 0; it < 16; ++it) {
    const double width = b - a;
    if (width <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b)) + 2.0 * pivmin) break;
    double sg[NCH];
    int c[NCH];
#pragma unroll
    for (int u = 0; u < NCH; ++u) sg[u] = a + width * ((double)(32 * NCH * wg + NCH * lane + u + 1) * INV);
    sturm_n<NCH>(m, d, e2, sg, pivmin, c);
    int nb = 0;  // points left of lam_j (counts are monotone in the point index)
#pragma unroll
    for (int u = 0; u < NCH; ++u) nb += __popc(__ballot_sync(0xffffffffu, c[u] <= j));
    if (WPE > 1) {
      if (lane == 0) s_nb[it & 1][warp] = nb;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * WPE) : "memory");
      nb = 0;
#pragma unroll
      for (int w = 0; w < WPE; ++w) nb += s_nb[it & 1][grp * WPE + w];
    }
    const double na = nb > 0 ? a + width * ((double)nb * INV) : a;
    const double nbb = nb < PT ? a + width * ((double)(nb + 1) * INV) : b;
    a = na;
    b = nbb;
  }
  if (lane == 0 && wg == 0) p.lam[j] = 0.5 * (a + b);
}

// ---------------------------------------------------------------------------
// 3. eigenvectors: inverse iteration (one warp per cluster)
// ---------------------------------------------------------------------------
// LU of T - lam I with partial pivoting (dgttrf): D (diag of U), DU, DU2 (supers of U),
// DL (multipliers), ipiv[i] = 1 if rows i, i+1 were swapped
// Pivoted LU of T - lam I (dgttf2) on one lane. The running row (its diagonal and super-diagonal
// entries) is carried in registers, so the dependent chain of a step is compare -> reciprocal ->
// FMA; through shared memory (the first version re-read D[i], DU[i] it had stored one step
// earlier) every step paid two store-to-load round trips. D is left raw: the caller inverts it with
// all lanes (gttrf_finish).
__device__ void gttrf(int m, const double* __restrict__ d, const double* __restrict__ e, double lam,
                      double* __restrict__ D, double* __restrict__ DL, double* __restrict__ DU,
                      double* __restrict__ DU2, int* __restrict__ ipiv, double tiny) {
  double di = d[0] - lam;          // row i after the eliminations so far: diagonal ...
  double dui = m > 1 ? e[0] : 0.0;  // ... and super-diagonal
  for (int i = 0; i + 1 < m; ++i) {
    const double dli = e[i];                       // sub-diagonal entry (i + 1, i)
    const double dn = d[i + 1] - lam;              // row i + 1 as given: diagonal ...
    const double dun = i + 2 < m ? e[i + 1] : 0.0;  // ... and super-diagonal
    if (fabs(di) >= fabs(dli)) {
      if (di == 0.0) di = tiny;
      const double f = dli * fast_rcp(di);
      D[i] = di;
      DL[i] = f;
      DU[i] = dui;
      DU2[i] = 0.0;
      ipiv[i] = 0;
      di = dn - f * dui;
      dui = dun;
    } else {  // rows i and i + 1 interchanged
      const double f = di * fast_rcp(dli);
      D[i] = dli;
      DL[i] = f;
      DU[i] = dn;
      DU2[i] = dun;
      ipiv[i] = 1;
      di = dui - f * dn;
      dui = -f * dun;
    }
  }
  D[m - 1] = di;
}
// D <- 1 / D (clamped away from zero) by the whole warp: the solves then chain FMAs only
__device__ void gttrf_finish(int m, double* D, double tiny, int lane) {
  for (int i = lane; i < m; i += 32) {
    double di = D[i];
    if (fabs(di) < tiny) di = di < 0.0 ? -tiny : tiny;
    D[i] = 1.0 / di;
  }
}

// the two substitutions (dgtts2) on one lane, the running entries in registers (one FMA per
// forward step, two FMAs and a multiply per backward step on the dependent chain)
__device__ void gtts2(int m, const double* __restrict__ D, const double* __restrict__ DL,
                      const double* __restrict__ DU, const double* __restrict__ DU2,
                      const int* __restrict__ ipiv, double* __restrict__ b) {
  double bi = b[0];
  for (int i = 0; i + 1 < m; ++i) {
    const double bn = b[i + 1], l = DL[i];
    if (!ipiv[i]) {
      b[i] = bi;
      bi = bn - l * bi;
    } else {
      b[i] = bn;
      bi = bi - l * bn;
    }
  }
  // D holds 1 / diag(U)
  double x1 = bi * D[m - 1], x2 = 0.0;  // x_{i+1}, x_{i+2}
  b[m - 1] = x1;
  for (int i = m - 2; i >= 0; --i) {
    const double xi = (b[i] - DU[i] * x1 - DU2[i] * x2) * D[i];
    b[i] = xi;
    x2 = x1;
    x1 = xi;
  }
}

// inverse-iteration steps per vector: the Sturm eigenvalue is accurate to O(eps ||T||), so
// the first solve already amplifies the wanted direction by ~1/eps; the second one (after the
// in-cluster Gram-Schmidt) is the dstein "extra" step
constexpr int kInvIters = 2;

__global__ void tri_eigvecs_kernel(TriArgs p) {
  const int m = p.m, lane = threadIdx.x & 31;
  const int cl = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // d, e in shared memory: the O(m) recurrences below run on one lane, where every L2 load
  // would be a serial round trip
  extern __shared__ double wsm[];
  double* sd = wsm;
  double* se = sd + m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sd[i] = p.d[i];
    se[i] = i + 1 < m ? p.e[i] : 0.0;
  }
  __syncthreads();
  if (cl >= m) return;
  double lo, hi, tnorm, pivmin;
  tri_bounds(m, sd, se, lo, hi, tnorm, pivmin);
  // reorthogonalisation threshold: dstein uses 1e-3 ||T||; inverse iteration leaves a
  // non-orthogonality of O(eps ||T|| / gap), so 1e-5 ||T|| already bounds it by ~1e-11 while
  // keeping FEAST's dense interior Ritz spectra from chaining into one long cluster
  const double ortol = 1e-5 * tnorm, eps = DBL_EPSILON;
  // vectors of the eigenvalues at or below the floor are not wanted (the truncation path of
  // reduced_gevp discards them): the near-null cluster of a graded mass matrix never forms
  int j0 = 0;
  if (p.vfloor > 0.0) {
    const double thr = p.vfloor * p.lam[m - 1];
    int lo_ = 0, hi_ = m;  // first index with lam > thr (ascending)
    while (lo_ < hi_) {
      const int mid = (lo_ + hi_) >> 1;
      if (p.lam[mid] > thr) hi_ = mid;
      else lo_ = mid + 1;
    }
    j0 = lo_;
  }
  if (cl < j0) {
    for (int i = lane; i < m; i += 32) p.z[i + (int64_t)cl * m] = 0.0;
    return;
  }
  if (cl > j0 && p.lam[cl] - p.lam[cl - 1] <= ortol) return;  // not the first of its cluster
  int cend = cl + 1;
  while (cend < m && p.lam[cend] - p.lam[cend - 1] <= ortol) ++cend;
  // per-warp shared scratch: LU bands, pivots, the iterate (the O(m) recurrences run on
  // lane 0 against shared memory, not L2)
  double* D = wsm + 2 * m + (threadIdx.x >> 5) * 6 * m;
  double* DL = D + m;
  double* DU = DL + m;
  double* DU2 = DU + m;
  double* zs = DU2 + m;
  int* ipiv = reinterpret_cast<int*>(zs + m);
  double prev = -1e300;
  for (int j = cl; j < cend; ++j) {
    double lam = p.lam[j];
    const double sep = 10.0 * eps * fmax(tnorm, 1e-300);
    if (j > cl && lam - prev < sep) lam = prev + sep;  // separate coincident shifts (dstein)
    prev = lam;
    if (lane == 0) gttrf(m, sd, se, lam, D, DL, DU, DU2, ipiv, eps * tnorm);
    __syncwarp();
    gttrf_finish(m, D, eps * tnorm, lane);
    double* zj = zs;
    for (int i = lane; i < m; i += 32) {  // deterministic pseudo-random start
      uint32_t h = (uint32_t)i * 2654435761u ^ ((uint32_t)j * 40503u + 12345u);
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      zj[i] = 0.5 + (double)(h & 0xffff) / 65536.0;
    }
    __syncwarp();
    for (int it = 0; it < kInvIters; ++it) {
      if (lane == 0) gtts2(m, D, DL, DU, DU2, ipiv, zj);
      __syncwarp();
      for (int k = cl; k < j; ++k) {  // modified Gram-Schmidt within the cluster
        const double* zk = p.z + (int64_t)k * m;
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += zk[i] * zj[i];
        s = warp_sum(s);
        for (int i = lane; i < m; i += 32) zj[i] -= s * zk[i];
        __syncwarp();
      }
      double nrm = 0.0;
      for (int i = lane; i < m; i += 32) nrm += zj[i] * zj[i];
      nrm = warp_sum(nrm);
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = lane; i < m; i += 32) zj[i] *= inv;
      __syncwarp();
    }
    // sign convention: largest-magnitude component positive (deterministic)
    double best = 0.0;
    int bi = 0;
    for (int i = lane; i < m; i += 32)
      if (fabs(zj[i]) > best) { best = fabs(zj[i]); bi = i; }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sgn = zj[bi] < 0.0 ? -1.0 : 1.0;
    __syncwarp();
    double* zout = p.z + (int64_t)j * m;
    for (int i = lane; i < m; i += 32) zout[i] = zj[i] * sgn;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// 4'. back-transformation for m <= 192 with every reflector resident in shared memory (packed:
//     reflector k holds rows k+1..m-1, m(m-1)/2 doubles = 147 KB at m = 192) and EIGHT lanes per
//     column (four columns per warp): the dot product per reflector is a 3-level shuffle over the
//     lane group instead of a 5-level warp reduction, and no reflector load waits on L2.
// ---------------------------------------------------------------------------
constexpr int TBS_NQ = 24;  // rows per lane: m <= 8 * 24 = 192
constexpr int TBS_NW = 1;   // warps per CTA: one (the chain is per warp; spread over m/4 SMs)
__global__ void __launch_bounds__(TBS_NW * 32, 1) tri_back_smem_kernel(int m, const double* __restrict__ hv,
                                                               const double* __restrict__ tau,
                                                               const double* __restrict__ z, double* v) {
  extern __shared__ double hs[];     // packed reflectors, then tau
  double* ts = hs + (size_t)m * (m - 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nref = m - 2;
  for (int k = warp; k < nref; k += TBS_NW) {  // reflector k: rows k+1..m-1 at hs[k m - k(k+1)/2 ...]
    double* dst = hs + (size_t)k * m - (size_t)k * (k + 1) / 2;
    for (int i = k + 1 + lane; i < m; i += 32) cp_async8z(dst + (i - k - 1), hv + i + (size_t)k * m, true);
  }
  for (int k = tid; k < nref; k += TBS_NW * 32) ts[k] = tau[k];
  const int sl = lane & 7, col = blockIdx.x * (4 * TBS_NW) + warp * 4 + (lane >> 3);
  const bool live = col < m;
  double x[TBS_NQ];
#pragma unroll
  for (int q = 0; q < TBS_NQ; ++q) {
    const int i = sl + 8 * q;
    x[q] = (live && i < m) ? z[i + (size_t)col * m] : 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  for (int k = nref - 1; k >= 0; --k) {
    const double* hk = hs + (size_t)k * m - (size_t)k * (k + 1) / 2 - (k + 1);  // hk[i], i > k
    double h[TBS_NQ];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int q = 0; q < TBS_NQ; ++q) {
      const int i = sl + 8 * q;
      h[q] = (i > k && i < m) ? hk[i] : 0.0;
      if ((q & 3) == 0) s0 = fma(h[q], x[q], s0);
      else if ((q & 3) == 1) s1 = fma(h[q], x[q], s1);
      else if ((q & 3) == 2) s2 = fma(h[q], x[q], s2);
      else s3 = fma(h[q], x[q], s3);
    }
    double sum = (s0 + s1) + (s2 + s3);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    sum *= ts[k];
#pragma unroll
    for (int q = 0; q < TBS_NQ; ++q) x[q] = fma(-sum, h[q], x[q]);
  }
  if (live) {
#pragma unroll
    for (int q = 0; q < TBS_NQ; ++q) {
      const int i = sl + 8 * q;
      if (i < m) v[i + (size_t)col * m] = x[q];
    }
  }
}

// ---------------------------------------------------------------------------
// 4. back-transformation V = H_0 ... H_{m-3} Z, one warp per column
// ---------------------------------------------------------------------------
// the column stays in registers (NQ per lane: m <= 32 NQ); the next PD reflectors are loaded
// while the current one is applied, so the only serial latency is the warp reduction
template <int NQ, int PD>
__global__ void tri_back_kernel(int m, const double* __restrict__ hv, const double* __restrict__ tau,
                                const double* __restrict__ z, double* v) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= m) return;
  double x[NQ], h[PD][NQ], tp[PD];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = lane + 32 * q;
    x[q] = i < m ? z[i + (int64_t)c * m] : 0.0;
  }
  // reflector k and its tau travel together PD reflectors ahead (a tau load issued at use sat
  // on the reduction's dependency chain: ~3x the kernel time)
  auto load = [&](int k, double* dst, double& tk) {
    const double* hk = hv + (int64_t)k * m;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      dst[q] = (k >= 0 && i > k && i < m) ? hk[i] : 0.0;
    }
    tk = k >= 0 ? tau[k] : 0.0;
  };
#pragma unroll
  for (int s = 0; s < PD; ++s) load(m - 3 - s, h[s], tp[s]);
  for (int k = m - 3; k >= 0; k -= PD) {
#pragma unroll
    for (int s = 0; s < PD; ++s) {
      const int kk = k - s;
      if (kk >= 0) {
        const double t = tp[s];
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) sum += h[s][q] * x[q];
        sum = warp_sum(sum) * t;
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q] -= sum * h[s][q];
      }
      load(kk - PD, h[s], tp[s]);  // refill this slot PD reflectors ahead
    }
  }
  double* vc = v + (int64_t)c * m;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = lane + 32 * q;
    if (i < m) vc[i] = x[q];
  }
}

// one-SM route while the packed matrix + v, w (2m) fit 226 KB of shared memory; the
// cooperative grid route beyond (tws holds 6m^2 + 3m doubles for either)
static int tri_smem_dim() { return 236; }
int tri_max_dim() { return 1024; }

// a (m x m, overwritten is allowed), eigenvalues ascending -> evals, vectors -> v (m x m)
cudaError_t tri_eig(int m, const double* a, double* evals, double* v, double* ws, int* iws, cudaStream_t st,
                    double vfloor, bool low_smem, cudaEvent_t ev_tridiag) {
  if (m < 1 || m > tri_max_dim()) return cudaErrorInvalidValue;
  double* d = ws;
  double* e = d + m;
  double* tau = e + m;
  double* hv = tau + m;            // m*m
  double* z = hv + (size_t)m * m;  // m*m
  double* gw = z + (size_t)m * m;  // 4*m*m: cooperative route scratch
  static bool attr = false;
  if (!attr) {
    // dynamic + static (the reduction scratch) must stay within the 227 KB opt-in limit
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    attr = true;
  }
  // route: the register-tile kernel for 3 <= m <= 192 (tridiag_tiles.cu), the one-SM
  // shared-memory kernel for m <= 2, the 16-CTA cluster while its layout fits (m <= ~840), the
  // cooperative grid beyond
  const bool use_tiles = m > 2 && m <= tri_tiles_max_dim();
  const bool use_cluster = !use_tiles && m > 2 && tcl_smem(m) <= 220 * 1024;
  const bool use_smem = !use_tiles && !use_cluster && m <= tri_smem_dim();
  if (use_tiles) {
    cudaError_t err = tridiag_tiles(m, a, d, e, hv, tau, st);
    if (err != cudaSuccess) return err;
  } else if (use_cluster) {
    const size_t ksm = tcl_smem(m);
    cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(TCL_P);
    cfg.blockDim = dim3(TCL_NT);
    cfg.dynamicSmemBytes = ksm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TCL_P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t err = cudaLaunchKernelEx(&cfg, tridiag_cluster_kernel, m, a, d, e, hv, tau);
    ++g_launches;
    if (err != cudaSuccess) return err;
  } else if (use_smem) {
    const size_t sm = sizeof(double) * ((size_t)m * (m + 1) / 2 + 2 * m);
    tridiag_kernel<<<1, 1024, sm, st>>>(m, a, d, e, hv, tau);
    ++g_launches;
  } else {
    static int grid = 0;
    const size_t csm = sizeof(double) * (size_t)(2 + TC_NW) * 1024;  // sized for m <= 1024
    if (!grid) {
      cudaFuncSetAttribute(tridiag_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
      int dev = 0, sms = 148, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tridiag_coop_kernel, TC_NT, csm);
      grid = sms * std::max(occ, 1);
      grid = std::min(grid, sms);  // one CTA per SM: more CTAs only add barrier cost
    }
    TriCoopArgs p{m, a, d, e, hv, tau, gw, nullptr, nullptr, nullptr, nullptr, nullptr};
    p.part = p.gps + (size_t)m * (m + 1) / 2;
    p.pcol = p.part + (size_t)grid * m;
    p.pvec = p.pcol + m;
    p.pvp = p.pvec + m;
    p.xn2 = p.pvp + grid;
    void* args[] = {&p};
    cudaError_t err = cudaLaunchCooperativeKernel((void*)tridiag_coop_kernel, grid, TC_NT, args, csm, st);
    ++g_launches;
    if (err != cudaSuccess) return err;
  }
  if (ev_tridiag) {
    const cudaError_t err = cudaEventRecord(ev_tridiag, st);
    if (err != cudaSuccess) return err;
  }
  TriArgs p{m, d, e, evals, z, nullptr, iws, vfloor};
  // one warp per CTA: these are serial per-warp chains, so spreading the m warps over all 148
  // SMs (instead of 4 per CTA on m/4 SMs) is what sets their time (ncu: issue-bound at 4 warps
  // per SM, 114 / 85 / 90 us for eigvals / eigvecs / back at m = 192)
  // eigenvalues: two 2-warp groups per CTA (each warp on its own SM sub-partition), two Sturm
  // chains per lane = 128 points per multisection step. The chain step is bound by MUFU.RCP64H
  // throughput, so fewer chains per lane on more sub-partitions win; measured at m = 192 (ncu,
  // cfg2): 116 us for one warp x 4 chains, 92 us for 2 warps x 4 chains, 78 us for 2 warps x 2
  // chains, 86 us for 3-4 warps x 2 chains, 264 us for 2 warps x 8 chains
  constexpr int kWpe = 2, kEpc = 2, kNch = 2;
  const unsigned evb = (unsigned)((m + kEpc - 1) / kEpc), evt = 32u * kWpe * kEpc;
  tri_eigvals_kernel<kWpe, kNch><<<evb, evt, sizeof(double) * 3 * m, st>>>(p);
  ++g_launches;
  const size_t vsm = sizeof(double) * (6 * m + 2 * m) + 64;
  if (vsm > 48 * 1024) cudaFuncSetAttribute(tri_eigvecs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm);
  tri_eigvecs_kernel<<<m, 32, vsm, st>>>(p);
  ++g_launches;
  // back-transformation: all reflectors in shared memory for m <= 192 (147 KB per CTA: a whole
  // SM, so not beside a concurrent kernel, low_smem); blocked (WY) above m = 384 (tri_back.cu; its
  // T factors live in the cooperative route's scratch gw, free by now); otherwise one warp per
  // column with the reflectors from L2 (m = 192: 83 us against 71 us from shared memory)
  if (m >= 3 && m <= 8 * TBS_NQ && !low_smem) {
    const size_t sm = sizeof(double) * ((size_t)m * (m - 1) / 2 + m);
    static bool battr = false;
    if (!battr) {
      cudaFuncSetAttribute(tri_back_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      battr = true;
    }
    tri_back_smem_kernel<<<(m + 4 * TBS_NW - 1) / (4 * TBS_NW), TBS_NW * 32, sm, st>>>(m, hv, tau, z, v);
    ++g_launches;
  } else if (m > 384) {
    cudaError_t err = tri_back_wy(m, hv, tau, z, v, gw, st);
    if (err != cudaSuccess) return err;
  } else {
    if (m <= 256) tri_back_kernel<8, 4><<<m, 32, 0, st>>>(m, hv, tau, z, v);
    else tri_back_kernel<16, 4><<<m, 32, 0, st>>>(m, hv, tau, z, v);
    ++g_launches;
  }
  return cudaGetLastError();
}

}  // namespace feastgpu
