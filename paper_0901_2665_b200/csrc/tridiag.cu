// tridiag.cu — symmetric eigendecomposition for the reduced problem when it fits one SM
// (m <= 240): the dense -> tridiagonal -> eigenpairs route of LAPACK's syevx, re-shaped for
// one B200 CTA plus a grid of warps. Used by sym_eig (jacobi.cu) in place of block Jacobi for
// those sizes; same contract as jacobi_eigh (eigh.hpp:84-163): eigenvalues ascending,
// orthonormal eigenvectors, repeated eigenvalues allowed.
//
//   tridiag_kernel      Householder reduction A = Q T Q^T (dsytd2, lower); the working
//                       matrix lives in packed lower-triangular SHARED memory (m(m+1)/2
//                       doubles, 148 KB at m = 192); one CTA of 1024 threads; reflectors out.
//   tri_eigvals_kernel  one warp per eigenvalue: 32-way multisection of the Sturm count of
//                       T - sigma I (dstebz) down to round-off; eigenvalue j is the j-th.
//   tri_eigvecs_kernel  one warp per cluster (|lam_i - lam_j| <= 1e-5 ||T||, cf. dstein):
//                       inverse iteration with the partial-pivot tridiagonal LU (dgttrf /
//                       dgtts2), modified Gram-Schmidt against earlier cluster members.
//   tri_back_kernel     V = H_0 H_1 ... H_{m-3} Z, one warp per column.

#include <cfloat>

#include "common.cuh"
#include "kernels.h"

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
  __shared__ double xn2s;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
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
    if (tid == 0) xn2s = s;
    __syncthreads();
  }

  // Three barriers per column: (A) reflector built, (C) p and p.v, (D) rank-2 update + the
  // next column's norm
  for (int k = 0; k + 2 < m; ++k) {
    const int r = m - k - 1;  // rows below the diagonal
    const double xn2 = xn2s;
    const double alpha = ps[pidx(k + 1, k, m)];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
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
          if (lane == 0) xn2s = nrm;
        } else {
          for (int i = j + lane; i < r; i += 32) col[i] -= v[i] * wj + w[i] * vj;
        }
      }
      __syncthreads();  // (D)
    } else {
      double part = 0.0;  // no reflection: the next column's norm directly
      for (int i = 2 + tid; i < r; i += nt) part += ps[pidx(k + 1 + i, k + 1, m)] * ps[pidx(k + 1 + i, k + 1, m)];
      const double s = tri_block_sum(part, red33);
      if (tid == 0) xn2s = s;
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

struct TriArgs {
  int m;
  const double* d;
  const double* e;
  double* lam;  // eigenvalues ascending
  double* z;    // m x m eigenvectors of T
  double* lu;   // 4*m per eigenpair (LU bands)
  int* piv;     // m per eigenpair
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

__global__ void tri_eigvals_kernel(TriArgs p) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e2 = d + p.m;
  const int m = p.m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    d[i] = p.d[i];
    if (i + 1 < m) e2[i] = p.e[i] * p.e[i];
  }
  __syncthreads();
  double lo, hi, tnorm, pivmin;
  tri_bounds(m, p.d, p.e, lo, hi, tnorm, pivmin);
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= m) return;
  double a = lo, b = hi;  // invariant: count(a) <= j < count(b)
  for (int it = 0; it < 24; ++it) {
    const double width = b - a;
    if (width <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b)) + 2.0 * pivmin) break;
    const double s = a + width * (double)(lane + 1) / 33.0;
    const int c = sturm(m, d, e2, s, pivmin);
    const int nb = __popc(__ballot_sync(0xffffffffu, c <= j));  // lanes left of lam_j (monotone)
    const double na = nb > 0 ? __shfl_sync(0xffffffffu, s, (nb > 0 ? nb : 1) - 1) : a;
    const double nbb = nb < 32 ? __shfl_sync(0xffffffffu, s, nb < 32 ? nb : 31) : b;
    a = na;
    b = nbb;
  }
  if (lane == 0) p.lam[j] = 0.5 * (a + b);
}

// ---------------------------------------------------------------------------
// 3. eigenvectors: inverse iteration (one warp per cluster)
// ---------------------------------------------------------------------------
// LU of T - lam I with partial pivoting (dgttrf): D (diag of U), DU, DU2 (supers of U),
// DL (multipliers), ipiv[i] = 1 if rows i, i+1 were swapped
__device__ void gttrf(int m, const double* d, const double* e, double lam, double* D, double* DL, double* DU,
                      double* DU2, int* ipiv, double tiny) {
  for (int i = 0; i < m; ++i) D[i] = d[i] - lam;
  for (int i = 0; i + 1 < m; ++i) {
    DL[i] = e[i];
    DU[i] = e[i];
    DU2[i] = 0.0;
    ipiv[i] = 0;
  }
  for (int i = 0; i + 1 < m; ++i) {
    if (fabs(D[i]) >= fabs(DL[i])) {
      if (D[i] == 0.0) D[i] = tiny;
      const double f = DL[i] * fast_rcp(D[i]);
      DL[i] = f;
      D[i + 1] -= f * DU[i];
    } else {
      const double f = D[i] * fast_rcp(DL[i]);
      D[i] = DL[i];
      DL[i] = f;
      const double t = DU[i];
      DU[i] = D[i + 1];
      D[i + 1] = t - f * D[i + 1];
      if (i + 2 < m) {
        DU2[i] = DU[i + 1];
        DU[i + 1] = -f * DU[i + 1];
      }
      ipiv[i] = 1;
    }
  }
  for (int i = 0; i < m; ++i) {  // store reciprocals: the solves then chain FMAs only
    double di = D[i];
    if (fabs(di) < tiny) di = di < 0.0 ? -tiny : tiny;
    D[i] = 1.0 / di;
  }
}

__device__ void gtts2(int m, const double* D, const double* DL, const double* DU, const double* DU2,
                      const int* ipiv, double* b) {
  for (int i = 0; i + 1 < m; ++i) {
    if (!ipiv[i]) {
      b[i + 1] -= DL[i] * b[i];
    } else {
      const double t = b[i];
      b[i] = b[i + 1];
      b[i + 1] = t - DL[i] * b[i];
    }
  }
  // D holds 1 / diag(U)
  b[m - 1] *= D[m - 1];
  if (m >= 2) b[m - 2] = (b[m - 2] - DU[m - 2] * b[m - 1]) * D[m - 2];
  for (int i = m - 3; i >= 0; --i) b[i] = (b[i] - DU[i] * b[i + 1] - DU2[i] * b[i + 2]) * D[i];
}

__global__ void tri_eigvecs_kernel(TriArgs p) {
  const int m = p.m, lane = threadIdx.x & 31;
  const int cl = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (cl >= m) return;
  double lo, hi, tnorm, pivmin;
  tri_bounds(m, p.d, p.e, lo, hi, tnorm, pivmin);
  // reorthogonalisation threshold: dstein uses 1e-3 ||T||; inverse iteration leaves a
  // non-orthogonality of O(eps ||T|| / gap), so 1e-5 ||T|| already bounds it by ~1e-11 while
  // keeping FEAST's dense interior Ritz spectra from chaining into one long cluster
  const double ortol = 1e-5 * tnorm, eps = DBL_EPSILON;
  if (cl > 0 && p.lam[cl] - p.lam[cl - 1] <= ortol) return;  // not the first of its cluster
  int cend = cl + 1;
  while (cend < m && p.lam[cend] - p.lam[cend - 1] <= ortol) ++cend;
  // per-warp shared scratch: LU bands, pivots, the iterate (the O(m) recurrences run on
  // lane 0 against shared memory, not L2)
  extern __shared__ double wsm[];
  double* D = wsm + (threadIdx.x >> 5) * 6 * m;
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
    if (lane == 0) gttrf(m, p.d, p.e, lam, D, DL, DU, DU2, ipiv, eps * tnorm);
    double* zj = zs;
    for (int i = lane; i < m; i += 32) {  // deterministic pseudo-random start
      uint32_t h = (uint32_t)i * 2654435761u ^ ((uint32_t)j * 40503u + 12345u);
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      zj[i] = 0.5 + (double)(h & 0xffff) / 65536.0;
    }
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
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
// 4. back-transformation V = H_0 ... H_{m-3} Z, one warp per column
// ---------------------------------------------------------------------------
// the column stays in registers (8 per lane: m <= 256); the next reflector is loaded while
// the current one is applied, so the only serial latency is the warp reduction
__global__ void tri_back_kernel(int m, const double* __restrict__ hv, const double* __restrict__ tau,
                                const double* __restrict__ z, double* v) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= m) return;
  constexpr int PD = 4;  // reflectors in flight (one L2 latency ~ a few reflector steps)
  double x[8], h[PD][8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = lane + 32 * q;
    x[q] = i < m ? z[i + (int64_t)c * m] : 0.0;
  }
  auto load = [&](int k, double* dst) {
    const double* hk = hv + (int64_t)k * m;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = lane + 32 * q;
      dst[q] = (k >= 0 && i > k && i < m) ? hk[i] : 0.0;
    }
  };
#pragma unroll
  for (int s = 0; s < PD; ++s) load(m - 3 - s, h[s]);
  for (int k = m - 3; k >= 0; k -= PD) {
#pragma unroll
    for (int s = 0; s < PD; ++s) {
      const int kk = k - s;
      if (kk >= 0) {
        const double t = tau[kk];
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += h[s][q] * x[q];
        sum = warp_sum(sum) * t;
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] -= sum * h[s][q];
      }
      load(kk - PD, h[s]);  // refill this slot PD reflectors ahead
    }
  }
  double* vc = v + (int64_t)c * m;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = lane + 32 * q;
    if (i < m) vc[i] = x[q];
  }
}

// packed m(m+1)/2 + v, w (2m) doubles <= 226 KB; 4 threads per trailing row (1024 threads)
int tri_max_dim() { return 236; }

// a (m x m, overwritten is allowed), eigenvalues ascending -> evals, vectors -> v (m x m)
cudaError_t tri_eig(int m, const double* a, double* evals, double* v, double* ws, int* iws, cudaStream_t st) {
  if (m < 1 || m > tri_max_dim()) return cudaErrorInvalidValue;
  double* d = ws;
  double* e = d + m;
  double* tau = e + m;
  double* hv = tau + m;            // m*m
  double* z = hv + (size_t)m * m;  // m*m
  double* lu = z + (size_t)m * m;  // 4*m*m
  const size_t sm = sizeof(double) * ((size_t)m * (m + 1) / 2 + 2 * m);
  static bool attr = false;
  if (!attr) {
    // dynamic + static (the reduction scratch) must stay within the 227 KB opt-in limit
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    attr = true;
  }
  tridiag_kernel<<<1, 1024, sm, st>>>(m, a, d, e, hv, tau);
  ++g_launches;
  TriArgs p{m, d, e, evals, z, lu, iws};
  const int wpb = 4;
  tri_eigvals_kernel<<<(m + wpb - 1) / wpb, 32 * wpb, sizeof(double) * 2 * m, st>>>(p);
  ++g_launches;
  tri_eigvecs_kernel<<<(m + wpb - 1) / wpb, 32 * wpb, sizeof(double) * 6 * m * wpb + 64, st>>>(p);
  ++g_launches;
  tri_back_kernel<<<(m + 7) / 8, 256, 0, st>>>(m, hv, tau, z, v);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
