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

#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

// ---------------------------------------------------------------------------
// Cholesky (single CTA, left-looking by columns)
// ---------------------------------------------------------------------------
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  return red[32];
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

// ---------------------------------------------------------------------------
// Block Jacobi symmetric eigensolver
// ---------------------------------------------------------------------------
struct EigWork {
  int mmax = 0;
  double* w = nullptr;     // mp x mp
  double* v = nullptr;     // mp x mp
  double* j = nullptr;     // npair * (2bs)^2
  double* part = nullptr;  // per-CTA partial sums
  int grid = 0;
};

static int eig_bs(int m) { return m <= 256 ? 16 : 32; }
static int eig_mp(int m) {
  const int bs = eig_bs(m);
  int nblk = (m + bs - 1) / bs;
  if (nblk < 2) nblk = 2;
  if (nblk & 1) ++nblk;
  return nblk * bs;
}

EigWork* eig_create(int mmax) {
  EigWork* w = new EigWork();
  w->mmax = mmax;
  const int mp = std::max(eig_mp(mmax), eig_mp(std::min(mmax, 256)));
  const int bs = 32;
  cudaMalloc(&w->w, sizeof(double) * mp * mp);
  cudaMalloc(&w->v, sizeof(double) * mp * mp);
  cudaMalloc(&w->j, sizeof(double) * (mp / 2 / 16 + 1) * (4 * bs * bs));
  cudaMalloc(&w->part, sizeof(double) * 1024);
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  w->grid = sms;
  return w;
}

void eig_destroy(EigWork* w) {
  if (!w) return;
  cudaFree(w->w);
  cudaFree(w->v);
  cudaFree(w->j);
  cudaFree(w->part);
  delete w;
}

// circle-method tournament: round r, pair i -> (blocks p, q)
__device__ __forceinline__ void tourney(int nblk, int r, int i, int& p, int& q) {
  auto pos = [&](int k) { return k == 0 ? 0 : 1 + (r + k - 1) % (nblk - 1); };
  p = pos(i);
  q = pos(nblk - 1 - i);
}

struct JacobiArgs {
  int m, mp, bs;
  const double* a;   // input m x m (ld m)
  double* w;
  double* v;
  double* jb;
  double* part;
  int max_sweeps;
};

// deterministic grid-wide sum: every CTA writes its partial, then every CTA adds them in order
__device__ double grid_sum(cg::grid_group& grid, double mine, double* part, double* red) {
  const double s = block_sum(mine, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  grid.sync();
  double tot = 0.0;
  for (int c = 0; c < (int)gridDim.x; ++c) tot += part[c];
  grid.sync();  // part[] may be reused afterwards
  return tot;
}

__global__ void __launch_bounds__(256) block_jacobi_kernel(JacobiArgs p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double jsm[];
  __shared__ double red[33];
  const int m = p.m, mp = p.mp, bs = p.bs, tb = 2 * bs, ldt = tb + 1;
  const int nblk = mp / bs, npair = nblk / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t gtid = blockIdx.x * (int64_t)nt + tid, gstride = (int64_t)gridDim.x * nt;
  constexpr double eps = DBL_EPSILON;

  // pad: W = [a 0; 0 0], V = I
  for (int64_t idx = gtid; idx < (int64_t)mp * mp; idx += gstride) {
    const int i = (int)(idx % mp), j = (int)(idx / mp);
    p.w[idx] = (i < m && j < m) ? p.a[i + (int64_t)j * m] : 0.0;
    p.v[idx] = i == j ? 1.0 : 0.0;
  }
  grid.sync();
  double fro = 0.0;
  for (int64_t idx = gtid; idx < (int64_t)mp * mp; idx += gstride) fro += p.w[idx] * p.w[idx];
  const double scale = fmax(sqrt(grid_sum(grid, fro, p.part, red)), DBL_MIN);
  const double tol_off = m * eps * scale;            // jacobi_eigh stopping rule (eigh.hpp:98)
  const double tiny = eps * scale / m;               // rotations below this are skipped

  double* S = jsm;                 // tb x ldt
  double* Jm = S + tb * ldt;       // tb x ldt
  double* rot = Jm + tb * ldt;     // bs x 4 (c, s_eff, ...)
  int* rp = reinterpret_cast<int*>(rot + 4 * bs);  // bs x 2
  __shared__ int any_rot;

  for (int sweep = 0; sweep < p.max_sweeps; ++sweep) {
    double off = 0.0;
    for (int64_t idx = gtid; idx < (int64_t)mp * mp; idx += gstride) {
      const int i = (int)(idx % mp), j = (int)(idx / mp);
      if (i != j) off += p.w[idx] * p.w[idx];
    }
    off = sqrt(grid_sum(grid, off, p.part, red));
    if (off <= tol_off) break;

    for (int r = 0; r < nblk - 1; ++r) {
      // ---------- phase A: diagonalise each pair's 2bs x 2bs sub-problem ----------
      for (int pi = blockIdx.x; pi < npair; pi += gridDim.x) {
        int P, Q;
        tourney(nblk, r, pi, P, Q);
        for (int idx = tid; idx < tb * tb; idx += nt) {
          const int u = idx % tb, v = idx / tb;
          const int gu = u < bs ? P * bs + u : Q * bs + u - bs;
          const int gv = v < bs ? P * bs + v : Q * bs + v - bs;
          S[u + v * ldt] = p.w[gu + (int64_t)gv * mp];
          Jm[u + v * ldt] = u == v ? 1.0 : 0.0;
        }
        __syncthreads();
        // one or two inner sweeps per pair visit: block Jacobi converges without fully
        // diagonalising each sub-problem, and every inner round costs two CTA barriers
        for (int isw = 0; isw < 2; ++isw) {
          if (tid == 0) any_rot = 0;
          __syncthreads();
          for (int ir = 0; ir < tb - 1; ++ir) {
            // rotation parameters (jacobi_eigh's formulas, eigh.hpp:104-124)
            for (int k = tid; k < bs; k += nt) {
              const int a0 = k == 0 ? 0 : 1 + (ir + k - 1) % (tb - 1);
              const int k2 = tb - 1 - k;
              const int b0 = k2 == 0 ? 0 : 1 + (ir + k2 - 1) % (tb - 1);
              const int pp = min(a0, b0), qq = max(a0, b0);
              const double apq = S[pp + qq * ldt];
              const double aa = fabs(apq);
              const double app = S[pp + pp * ldt], aqq = S[qq + qq * ldt];
              double c = 1.0, sph = 0.0, phc = 1.0;
              // skip rotations below the global stopping floor (their squares sum to at
              // most (eps*scale)^2 < tol_off^2) or at round-off relative to the diagonal
              if (aa > tiny && aa > eps * 0.5 * (fabs(app) + fabs(aqq))) {
                const double ph = apq > 0.0 ? 1.0 : -1.0;
                const double tau = (aqq - app) / (2.0 * aa);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + hypot(1.0, tau));
                c = 1.0 / sqrt(1.0 + t * t);
                const double s = t * c;
                sph = ph * s;
                phc = ph * c;
                rot[4 * k + 3] = s;
                any_rot = 1;
              } else {
                rot[4 * k + 3] = 0.0;
              }
              rot[4 * k + 0] = c;
              rot[4 * k + 1] = sph;
              rot[4 * k + 2] = phc;
              rp[2 * k] = pp;
              rp[2 * k + 1] = qq;
            }
            __syncthreads();
            // S <- R^T S R on 2x2 blocks; R = [[c, s], [-ph s, ph c]]
            for (int t = tid; t < bs * bs; t += nt) {
              const int ka = t % bs, kb = t / bs;
              const int pa = rp[2 * ka], qa = rp[2 * ka + 1], pb = rp[2 * kb], qb = rp[2 * kb + 1];
              const double ca = rot[4 * ka], sa = rot[4 * ka + 3], mpsa = -rot[4 * ka + 1], pca = rot[4 * ka + 2];
              const double cb = rot[4 * kb], sb = rot[4 * kb + 3], mpsb = -rot[4 * kb + 1], pcb = rot[4 * kb + 2];
              const double x00 = S[pa + pb * ldt], x01 = S[pa + qb * ldt];
              const double x10 = S[qa + pb * ldt], x11 = S[qa + qb * ldt];
              const double y00 = x00 * cb + x01 * mpsb, y01 = x00 * sb + x01 * pcb;
              const double y10 = x10 * cb + x11 * mpsb, y11 = x10 * sb + x11 * pcb;
              double z00 = ca * y00 + mpsa * y10, z01 = ca * y01 + mpsa * y11;
              double z10 = sa * y00 + pca * y10, z11 = sa * y01 + pca * y11;
              if (ka == kb) { z01 = 0.0; z10 = 0.0; }
              S[pa + pb * ldt] = z00;
              S[pa + qb * ldt] = z01;
              S[qa + pb * ldt] = z10;
              S[qa + qb * ldt] = z11;
            }
            for (int t = tid; t < tb * bs; t += nt) {
              const int row = t % tb, kb = t / tb;
              const int pb = rp[2 * kb], qb = rp[2 * kb + 1];
              const double cb = rot[4 * kb], sb = rot[4 * kb + 3], mpsb = -rot[4 * kb + 1], pcb = rot[4 * kb + 2];
              const double x0 = Jm[row + pb * ldt], x1 = Jm[row + qb * ldt];
              Jm[row + pb * ldt] = x0 * cb + x1 * mpsb;
              Jm[row + qb * ldt] = x0 * sb + x1 * pcb;
            }
            __syncthreads();
          }
          if (!any_rot) break;
        }
        double* J = p.jb + (int64_t)pi * tb * tb;
        for (int idx = tid; idx < tb * tb; idx += nt) J[idx] = Jm[(idx % tb) + (idx / tb) * ldt];
        __syncthreads();
      }
      grid.sync();
      // ---------- phase B: W <- J^T W J (block pairs), V <- V J ----------
      double* X = jsm;               // tb x ldt
      double* Ja = X + tb * ldt;     // tb x ldt
      double* Jb = Ja + tb * ldt;    // tb x ldt
      double* Y = Jb + tb * ldt;     // tb x ldt
      const int nrc = mp / tb;       // V row chunks
      const int ntask = npair * npair + nrc * npair;
      for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
        if (task < npair * npair) {
          const int ia = task % npair, ib = task / npair;
          int Pa, Qa, Pb, Qb;
          tourney(nblk, r, ia, Pa, Qa);
          tourney(nblk, r, ib, Pb, Qb);
          const double* JA = p.jb + (int64_t)ia * tb * tb;
          const double* JB = p.jb + (int64_t)ib * tb * tb;
          for (int idx = tid; idx < tb * tb; idx += nt) {
            const int u = idx % tb, v = idx / tb;
            const int gu = u < bs ? Pa * bs + u : Qa * bs + u - bs;
            const int gv = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            X[u + v * ldt] = p.w[gu + (int64_t)gv * mp];
            Ja[u + v * ldt] = JA[idx];
            Jb[u + v * ldt] = JB[idx];
          }
          __syncthreads();
          for (int idx = tid; idx < tb * tb; idx += nt) {  // Y = X Jb
            const int u = idx % tb, v = idx / tb;
            double s = 0.0;
            for (int k = 0; k < tb; ++k) s += X[u + k * ldt] * Jb[k + v * ldt];
            Y[u + v * ldt] = s;
          }
          __syncthreads();
          for (int idx = tid; idx < tb * tb; idx += nt) {  // W = Ja^T Y
            const int u = idx % tb, v = idx / tb;
            double s = 0.0;
            for (int k = 0; k < tb; ++k) s += Ja[k + u * ldt] * Y[k + v * ldt];
            const int gu = u < bs ? Pa * bs + u : Qa * bs + u - bs;
            const int gv = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            p.w[gu + (int64_t)gv * mp] = s;
          }
          __syncthreads();
        } else {
          const int t2 = task - npair * npair;
          const int rc = t2 % nrc, ib = t2 / nrc;
          int Pb, Qb;
          tourney(nblk, r, ib, Pb, Qb);
          const double* JB = p.jb + (int64_t)ib * tb * tb;
          for (int idx = tid; idx < tb * tb; idx += nt) {
            const int u = idx % tb, v = idx / tb;
            const int gv = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            X[u + v * ldt] = p.v[(rc * tb + u) + (int64_t)gv * mp];
            Jb[u + v * ldt] = JB[idx];
          }
          __syncthreads();
          for (int idx = tid; idx < tb * tb; idx += nt) {
            const int u = idx % tb, v = idx / tb;
            double s = 0.0;
            for (int k = 0; k < tb; ++k) s += X[u + k * ldt] * Jb[k + v * ldt];
            const int gv = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            p.v[(rc * tb + u) + (int64_t)gv * mp] = s;
          }
          __syncthreads();
        }
      }
      grid.sync();
    }
  }
}

// ascending stable sort of diag(W)[0..m) with the eigenvector columns (eigh.hpp:152-162)
__global__ void eig_sort_kernel(int m, int mp, const double* w, const double* v, double* evals,
                                double* vout) {
  const int i = blockIdx.x;
  __shared__ int rank_s;
  const double di = w[i + (int64_t)i * mp];
  int cnt = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double dj = w[j + (int64_t)j * mp];
    cnt += (dj < di || (dj == di && j < i)) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int wc[32];
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += wc[k];
    rank_s = t;
    evals[t] = di;
  }
  __syncthreads();
  const int rk = rank_s;
  for (int r = threadIdx.x; r < m; r += blockDim.x) vout[r + (int64_t)rk * m] = v[r + (int64_t)i * mp];
}

cudaError_t sym_eig(EigWork* w, int m, double* a, double* evals, double* v, cudaStream_t st) {
  if (m < 1 || m > w->mmax) return cudaErrorInvalidValue;
  const int bs = eig_bs(m), mp = eig_mp(m), tb = 2 * bs, ldt = tb + 1;
  JacobiArgs p{m, mp, bs, a, w->w, w->v, w->j, w->part, 60};
  const size_t smA = sizeof(double) * (2 * tb * ldt + 4 * bs) + sizeof(int) * 2 * bs;
  const size_t smB = sizeof(double) * 4 * tb * ldt;
  const size_t sm = std::max(smA, smB);
  cudaFuncSetAttribute(block_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, block_jacobi_kernel, 256, sm);
  const int npair = mp / bs / 2;
  const int ntask = npair * npair + (mp / tb) * npair;
  int grid = std::min(w->grid * std::max(occ, 1), std::max(ntask, npair));
  grid = std::min(grid, 1024);
  void* args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)block_jacobi_kernel, grid, 256, args, sm, st);
  ++g_launches;
  if (e != cudaSuccess) return e;
  eig_sort_kernel<<<m, 128, 0, st>>>(m, mp, w->w, w->v, evals, v);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
