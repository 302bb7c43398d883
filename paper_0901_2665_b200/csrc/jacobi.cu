// jacobi.cu — symmetric eigendecomposition of the reduced matrix on device (the role of
// jacobi_eigh, eigh.hpp:84-163): eigenvalues ascending in a stable order, orthonormal
// eigenvectors. Same method class as the reference — cyclic Jacobi, so repeated and tiny
// eigenvalues come out as accurately — re-shaped for 148 SMs as BLOCK Jacobi:
//
//   * the m x m matrix is cut into 2k blocks of bs rows (padded with decoupled zeros);
//   * each outer round pairs the blocks by the circle method; every pair's 2bs x 2bs
//     sub-problem is swept once in shared memory by parallel round-robin Jacobi (phase A:
//     one CTA per pair, ONE barrier per inner round — the sub-matrix is double-buffered and
//     every thread recomputes the two rotations its 2x2 block needs);
//   * the accumulated pair rotations are applied to W (J_a^T W_ab J_b) and V (V_b J_b) as
//     small GEMM tiles by all CTAs (phase B);
//   * one cooperative kernel; two grid barriers per outer round, a fixed-order grid
//     reduction of the off-diagonal norm per sweep (the stopping rule of eigh.hpp:98).

#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include <mutex>
#include <vector>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

// fixed-order block reduction (run-to-run deterministic)
static __device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  return red[32];
}

int tri_max_dim();
cudaError_t tri_eig(int m, const double* a, double* evals, double* v, double* ws, int* iws, cudaStream_t st,
                    double vfloor);

struct EigWork {
  int mmax = 0;
  double* w = nullptr;     // mp x mp
  double* v = nullptr;     // mp x mp
  double* j = nullptr;     // npair * (2bs)^2
  double* part = nullptr;  // per-CTA partial sums
  unsigned long long* dbg = nullptr;
  double* tws = nullptr;   // tridiagonal route (m <= tri_max_dim): 6m^2 + 3m
  int* tiws = nullptr;     // m^2
  int grid = 0;
  int dev = 0;
};

// Process-wide cache of released workspaces: a fresh context (every end-to-end solve opens one)
// takes a cached set of the same size instead of seven cudaMalloc calls, and a destroyed one
// parks its set instead of seven device-synchronising cudaFree calls.
static std::mutex g_eig_mu;
static std::vector<EigWork*> g_eig_cache;
constexpr size_t kEigCacheMax = 4;

static int eig_bs(int m) { return m <= 256 ? 16 : 32; }
static int eig_mp(int m) {
  const int bs = eig_bs(m);
  int nblk = (m + bs - 1) / bs;
  if (nblk < 2) nblk = 2;
  if (nblk & 1) ++nblk;
  return nblk * bs;
}

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
  const int mp = std::max(eig_mp(mmax), eig_mp(std::min(mmax, 256)));
  cudaMalloc(&w->w, sizeof(double) * mp * mp);
  cudaMalloc(&w->v, sizeof(double) * mp * mp);
  cudaMalloc(&w->j, sizeof(double) * (mp / 32 + 2) * (4 * 32 * 32));
  cudaMalloc(&w->part, sizeof(double) * 1024);
  cudaMalloc(&w->dbg, sizeof(unsigned long long) * 8);
  const size_t tm = (size_t)std::min(mmax, tri_max_dim());
  cudaMalloc(&w->tws, sizeof(double) * (6 * tm * tm + 3 * tm));
  cudaMalloc(&w->tiws, sizeof(int) * tm * tm);
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  w->grid = sms;
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
  cudaFree(w->w);
  cudaFree(w->v);
  cudaFree(w->j);
  cudaFree(w->part);
  cudaFree(w->dbg);
  cudaFree(w->tws);
  cudaFree(w->tiws);
  delete w;
}

// circle-method tournament of n players: round r, pair i -> (p, q)
__device__ __forceinline__ void tourney(int n, int r, int i, int& p, int& q) {
  p = i == 0 ? 0 : 1 + (r + i - 1) % (n - 1);
  const int k2 = n - 1 - i;
  q = k2 == 0 ? 0 : 1 + (r + k2 - 1) % (n - 1);
  if (p > q) { const int t = p; p = q; q = t; }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct JacobiArgs {
  int m, mp, bs;
  const double* a;  // input m x m (ld m)
  double* w;
  double* v;
  double* jb;
  double* part;
  int max_sweeps;
  unsigned long long* dbg;  // optional: ns in phase A, phase B, sweeps, rounds
};

// deterministic grid-wide sum: every CTA writes its partial, then every CTA adds them in order
__device__ double grid_sum(cg::grid_group& grid, double mine, double* part, double* red) {
  const double s = block_sum(mine, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  grid.sync();
  double tot = 0.0;
  for (int c = 0; c < (int)gridDim.x; ++c) tot += part[c];
  grid.sync();
  return tot;
}

// Jacobi rotation for (app, aqq, apq) with jacobi_eigh's formulas (eigh.hpp:116-124), as
// R = [[c, s], [-ph s, ph c]] (rows: old p, q; columns: new p, q). Identity below the floor.
struct Rot {
  double c, s, mps, pc;  // c, s, -ph*s, ph*c
};
__device__ __forceinline__ Rot make_rot(double app, double aqq, double apq, double tiny) {
  Rot r{1.0, 0.0, 0.0, 1.0};
  const double aa = fabs(apq);
  if (aa > tiny && aa > DBL_EPSILON * 0.5 * (fabs(app) + fabs(aqq))) {
    const double ph = apq > 0.0 ? 1.0 : -1.0;
    const double tau = (aqq - app) / (2.0 * aa);
    const double at = fabs(tau);
    // t = sign(tau) / (|tau| + sqrt(1 + tau^2)); for huge |tau| sqrt would overflow
    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (at < 1e150 ? at + sqrt(1.0 + tau * tau) : 2.0 * at);
    const double c = rsqrt(1.0 + t * t);
    const double s = t * c;
    r.c = c;
    r.s = s;
    r.mps = -ph * s;
    r.pc = ph * c;
  }
  return r;
}

__global__ void __launch_bounds__(256) block_jacobi_kernel(JacobiArgs p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double jsm[];
  __shared__ double red[33];
  __shared__ unsigned char ptab[63 * 32 * 2];  // inner tournament: (tb-1) rounds x bs pairs
  __shared__ Rot rot[32];
  const int m = p.m, mp = p.mp, bs = p.bs, tb = 2 * bs, ldt = tb + 1;
  const int nblk = mp / bs, npair = nblk / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t gtid = blockIdx.x * (int64_t)nt + tid, gstride = (int64_t)gridDim.x * nt;
  const bool prof = p.dbg && blockIdx.x == 0 && tid == 0;
  unsigned long long tA = 0, tB = 0, t0 = 0;
  int nsweeps = 0, nrounds = 0;

  for (int e = tid; e < (tb - 1) * bs; e += nt) {
    int pp, qq;
    tourney(tb, e / bs, e % bs, pp, qq);
    ptab[2 * e] = (unsigned char)pp;
    ptab[2 * e + 1] = (unsigned char)qq;
  }
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
  const double tol_off = m * DBL_EPSILON * scale;  // jacobi_eigh stopping rule (eigh.hpp:98)
  const double tiny = DBL_EPSILON * scale / m;     // rotations below this are skipped

  double* S0 = jsm;              // tb x ldt, double-buffered sub-problem
  double* S1 = S0 + tb * ldt;
  double* Jm = S1 + tb * ldt;    // tb x ldt accumulated rotation

  for (int sweep = 0; sweep < p.max_sweeps; ++sweep) {
    double off = 0.0;
    for (int64_t idx = gtid; idx < (int64_t)mp * mp; idx += gstride) {
      const int i = (int)(idx % mp), j = (int)(idx / mp);
      if (i != j) off += p.w[idx] * p.w[idx];
    }
    off = sqrt(grid_sum(grid, off, p.part, red));
    if (off <= tol_off) break;
    ++nsweeps;

    for (int r = 0; r < nblk - 1; ++r) {
      ++nrounds;
      if (prof) t0 = gtime();
      // ---------- phase A: one parallel Jacobi sweep over each pair's sub-problem ----------
      for (int pi = blockIdx.x; pi < npair; pi += gridDim.x) {
        int P, Q;
        tourney(nblk, r, pi, P, Q);
        for (int idx = tid; idx < tb * tb; idx += nt) {
          const int u = idx % tb, v = idx / tb;
          const int gu = u < bs ? P * bs + u : Q * bs + u - bs;
          const int gv = v < bs ? P * bs + v : Q * bs + v - bs;
          cp_async8z(S0 + u + v * ldt, p.w + gu + (int64_t)gv * mp, true);
          Jm[u + v * ldt] = u == v ? 1.0 : 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        double* Sc = S0;
        double* Sn = S1;
        for (int ir = 0; ir < tb - 1; ++ir) {
          const unsigned char* pr = ptab + 2 * ir * bs;
          // rotations of this inner round, one thread per pair (the FP64 div/sqrt chain is
          // the latency floor of an inner round, so it is computed once, not per use)
          if (tid < bs) {
            const int pp = pr[2 * tid], qq = pr[2 * tid + 1];
            rot[tid] = make_rot(Sc[pp + pp * ldt], Sc[qq + qq * ldt], Sc[pp + qq * ldt], tiny);
          }
          __syncthreads();
          // S_next = R^T S R on 2x2 blocks
          for (int t = tid; t < bs * bs; t += nt) {
            const int ka = t % bs, kb = t / bs;
            const int pa = pr[2 * ka], qa = pr[2 * ka + 1], pb = pr[2 * kb], qb = pr[2 * kb + 1];
            const Rot ra = rot[ka];
            const Rot rb = rot[kb];
            const double x00 = Sc[pa + pb * ldt], x01 = Sc[pa + qb * ldt];
            const double x10 = Sc[qa + pb * ldt], x11 = Sc[qa + qb * ldt];
            const double y00 = x00 * rb.c + x01 * rb.mps, y01 = x00 * rb.s + x01 * rb.pc;
            const double y10 = x10 * rb.c + x11 * rb.mps, y11 = x10 * rb.s + x11 * rb.pc;
            double z00 = ra.c * y00 + ra.mps * y10, z01 = ra.c * y01 + ra.mps * y11;
            double z10 = ra.s * y00 + ra.pc * y10, z11 = ra.s * y01 + ra.pc * y11;
            if (ka == kb && ra.s != 0.0) { z01 = 0.0; z10 = 0.0; }
            Sn[pa + pb * ldt] = z00;
            Sn[pa + qb * ldt] = z01;
            Sn[qa + pb * ldt] = z10;
            Sn[qa + qb * ldt] = z11;
          }
          // J <- J R (columns pb, qb)
          for (int t = tid; t < tb * bs; t += nt) {
            const int row = t % tb, kb = t / tb;
            const int pb = pr[2 * kb], qb = pr[2 * kb + 1];
            const Rot rb = rot[kb];
            const double x0 = Jm[row + pb * ldt], x1 = Jm[row + qb * ldt];
            Jm[row + pb * ldt] = x0 * rb.c + x1 * rb.mps;
            Jm[row + qb * ldt] = x0 * rb.s + x1 * rb.pc;
          }
          __syncthreads();
          double* t2 = Sc;
          Sc = Sn;
          Sn = t2;
        }
        double* J = p.jb + (int64_t)pi * tb * tb;
        for (int idx = tid; idx < tb * tb; idx += nt) J[idx] = Jm[(idx % tb) + (idx / tb) * ldt];
        __syncthreads();
      }
      if (prof) { const unsigned long long t1 = gtime(); tA += t1 - t0; t0 = t1; }
      grid.sync();
      // ---------- phase B: W <- J^T W J (block pairs), V <- V J ----------
      double* X = jsm;               // tb x ldt
      double* Ja = X + tb * ldt;     // tb x ldt
      double* Jb = Ja + tb * ldt;    // tb x ldt
      double* Y = Jb + tb * ldt;     // tb x ldt
      const int nrc = mp / tb;       // V row chunks
      const int ntask = npair * npair + nrc * npair;
      for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
        const bool wt = task < npair * npair;
        int ia = 0, ib, rc = 0;
        if (wt) { ia = task % npair; ib = task / npair; }
        else { const int t2 = task - npair * npair; rc = t2 % nrc; ib = t2 / nrc; }
        int Pa = 0, Qa = 0, Pb, Qb;
        if (wt) tourney(nblk, r, ia, Pa, Qa);
        tourney(nblk, r, ib, Pb, Qb);
        const double* JA = p.jb + (int64_t)ia * tb * tb;
        const double* JB = p.jb + (int64_t)ib * tb * tb;
        for (int idx = tid; idx < tb * tb; idx += nt) {
          const int u = idx % tb, v = idx / tb;
          const int gv = v < bs ? Pb * bs + v : Qb * bs + v - bs;
          if (wt) {
            const int gu = u < bs ? Pa * bs + u : Qa * bs + u - bs;
            cp_async8z(X + u + v * ldt, p.w + gu + (int64_t)gv * mp, true);
            cp_async8z(Ja + u + v * ldt, JA + idx, true);
          } else {
            cp_async8z(X + u + v * ldt, p.v + (rc * tb + u) + (int64_t)gv * mp, true);
          }
          cp_async8z(Jb + u + v * ldt, JB + idx, true);
        }
        cp_async_wait_all();
        __syncthreads();
        // Y = X Jb; 2x2 register tile per thread
        for (int t = tid; t < (tb / 2) * (tb / 2); t += nt) {
          const int u = 2 * (t % (tb / 2)), v = 2 * (t / (tb / 2));
          double s00 = 0, s01 = 0, s10 = 0, s11 = 0;
          for (int k = 0; k < tb; ++k) {
            const double x0 = X[u + k * ldt], x1 = X[u + 1 + k * ldt];
            const double j0 = Jb[k + v * ldt], j1 = Jb[k + (v + 1) * ldt];
            s00 += x0 * j0; s01 += x0 * j1; s10 += x1 * j0; s11 += x1 * j1;
          }
          if (wt) {
            Y[u + v * ldt] = s00; Y[u + (v + 1) * ldt] = s01;
            Y[u + 1 + v * ldt] = s10; Y[u + 1 + (v + 1) * ldt] = s11;
          } else {
            const int gv0 = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            const int gv1 = v + 1 < bs ? Pb * bs + v + 1 : Qb * bs + v + 1 - bs;
            double* vv = p.v + rc * tb + u;
            vv[(int64_t)gv0 * mp] = s00; vv[1 + (int64_t)gv0 * mp] = s10;
            vv[(int64_t)gv1 * mp] = s01; vv[1 + (int64_t)gv1 * mp] = s11;
          }
        }
        if (wt) {
          __syncthreads();
          for (int t = tid; t < (tb / 2) * (tb / 2); t += nt) {  // W = Ja^T Y
            const int u = 2 * (t % (tb / 2)), v = 2 * (t / (tb / 2));
            double s00 = 0, s01 = 0, s10 = 0, s11 = 0;
            for (int k = 0; k < tb; ++k) {
              const double a0 = Ja[k + u * ldt], a1 = Ja[k + (u + 1) * ldt];
              const double y0 = Y[k + v * ldt], y1 = Y[k + (v + 1) * ldt];
              s00 += a0 * y0; s01 += a0 * y1; s10 += a1 * y0; s11 += a1 * y1;
            }
            const int gu0 = u < bs ? Pa * bs + u : Qa * bs + u - bs;
            const int gu1 = u + 1 < bs ? Pa * bs + u + 1 : Qa * bs + u + 1 - bs;
            const int gv0 = v < bs ? Pb * bs + v : Qb * bs + v - bs;
            const int gv1 = v + 1 < bs ? Pb * bs + v + 1 : Qb * bs + v + 1 - bs;
            p.w[gu0 + (int64_t)gv0 * mp] = s00; p.w[gu0 + (int64_t)gv1 * mp] = s01;
            p.w[gu1 + (int64_t)gv0 * mp] = s10; p.w[gu1 + (int64_t)gv1 * mp] = s11;
          }
        }
        __syncthreads();
      }
      if (prof) { const unsigned long long t1 = gtime(); tB += t1 - t0; }
      grid.sync();
    }
  }
  if (prof) {
    p.dbg[0] = tA;
    p.dbg[1] = tB;
    p.dbg[2] = nsweeps;
    p.dbg[3] = nrounds;
  }
}

// ascending stable sort of diag(W)[0..m) with the eigenvector columns (eigh.hpp:152-162)
__global__ void eig_sort_kernel(int m, int mp, const double* w, const double* v, double* evals,
                                double* vout) {
  const int i = blockIdx.x;
  __shared__ int rank_s;
  __shared__ int wc[32];
  const double di = w[i + (int64_t)i * mp];
  int cnt = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double dj = w[j + (int64_t)j * mp];
    cnt += (dj < di || (dj == di && j < i)) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
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

cudaError_t sym_eig(EigWork* w, int m, double* a, double* evals, double* v, cudaStream_t st, double vfloor) {
  if (m < 1 || m > w->mmax) return cudaErrorInvalidValue;
  // tridiagonal route up to m = 1024 (shared-memory reduction, preceded by an L2-resident
  // stage for m > 236; FEAST_EIG=jacobi
  // forces block Jacobi for comparison)
  static const char* force = getenv("FEAST_EIG");
  const bool jacobi_only = force && force[0] == 'j';
  if (m <= tri_max_dim() && !jacobi_only) return tri_eig(m, a, evals, v, w->tws, w->tiws, st, vfloor);
  static const bool debug = getenv("FEAST_EIG_DEBUG") != nullptr;
  const int bs = eig_bs(m), mp = eig_mp(m), tb = 2 * bs, ldt = tb + 1;
  JacobiArgs p{m, mp, bs, a, w->w, w->v, w->j, w->part, 60, debug ? w->dbg : nullptr};
  const size_t sm = sizeof(double) * 4 * tb * ldt;
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
  if (debug) {
    unsigned long long h[4];
    cudaMemcpyAsync(h, w->dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[sym_eig m=%d bs=%d grid=%d] sweeps=%llu rounds=%llu phaseA=%.1fus phaseB=%.1fus\n", m, bs,
            grid, h[2], h[3], h[0] * 1e-3, h[1] * 1e-3);
  }
  return cudaGetLastError();
}

}  // namespace feastgpu
