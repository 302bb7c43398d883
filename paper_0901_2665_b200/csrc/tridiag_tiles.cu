// tridiag_tiles.cu — Householder tridiagonalisation (dsytd2, lower) of the reduced matrix
// for m <= 192 on ONE SM with the matrix resident in REGISTERS.
//
// Same output contract as tridiag_kernel (tridiag.cu): d[m], e[m-1], tau[m], hv (m x m,
// column k holds v_k in rows k+1.., v_k[k+1] = 1). The arithmetic per column is the
// reference-style reflector (beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta) applied
// as A22 -= v w^T + w v^T, w = p - (tau/2)(p.v) v, p = tau A22 v; the eigenvalues agree with
// jacobi_eigh (eigh.hpp:84-163) to rounding (tests/test_gpu_parity.py).
//
// Layout: the (padded) matrix is cut into 16 x 16 tiles; the nb(nb+1)/2 lower tiles (both
// triangles of the diagonal tiles) are dealt to 16 warps, at most 5 per warp, in order of
// decreasing tile column, so a warp's active (trailing) tiles are always a prefix of its slots
// and stay spread over all warps as the reduction advances. Lane l holds the 2 x 4 sub-block
// rows 2(l & 7) + {0,1}, columns 4(l >> 3) + {0..3} of each of its tiles: 40 doubles per lane,
// never spilled, never re-read from shared memory.
//
// Per column k, two block barriers:
//   (a) every warp applies the pending rank-2 update (v_{k-1}, w_{k-1}) to its active tiles
//       (all of them interleaved: one straight-line body per active count), hands column k+1
//       to warp 0, and leaves the tile partials of A22 v_k: row part (8 FMAs, 2 shuffles),
//       column part (8 FMAs, a 4-shuffle reduce-scatter over the 8 row-pair lanes);
//   (b) the row warps (one row per lane) sum each row's tile partials in a fixed order
//       (deterministic) into p, form p.v, w_k = p - (tau/2)(p.v) v_k, bring column k+1 up to
//       date with (v_k, w_k) and form the reflector v_{k+1} (d, e, tau, hv): two named-barrier
//       exchanges among those warps, the reflector scalars computed identically by each.
// Rows/columns <= k carry v = w = 0, so finished entries are never changed and no per-element
// masking is needed. Diagonal tiles are updated with the same FMAs as the others, so their two
// triangles may drift apart by rounding; their row part uses the full tile.

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

constexpr int TT_NW = 16;                      // warps
constexpr int TT_NT = TT_NW * 32;              // threads
constexpr int TT_SLOTS = 5;                    // tiles per warp (16 * 5 >= 78)
constexpr int TT_MAXNB = 12;                   // tile rows: m <= 192
constexpr int TT_MP = 16 * TT_MAXNB;           // padded dimension
constexpr int TT_NTILES = TT_MAXNB * (TT_MAXNB + 1) / 2;
constexpr int TT_NQ = TT_MP / 32;              // rows per lane of warp 0

int tri_tiles_max_dim() { return TT_MP; }

#ifdef TT_PROFILE  // tools/microbench/tt_phases.cu: per-phase cycle sums seen by thread 0
__device__ unsigned long long tt_prof[16];
__shared__ long long tt_acc[16];
#define TT_MARK(i)                                 \
  if (threadIdx.x == 0) {                          \
    const long long now = clock64();               \
    if (i > 0) tt_acc[i] += now - tt_acc[0];       \
    tt_acc[0] = now;                               \
  }
#else
#define TT_MARK(i)
#endif

__device__ __forceinline__ int tt_id(int I, int J) { return I * (I + 1) / 2 + J; }
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ double2 tt_ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// phase (a) on slots S0 .. S0+NS-1 of this warp, interleaved (straight-line). A slot without a
// tile (tIJ < 0) runs on zeros and dumps its partials into the spare row TT_NTILES; an active
// slot's partner that is already inactive is harmless: it only touches finished columns.
template <int S0, int NS>
__device__ __forceinline__ void tt_tiles(double (&A)[TT_SLOTS][8], const int (&tIJ)[TT_SLOTS], int k, int lane,
                                         const double* vo, const double* wo, const double* vn, double* colbuf,
                                         double* part) {
  const int rho = lane & 7, gam = lane >> 3;
  const int kn = k + 1, Jn = kn >> 4, gn = (kn & 15) >> 2, cn = kn & 3;
  const bool g0 = lane & 8, b4 = lane & 4, b2 = lane & 2;
#pragma unroll
  for (int s = S0; s < S0 + NS; ++s) {
    const bool real = tIJ[s] >= 0;
    const int I = real ? tIJ[s] >> 4 : 0, J = real ? tIJ[s] & 15 : 0;
    const int r0 = 16 * I + 2 * rho, c0 = 16 * J + 4 * gam;
    const double2 voI = tt_ld2(vo + r0), woI = tt_ld2(wo + r0), vnI = tt_ld2(vn + r0);
    const double2 vo0 = tt_ld2(vo + c0), vo1 = tt_ld2(vo + c0 + 2);
    const double2 wo0 = tt_ld2(wo + c0), wo1 = tt_ld2(wo + c0 + 2);
    const double2 vn0 = tt_ld2(vn + c0), vn1 = tt_ld2(vn + c0 + 2);
    const double voJ[4] = {vo0.x, vo0.y, vo1.x, vo1.y}, woJ[4] = {wo0.x, wo0.y, wo1.x, wo1.y};
    const double vnJ[4] = {vn0.x, vn0.y, vn1.x, vn1.y};
    const double vr[2] = {voI.x, voI.y}, wr[2] = {woI.x, woI.y}, nr[2] = {vnI.x, vnI.y};
    double rp[2] = {0.0, 0.0}, cp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double x = fma(-vr[a], woJ[c], fma(-wr[a], voJ[c], A[s][4 * a + c]));
        A[s][4 * a + c] = x;
        rp[a] = fma(x, vnJ[c], rp[a]);
        cp[c] = fma(x, nr[a], cp[c]);
      }
    if (real && J == Jn && gam == gn) {  // column k+1 (one update behind) for warp 0
      double x0 = A[s][0], x1 = A[s][4];
#pragma unroll
      for (int c = 1; c < 4; ++c)
        if (c == cn) x0 = A[s][c], x1 = A[s][4 + c];
      colbuf[r0] = x0;
      colbuf[r0 + 1] = x1;
    }
    // partials of row i from partner block X go to part[X * TT_MP + i]: the row part of tile
    // (I, J) to part[J][16I + r], its column part to part[I][16J + c] (diagonal tiles: row part
    // only; slots without a tile write the spare row TT_MAXNB)
    const int prow_at = real ? J * TT_MP + 16 * I : TT_MAXNB * TT_MP;
    const int pcol_at = (real && I != J) ? I * TT_MP + 16 * J : TT_MAXNB * TT_MP;
    // row part: 2 rows over the 4 column-quad lanes (xor 8, 16)
    double rk = (g0 ? rp[1] : rp[0]) + __shfl_xor_sync(0xffffffffu, g0 ? rp[0] : rp[1], 8);
    rk += __shfl_xor_sync(0xffffffffu, rk, 16);
    if (lane < 16) part[prow_at + 2 * rho + (g0 ? 1 : 0)] = rk;
    // column part: 4 columns over the 8 row-pair lanes (xor 4, 2, 1)
    double c2[2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
      c2[j] = (b4 ? cp[j + 2] : cp[j]) + __shfl_xor_sync(0xffffffffu, b4 ? cp[j] : cp[j + 2], 4);
    double c1 = (b2 ? c2[1] : c2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? c2[0] : c2[1], 2);
    c1 += __shfl_xor_sync(0xffffffffu, c1, 1);
    if (!(lane & 1)) part[pcol_at + 4 * gam + (b4 ? 2 : 0) + (b2 ? 1 : 0)] = c1;
  }
}

__global__ void __launch_bounds__(TT_NT, 1) tridiag_tiles_kernel(int m, const double* __restrict__ a,
                                                                 double* __restrict__ d, double* __restrict__ e,
                                                                 double* __restrict__ hv, double* __restrict__ tau) {
  __shared__ __align__(16) double vbuf[2][TT_MP];
  __shared__ __align__(16) double wbuf[TT_MP];
  __shared__ double colbuf[TT_MP];
  __shared__ double part[(TT_MAXNB + 1) * TT_MP];  // [partner block X][row]; + a spare row
  __shared__ double redp[TT_MP / 32], redx[TT_MP / 32], sc[3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (m + 15) >> 4, mp = nb * 16;

  // tile assignment: order by J descending, I ascending; tile t -> warp t % 16, slot t / 16
  int tIJ[TT_SLOTS];  // I * 16 + J, or -1
  {
    int t = 0;
#pragma unroll
    for (int s = 0; s < TT_SLOTS; ++s) tIJ[s] = -1;
    for (int J = nb - 1; J >= 0; --J)
      for (int I = J; I < nb; ++I, ++t) {
        const int w = t % TT_NW, s = t / TT_NW;
#pragma unroll
        for (int q = 0; q < TT_SLOTS; ++q)
          if (w == warp && s == q) tIJ[q] = I * 16 + J;
      }
  }
  double A[TT_SLOTS][8];
#pragma unroll
  for (int s = 0; s < TT_SLOTS; ++s) {
    const int r0 = 16 * (tIJ[s] >> 4) + 2 * (lane & 7), c0 = 16 * (tIJ[s] & 15) + 4 * (lane >> 3);
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int row = r0 + (x >> 2), col = c0 + (x & 3);
      A[s][x] = (tIJ[s] >= 0 && row < m && col < m) ? a[row + (size_t)col * m] : 0.0;
    }
  }
  for (int i = tid; i < TT_MP; i += TT_NT) {
    vbuf[0][i] = vbuf[1][i] = wbuf[i] = 0.0;
    colbuf[i] = i < m ? a[i] : 0.0;
  }
  for (int i = tid; i < (TT_MAXNB + 1) * TT_MP; i += TT_NT) part[i] = 0.0;
  __syncthreads();
#ifdef TT_PROFILE
  if (tid < 16) tt_acc[tid] = 0;
  __syncthreads();
#endif

  // Step k = -1 .. m-2: (a) [k >= 0] all warps: pending update, column k+1, partials of A22 v_k;
  // (b) row warps: p = tau_k A22 v_k, w_k, column k+1 brought up to date, reflector v_{k+1}.
  // At k = -1 every vector is zero, so (b) reduces to the first reflector from column 0.
  double tk = 0.0;  // row warps: tau_k
  const int nbw = (mp + 31) >> 5;  // warps that own rows in phase (b)
  for (int k = -1; k + 1 < m; ++k) {
    const double* vo = vbuf[(k + 1) & 1];  // v_{k-1}
    const double* vn = vbuf[k & 1];        // v_k
    TT_MARK(0);
    if (k >= 0) {
      int na = 0;  // active slots: a prefix (slots are in decreasing tile column order)
#pragma unroll
      for (int s = 0; s < TT_SLOTS; ++s) na += (tIJ[s] >= 0 && 16 * (tIJ[s] & 15) + 15 > k) ? 1 : 0;
      if (na > 0) tt_tiles<0, 2>(A, tIJ, k, lane, vo, wbuf, vn, colbuf, part);
      if (na > 2) tt_tiles<2, 2>(A, tIJ, k, lane, vo, wbuf, vn, colbuf, part);
      if (na > 4) tt_tiles<4, 1>(A, tIJ, k, lane, vo, wbuf, vn, colbuf, part);
      TT_MARK(1);
      __syncthreads();  // (a)
      TT_MARK(2);
    }
    if (warp < nbw) {
      // (b) on the warps of the row threads, one row per lane (i = 32 warp + lane): each lane
      // sums its row's tile partials, two named-barrier exchanges (p.v, then ||x||^2 and the
      // pivot / alpha entries) and every warp forms the same reflector scalars
      const int i = 32 * warp + lane, Jc = (k + 1) >> 4, kc = k + 1;
      double pi = 0.0, pj = 0.0;  // fixed order (even / odd partner blocks), no masking
      {
        int X = Jc;
#pragma unroll 1
        for (; X + 1 < nb; X += 2) {
          pi += part[X * TT_MP + i];
          pj += part[(X + 1) * TT_MP + i];
        }
        if (X < nb) pi += part[X * TT_MP + i];
        pi += pj;
      }
      pi = (i > k && i < m) ? tk * pi : 0.0;
      const double vi = vn[i];
      const double pvw = warp_sum(pi * vi);
      if (lane == 0) redp[warp] = pvw;
      if (i == kc) sc[2] = pi;  // p_k[k+1] for w_k[k+1]
      named_sync(1, 32 * nbw);
      double pv = 0.0;
      for (int w = 0; w < nbw; ++w) pv += redp[w];
      const double c = -0.5 * tk * pv;
      const double wi = fma(c, vi, pi);
      wbuf[i] = wi;
      const double vk1 = vn[kc];                 // v_k[k+1]
      const double wk1 = fma(c, vk1, sc[2]);    // w_k[k+1]
      const double coli = colbuf[i] - (vi * wk1 + wi * vk1);  // column k+1, row i, up to date
      const double xw = warp_sum((i >= kc + 2 && i < m) ? coli * coli : 0.0);
      if (lane == 0) redx[warp] = xw;
      if (i == kc) sc[0] = coli;
      if (i == kc + 1) sc[1] = coli;
      named_sync(1, 32 * nbw);
      double xn2 = 0.0;
      for (int w = 0; w < nbw; ++w) xn2 += redx[w];
      const double dk = sc[0], alpha = kc + 1 < m ? sc[1] : 0.0;
      TT_MARK(6);
      double t = 0.0, beta = alpha, scal = 0.0;
      if (xn2 > 0.0) {  // identical on every lane of every row warp (same inputs)
        // nu = ||(alpha, x)||, beta = -sign(alpha) nu, tau = (beta - alpha) / beta = 1 + |alpha| / nu,
        // scal = 1 / (alpha - beta) = sign(alpha) / (|alpha| + nu): one rsqrt and one division
        // on the serial path instead of a sqrt and two divisions
        const double s2 = fma(alpha, alpha, xn2), rn = rsqrt(s2), nu = s2 * rn, aa = fabs(alpha);
        beta = -copysign(nu, alpha);
        t = fma(aa, rn, 1.0);
        scal = copysign(1.0, alpha) / (aa + nu);
      }
      TT_MARK(7);
      if (i == 0) {
        d[kc] = dk;
        if (kc + 1 < m) e[kc] = beta;
        tau[kc] = t;
      }
      const double vnew = i == kc + 1 ? 1.0 : ((i > kc + 1 && i < m && t != 0.0) ? coli * scal : 0.0);
      vbuf[kc & 1][i] = t != 0.0 ? vnew : 0.0;  // zero beyond m
      if (i > kc && i < m) hv[i + (size_t)kc * m] = vnew;
      tk = t;
    }
    TT_MARK(3);
    __syncthreads();  // (b)
    TT_MARK(4);
  }
#ifdef TT_PROFILE
  if (tid < 16) tt_prof[tid] += tt_acc[tid];
#endif
}

cudaError_t tridiag_tiles(int m, const double* a, double* d, double* e, double* hv, double* tau,
                          cudaStream_t st) {
  if (m < 3 || m > TT_MP) return cudaErrorInvalidValue;
  tridiag_tiles_kernel<<<1, TT_NT, 0, st>>>(m, a, d, e, hv, tau);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
