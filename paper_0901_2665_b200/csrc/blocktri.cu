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

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

int64_t g_launches = 0;

// ---------------------------------------------------------------------------
// Small blocks (b = 16, 32, 64): one CTA per node and chain direction.
//
// Twisted recursion (kmid >= 0): a cluster of two CTAs per node eliminates from both ends.
//   top    (rank 0), l = 0 .. kmid-1 : S_l = M_l - C_{l-1} G_{l-1}; G_l = S_l^{-1} C_l^T -> g[l],
//                                      H_l = S_l^{-1} C_{l-1} -> h[l-1]
//   bottom (rank 1), l = L-1 .. kmid+1: R_l = M_l - C_l^T G'_{l+1}; G'_l = R_l^{-1} C_{l-1} -> g[l-1],
//                                      H'_l = R_l^{-1} C_l^T -> h[l]
//   middle (rank 0, after a cluster barrier), l = kmid:
//     T = M_k - C_{k-1} G_{k-1} - C_k^T G'_{k+1};  T^{-1} -> sinv[k], T^{-1} C_{k-1} -> h[k-1],
//     T^{-1} C_k^T -> h[k]
// so the dependency chain is ~L/2 layers long instead of L (and the sweep's 2L-1 steps become
// ~L). Both directions are the same code: a layer's "in" coupling is the neighbour already
// eliminated, its "out" coupling the one still ahead. kmid < 0: the plain top-down chain.
//
// Per layer: S = M - Cin Gprev (DMMA tiles, operands converted from the (A, B) pairs on the
// fly), S^{-1} by Gauss-Jordan with partial pivoting (largest |.|^2, first index on ties)
// in place — rows spread over the CTA's threads for b <= 32 (gj_cta), in shared memory for
// b = 64 — then H = S^{-1} Cin and G = S^{-1} Cout (DMMA). For b <= 32 the next layer's raw
// blocks are prefetched with cp.async while this one is processed.
// ---------------------------------------------------------------------------
template <int B>
struct FacShape {
  static constexpr int NT = B == 16 ? 128 : 256;
  static constexpr int LDS = B + 4;        // Sv / Gp column stride (double2)
  static constexpr bool RAW_SMEM = B <= 32;
  static constexpr size_t smem_bytes() {
    return sizeof(double2) * (2 * (size_t)B * LDS + B + (RAW_SMEM ? 5 * (size_t)B * B : 0));
  }
};

FEAST_DEV double2 czb(double2 e, double2 z) { return make_double2(z.x * e.y - e.x, z.y * e.y); }

// acc tiles of X(B x B) * Y(B x B) over the CTA's warps; out(i, j, v) per element
template <int B, class FA, class FB, class FO>
FEAST_DEV void cgemm_tiles(int warp, int nwarps, int lane, FA fa, FB fb, FO out) {
  constexpr int MT = B / 8;
  const int g = lane >> 2, t4 = lane & 3;
  for (int tile = warp; tile < MT * MT; tile += nwarps) {
    const int r0 = 8 * (tile % MT), c0 = 8 * (tile / MT);
    CAcc acc, acc2;
    acc.zero();
    acc2.zero();
#pragma unroll
    for (int k = 0; k < B; k += 8) {
      cmma(acc, fa(r0 + g, k + t4), fb(k + t4, c0 + g));
      cmma(acc2, fa(r0 + g, k + 4 + t4), fb(k + 4 + t4, c0 + g));
    }
    out(r0 + g, c0 + 2 * t4, make_double2(acc.r0 + acc2.r0, acc.i0 + acc2.i0));
    out(r0 + g, c0 + 2 * t4 + 1, make_double2(acc.r1 + acc2.r1, acc.i1 + acc2.i1));
  }
}

// In-place Gauss-Jordan inverse of Sv (B x B, column stride lds) by the whole CTA (NT = B x NG
// threads: thread t owns row t % B and NCOL = B / NG columns of it) with IMPLICIT partial pivoting:
// the pivot row of column k is never moved; at the end the row that pivoted column k holds row k of
// (P S)^{-1}, and S^{-1}[i, p_t] = that row's element t. No row swaps, no dynamically indexed
// registers, the k loop stays rolled.
//   * Pivot search: ONE warp-wide integer max (REDUX) per step on a 32-bit key, the top 27 bits of
//     |a_ik|^2 (its binary64 pattern orders like the value) over B - 1 - i in the low bits: the
//     unused row with the largest modulus to within 2^-15 relative, lowest index among those
//     (threshold partial pivoting with a threshold of 1 - 3e-5). Every warp repeats it on its own
//     lanes (same result, no exchange). The shuffle arg-max it replaces (4 dependent levels of 64-bit
//     shuffles and FP64 compares) was the longest dependent chain of a pivot step.
//   * Two block barriers per pivot step separate the reads of the pivot row and column from their
//     overwriting. (One warp doing the whole elimination, the first version, left the other three
//     waiting for two thirds of the kernel: ncu, profiles/r02_summary.md.)
template <int B, int NT>
FEAST_DEV void gj_cta(double2* Sv, int lds, int* pivs, int* status) {
  constexpr int NG = NT / B, NCOL = B / NG;
  static_assert(NT % B == 0 && B % NG == 0 && B <= 32, "gj_cta: one row per lane group");
  const int tid = threadIdx.x;
  const int r = tid % B, j0 = (tid / B) * NCOL;
  bool used = false, bad = false;
  int mystep = 0;
#pragma unroll 1
  for (int k = 0; k < B; ++k) {
    const double2 ak = Sv[r + k * lds];
    // (lanes r and r + B of a warp hold the same row when B = 16: the warp-wide max is the 16-row max)
    const unsigned key =
        used ? 0u : (((unsigned)__double2hiint(ak.x * ak.x + ak.y * ak.y) & ~(unsigned)(B - 1)) | (unsigned)(B - 1 - r));
    const int p = B - 1 - (int)(__reduce_max_sync(0xffffffffu, key) & (unsigned)(B - 1));
    const bool isp = r == p;
    used |= isp;
    mystep = isp ? k : mystep;
    if (tid == 0) pivs[k] = p;
    // 1 / a_pk = conj(a_pk) / |a_pk|^2
    const double2 apk = Sv[p + k * lds];
    const double best = apk.x * apk.x + apk.y * apk.y;
    bad |= !(best > 0.0);
    const double rn = 1.0 / best;
    const double2 inv = make_double2(apk.x * rn, -apk.y * rn);
    double2 piv[NCOL], a0[NCOL];
#pragma unroll
    for (int jj = 0; jj < NCOL; ++jj) {
      piv[jj] = Sv[p + (j0 + jj) * lds];
      a0[jj] = Sv[r + (j0 + jj) * lds];
    }
    __syncthreads();  // every thread holds the pivot row / column entries it needs
    const double2 mk = make_double2(-ak.x, -ak.y);
#pragma unroll
    for (int jj = 0; jj < NCOL; ++jj) {
      const bool jk = j0 + jj == k;
      const double2 pv = jk ? inv : cmul(piv[jj], inv);   // scaled pivot row
      const double2 a = jk ? make_double2(0.0, 0.0) : a0[jj];
      const double2 upd = make_double2(a.x + mk.x * pv.x - mk.y * pv.y, a.y + mk.x * pv.y + mk.y * pv.x);
      Sv[r + (j0 + jj) * lds] = isp ? pv : upd;
    }
    __syncthreads();
  }
  double2 mine[NCOL];
#pragma unroll
  for (int jj = 0; jj < NCOL; ++jj) mine[jj] = Sv[r + (j0 + jj) * lds];
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < NCOL; ++jj) Sv[mystep + pivs[j0 + jj] * lds] = mine[jj];
  if (bad && tid == 0) atomicExch(status, 1);
}

// the same elimination by the whole CTA in shared memory (b = 64)
template <int B, int NT>
FEAST_DEV void gj_smem(double2* Sv, int lds, int* pivs, int* cpos, int* status) {
  constexpr int PER = B * B / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2 v[PER];
  for (int k = 0; k < B; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int p = B;
      for (int i = k + lane; i < B; i += 32) {
        const double2 e = Sv[i + k * lds];
        const double m = e.x * e.x + e.y * e.y;
        if (m > best) {
          best = m;
          p = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (ob > best || (ob == best && op < p)) {
          best = ob;
          p = op;
        }
      }
      if (lane == 0) {
        pivs[k] = p;
        if (!(best > 0.0)) atomicExch(status, 1);
      }
    }
    __syncthreads();
    const int p = pivs[k];
    if (p != k)
      for (int jj = tid; jj < B; jj += NT) {
        const double2 t = Sv[k + jj * lds];
        Sv[k + jj * lds] = Sv[p + jj * lds];
        Sv[p + jj * lds] = t;
      }
    __syncthreads();
    const double2 inv = cdiv(make_double2(1.0, 0.0), Sv[k + k * lds]);
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int idx = tid + e * NT, i = idx % B, jj = idx / B;
      const double2 rk = cmul(jj == k ? make_double2(1.0, 0.0) : Sv[k + jj * lds], inv);
      v[e] = i == k ? rk
                    : csub(jj == k ? make_double2(0.0, 0.0) : Sv[i + jj * lds], cmul(Sv[i + k * lds], rk));
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int idx = tid + e * NT;
      Sv[idx % B + (idx / B) * lds] = v[e];
    }
    __syncthreads();
  }
  if (tid < B) {
    int pos = tid;
    for (int k = B - 1; k >= 0; --k) {
      const int p = pivs[k];
      if (pos == k) pos = p;
      else if (pos == p) pos = k;
    }
    cpos[tid] = pos;
  }
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int idx = tid + e * NT;
    v[e] = Sv[idx % B + (idx / B) * lds];
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int idx = tid + e * NT;
    Sv[idx % B + cpos[idx / B] * lds] = v[e];
  }
}

template <int B>
__global__ void __launch_bounds__(FacShape<B>::NT) bt_factor_small_kernel(BtFactorArgs a) {
  using Sh = FacShape<B>;
  constexpr int NT = Sh::NT, LDS = Sh::LDS, NW = NT / 32;
  constexpr bool RAW = Sh::RAW_SMEM;
  constexpr size_t BB = (size_t)B * B;
  const bool tw = a.kmid >= 0;
  const int node = tw ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // factor slot (node, chunk)
  const int half = tw ? (int)(blockIdx.x & 1) : 0;
  const int L = a.L, kmid = tw ? a.kmid : L - 1;
  const int nsteps = half == 0 ? kmid + 1 : L - 1 - kmid;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double2 z = a.z[node / a.chunks];
  // this chunk's layers of the pencil (chunks == 1: the whole chain)
  const size_t lay0 = (size_t)(node % a.chunks) * L;
  const double2* abdiag = a.abdiag + lay0 * BB;
  const double2* ablow = a.ablow + lay0 * BB;
  extern __shared__ __align__(16) double2 fsm[];
  double2* Sv = fsm;                  // B x LDS: S, then S^{-1}
  double2* Gp = Sv + B * LDS;         // B x LDS: G of the previous layer (B operand of the S update)
  double2* colbuf = Gp + B * LDS;     // B
  double2* rawD = colbuf + B;         // RAW: 2 x BB (A, B) pairs of the diagonal block
  double2* rawC = rawD + 2 * BB;      // RAW: 3 x BB (A, B) pairs of the out coupling
  __shared__ int pivs[B], cpos[B];
  double2* sinv = a.sinv + (size_t)node * L * BB;
  double2* gm = a.g + (size_t)node * (L > 1 ? L - 1 : 0) * BB;
  double2* hm = a.h + (size_t)node * (L > 1 ? L - 1 : 0) * BB;
  // b <= 32: factors stored row-swizzled for the bulk-copy sweep (sweep_small.cu): row i of
  // column j at j*B + (i ^ 2(j & 3)); b = 64: plain column-major (sweep.cu)
  auto fidx = [&](int i, int j) { return RAW ? j * B + (i ^ ((j & 3) << 1)) : j * B + i; };

  auto layer_of = [&](int r) { return half == 0 ? r : L - 1 - r; };
  auto has_out = [&](int l) { return half == 0 ? l + 1 < L : true; };
  auto prefetch = [&](int r) {
    if (RAW && r < nsteps) {
      const int l = layer_of(r);
      const double2* d = abdiag + (size_t)l * BB;
      double2* dd = rawD + (r & 1) * BB;
      for (int e = tid; e < (int)BB; e += NT) cp_async16(dd + e, d + e);
      if (has_out(l)) {
        const double2* c = ablow + (size_t)(half == 0 ? l : l - 1) * BB;
        double2* cd = rawC + (r % 3) * BB;
        for (int e = tid; e < (int)BB; e += NT) cp_async16(cd + e, c + e);
      }
    }
    cp_async_commit();
  };

  prefetch(0);
  for (int r = 0; r < nsteps; ++r) {
    const int l = layer_of(r);
    prefetch(r + 1);
    cp_async_wait<1>();
    __syncthreads();
    const double2* dsrc = RAW ? rawD + (r & 1) * BB : abdiag + (size_t)l * BB;
    // raw (A, B) pairs of the in / out couplings (as stored: C_c = M(c+1, c), col-major)
    const double2* cin = r == 0 ? nullptr
                         : RAW ? rawC + ((r + 2) % 3) * BB
                               : ablow + (size_t)(half == 0 ? l - 1 : l) * BB;
    const double2* cout = !has_out(l) ? nullptr
                          : RAW ? rawC + (r % 3) * BB
                                : ablow + (size_t)(half == 0 ? l : l - 1) * BB;
    // top: Cin = C_{l-1}, Cout = C_l^T ; bottom: Cin = C_l^T, Cout = C_{l-1}
    auto Ci = [&](int i, int t) { return czb(half == 0 ? cin[i + t * B] : cin[t + i * B], z); };
    auto Co = [&](int i, int t) { return czb(half == 0 ? cout[t + i * B] : cout[i + t * B], z); };
    auto Gop = [&](int t, int j) { return Gp[t + j * LDS]; };
    auto Sop = [&](int i, int t) { return Sv[i + t * LDS]; };

    // (1) S = M_l - Cin G_prev   [- Cout G'_{k+1} at the middle layer]
    if (r == 0) {
      for (int e = tid; e < (int)BB; e += NT) Sv[e % B + (e / B) * LDS] = czb(dsrc[e], z);
    } else {
      cgemm_tiles<B>(warp, NW, lane, Ci, Gop,
                     [&](int i, int j, double2 v) { Sv[i + j * LDS] = csub(czb(dsrc[i + j * B], z), v); });
    }
    const bool middle = tw && half == 0 && l == kmid;
    if (middle) {
      __syncthreads();                    // S complete, G_{k-1} no longer read
      __threadfence();
      cg::this_cluster().sync();          // the bottom CTA has stored G'_{k+1} = g[kmid]
      for (int e = tid; e < (int)BB; e += NT)
        Gp[e % B + (e / B) * LDS] = __ldcg(gm + (size_t)kmid * BB + fidx(e % B, e / B));
      __syncthreads();
      cgemm_tiles<B>(warp, NW, lane, Co, Gop,
                     [&](int i, int j, double2 v) { Sv[i + j * LDS] = csub(Sv[i + j * LDS], v); });
    }
    __syncthreads();

    // (2) S^{-1} in place
    if constexpr (RAW) {
      gj_cta<B, NT>(Sv, LDS, pivs, a.status);
    } else {
      gj_smem<B, NT>(Sv, LDS, pivs, cpos, a.status);
    }
    __syncthreads();

    // (3) outputs: S^{-1}, H = S^{-1} Cin, G = S^{-1} Cout (kept for the next layer)
    double2* so = sinv + (size_t)l * BB;
    for (int e = tid; e < (int)BB; e += NT) so[fidx(e % B, e / B)] = Sv[e % B + (e / B) * LDS];
    if (r > 0) {
      double2* ho = hm + (size_t)(half == 0 ? l - 1 : l) * BB;
      cgemm_tiles<B>(warp, NW, lane, Sop, [&](int t, int j) { return Ci(t, j); },
                     [&](int i, int j, double2 v) { ho[fidx(i, j)] = v; });
    }
    if (cout) {
      double2* go = middle ? hm + (size_t)kmid * BB : gm + (size_t)(half == 0 ? l : l - 1) * BB;
      cgemm_tiles<B>(warp, NW, lane, Sop, [&](int t, int j) { return Co(t, j); },
                     [&](int i, int j, double2 v) {
                       go[fidx(i, j)] = v;
                       Gp[i + j * LDS] = v;
                     });
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if (tw && half == 1) {
    __threadfence();
    cg::this_cluster().sync();  // releases g[kmid] to the top CTA's middle layer
  }
}

template <int B>
static cudaError_t launch_factor_small(const BtFactorArgs& a, cudaStream_t st) {
  using Sh = FacShape<B>;
  const size_t sm = Sh::smem_bytes();
  auto kern = bt_factor_small_kernel<B>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const bool tw = a.kmid >= 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.nodes * (tw ? 2 : 1)));
  cfg.blockDim = dim3(Sh::NT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = tw ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

int bt_twist_layer(int L, int b, bool enable) { return (enable && b <= 64 && L >= 4) ? L / 2 : -1; }

// ---------------------------------------------------------------------------
// Large blocks (b >= 128): the same recursion, every dense b x b operation batched over the
// nodes and run on the DMMA GEMM / batched-LU kernels (one layer at a time):
//   S_l = M_l - C_{l-1} G_{l-1}  (zgemm) ;  S_l^{-1} by block Gauss-Jordan in place (below) ;
//   H_l = S_l^{-1} C_{l-1} ;  G_l = S_l^{-1} C_l^T  (zgemm) ; all three packed into panels
// ---------------------------------------------------------------------------
cudaError_t zgemm_batched(int m, int n, int k, double2 alpha, const double2* a, int lda, int64_t sa,
                          const double2* b, int ldb, int64_t sb, double2 beta, double2* c, int ldc,
                          int64_t sc, int batch, cudaStream_t st);
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

static cudaError_t bt_factor_big(const BtFactorArgs& a, cudaStream_t st) {
  const int L = a.L, b = a.b, nodes = a.nodes;
  const int64_t bb = (int64_t)b * b, lnode = (int64_t)L * bb, gnode = (int64_t)(L > 1 ? L - 1 : 0) * bb;
  double2* S = a.work;                 // S_l, then S_l^{-1}   (nodes x bb)
  double2* Cp = S + nodes * bb;        // C_{l-1}, then C_l
  double2* CT = Cp + nodes * bb;       // C_l^T
  double2* X = CT + nodes * bb;        // S_l^{-1}
  double2* scr = X + nodes * bb;       // G_l (col-major) until the next Schur update; I - S X
  double2* gjw = scr + nodes * bb;     // Gauss-Jordan work
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0), zero = make_double2(0.0, 0.0);
  dim3 g((unsigned)std::min<int64_t>((bb + 255) / 256, 512), nodes);
  // factors leave in the sweep's panel layout; G_l also stays col-major in scr until the
  // next layer's Schur update has used it (the refinement reuses scr only after that)
  const int rb = bt_panel_rows(b);
  auto pack = [&](const double2* src, double2* dst, int64_t dstride) {
    pack_panels_kernel<<<g, 256, 0, st>>>(src, dst, dstride, b, rb);
    ++g_launches;
  };
  for (int l = 0; l < L; ++l) {
    bt_make_kernel<<<g, 256, 0, st>>>(b, a.abdiag + l * bb, a.z, S, 0);
    ++g_launches;
    if (l > 0) zgemm_batched(b, b, b, mone, Cp, b, bb, scr, b, bb, one, S, b, bb, nodes, st);
    {
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
  return (size_t)nodes * (5 * (size_t)b * b + 2 * (size_t)b * GJ_NB + (size_t)GJ_NB * GJ_NB);  // S Cp CT X scr + GJ
}

cudaError_t bt_factor(const BtFactorArgs& a, cudaStream_t st) {
  switch (a.b) {
    case 16: return launch_factor_small<16>(a, st);
    case 32: return launch_factor_small<32>(a, st);
    case 64: return launch_factor_small<64>(a, st);
  }
  return bt_factor_big(a, st);
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
