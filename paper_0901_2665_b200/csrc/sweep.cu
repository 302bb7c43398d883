// sweep.cu — block-Thomas forward/backward sweeps for all contour nodes, fused with the
// quadrature epilogue of accumulate_subspace_real (core.hpp:170-180).
//
// With the factors of blocktri.cu (S_l^{-1}, H_l = S_l^{-1} C_{l-1}, G_l = S_l^{-1} C_l^T):
//   forward : y_l = S_l^{-1} Y_l - H_l y_{l-1}           (H_0 = 0)
//   backward: x_{L-1} = y_{L-1},  x_l = y_l - G_l x_{l+1}
//   epilogue: T_e = Re(c_e x)  (real mode)  or  W_e = x (complex mode, ShiftSystem shim)
// Each chain step is ONE complex GEMM on FP64 DMMA tiles: the forward step streams the
// concatenated [S_l^{-1} | H_l] (K = 2B) against [Y_l ; y_{l-1}], the backward step streams
// G_l (K = B) against x_{l+1}.
//
// CTA = (column block of NC right-hand sides, node slot); the whole chain of one column
// block runs in one CTA with no grid-level synchronisation. Matrix chunks AND the
// right-hand-side rows each step needs (Y_l forward, y_l backward) ride the same cp.async
// ring, issued NSTAGE-1 chunks ahead, so no global-memory latency sits on the dependency
// chain; the running vector is double-buffered in shared memory (one barrier per chunk).
// The block size B is a template parameter (powers of two, 16..512), so all index math is
// shifts and the inner loops unroll; small blocks split every accumulator in two (even /
// odd k) to halve the DMMA dependency chain.

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

// chunk widths: whole matrices while a chunk (the CTA's RB = B/P rows) fits 32 KB, else the
// largest power of two that does
template <int B, int P>
struct SweepShape {
  static constexpr int RB = B / P;
  static constexpr int KCB = (B * RB * 16 <= 32 * 1024) ? B : (32 * 1024) / (RB * 16);
  static constexpr int KCF = (2 * B * RB * 16 <= 32 * 1024) ? 2 * B : KCB;
  static constexpr int NCHF = 2 * B / KCF, NCHB = B / KCB;
  static constexpr int KCMAX = KCF > KCB ? KCF : KCB;
  static constexpr int SA = RB + 2;  // stage column stride (double2), conflict-free LDS.128
  static constexpr int SV = B + 4;   // vector [col][k] stride (double2)
  static constexpr int SY = B + 4;   // real vector stride (double), conflict-free LDS.64
};

// P > 1: a thread-block cluster of P CTAs shares one column block; CTA rank p computes rows
// [p*B/P, (p+1)*B/P) of every chain step and stores them into all P CTAs' running-vector
// buffers through distributed shared memory, one cluster barrier per step (finer work units
// for the 148 SMs, and enough CTAs when a GPU owns a single contour node).
template <int B, int P, int NC, int TPW, int NSTAGE, bool CPLX_IN>
__global__ void __launch_bounds__(NC * B / 64 / P / TPW * 32) bt_sweep_kernel(BtSweepArgs a) {
  using Sh = SweepShape<B, P>;
  constexpr int RB = Sh::RB;
  constexpr int KCF = Sh::KCF, KCB = Sh::KCB, NCHF = Sh::NCHF, NCHB = Sh::NCHB, KCMAX = Sh::KCMAX;
  constexpr int SA = Sh::SA, SV = Sh::SV, SY = Sh::SY;
  // small blocks: vectors prefetched through NSTAGE slots and a double-buffered running
  // vector; big blocks (one step = many chunks, latency amortised): one slot loaded at the
  // step start, y_l read back by its own lane, and for B = 512 a single running buffer
  constexpr bool VPRE = B <= 128;
  constexpr bool VDB = B * NC <= 2048;
  constexpr int VS = VPRE ? NSTAGE : 1;               // vector slots
  // the backward's y_l rows are prefetched NSTAGE-1 chunks ahead: with one chunk per step
  // that reaches back into the forward sweep, and only y_{L-2} (read from the running
  // buffer below) may still be unwritten then
  static_assert(!VPRE || NSTAGE <= 3, "deeper rings would prefetch y_l before the forward sweep writes it");
  constexpr int MT = RB / 8;                          // local m-tiles
  constexpr int NWARPS = MT * (NC / 8) / TPW;
  constexpr int NT = NWARPS * 32;
  constexpr bool SPLIT = TPW <= 2;                    // two accumulator sets
  constexpr size_t BB = (size_t)B * B;
  const int s = blockIdx.y;
  const int prank = P > 1 ? (int)(blockIdx.x % P) : 0;
  const int c0 = (blockIdx.x / P) * NC;
  const int row0 = prank * RB;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  extern __shared__ __align__(16) double2 smem[];
  double2* Vs0 = smem;                  // running vector, double-buffered [col][k]
  double2* Vs1 = VDB ? Vs0 + NC * SV : Vs0;
  double2* Vslot = Vs1 + NC * SV;       // VS slots: Y_l (real [col][k], ld SY) / y_l (complex)
  double2* St = Vslot + VS * NC * SV;   // NSTAGE stages of KCMAX x SA
  const double2 coeff = a.coeff[s];
  const double2* sinv = a.sinv + (size_t)s * L * BB;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  double2* W = a.w + (size_t)s * ldv * m;
  double* T = a.complex_mode ? nullptr : a.t + (size_t)s * ldv * m;
  const int total = L * NCHF + (L - 1) * NCHB;

  for (int i = tid; i < (VDB ? 2 : 1) * NC * SV; i += NT) Vs0[i] = make_double2(0.0, 0.0);
  // every CTA of the cluster has zeroed its buffers before anyone stores into them remotely
  if (P > 1) cg::this_cluster().sync();

  // -------- producer: chunk q (+ the step's right-hand-side rows with its first chunk) --------
  auto issue = [&](int q) {
    if (q < total) {
      double2* dst = St + (q % NSTAGE) * KCMAX * SA;
      int l, j, vseq;
      const bool fwd = q < L * NCHF;
      if (fwd) {
        l = q / NCHF;
        j = q - l * NCHF;
        vseq = l;
        const int k0 = j * KCF;
#pragma unroll
        for (int e0 = 0; e0 < KCF * RB; e0 += NT) {
          const int e = e0 + tid;
          if (KCF * RB % NT == 0 || e < KCF * RB) {
            const int k = e / RB, i = e % RB, kg = k0 + k;
            const bool v = kg < B || l > 0;
            const double2* src = kg < B ? sinv + (size_t)l * BB + (size_t)kg * B + row0 + i
                                        : hm + (size_t)(l - 1) * BB + (size_t)(kg - B) * B + row0 + i;
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + k * SA + i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(v ? src : sinv),
                         "r"(v ? 16 : 0));
          }
        }
      } else {
        const int q2 = q - L * NCHF;
        l = L - 2 - q2 / NCHB;
        j = q2 - (q2 / NCHB) * NCHB;
        vseq = L + (L - 2 - l);
        const double2* src = gm + (size_t)l * BB + (size_t)j * KCB * B + row0;
#pragma unroll
        for (int e0 = 0; e0 < KCB * RB; e0 += NT) {
          const int e = e0 + tid;
          if (KCB * RB % NT == 0 || e < KCB * RB) {
            const int k = e / RB, i = e % RB;
            cp_async16(dst + k * SA + i, src + (size_t)k * B + i);
          }
        }
      }
      if (VPRE && j == 0) {
        double2* vd = Vslot + (vseq % VS) * NC * SV;
        const size_t rbase = (size_t)l * B;
#pragma unroll
        for (int e0 = 0; e0 < NC * B; e0 += NT) {
          const int e = e0 + tid;
          if (NC * B % NT == 0 || e < NC * B) {
            const int col = e / B, i = e % B;
            const int gc = c0 + col;
            const bool v = gc < m;
            const size_t off = rbase + i + (size_t)(v ? gc : 0) * ldv;
            if (fwd && !CPLX_IN) {
              double* vdd = reinterpret_cast<double*>(vd);
              const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(vdd + col * SY + i));
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(a.y + off),
                           "r"(v ? 8 : 0));
            } else {
              const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(vd + col * SV + i));
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(W + off),
                           "r"(v ? 16 : 0));
            }
          }
        }
      }
    }
    cp_async_commit();
  };
  int qc = 0;
#pragma unroll
  for (int p = 0; p < NSTAGE - 1; ++p) issue(p);
  auto acquire = [&]() -> const double2* {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    issue(qc + NSTAGE - 1);
    const double2* p = St + (qc % NSTAGE) * KCMAX * SA;
    ++qc;
    return p;
  };

  CAcc acc[TPW], acc2[SPLIT ? TPW : 1];
  // fragment offsets: A row 8*mt+g within this CTA's rows (arow), the same row within the
  // layer (grow = row0 + arow), B column 8*nt+g
  int arow[TPW], grow[TPW], bcol[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tt = warp + NWARPS * j;
    arow[j] = 8 * (tt % MT) + g;
    grow[j] = row0 + arow[j];
    bcol[j] = 8 * (tt / MT) + g;
  }
  // this step's result rows go to every CTA of the cluster (DSMEM) or just here
  auto put = [&](double2* Vout, int idx, double2 val) {
    if (P == 1) {
      Vout[idx] = val;
    } else {
      cg::cluster_group cl = cg::this_cluster();
#pragma unroll
      for (int q = 0; q < P; ++q) cl.map_shared_rank(Vout, q)[idx] = val;
    }
  };
  auto step_barrier = [&]() {
    if (P > 1) cg::this_cluster().sync();
  };
  auto zero_acc = [&]() {
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      acc[j].zero();
      if (SPLIT) acc2[j].zero();
    }
  };
  auto fold_acc = [&]() {
    if (SPLIT) {
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        acc[j].r0 += acc2[j].r0; acc[j].r1 += acc2[j].r1;
        acc[j].i0 += acc2[j].i0; acc[j].i1 += acc2[j].i1;
      }
    }
  };

  // ---------------- forward sweep ----------------
  for (int l = 0; l < L; ++l) {
    const double2* Bv = (l & 1) ? Vs0 : Vs1;  // y_{l-1}
    double2* Vout = (l & 1) ? Vs1 : Vs0;
    const double2* Ys = Vslot + (l % VS) * NC * SV;
    const double* Ysr = reinterpret_cast<const double*>(Ys);
    if (!VPRE) {  // Y_l into the single slot (previous readers are done after the barrier)
      __syncthreads();
      for (int e = tid; e < NC * B; e += NT) {
        const int col = e / B, i = e % B, gc = c0 + col;
        const size_t off = (size_t)l * B + i + (size_t)(gc < m ? gc : 0) * ldv;
        if (CPLX_IN) Vslot[col * SV + i] = gc < m ? W[off] : make_double2(0.0, 0.0);
        else reinterpret_cast<double*>(Vslot)[col * SY + i] = gc < m ? a.y[off] : 0.0;
      }
    }
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHF; ++c) {
      const double2* As = acquire();
#pragma unroll
      for (int kk = 0; kk < KCF; kk += 4) {
        const int kg = c * KCF + kk;  // warp-uniform
        CAcc* ac = (SPLIT && ((kk >> 2) & 1)) ? acc2 : acc;
        if (kg < B) {  // S_l^{-1} Y_l
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            const double2 av = As[(kk + t4) * SA + arow[j]];
            if (CPLX_IN) {
              cmma(ac[j], av, Ys[bcol[j] * SV + kg + t4]);
            } else {
              const double yv = Ysr[bcol[j] * SY + kg + t4];
              dmma884(ac[j].r0, ac[j].r1, av.x, yv);
              dmma884(ac[j].i0, ac[j].i1, av.y, yv);
            }
          }
        } else {       // - H_l y_{l-1}
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            const double2 av = As[(kk + t4) * SA + arow[j]];
            cmma(ac[j], make_double2(-av.x, -av.y), Bv[bcol[j] * SV + kg - B + t4]);
          }
        }
      }
    }
    fold_acc();
    if (!VDB) {  // single running buffer: every warp (of every cluster CTA) is done with y_{l-1}
      if (P > 1) step_barrier();
      else __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      put(Vout, (cl0 + 0) * SV + grow[j], y0);
      put(Vout, (cl0 + 1) * SV + grow[j], y1);
      if (l + 1 < L) {
        const size_t row = (size_t)l * B + grow[j];
        if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
        if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
      }
    }
    step_barrier();
  }

  // ---------------- backward sweep ----------------
  auto epilogue = [&](int l, int j, double2 x0, double2 x1) {
    const size_t row = (size_t)l * B + grow[j];
    const int col = c0 + bcol[j] - g + 2 * t4;
    if (a.complex_mode) {
      if (col < m) W[row + (size_t)col * ldv] = x0;
      if (col + 1 < m) W[row + (size_t)(col + 1) * ldv] = x1;
    } else {
      if (col < m) T[row + (size_t)col * ldv] = coeff.x * x0.x - coeff.y * x0.y;
      if (col + 1 < m) T[row + (size_t)(col + 1) * ldv] = coeff.x * x1.x - coeff.y * x1.y;
    }
  };
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    epilogue(L - 1, j, make_double2(acc[j].r0, acc[j].i0), make_double2(acc[j].r1, acc[j].i1));

  for (int l = L - 2; l >= 0; --l) {
    const double2* Bv = (l & 1) ? Vs0 : Vs1;  // x_{l+1}
    double2* Vout = (l & 1) ? Vs1 : Vs0;
    // y_l from its prefetched slot, except y_{L-2}: the forward sweep finished it only one
    // step ago (possibly after its slot was issued); it still sits in the running-vector
    // buffer this step writes x_{L-2} into (same lane, same element)
    const double2* Ys = (l == L - 2) ? Vout : Vslot + ((L + (L - 2 - l)) % VS) * NC * SV;
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHB; ++c) {
      const double2* As = acquire();
#pragma unroll
      for (int kk = 0; kk < KCB; kk += 4) {
        const int kg = c * KCB + kk;
        CAcc* ac = (SPLIT && ((kk >> 2) & 1)) ? acc2 : acc;
#pragma unroll
        for (int j = 0; j < TPW; ++j)
          cmma(ac[j], As[(kk + t4) * SA + arow[j]], Bv[bcol[j] * SV + kg + t4]);
      }
    }
    fold_acc();
    if (!VDB) {  // single running buffer: every warp (of every cluster CTA) is done with x_{l+1}
      if (P > 1) step_barrier();
      else __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const int r = grow[j];
      double2 y0, y1;
      if (VPRE) {
        y0 = Ys[(cl0 + 0) * SV + r];
        y1 = Ys[(cl0 + 1) * SV + r];
      } else {  // written by this very lane in the forward sweep
        const size_t row = (size_t)l * B + r;
        y0 = c0 + cl0 < m ? W[row + (size_t)(c0 + cl0) * ldv] : make_double2(0.0, 0.0);
        y1 = c0 + cl0 + 1 < m ? W[row + (size_t)(c0 + cl0 + 1) * ldv] : make_double2(0.0, 0.0);
      }
      const double2 x0 = make_double2(y0.x - acc[j].r0, y0.y - acc[j].i0);
      const double2 x1 = make_double2(y1.x - acc[j].r1, y1.y - acc[j].i1);
      put(Vout, (cl0 + 0) * SV + r, x0);
      put(Vout, (cl0 + 1) * SV + r, x1);
      epilogue(l, j, x0, x1);
    }
    step_barrier();
  }
  cp_async_wait<0>();
}

template <int B, int P, int NC, int TPW, int NSTAGE>
static cudaError_t launch_sweep(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = SweepShape<B, P>;
  constexpr int NWARPS = (B / 8 / P) * (NC / 8) / TPW;
  constexpr int nvec = (B * NC <= 2048 ? 2 : 1) + (B <= 128 ? NSTAGE : 1);
  const size_t sm = sizeof(double2) * ((size_t)nvec * NC * Sh::SV + (size_t)NSTAGE * Sh::KCMAX * Sh::SA);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.m + NC - 1) / NC * P), (unsigned)a.nodes);
  cfg.blockDim = dim3(NWARPS * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (a.complex_mode) {
    auto kern = bt_sweep_kernel<B, P, NC, TPW, NSTAGE, true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    auto kern = bt_sweep_kernel<B, P, NC, TPW, NSTAGE, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

bool bt_block_supported(int b) {
  return b == 16 || b == 32 || b == 64 || b == 128 || b == 256 || b == 512;
}

cudaError_t bt_sweep_tma(const BtSweepArgs& a, cudaStream_t st);

cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st) {
  // b >= 128: panel-layout factors and the bulk-copy pipeline of sweep_tma.cu
  if (bt_panel_rows(a.b) > 0) return bt_sweep_tma(a, st);
  switch (a.b) {
    case 16: return launch_sweep<16, 1, 16, 1, 3>(a, st);    // 4 warps
    case 32: return launch_sweep<32, 1, 16, 1, 3>(a, st);    // 8 warps
    case 64: return launch_sweep<64, 1, 16, 2, 3>(a, st);    // 8 warps
  }
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
