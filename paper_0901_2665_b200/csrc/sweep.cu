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
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace feastgpu {

// chunk widths: whole matrices while a chunk fits 32 KB, else the largest power of two that does
template <int B>
struct SweepShape {
  static constexpr int KCB = (B * B * 16 <= 32 * 1024) ? B : (32 * 1024) / (B * 16);
  static constexpr int KCF = (2 * B * B * 16 <= 32 * 1024) ? 2 * B : KCB;
  static constexpr int KCM = (3 * B * B * 16 <= 32 * 1024) ? 3 * B : KCB;  // twisted middle step
  static constexpr int NCHF = 2 * B / KCF, NCHB = B / KCB;
  static constexpr int KCMAX = KCM > KCF ? KCM : KCF;
  static constexpr int SA = B + 2;   // stage column stride (double2), conflict-free LDS.128
  static constexpr int SV = B + 4;   // vector [col][k] stride (double2)
  static constexpr int SY = B + 4;   // real vector stride (double), conflict-free LDS.64
};

// One CTA walks the whole chain of one column block (NC right-hand sides) of one node.
// Steps, in order: H forward steps, the middle step, H backward steps.
//   plain   (TW = false): H = L-1 forward layers 0..L-2, middle = layer L-1 (K = 2B)
//   twisted (TW = true) : a cluster of two CTAs per column block. Rank 0 runs the top half
//     (forward l = 0..kmid-1, backward l = kmid-1..0), rank 1 the bottom half (forward
//     l = L-1..kmid+1, backward l = kmid+1..L-1), with the factors of bt_factor's twisted
//     recursion. After their forward halves the two CTAs swap the last forward vectors through
//     DSMEM and both compute the middle layer
//       x_k = T^{-1} Y_k - (T^{-1} C_{k-1}) y_{k-1} - (T^{-1} C_k^T) u_{k+1}    (K = 3B)
//     so the dependency chain is L+1 steps instead of 2L-1.
template <int B, int NC, int TPW, int NSTAGE, bool CPLX_IN, bool TW>
__global__ void __launch_bounds__(NC * B / 64 / TPW * 32) bt_sweep_kernel(BtSweepArgs a) {
  using Sh = SweepShape<B>;
  constexpr int KCF = Sh::KCF, KCB = Sh::KCB, KCM = TW ? Sh::KCM : Sh::KCF;
  constexpr int NCHF = Sh::NCHF, NCHB = Sh::NCHB, NCHM = (TW ? 3 : 2) * B / KCM;
  constexpr int KCMAX = Sh::KCMAX, SA = Sh::SA, SV = Sh::SV, SY = Sh::SY;
  constexpr int VS = NSTAGE;                          // vector slots (prefetched RHS rows)
  // the backward's y_l rows are prefetched NSTAGE-1 chunks ahead: with one chunk per step
  // that reaches back into the forward sweep, and only the last forward vector (read from the
  // running buffer below) may still be unwritten then
  static_assert(NSTAGE <= 3, "deeper rings would prefetch y_l before the forward sweep writes it");
  constexpr int MT = B / 8;                           // m-tiles
  constexpr int NWARPS = MT * (NC / 8) / TPW;
  constexpr int NT = NWARPS * 32;
  constexpr bool SPLIT = TPW <= 2;                    // two accumulator sets
  constexpr size_t BB = (size_t)B * B;
  const int s = blockIdx.y;
  const int half = TW ? (int)(blockIdx.x & 1) : 0;
  const int c0 = (int)(TW ? blockIdx.x >> 1 : blockIdx.x) * NC;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int kmid = TW ? a.kmid : L - 1;
  const int H = half == 0 ? kmid : L - 1 - kmid;    // forward (and backward) steps
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  extern __shared__ __align__(16) double2 smem[];
  double2* Vs0 = smem;                  // running vector, double-buffered [col][k]
  double2* Vs1 = Vs0 + NC * SV;
  double2* Xb = Vs1 + NC * SV;          // TW: the partner's last forward vector
  double2* Vslot = Xb + (TW ? NC * SV : 0);  // VS slots: Y_l (real [col][k], ld SY) / y_l (complex)
  double2* St = Vslot + VS * NC * SV;   // NSTAGE stages of KCMAX x SA
  const double2 coeff = a.coeff[s];
  const double2* sinv = a.sinv + (size_t)s * L * BB;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  double2* W = a.w + (size_t)s * ldv * m;
  double* T = a.complex_mode ? nullptr : a.t + (size_t)s * ldv * m;
  const int nfwd = H * NCHF, total = nfwd + NCHM + H * NCHB;
  auto layer_of = [&](int r) { return half == 0 ? r : L - 1 - r; };
  auto buf = [&](int v) { return (v & 1) ? Vs1 : Vs0; };  // output buffer of step v

  for (int i = tid; i < 2 * NC * SV; i += NT) Vs0[i] = make_double2(0.0, 0.0);

  // -------- producer: chunk q (+ the step's right-hand-side rows with its first chunk) --------
  auto issue = [&](int q) {
    if (q < total) {
      double2* dst = St + (q % NSTAGE) * KCMAX * SA;
      int l, j, vseq, kc, kind;  // kind 0 forward, 1 middle, 2 backward, 3 first forward step
      if (q < nfwd) {
        const int r = q / NCHF;
        j = q - r * NCHF;
        l = layer_of(r);
        vseq = r;
        kc = KCF;
        kind = r == 0 ? 3 : 0;
      } else if (q < nfwd + NCHM) {
        j = q - nfwd;
        l = kmid;
        vseq = H;
        kc = KCM;
        kind = 1;
      } else {
        const int q2 = q - nfwd - NCHM, rb = q2 / NCHB;
        j = q2 - rb * NCHB;
        l = layer_of(H - 1 - rb);
        vseq = H + 1 + rb;
        kc = KCB;
        kind = 2;
      }
      const int k0 = j * kc;
#pragma unroll
      for (int e0 = 0; e0 < KCMAX * B; e0 += NT) {
        const int e = e0 + tid;
        const int k = e / B, i = e % B, kg = k0 + k;
        if (k < kc) {
          const double2* src = sinv;
          bool v = true;
          if (kind == 2) {
            src = gm + (size_t)(half == 0 ? l : l - 1) * BB + (size_t)kg * B + i;
          } else if (kg < B) {
            src = sinv + (size_t)l * BB + (size_t)kg * B + i;
          } else if (kind == 1) {  // middle: [T^{-1} | T^{-1} C_{k-1} | T^{-1} C_k^T]
            v = kg >= 2 * B || H > 0;
            src = !v ? sinv
                 : kg < 2 * B ? hm + (size_t)(kmid - 1) * BB + (size_t)(kg - B) * B + i
                              : hm + (size_t)kmid * BB + (size_t)(kg - 2 * B) * B + i;
          } else {  // forward H part (none on the first step)
            v = kind == 0;
            src = v ? hm + (size_t)(half == 0 ? l - 1 : l) * BB + (size_t)(kg - B) * B + i : sinv;
          }
          const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + k * SA + i));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(v ? 16 : 0));
        }
      }
      if (j == 0) {
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
            if (kind != 2 && !CPLX_IN) {
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
  int arow[TPW], bcol[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tt = warp + NWARPS * j;
    arow[j] = 8 * (tt % MT) + g;
    bcol[j] = 8 * (tt / MT) + g;
  }
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
  // acc += chunk (KC columns, global K offset kc_base) x operand, K segments:
  //   [0, B) the RHS slot, [B, 2B) -(.) x Bv, [2B, 3B) -(.) x Bo
  auto mma_chunk = [&](const double2* As, int kc_base, auto KCc, const double2* Ys, const double2* Bv,
                       const double2* Bo) {
    constexpr int KC = decltype(KCc)::value;
    const double* Ysr = reinterpret_cast<const double*>(Ys);
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const int kg = kc_base + kk;  // warp-uniform
      CAcc* ac = (SPLIT && ((kk >> 2) & 1)) ? acc2 : acc;
      if (kg < B) {
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
      } else {
        const double2* Bx = kg < 2 * B ? Bv : Bo;
        const int kb = kg < 2 * B ? kg - B : kg - 2 * B;
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const double2 av = As[(kk + t4) * SA + arow[j]];
          cmma(ac[j], make_double2(-av.x, -av.y), Bx[bcol[j] * SV + kb + t4]);
        }
      }
    }
  };
  auto epilogue = [&](int l, int j, double2 x0, double2 x1) {
    const size_t row = (size_t)l * B + arow[j];
    const int col = c0 + bcol[j] - g + 2 * t4;
    if (a.complex_mode) {
      if (col < m) W[row + (size_t)col * ldv] = x0;
      if (col + 1 < m) W[row + (size_t)(col + 1) * ldv] = x1;
    } else {
      if (col < m) T[row + (size_t)col * ldv] = coeff.x * x0.x - coeff.y * x0.y;
      if (col + 1 < m) T[row + (size_t)(col + 1) * ldv] = coeff.x * x1.x - coeff.y * x1.y;
    }
  };

  // ---------------- forward half ----------------
  for (int r = 0; r < H; ++r) {
    const int l = layer_of(r);
    const double2* Bv = buf(r - 1);
    double2* Vout = buf(r);
    const double2* Ys = Vslot + (r % VS) * NC * SV;
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHF; ++c) {
      const double2* As = acquire();
      mma_chunk(As, c * KCF, std::integral_constant<int, KCF>{}, Ys, Bv, Bv);
    }
    fold_acc();
    const bool last = r == H - 1;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      Vout[(cl0 + 0) * SV + arow[j]] = y0;
      Vout[(cl0 + 1) * SV + arow[j]] = y1;
      if (TW && last) {  // the partner's middle step needs this vector
        double2* px = cg::this_cluster().map_shared_rank(Xb, half ^ 1);
        px[(cl0 + 0) * SV + arow[j]] = y0;
        px[(cl0 + 1) * SV + arow[j]] = y1;
      }
      const size_t row = (size_t)l * B + arow[j];
      if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
      if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
    }
  }

  // ---------------- middle layer ----------------
  if (TW) {
    // every prefetch that reads W row kmid (the complex-mode RHS) has landed before the top
    // CTA may overwrite it with x_k, and the partner's vector is in Xb
    cp_async_wait<0>();
    cg::this_cluster().sync();
  }
  {
    const double2* Bprev = buf(H - 1);
    double2* Vout = buf(H);
    const double2* Ys = Vslot + (H % VS) * NC * SV;
    const double2* By = TW && half == 1 ? Xb : Bprev;  // y_{k-1}
    const double2* Bu = TW && half == 1 ? Bprev : Xb;  // u_{k+1}
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHM; ++c) {
      const double2* As = acquire();
      mma_chunk(As, c * KCM, std::integral_constant<int, KCM>{}, Ys, By, Bu);
    }
    fold_acc();
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const double2 x0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 x1 = make_double2(acc[j].r1, acc[j].i1);
      Vout[(cl0 + 0) * SV + arow[j]] = x0;
      Vout[(cl0 + 1) * SV + arow[j]] = x1;
      if (half == 0) epilogue(kmid, j, x0, x1);
    }
  }

  // ---------------- backward half ----------------
  for (int rb = 0; rb < H; ++rb) {
    const int r = H - 1 - rb, l = layer_of(r), v = H + 1 + rb;
    const double2* Bv = buf(v - 1);  // x of the neighbour towards the middle
    double2* Vout = buf(v);
    // y_l from its prefetched slot, except the last forward vector (rb = 0): it was finished
    // only one step before the middle and sits in the buffer this step writes (same lane,
    // same element)
    const double2* Ys = rb == 0 ? Vout : Vslot + (v % VS) * NC * SV;
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHB; ++c) {
      const double2* As = acquire();
      mma_chunk(As, c * KCB + B, std::integral_constant<int, KCB>{}, Ys, Bv, Bv);
    }
    fold_acc();
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const int rr = arow[j];
      const double2 y0 = Ys[(cl0 + 0) * SV + rr];
      const double2 y1 = Ys[(cl0 + 1) * SV + rr];
      // mma_chunk accumulated -G x (the segment-1 sign), so x = y + acc
      const double2 x0 = make_double2(y0.x + acc[j].r0, y0.y + acc[j].i0);
      const double2 x1 = make_double2(y1.x + acc[j].r1, y1.y + acc[j].i1);
      Vout[(cl0 + 0) * SV + rr] = x0;
      Vout[(cl0 + 1) * SV + rr] = x1;
      epilogue(l, j, x0, x1);
    }
  }
  cp_async_wait<0>();  // (the partner's DSMEM stores into Xb all precede the middle barrier)
}

template <int B, int NC, int TPW, int NSTAGE, bool TW>
static cudaError_t launch_sweep(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = SweepShape<B>;
  constexpr int NWARPS = (B / 8) * (NC / 8) / TPW;
  constexpr int nvec = 2 + (TW ? 1 : 0) + NSTAGE;
  const size_t sm = sizeof(double2) * ((size_t)nvec * NC * Sh::SV + (size_t)NSTAGE * Sh::KCMAX * Sh::SA);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.m + NC - 1) / NC * (TW ? 2 : 1)), (unsigned)a.nodes);
  cfg.blockDim = dim3(NWARPS * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TW ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (a.complex_mode) {
    auto kern = bt_sweep_kernel<B, NC, TPW, NSTAGE, true, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    auto kern = bt_sweep_kernel<B, NC, TPW, NSTAGE, false, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int B, int NC, int TPW, int NSTAGE>
static cudaError_t launch_sweep_any(const BtSweepArgs& a, cudaStream_t st) {
  return a.kmid >= 0 ? launch_sweep<B, NC, TPW, NSTAGE, true>(a, st)
                     : launch_sweep<B, NC, TPW, NSTAGE, false>(a, st);
}

bool bt_block_supported(int b) {
  return b == 16 || b == 32 || b == 64 || b == 128 || b == 256 || b == 512;
}

cudaError_t bt_sweep_tma(const BtSweepArgs& a, cudaStream_t st);
cudaError_t bt_sweep_small(const BtSweepArgs& a, cudaStream_t st);

cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st) {
  // b >= 128: panel-layout factors and the bulk-copy pipeline of sweep_tma.cu
  if (bt_panel_rows(a.b) > 0) return bt_sweep_tma(a, st);
  // b = 16, 32: swizzled factors and the bulk-copy pipeline of sweep_small.cu
  if (a.b == 16 || a.b == 32) return bt_sweep_small(a, st);
  if (a.b == 64) return launch_sweep_any<64, 16, 2, 3>(a, st);  // 8 warps, cp.async ring
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
