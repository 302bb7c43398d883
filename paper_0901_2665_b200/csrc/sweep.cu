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

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

// chunk widths: whole matrices while they fit 32 KB, else the largest power of two that does
template <int B>
struct SweepShape {
  static constexpr int KCB = (B * B * 16 <= 32 * 1024) ? B : (32 * 1024) / (B * 16);
  static constexpr int KCF = (2 * B * B * 16 <= 32 * 1024) ? 2 * B : KCB;
  static constexpr int NCHF = 2 * B / KCF, NCHB = B / KCB;
  static constexpr int KCMAX = KCF > KCB ? KCF : KCB;
  static constexpr int SA = B + 2;  // stage column stride (double2), conflict-free LDS.128
  static constexpr int SV = B + 4;  // vector [col][k] stride (double2)
  static constexpr int SY = B + 4;  // real vector stride (double), conflict-free LDS.64
};

template <int B, int NC, int TPW, int NSTAGE, bool CPLX_IN>
__global__ void __launch_bounds__(NC * B / 64 / TPW * 32) bt_sweep_kernel(BtSweepArgs a) {
  using Sh = SweepShape<B>;
  constexpr int KCF = Sh::KCF, KCB = Sh::KCB, NCHF = Sh::NCHF, NCHB = Sh::NCHB, KCMAX = Sh::KCMAX;
  constexpr int SA = Sh::SA, SV = Sh::SV, SY = Sh::SY;
  // small blocks: vectors prefetched through NSTAGE slots and a double-buffered running
  // vector; big blocks (one step = many chunks, latency amortised): one slot loaded at the
  // step start, y_l read back by its own lane, and for B = 512 a single running buffer
  constexpr bool VPRE = B <= 128;
  constexpr bool VDB = B * NC <= 2048;
  constexpr int VS = VPRE ? NSTAGE : 1;               // vector slots
  constexpr int MT = B / 8;                           // m-tiles
  constexpr int NWARPS = (B / 8) * (NC / 8) / TPW;
  constexpr int NT = NWARPS * 32;
  constexpr bool SPLIT = TPW <= 2;                    // two accumulator sets
  constexpr size_t BB = (size_t)B * B;
  const int s = blockIdx.y;
  const int c0 = blockIdx.x * NC;
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
        for (int e0 = 0; e0 < KCF * B; e0 += NT) {
          const int e = e0 + tid;
          if (KCF * B % NT == 0 || e < KCF * B) {
            const int k = e / B, i = e % B, kg = k0 + k;
            const bool v = kg < B || l > 0;
            const double2* src = kg < B ? sinv + (size_t)l * BB + (size_t)kg * B + i
                                        : hm + (size_t)(l - 1) * BB + (size_t)(kg - B) * B + i;
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
        const double2* src = gm + (size_t)l * BB + (size_t)j * KCB * B;
#pragma unroll
        for (int e0 = 0; e0 < KCB * B; e0 += NT) {
          const int e = e0 + tid;
          if (KCB * B % NT == 0 || e < KCB * B) cp_async16(dst + (e / B) * SA + e % B, src + e);
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
  int arow[TPW], bcol[TPW];  // fragment offsets: A row 8*mt+g, B column 8*nt+g
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
    if (!VDB) __syncthreads();  // single running buffer: every warp is done reading y_{l-1}
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      Vout[(cl0 + 0) * SV + arow[j]] = y0;
      Vout[(cl0 + 1) * SV + arow[j]] = y1;
      if (l + 1 < L) {
        const size_t row = (size_t)l * B + arow[j];
        if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
        if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
      }
    }
  }

  // ---------------- backward sweep ----------------
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
    if (!VDB) __syncthreads();  // single running buffer: every warp is done reading x_{l+1}
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const int r = arow[j];
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
      Vout[(cl0 + 0) * SV + r] = x0;
      Vout[(cl0 + 1) * SV + r] = x1;
      epilogue(l, j, x0, x1);
    }
  }
  cp_async_wait<0>();
}

template <int B, int NC, int TPW, int NSTAGE>
static cudaError_t launch_sweep(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = SweepShape<B>;
  constexpr int NWARPS = (B / 8) * (NC / 8) / TPW;
  constexpr int nvec = (B * NC <= 2048 ? 2 : 1) + (B <= 128 ? NSTAGE : 1);
  const size_t sm = sizeof(double2) * ((size_t)nvec * NC * Sh::SV + (size_t)NSTAGE * Sh::KCMAX * Sh::SA);
  dim3 grid((a.m + NC - 1) / NC, a.nodes);
  cudaError_t e;
  if (a.complex_mode) {
    auto kern = bt_sweep_kernel<B, NC, TPW, NSTAGE, true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, NWARPS * 32, sm, st>>>(a);
  } else {
    auto kern = bt_sweep_kernel<B, NC, TPW, NSTAGE, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, NWARPS * 32, sm, st>>>(a);
  }
  ++g_launches;
  return cudaGetLastError();
}

bool bt_block_supported(int b) {
  return b == 16 || b == 32 || b == 64 || b == 128 || b == 256 || b == 512;
}

cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st) {
  switch (a.b) {
    case 16: return launch_sweep<16, 16, 1, 3>(a, st);    // 4 warps
    case 32: return launch_sweep<32, 16, 1, 3>(a, st);    // 8 warps
    case 64: return launch_sweep<64, 16, 2, 3>(a, st);    // 8 warps
    case 128: return launch_sweep<128, 8, 2, 3>(a, st);   // 8 warps
    case 256: return launch_sweep<256, 16, 8, 2>(a, st);  // 8 warps; 16 columns halve L2 bytes/flop
    case 512: return launch_sweep<512, 8, 8, 2>(a, st);   // 8 warps
  }
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
