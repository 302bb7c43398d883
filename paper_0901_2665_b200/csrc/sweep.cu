// sweep.cu — block-Thomas forward/backward sweeps for all contour nodes, fused with the
// quadrature epilogue of accumulate_subspace_real (core.hpp:170-180).
//
// With the factors of blocktri.cu (S_l^{-1}, H_l = S_l^{-1} C_{l-1}, G_l = S_l^{-1} C_l^T):
//   forward : y_l = S_l^{-1} Y_l - H_l y_{l-1}           (H_0 = 0)
//   backward: x_{L-1} = y_{L-1},  x_l = y_l - G_l x_{l+1}
//   epilogue: T_e = Re(c_e x)  (real mode)  or  W_e = x (complex mode, ShiftSystem shim)
// Each chain step is ONE complex GEMM on FP64 DMMA tiles: the forward step streams the
// concatenated [S_l^{-1} | H_l] (K = 2b) against [Y_l ; y_{l-1}], the backward step streams
// G_l (K = b) against x_{l+1}.
//
// CTA = (column block of NC right-hand sides, node slot); the whole chain of one column
// block runs in one CTA with no grid-level synchronisation. Matrix chunks AND the
// right-hand-side rows each step needs (Y_l forward, y_l backward) ride the same cp.async
// ring, issued NSTAGE-1 chunks ahead, so no global-memory latency sits on the dependency
// chain; the running vector is double-buffered in shared memory (one barrier per chunk).

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

template <int NC, int TPW, int NSTAGE, bool CPLX_IN>
__global__ void __launch_bounds__(TPW >= 4 ? 256 : 512) bt_sweep_kernel(BtSweepArgs a, int kcf, int kcb) {
  constexpr int VS = NSTAGE;  // vector slots
  const int s = blockIdx.y;
  const int c0 = blockIdx.x * NC;
  const int L = a.L, b = a.b, m = a.m, ldv = a.ldv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int nwarps = blockDim.x >> 5;
  const int mtiles = b >> 3;
  const int SA = b + 2, SV = b + 4;
  const int kcmax = kcf > kcb ? kcf : kcb;
  extern __shared__ __align__(16) double2 smem[];
  double2* Vs0 = smem;                      // running vector, double-buffered [col][k]
  double2* Vs1 = Vs0 + NC * SV;
  double2* Vslot = Vs1 + NC * SV;           // VS slots: Y_l (real, [col][k], ld SV*2) / y_l (complex)
  double2* St = Vslot + VS * NC * SV;       // NSTAGE stages of kcmax x SA
  const double2 coeff = a.coeff[s];
  const size_t bb = (size_t)b * b;
  const double2* sinv = a.sinv + (size_t)s * L * bb;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * bb;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * bb;
  double2* W = a.w + (size_t)s * ldv * m;
  double* T = a.complex_mode ? nullptr : a.t + (size_t)s * ldv * m;
  const int nchf = 2 * b / kcf, nchb = b / kcb;
  const int total = L * nchf + (L - 1) * nchb;

  for (int i = threadIdx.x; i < 2 * NC * SV; i += blockDim.x) Vs0[i] = make_double2(0.0, 0.0);

  // -------- producer: chunk q (+ the step's vector with its first chunk) --------
  auto issue = [&](int q) {
    if (q < total) {
      double2* dst = St + (size_t)(q % NSTAGE) * kcmax * SA;
      int l, j, vseq;
      bool fwd = q < L * nchf;
      if (fwd) {
        l = q / nchf; j = q % nchf; vseq = l;
        const int k0 = j * kcf;
        for (int e = threadIdx.x; e < kcf * b; e += blockDim.x) {
          const int k = e / b, i = e - k * b, kg = k0 + k;
          const double2* src = kg < b ? sinv + (size_t)l * bb + (size_t)kg * b + i
                                      : hm + (size_t)(l - 1) * bb + (size_t)(kg - b) * b + i;
          const bool v = kg < b || l > 0;
          const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + k * SA + i));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                       "l"(v ? src : sinv), "r"(v ? 16 : 0));
        }
      } else {
        const int q2 = q - L * nchf;
        l = L - 2 - q2 / nchb; j = q2 % nchb; vseq = L + (L - 2 - l);
        const double2* src = gm + (size_t)l * bb + (size_t)j * kcb * b;
        for (int e = threadIdx.x; e < kcb * b; e += blockDim.x) {
          const int k = e / b, i = e - k * b;
          cp_async16(dst + k * SA + i, src + e);
        }
      }
      if (j == 0) {  // the right-hand-side rows of this chain step
        double2* vd = Vslot + (size_t)(vseq % VS) * NC * SV;
        for (int e = threadIdx.x; e < NC * b; e += blockDim.x) {
          const int col = e / b, i = e - col * b;
          const int gc = c0 + col;
          const bool v = gc < m;
          const size_t off = (size_t)l * b + i + (size_t)(v ? gc : 0) * ldv;
          if (fwd && !CPLX_IN) {  // real Y_l -> doubles at [col][k] (ld b+4: conflict-free LDS.64)
            double* vdd = reinterpret_cast<double*>(vd);
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(vdd + col * (b + 4) + i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(a.y + off),
                         "r"(v ? 8 : 0));
          } else {                // complex y_l (backward) or complex input (forward)
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(vd + col * SV + i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(W + off),
                         "r"(v ? 16 : 0));
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
    const double2* p = St + (size_t)(qc % NSTAGE) * kcmax * SA;
    ++qc;
    return p;
  };

  CAcc acc[TPW];
  int mt[TPW], ntl[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tt = warp + nwarps * j;
    mt[j] = tt % mtiles;
    ntl[j] = tt / mtiles;
  }

  // ---------------- forward sweep ----------------
  for (int l = 0; l < L; ++l) {
    const double2* Bv = (l & 1) ? Vs0 : Vs1;  // y_{l-1}
    double2* Vout = (l & 1) ? Vs1 : Vs0;
    const double2* Ys = Vslot + (size_t)(l % VS) * NC * SV;
    const double* Ysr = reinterpret_cast<const double*>(Ys);
#pragma unroll
    for (int j = 0; j < TPW; ++j) acc[j].zero();
    for (int c = 0; c < nchf; ++c) {
      const double2* As = acquire();
      for (int kk = 0; kk < kcf; kk += 4) {
        const int kg = c * kcf + kk;  // warp-uniform
        if (kg < b) {  // S_l^{-1} Y_l
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            const double2 av = As[(kk + t4) * SA + 8 * mt[j] + g];
            if (CPLX_IN) {
              cmma(acc[j], av, Ys[(8 * ntl[j] + g) * SV + kg + t4]);
            } else {
              const double yv = Ysr[(8 * ntl[j] + g) * (b + 4) + kg + t4];
              dmma884(acc[j].r0, acc[j].r1, av.x, yv);
              dmma884(acc[j].i0, acc[j].i1, av.y, yv);
            }
          }
        } else {       // - H_l y_{l-1}
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            const double2 av = As[(kk + t4) * SA + 8 * mt[j] + g];
            cmma(acc[j], make_double2(-av.x, -av.y), Bv[(8 * ntl[j] + g) * SV + kg - b + t4]);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = 8 * ntl[j] + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      Vout[(cl0 + 0) * SV + 8 * mt[j] + g] = y0;
      Vout[(cl0 + 1) * SV + 8 * mt[j] + g] = y1;
      if (l + 1 < L) {
        const int row = l * b + 8 * mt[j] + g;
        if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
        if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
      }
    }
  }

  // ---------------- backward sweep ----------------
  auto epilogue = [&](int l, int j, double2 x0, double2 x1) {
    const int row = l * b + 8 * mt[j] + g;
    const int col = c0 + 8 * ntl[j] + 2 * t4;
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
    // y_l: from its prefetched slot, except y_{L-2}, which the forward sweep finished
    // only one step ago (possibly after its slot was issued) and which still sits in the
    // running-vector buffer this step writes x_{L-2} into (same lane, same element)
    const double2* Ys = (l == L - 2) ? Vout : Vslot + (size_t)((L + (L - 2 - l)) % VS) * NC * SV;
#pragma unroll
    for (int j = 0; j < TPW; ++j) acc[j].zero();
    for (int c = 0; c < nchb; ++c) {
      const double2* As = acquire();
      for (int kk = 0; kk < kcb; kk += 4) {
        const int kg = c * kcb + kk;
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const double2 av = As[(kk + t4) * SA + 8 * mt[j] + g];
          cmma(acc[j], av, Bv[(8 * ntl[j] + g) * SV + kg + t4]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = 8 * ntl[j] + 2 * t4;
      const int r = 8 * mt[j] + g;
      const double2 y0 = Ys[(cl0 + 0) * SV + r], y1 = Ys[(cl0 + 1) * SV + r];
      const double2 x0 = make_double2(y0.x - acc[j].r0, y0.y - acc[j].i0);
      const double2 x1 = make_double2(y1.x - acc[j].r1, y1.y - acc[j].i1);
      Vout[(cl0 + 0) * SV + r] = x0;
      Vout[(cl0 + 1) * SV + r] = x1;
      epilogue(l, j, x0, x1);
    }
  }
  cp_async_wait<0>();
}

template <int NC, int TPW, int NSTAGE>
static cudaError_t launch_sweep(const BtSweepArgs& a, int kcf, int kcb, int warps, cudaStream_t st) {
  const int SA = a.b + 2, SV = a.b + 4;
  const int kcmax = kcf > kcb ? kcf : kcb;
  const size_t sm = sizeof(double2) * ((size_t)(2 + NSTAGE) * NC * SV + (size_t)NSTAGE * kcmax * SA);
  dim3 grid((a.m + NC - 1) / NC, a.nodes);
  cudaError_t e;
  if (a.complex_mode) {
    auto kern = bt_sweep_kernel<NC, TPW, NSTAGE, true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, warps * 32, sm, st>>>(a, kcf, kcb);
  } else {
    auto kern = bt_sweep_kernel<NC, TPW, NSTAGE, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<grid, warps * 32, sm, st>>>(a, kcf, kcb);
  }
  ++g_launches;
  return cudaGetLastError();
}

// chunk widths: one chunk per matrix while it fits 32 KB, else the largest power of two
static int pick_kc(int width, int b) {
  int kc = 4;
  for (int c = 4; c <= width; c *= 2)
    if (width % c == 0 && (size_t)c * b * 16 <= 32 * 1024) kc = c;
  return kc;
}

cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st) {
  const int b = a.b;
  if (b % 16 != 0) return cudaErrorInvalidValue;
  int kcf = pick_kc(2 * b, b), kcb = pick_kc(b, b);
  if (kcf > b && (2 * b) % kcf) kcf = kcb;
  const bool wide = b <= 64;
  const int tiles = (b / 8) * (wide ? 2 : 1);
  int tpw = 1;
  while (tiles / tpw > 16 || tiles % tpw != 0) tpw *= 2;
  const int warps = tiles / tpw;
  if (tpw > 8) return cudaErrorInvalidValue;
  if (wide) {
    switch (tpw) {
      case 1: return launch_sweep<16, 1, 3>(a, kcf, kcb, warps, st);
      case 2: return launch_sweep<16, 2, 3>(a, kcf, kcb, warps, st);
      default: return cudaErrorInvalidValue;
    }
  }
  // NC = 8 for big blocks (shared memory); two stages once b >= 384
  switch (tpw) {
    case 1: return launch_sweep<8, 1, 3>(a, kcf, kcb, warps, st);
    case 2: return launch_sweep<8, 2, 3>(a, kcf, kcb, warps, st);
    case 4: return b >= 384 ? launch_sweep<8, 4, 2>(a, kcf, kcb, warps, st) : launch_sweep<8, 4, 3>(a, kcf, kcb, warps, st);
    case 8: return b >= 384 ? launch_sweep<8, 8, 2>(a, kcf, kcb, warps, st) : launch_sweep<8, 8, 3>(a, kcf, kcb, warps, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
