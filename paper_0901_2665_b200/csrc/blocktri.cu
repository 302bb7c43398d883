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

#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

int64_t g_launches = 0;

// ---------------------------------------------------------------------------
// Factor: one CTA per node walks the L-step chain. v0: any b; [S | I] lives in shared
// memory for b <= 64 and in global scratch otherwise.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) bt_factor_kernel(BtFactorArgs a) {
  const int s = blockIdx.x;
  const int L = a.L, b = a.b, tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const double2 z = a.z[s];
  const int ld = b + 1;
  extern __shared__ __align__(16) double2 fsm[];
  double2* f = fsm;                                   // b
  double2* aug = (b <= 64) ? fsm + b : a.scratch + (size_t)s * b * 2 * ld;
  __shared__ int piv_s;
  __shared__ int bad_s;
  const size_t bb = (size_t)b * b;
  double2* sinv = a.sinv + (size_t)s * L * bb;
  double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * bb;
  if (tid == 0) bad_s = 0;

  for (int l = 0; l < L; ++l) {
    // (a) S_l = M_l - C_{l-1} G_{l-1};  right half = I
    const double2* ab = a.abdiag + (size_t)l * bb;
    for (int idx = tid; idx < b * b; idx += nt) {
      const int i = idx % b, j = idx / b;
      const double2 e = ab[idx];
      double2 v = make_double2(z.x * e.y - e.x, z.y * e.y);
      if (l > 0) {
        const double2* cl = a.ablow + (size_t)(l - 1) * bb;
        const double2* gp = gm + (size_t)(l - 1) * bb;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < b; ++k) {
          const double2 ce = cl[i + (size_t)k * b];
          const double2 c = make_double2(z.x * ce.y - ce.x, z.y * ce.y);
          acc = cadd(acc, cmul(c, gp[k + (size_t)j * b]));
        }
        v = csub(v, acc);
      }
      aug[i + (size_t)j * ld] = v;
      aug[i + (size_t)(b + j) * ld] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();

    // (b) Gauss-Jordan with partial pivoting (largest |.|, first index on ties,
    //     the DenseLU / BandedLU rule of lu.hpp:29-38)
    for (int k = 0; k < b; ++k) {
      if (warp == 0) {
        double best = -1.0;
        int bi = b;
        for (int i = k + lane; i < b; i += 32) {
          const double v = cabs_(aug[i + (size_t)k * ld]);
          if (v > best) { best = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) {
          piv_s = bi;
          if (!(best > 0.0)) bad_s = 1;
        }
      }
      __syncthreads();
      if (bad_s) {
        if (tid == 0) atomicExch(a.status, 1);
        return;
      }
      const int p = piv_s;
      if (p != k)
        for (int j = k + tid; j < 2 * b; j += nt) {
          const double2 t0 = aug[k + (size_t)j * ld];
          aug[k + (size_t)j * ld] = aug[p + (size_t)j * ld];
          aug[p + (size_t)j * ld] = t0;
        }
      __syncthreads();
      const double2 pv = aug[k + (size_t)k * ld];
      __syncthreads();
      for (int j = k + 1 + tid; j < 2 * b; j += nt)
        aug[k + (size_t)j * ld] = cdiv(aug[k + (size_t)j * ld], pv);
      for (int i = tid; i < b; i += nt) f[i] = aug[i + (size_t)k * ld];
      __syncthreads();
      const int ncol = 2 * b - k - 1;
      for (int idx = tid; idx < b * ncol; idx += nt) {
        const int i = idx % b, j = k + 1 + idx / b;
        if (i == k) continue;
        aug[i + (size_t)j * ld] = csub(aug[i + (size_t)j * ld], cmul(f[i], aug[k + (size_t)j * ld]));
      }
      __syncthreads();
    }

    // Sinv_l out
    double2* si = sinv + (size_t)l * bb;
    for (int idx = tid; idx < b * b; idx += nt) {
      const int i = idx % b, j = idx / b;
      si[idx] = aug[i + (size_t)(b + j) * ld];
    }
    // (c) G_l = S_l^{-1} C_l^T
    if (l + 1 < L) {
      const double2* cl = a.ablow + (size_t)l * bb;
      double2* gp = gm + (size_t)l * bb;
      for (int idx = tid; idx < b * b; idx += nt) {
        const int i = idx % b, j = idx / b;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < b; ++k) {
          const double2 ce = cl[j + (size_t)k * b];   // C_l(j, k)
          const double2 c = make_double2(z.x * ce.y - ce.x, z.y * ce.y);
          acc = cadd(acc, cmul(aug[i + (size_t)(b + k) * ld], c));
        }
        gp[idx] = acc;
      }
    }
    __syncthreads();
  }
}

cudaError_t bt_factor(const BtFactorArgs& a, cudaStream_t st) {
  size_t sm = sizeof(double2) * (size_t)a.b;
  if (a.b <= 64) sm += sizeof(double2) * (size_t)a.b * 2 * (a.b + 1);
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(bt_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  bt_factor_kernel<<<a.nodes, 256, sm, st>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Sweeps. CTA = (column block of NC right-hand sides, node slot). The whole forward and
// backward chain of one column block runs inside one CTA with no grid-level sync; the
// b x b factor blocks are streamed through a cp.async ring of NSTAGE chunks (kc columns
// each) that runs ahead of the dependency chain, so only the in-SM GEMM latency is
// serial. Each warp owns TPW 8x8 complex output tiles (4 DMMAs per k4 step each).
// ---------------------------------------------------------------------------
template <int NC, int TPW, int NSTAGE>
__global__ void __launch_bounds__(TPW >= 4 ? 256 : 512) bt_sweep_kernel(BtSweepArgs a, int kc) {
  const int s = blockIdx.y;
  const int c0 = blockIdx.x * NC;
  const int L = a.L, b = a.b, m = a.m, ldv = a.ldv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int nwarps = blockDim.x >> 5;
  const int mtiles = b >> 3;
  const int SA = b + 2, SV = b + 4;
  extern __shared__ __align__(16) double2 smem[];
  double2* Vs = smem;
  double2* Ts = Vs + NC * SV;
  double2* St = Ts + NC * SV;
  const double2 z = a.z[s];
  const double2 coeff = a.coeff[s];
  const int nch = b / kc;
  const size_t bb = (size_t)b * b;
  const double2* sinv = a.sinv + (size_t)s * L * bb;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * bb;
  double2* W = a.w + (size_t)s * ldv * m;
  double* T = a.complex_mode ? nullptr : a.t + (size_t)s * ldv * m;
  const int total = nch * (3 * L - 2);

  auto chunk_src = [&](int q) -> const double2* {
    if (q < nch) return sinv + (size_t)q * kc * b;
    q -= nch;
    if (q < 2 * nch * (L - 1)) {
      const int l = 1 + q / (2 * nch), r = q % (2 * nch);
      if (r < nch) return a.ablow + (size_t)(l - 1) * bb + (size_t)r * kc * b;
      return sinv + (size_t)l * bb + (size_t)(r - nch) * kc * b;
    }
    q -= 2 * nch * (L - 1);
    const int l = L - 2 - q / nch;
    return gm + (size_t)l * bb + (size_t)(q % nch) * kc * b;
  };
  auto issue = [&](int q) {
    if (q < total) {
      const double2* src = chunk_src(q);
      double2* dst = St + (size_t)(q % NSTAGE) * kc * SA;
      for (int e = threadIdx.x; e < kc * b; e += blockDim.x) {
        const int k = e / b, i = e - k * b;
        cp_async16(dst + k * SA + i, src + e);
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
    const double2* p = St + (size_t)(qc % NSTAGE) * kc * SA;
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
  // GEMM acc = M * Bop over one b x b complex matrix streamed as nch chunks.
  // COUPLING: M holds (A, B) real pairs and the operand is C = zB - A.
  auto gemm = [&](const double2* Bop, bool coupling) {
#pragma unroll
    for (int j = 0; j < TPW; ++j) acc[j].zero();
    for (int c = 0; c < nch; ++c) {
      const double2* As = acquire();
      for (int kk = 0; kk < kc; kk += 4) {
        const int kg = c * kc + kk + t4;
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          double2 av = As[(kk + t4) * SA + 8 * mt[j] + g];
          if (coupling) av = make_double2(z.x * av.y - av.x, z.y * av.y);
          const double2 bv = Bop[(8 * ntl[j] + g) * SV + kg];
          cmma(acc[j], av, bv);
        }
      }
    }
  };

  // ---------------- forward sweep ----------------
  for (int l = 0; l < L; ++l) {
    if (l > 0) gemm(Vs, true);
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int row = l * b + 8 * mt[j] + g;
      const int cl0 = 8 * ntl[j] + 2 * t4;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + cl0 + h;
        double2 y = make_double2(0.0, 0.0);
        if (col < m) {
          if (a.complex_mode) y = W[row + (size_t)col * ldv];
          else y.x = a.y[row + (size_t)col * ldv];
        }
        const double ar = (l > 0) ? (h ? acc[j].r1 : acc[j].r0) : 0.0;
        const double ai = (l > 0) ? (h ? acc[j].i1 : acc[j].i0) : 0.0;
        Ts[(cl0 + h) * SV + 8 * mt[j] + g] = make_double2(y.x - ar, y.y - ai);
      }
    }
    gemm(Ts, false);  // y_l = S_l^{-1} t
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int row = l * b + 8 * mt[j] + g;
      const int cl0 = 8 * ntl[j] + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      Vs[(cl0 + 0) * SV + 8 * mt[j] + g] = y0;
      Vs[(cl0 + 1) * SV + 8 * mt[j] + g] = y1;
      if (l + 1 < L) {
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
    gemm(Vs, false);  // G_l x_{l+1}
    double2 x[TPW][2];
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int row = l * b + 8 * mt[j] + g;
      const int col = c0 + 8 * ntl[j] + 2 * t4;
      const double2 y0 = col < m ? W[row + (size_t)col * ldv] : make_double2(0.0, 0.0);
      const double2 y1 = col + 1 < m ? W[row + (size_t)(col + 1) * ldv] : make_double2(0.0, 0.0);
      x[j][0] = make_double2(y0.x - acc[j].r0, y0.y - acc[j].i0);
      x[j][1] = make_double2(y1.x - acc[j].r1, y1.y - acc[j].i1);
    }
    __syncthreads();  // every warp is done reading Vs
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = 8 * ntl[j] + 2 * t4;
      Vs[(cl0 + 0) * SV + 8 * mt[j] + g] = x[j][0];
      Vs[(cl0 + 1) * SV + 8 * mt[j] + g] = x[j][1];
      epilogue(l, j, x[j][0], x[j][1]);
    }
  }
  cp_async_wait<0>();
}

template <int NC, int TPW, int NSTAGE>
static cudaError_t launch_sweep(const BtSweepArgs& a, int kc, int warps, cudaStream_t st) {
  const int SA = a.b + 2, SV = a.b + 4;
  const size_t sm = sizeof(double2) * ((size_t)2 * NC * SV + (size_t)NSTAGE * kc * SA);
  auto kern = bt_sweep_kernel<NC, TPW, NSTAGE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dim3 grid((a.m + NC - 1) / NC, a.nodes);
  kern<<<grid, warps * 32, sm, st>>>(a, kc);
  ++g_launches;
  return cudaGetLastError();
}

static int pick_kc(int b) {
  int kc = 4;
  for (int c = 4; c <= b; c *= 2)
    if (b % c == 0 && (size_t)c * b * 16 <= 32 * 1024) kc = c;
  return kc;
}

cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st) {
  const int b = a.b;
  if (b % 16 != 0) return cudaErrorInvalidValue;
  const int kc = pick_kc(b);
  // NC = 16 while b is small (more reuse of each streamed block), 8 for big blocks (smem)
  const bool wide = b <= 64;
  const int tiles = (b / 8) * (wide ? 2 : 1);
  int tpw = 1;
  while (tiles / tpw > 16 || tiles % tpw != 0) tpw *= 2;
  const int warps = tiles / tpw;
  if (tpw > 8) return cudaErrorInvalidValue;
  const bool big = b >= 384;
  if (wide) {
    switch (tpw) {
      case 1: return launch_sweep<16, 1, 3>(a, kc, warps, st);
      case 2: return launch_sweep<16, 2, 3>(a, kc, warps, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (tpw) {
    case 1: return launch_sweep<8, 1, 3>(a, kc, warps, st);
    case 2: return launch_sweep<8, 2, 3>(a, kc, warps, st);
    case 4: return big ? launch_sweep<8, 4, 2>(a, kc, warps, st) : launch_sweep<8, 4, 3>(a, kc, warps, st);
    case 8: return big ? launch_sweep<8, 8, 2>(a, kc, warps, st) : launch_sweep<8, 8, 3>(a, kc, warps, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Q = -sum_s T_s, ascending s from zero (the ordered reduction of core.hpp:181-183)
// ---------------------------------------------------------------------------
__global__ void reduce_terms_kernel(const double* __restrict__ t, int nodes, int64_t slice, int n,
                                    int m, int ld, double* __restrict__ q) {
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const int64_t off = i + j * ld;
    double acc = 0.0;
    for (int s = 0; s < nodes; ++s) acc -= t[s * slice + off];
    q[off] = acc;
  }
}

cudaError_t reduce_terms(const double* t, int nodes, int64_t slice, int n, int m, int ld, double* q,
                         cudaStream_t st) {
  const int64_t total = (int64_t)n * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  reduce_terms_kernel<<<blocks, 256, 0, st>>>(t, nodes, slice, n, m, ld, q);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Y = Op X for a block-tridiagonal real operator (v0: one thread per output entry).
// ---------------------------------------------------------------------------
__global__ void bt_apply_kernel(int L, int b, const double2* __restrict__ abdiag,
                                const double2* __restrict__ ablow, int which,
                                const double* __restrict__ x, int ldx, double* __restrict__ y,
                                int ldy, int m) {
  const int64_t n = (int64_t)L * b;
  const int64_t total = n * m;
  const size_t bb = (size_t)b * b;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, j = idx / n;
    const int l = (int)(r / b), i = (int)(r % b);
    const double* xc = x + j * ldx;
    double acc = 0.0;
    const double* d = reinterpret_cast<const double*>(abdiag + l * bb) + which;
    for (int k = 0; k < b; ++k) acc += d[2 * (i + (size_t)k * b)] * xc[(int64_t)l * b + k];
    if (l > 0) {  // C_{l-1} (row i of block (l, l-1))
      const double* c = reinterpret_cast<const double*>(ablow + (l - 1) * bb) + which;
      for (int k = 0; k < b; ++k) acc += c[2 * (i + (size_t)k * b)] * xc[(int64_t)(l - 1) * b + k];
    }
    if (l + 1 < L) {  // C_l^T: (l, l+1) entry (i, k) = C_l(k, i)
      const double* c = reinterpret_cast<const double*>(ablow + l * bb) + which;
      for (int k = 0; k < b; ++k) acc += c[2 * (k + (size_t)i * b)] * xc[(int64_t)(l + 1) * b + k];
    }
    y[r + j * ldy] = acc;
  }
}

cudaError_t bt_apply(int L, int b, const double2* abdiag, const double2* ablow, int which,
                     const double* x, int ldx, double* y, int ldy, int m, cudaStream_t st) {
  const int64_t total = (int64_t)L * b * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  bt_apply_kernel<<<blocks, 256, 0, st>>>(L, b, abdiag, ablow, which, x, ldx, y, ldy, m);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
