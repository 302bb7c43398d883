// band_apply.cu — the block-tridiagonal operator applies of the Rayleigh-Ritz step
// (SymmetricOperator::apply, operator.hpp:132-158: A Q, B Q, B X) for small blocks (b = 16, 32),
// from a band-row copy of the operator built once per pencil:
//
//   band row r = l b + i  =  [ C_{l-1}(i, :) | D_l(i, :) | C_l^T(i, :) ]   (3b doubles)
//
// so the rows of one layer are a dense b x 3b tile and Y_l = band_l X[(l-1)b : (l+2)b, :] is a
// K = 3b DMMA product with no zero blocks (the older bt_apply_small_kernel multiplies a 64 x 96
// window, twice the work). A CTA owns 64 rows x 64 columns: the X window (64 + 2b rows) and the
// band tiles arrive by 16-byte cp.async, the results leave through shared memory as 16-byte
// coalesced stores. TWO = A and B from the same X window in one pass (A Q and B Q).

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

FEAST_DEV void cp_async16z(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0));
}

__global__ void band_rows_kernel(int L, int B, const double* __restrict__ diag, const double* __restrict__ low,
                                 double* __restrict__ ab) {
  const int W = 3 * B;
  const int64_t BB = (int64_t)B * B, total = (int64_t)L * B * W;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / W;
    const int k = (int)(e % W), l = (int)(r / B), i = (int)(r % B), seg = k / B, j = k % B;
    double v = 0.0;
    if (seg == 0) v = l >= 1 ? low[(l - 1) * BB + i + (int64_t)j * B] : 0.0;  // M(l, l-1) = C_{l-1}
    else if (seg == 1) v = diag[l * BB + i + (int64_t)j * B];                 // D_l
    else v = l + 1 < L ? low[l * BB + j + (int64_t)i * B] : 0.0;              // M(l, l+1) = C_l^T
    ab[e] = v;
  }
}

template <int B, bool TWO>
__global__ void __launch_bounds__(256) band_apply_kernel(int n, int rbeg, int rend, const double* __restrict__ ab1,
                                                         const double* __restrict__ ab2,
                                                         const double* __restrict__ x, int ldx, double* y1,
                                                         double* y2, int ldy, int m) {
  constexpr int RT = 64, NCOL = 64, W = 3 * B, XR = RT + 2 * B, SX = XR + 4, SA = W + 4, SY = RT + 4;
  constexpr int LAYERS = RT / B, WPL = 8 / LAYERS, COLS = NCOL / WPL, MF = B / 8, NF = COLS / 8;
  extern __shared__ __align__(16) double sm[];
  double* Xs = sm;                  // [NCOL][SX]: X(c0 + k, n0 + col) at Xs[col * SX + k]
  double* As1 = Xs + NCOL * SX;     // [RT][SA]: band row r0 + rr at As1[rr * SA]
  double* As2 = As1 + RT * SA;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int r0 = rbeg + blockIdx.y * RT, n0 = blockIdx.x * NCOL, c0 = r0 - B;
  for (int e = tid; e < NCOL * (XR / 2); e += 256) {
    const int col = e / (XR / 2), ch = e - col * (XR / 2), row = c0 + 2 * ch, gc = n0 + col;
    const bool v = gc < m && row >= 0 && row < n;
    cp_async16z(Xs + col * SX + 2 * ch, v ? x + row + (int64_t)gc * ldx : x, v);
  }
  for (int e = tid; e < RT * (W / 2); e += 256) {
    const int rr = e / (W / 2), ch = e - rr * (W / 2);
    const bool v = r0 + rr < rend;
    cp_async16z(As1 + rr * SA + 2 * ch, v ? ab1 + (int64_t)(r0 + rr) * W + 2 * ch : ab1, v);
    if (TWO) cp_async16z(As2 + rr * SA + 2 * ch, v ? ab2 + (int64_t)(r0 + rr) * W + 2 * ch : ab2, v);
  }
  cp_async_wait_all();
  __syncthreads();
  const int ly = warp / WPL, cb = (warp % WPL) * COLS;
  double acc1[MF][NF][2] = {}, acc2[MF][NF][2] = {};
#pragma unroll 4
  for (int kk = 0; kk < W; kk += 4) {
    double a1[MF], a2[MF], bf[NF];
#pragma unroll
    for (int i = 0; i < MF; ++i) {
      a1[i] = As1[(ly * B + 8 * i + g) * SA + kk + t4];
      if (TWO) a2[i] = As2[(ly * B + 8 * i + g) * SA + kk + t4];
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) bf[j] = Xs[(cb + 8 * j + g) * SX + ly * B + kk + t4];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        dmma884(acc1[i][j][0], acc1[i][j][1], a1[i], bf[j]);
        if (TWO) dmma884(acc2[i][j][0], acc2[i][j][1], a2[i], bf[j]);
      }
  }
  // epilogue through shared memory (the X window is dead): Ys[col * SY + row], 16-byte stores
  double* Ys = Xs;
#pragma unroll
  for (int pass = 0; pass < (TWO ? 2 : 1); ++pass) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          Ys[(cb + 8 * j + 2 * t4 + h) * SY + ly * B + 8 * i + g] = pass ? acc2[i][j][h] : acc1[i][j][h];
    __syncthreads();
    double* y = pass ? y2 : y1;
    for (int e = tid; e < NCOL * (RT / 2); e += 256) {
      const int col = e / (RT / 2), pr = e - col * (RT / 2), row = r0 + 2 * pr, gc = n0 + col;
      if (gc < m && row < rend)
        *reinterpret_cast<double2*>(y + row + (int64_t)gc * ldy) = *reinterpret_cast<const double2*>(Ys + col * SY + 2 * pr);
    }
  }
}

cudaError_t band_rows(int L, int b, const double* diag, const double* low, double* ab, cudaStream_t st) {
  const int64_t total = (int64_t)L * b * 3 * b;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  band_rows_kernel<<<blocks, 256, 0, st>>>(L, b, diag, low, ab);
  ++g_launches;
  return cudaGetLastError();
}

template <int B, bool TWO>
static cudaError_t launch_band(int n, int rbeg, int rend, const double* ab1, const double* ab2, const double* x,
                               int ldx, double* y1, double* y2, int ldy, int m, cudaStream_t st) {
  constexpr int RT = 64, NCOL = 64, W = 3 * B, XR = RT + 2 * B;
  const int sm = (int)sizeof(double) * (NCOL * (XR + 4) + (TWO ? 2 : 1) * RT * (W + 4));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(band_apply_kernel<B, TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    attr = true;
  }
  if (rend <= rbeg || m <= 0) return cudaSuccess;
  dim3 grid((m + NCOL - 1) / NCOL, (rend - rbeg + RT - 1) / RT);
  band_apply_kernel<B, TWO><<<grid, 256, sm, st>>>(n, rbeg, rend, ab1, ab2, x, ldx, y1, y2, ldy, m);
  ++g_launches;
  return cudaGetLastError();
}

// rows [l0 b, l1 b) of y1 = A x (and y2 = B x when ab2 != nullptr); b = 16 or 32, n = L b,
// ldx / ldy even; x is read on rows [l0 b - b, l1 b + b) within [0, n)
cudaError_t band_apply(int L, int b, const double* ab1, const double* ab2, const double* x, int ldx, double* y1,
                       double* y2, int ldy, int m, cudaStream_t st, int l0, int l1) {
  const int n = L * b;
  if (l1 < 0) l1 = L;
  const int rb = l0 * b, re = l1 * b;
  if (b == 16) return ab2 ? launch_band<16, true>(n, rb, re, ab1, ab2, x, ldx, y1, y2, ldy, m, st)
                          : launch_band<16, false>(n, rb, re, ab1, ab2, x, ldx, y1, y2, ldy, m, st);
  if (b == 32) return ab2 ? launch_band<32, true>(n, rb, re, ab1, ab2, x, ldx, y1, y2, ldy, m, st)
                          : launch_band<32, false>(n, rb, re, ab1, ab2, x, ldx, y1, y2, ldy, m, st);
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
