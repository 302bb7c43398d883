// gemm.cu — FP64 DMMA GEMMs for sm_100a (mma.sync.m8n8k4.f64; tcgen05 has no f64 kind).
//
//  zgemm_batched : complex, column-major, C = alpha*A*B + beta*C, batched over contour
//                  nodes (blockIdx.z). Used by the dense LU trailing update
//                  (lu.hpp:44-50 restated blocked), the U12 = L11^{-1} A12 panel solve
//                  and both blocked triangular sweeps of the multi-RHS solve (lu.hpp:56-95).
//  dgemm         : real, C = alpha*op(A)*op(B) + beta*C with op in {N, T}; split-K with a
//                  fixed-order reduction (deterministic) for the tall-skinny projections
//                  Q^T (AQ), Q^T (BQ) of rayleigh_ritz (core.hpp:233-234, dense.hpp:76-90),
//                  X = Q Phi (dense.hpp:59-73) and dense operator applies (operator.hpp:132).
//
// Tiles: 64x64 per CTA, 8 warps as 2 (m) x 4 (n), warp tile 32x16 = 4x2 DMMA 8x8 tiles,
// 3-stage cp.async ring. Shared layouts are padded so fragment loads are conflict-free:
// A as [k][m] (stride 64+2 complex / 64+4 real), B as [n][k] (stride BK+4).

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

FEAST_DEV void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
FEAST_DEV void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}

// ===========================================================================
// complex
// ===========================================================================
namespace zg {
constexpr int BM = 64, BN = 64, BK = 16, NS = 3;
constexpr int SA = BM + 2;  // [k][m] double2
constexpr int SB = BK + 4;  // [n][k] double2
constexpr int STAGE = BK * SA + BN * SB;
}  // namespace zg

struct ZgemmArgs {
  int m, n, k;
  double2 alpha, beta;
  const double2* a;
  int lda;
  int64_t sa;
  const double2* b;
  int ldb;
  int64_t sb;
  double2* c;
  int ldc;
  int64_t sc;
  int splits = 1;  // split-K: blockIdx.z = batch * splits + slice; slice s covers K [s ksplit, ..)
  int ksplit = 0;
};

__global__ void __launch_bounds__(256, 2) zgemm_kernel(ZgemmArgs p) {
  using namespace zg;
  extern __shared__ __align__(16) double2 zsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int bz = blockIdx.z / p.splits, ks = blockIdx.z % p.splits;
  const int kbeg = ks * p.ksplit;
  const double2* A = p.a + bz * p.sa + (int64_t)kbeg * p.lda;
  const double2* B = p.b + bz * p.sb + kbeg;
  double2* C = p.c + blockIdx.z * p.sc;  // (split-K: slot of this batch entry and slice)
  const int kloc = p.splits > 1 ? min(p.ksplit, p.k - kbeg) : p.k;
  const int nk = (kloc + BK - 1) / BK;

  auto load = [&](int kt) {
    if (kt < nk) {
      double2* As = zsm + (kt % NS) * STAGE;
      double2* Bs = As + BK * SA;
      const int k0 = kt * BK;
      // A tile: BM x BK, element (m, k); 1024 entries, 4 per thread
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + r * 256;
        const int mm = e & (BM - 1), kk = e >> 6;
        const bool v = (m0 + mm < p.m) && (k0 + kk < kloc);
        const double2* src = v ? A + (m0 + mm) + (int64_t)(k0 + kk) * p.lda : A;
        cp_async16_zfill(As + kk * SA + mm, src, v);
      }
      // B tile: BK x BN, element (k, n)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + r * 256;
        const int kk = e & (BK - 1), nn = e >> 4;
        const bool v = (n0 + nn < p.n) && (k0 + kk < kloc);
        const double2* src = v ? B + (k0 + kk) + (int64_t)(n0 + nn) * p.ldb : B;
        cp_async16_zfill(Bs + nn * SB + kk, src, v);
      }
    }
    cp_async_commit();
  };

  CAcc acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j].zero();

#pragma unroll
  for (int s = 0; s < NS - 1; ++s) load(s);
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NS - 2>();
    __syncthreads();
    load(kt + NS - 1);
    const double2* As = zsm + (kt % NS) * STAGE;
    const double2* Bs = As + BK * SA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double2 af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[(kk + t4) * SA + wm * 32 + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[(wn * 16 + j * 8 + g) * SB + kk + t4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) cmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // B may alias C (in-place triangular apply): all reads done before writes

  const bool beta0 = p.beta.x == 0.0 && p.beta.y == 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 16 + j * 8 + 2 * t4 + h;
        if (col >= p.n) continue;
        const double2 v = make_double2(h ? acc[i][j].r1 : acc[i][j].r0, h ? acc[i][j].i1 : acc[i][j].i0);
        double2* cp = C + row + (int64_t)col * p.ldc;
        double2 out = cmul(p.alpha, v);
        if (!beta0) out = cadd(out, cmul(p.beta, *cp));
        *cp = out;
      }
    }
  }
}

// C = alpha sum_s P_s + beta C over the split-K slots P (m x n, ld m, slot (batch, slice)),
// slices added in order (deterministic)
__global__ void zsplitk_reduce_kernel(const double2* __restrict__ w, int splits, int m, int n, double2 alpha,
                                      double2 beta, double2* c, int ldc, int64_t sc) {
  const int bz = blockIdx.y;
  const int64_t slot = (int64_t)m * n, total = slot;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double2* src = w + (int64_t)bz * splits * slot + e;
    double2 acc = src[0];
    for (int s = 1; s < splits; ++s) acc = cadd(acc, src[s * slot]);
    double2* cp = c + bz * sc + i + j * ldc;
    double2 out = cmul(alpha, acc);
    if (beta.x != 0.0 || beta.y != 0.0) out = cadd(out, cmul(beta, *cp));
    *cp = out;
  }
}

// split-K workspace, per device, grown on demand from the stream-ordered pool (never freed)
static double2* zsplitk_ws(size_t count, cudaStream_t st) {
  static double2* ws[16] = {};
  static size_t cap[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16) return nullptr;
  if (cap[dev] < count) {
    if (ws[dev]) cudaFreeAsync(ws[dev], st);
    ws[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws[dev]), sizeof(double2) * count, st) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cap[dev] = count;
  }
  return ws[dev];
}

cudaError_t zgemm_batched(int m, int n, int k, double2 alpha, const double2* a, int lda, int64_t sa,
                          const double2* b, int ldb, int64_t sb, double2 beta, double2* c, int ldc,
                          int64_t sc, int batch, cudaStream_t st) {
  if (m <= 0 || n <= 0 || batch <= 0) return cudaSuccess;
  static bool attr = false;
  const int smem = zg::NS * zg::STAGE * (int)sizeof(double2);
  if (!attr) {
    cudaFuncSetAttribute(zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  // split-K when the whole grid cannot fill the GPU (the block factor's b x b products with a few
  // nodes: streamed node batches, one node per GPU) and K is long enough. The slice count is a
  // function of the per-entry shape only, so two batch sizes that both split use the same slices.
  // (Splitting a full grid only adds partial-sum traffic: the 16-node b = 512 factor ran 0.78 s
  // unsplit against 1.33 s split three ways.)
  const int tiles = ((n + zg::BN - 1) / zg::BN) * ((m + zg::BM - 1) / zg::BM);
  int splits = 1;
  if (tiles * batch < 148 && k >= 128) splits = std::min({(148 + tiles - 1) / tiles, k / 64, 8});
  if (splits > 1) {
    const int ksplit = ((k + splits - 1) / splits + zg::BK - 1) / zg::BK * zg::BK;
    splits = (k + ksplit - 1) / ksplit;
    const int64_t slot = (int64_t)m * n;
    double2* w = zsplitk_ws((size_t)slot * splits * batch, st);
    if (w) {
      ZgemmArgs p{m, n, k, make_double2(1.0, 0.0), make_double2(0.0, 0.0), a, lda, sa, b, ldb, sb, w, m, slot,
                  splits, ksplit};
      dim3 grid((n + zg::BN - 1) / zg::BN, (m + zg::BM - 1) / zg::BM, batch * splits);
      zgemm_kernel<<<grid, 256, smem, st>>>(p);
      ++g_launches;
      dim3 rg((unsigned)std::min<int64_t>((slot + 255) / 256, 1024), batch);
      zsplitk_reduce_kernel<<<rg, 256, 0, st>>>(w, splits, m, n, alpha, beta, c, ldc, sc);
      ++g_launches;
      return cudaGetLastError();
    }
  }
  ZgemmArgs p{m, n, k, alpha, beta, a, lda, sa, b, ldb, sb, c, ldc, sc};
  dim3 grid((n + zg::BN - 1) / zg::BN, (m + zg::BM - 1) / zg::BM, batch);
  zgemm_kernel<<<grid, 256, smem, st>>>(p);
  ++g_launches;
  return cudaGetLastError();
}

// ===========================================================================
// real
// ===========================================================================
namespace dg {
constexpr int BM = 64, BN = 64, BK = 32, NS = 3;
constexpr int SA = BM + 4;   // N-layout A: [k][m];   T-layout A: [m][k] with stride BK+4
constexpr int SAT = BK + 4;
constexpr int SB = BK + 4;   // N-layout B: [n][k];   T-layout B: [k][n] with stride BN+4
constexpr int SBT = BN + 4;
constexpr int A_ELEMS = BK * SA > BM * SAT ? BK * SA : BM * SAT;
constexpr int B_ELEMS = BN * SB > BK * SBT ? BN * SB : BK * SBT;
constexpr int STAGE = A_ELEMS + B_ELEMS;
}  // namespace dg

struct DgemmArgs {
  int m, n, k;
  int kslice;  // K per z-slice (split-K mode)
  const double* a;
  int lda;
  const double* b;
  int ldb;
  double* c;
  int ldc;
  int64_t sc;  // stride between z-slices of the output
  double alpha, beta;
  int batched;     // z indexes independent problems instead of K slices
  int64_t sa, sb;  // batch strides of A and B
  int symhalf = 0;  // > 0: C = [S1 | S2] of symmetric symhalf x symhalf halves: lower tiles skipped
};

// V16: 16-byte copies (pairs along each operand's contiguous dimension; the launcher checks
// even dimensions / leading dimensions and 16-byte aligned bases): half the copy instructions
template <bool TA, bool TB, bool V16>
__global__ void __launch_bounds__(256, 2) dgemm_kernel(DgemmArgs p) {
  using namespace dg;
  extern __shared__ __align__(16) double dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (p.symhalf && m0 / BM > (n0 % p.symhalf) / BN) return;  // mirrored by symmetrize_tiles
  const int kbeg = p.batched ? 0 : blockIdx.z * p.kslice;
  const int kend = p.batched ? p.k : min(p.k, kbeg + p.kslice);
  const int nk = (kend - kbeg + BK - 1) / BK;
  double* C = p.c + blockIdx.z * p.sc;
  if (p.batched) {
    p.a += blockIdx.z * p.sa;
    p.b += blockIdx.z * p.sb;
  }

  auto load = [&](int kt) {
    if (kt < nk) {
      double* As = dsm + (kt % NS) * STAGE;
      double* Bs = As + A_ELEMS;
      const int k0 = kbeg + kt * BK;
      if (V16) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int c = tid + r * 256;
          if (!TA) {
            const int mm = (c & (BM / 2 - 1)) * 2, kk = c / (BM / 2);
            const bool v = (m0 + mm < p.m) && (k0 + kk < kend);
            cp_async16_zfill(As + kk * SA + mm, v ? p.a + (m0 + mm) + (int64_t)(k0 + kk) * p.lda : p.a, v);
          } else {
            const int kk = (c & (BK / 2 - 1)) * 2, mm = c / (BK / 2);
            const bool v = (m0 + mm < p.m) && (k0 + kk < kend);
            cp_async16_zfill(As + mm * SAT + kk, v ? p.a + (k0 + kk) + (int64_t)(m0 + mm) * p.lda : p.a, v);
          }
          if (!TB) {
            const int kk = (c & (BK / 2 - 1)) * 2, nn = c / (BK / 2);
            const bool v = (n0 + nn < p.n) && (k0 + kk < kend);
            cp_async16_zfill(Bs + nn * SB + kk, v ? p.b + (k0 + kk) + (int64_t)(n0 + nn) * p.ldb : p.b, v);
          } else {
            const int nn = (c & (BN / 2 - 1)) * 2, kk = c / (BN / 2);
            const bool v = (n0 + nn < p.n) && (k0 + kk < kend);
            cp_async16_zfill(Bs + kk * SBT + nn, v ? p.b + (n0 + nn) + (int64_t)(k0 + kk) * p.ldb : p.b, v);
          }
        }
        cp_async_commit();
        return;
      }
      // A tile (BM x BK), 2048 doubles, 8 per thread
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int e = tid + r * 256;
        if (!TA) {  // A(m, k) at a[m + k*lda] -> As[k][m]
          const int mm = e & (BM - 1), kk = e >> 6;
          const bool v = (m0 + mm < p.m) && (k0 + kk < kend);
          const double* src = v ? p.a + (m0 + mm) + (int64_t)(k0 + kk) * p.lda : p.a;
          cp_async8_zfill(As + kk * SA + mm, src, v);
        } else {    // op(A)(m, k) = a[k + m*lda] -> As[m][k]
          const int kk = e & (BK - 1), mm = e >> 5;
          const bool v = (m0 + mm < p.m) && (k0 + kk < kend);
          const double* src = v ? p.a + (k0 + kk) + (int64_t)(m0 + mm) * p.lda : p.a;
          cp_async8_zfill(As + mm * SAT + kk, src, v);
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int e = tid + r * 256;
        if (!TB) {  // B(k, n) at b[k + n*ldb] -> Bs[n][k]
          const int kk = e & (BK - 1), nn = e >> 5;
          const bool v = (n0 + nn < p.n) && (k0 + kk < kend);
          const double* src = v ? p.b + (k0 + kk) + (int64_t)(n0 + nn) * p.ldb : p.b;
          cp_async8_zfill(Bs + nn * SB + kk, src, v);
        } else {    // op(B)(k, n) = b[n + k*ldb] -> Bs[k][n]
          const int nn = e & (BN - 1), kk = e >> 6;
          const bool v = (n0 + nn < p.n) && (k0 + kk < kend);
          const double* src = v ? p.b + (n0 + nn) + (int64_t)(k0 + kk) * p.ldb : p.b;
          cp_async8_zfill(Bs + kk * SBT + nn, src, v);
        }
      }
    }
    cp_async_commit();
  };

  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NS - 1; ++s) load(s);
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NS - 2>();
    __syncthreads();
    load(kt + NS - 1);
    const double* As = dsm + (kt % NS) * STAGE;
    const double* Bs = As + A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mm = wm * 32 + i * 8 + g;
        af[i] = TA ? As[mm * SAT + kk + t4] : As[(kk + t4) * SA + mm];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int nn = wn * 16 + j * 8 + g;
        bf[j] = TB ? Bs[(kk + t4) * SBT + nn] : Bs[nn * SB + kk + t4];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 16 + j * 8 + 2 * t4 + h;
        if (col >= p.n) continue;
        double* cp = C + row + (int64_t)col * p.ldc;
        const double v = p.alpha * acc[i][j][h];
        *cp = p.beta == 0.0 ? v : v + p.beta * *cp;
      }
  }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ w, int slices, int64_t slice, int m,
                                     int n, double alpha, double beta, double* __restrict__ c,
                                     int ldc) {
  const int64_t total = (int64_t)m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    double s = 0.0;
    for (int z = 0; z < slices; ++z) s += w[z * slice + i + j * m];
    double* cp = c + i + j * ldc;
    *cp = beta == 0.0 ? alpha * s : alpha * s + beta * *cp;
  }
}

template <bool TA, bool TB, bool V16>
static void set_attr_once() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(dgemm_kernel<TA, TB, V16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         dg::NS * dg::STAGE * (int)sizeof(double));
    done = true;
  }
}
template <bool TA, bool TB>
static void launch_dgemm(bool v16, dim3 grid, int smem, cudaStream_t st, const DgemmArgs& p) {
  if (v16) {
    set_attr_once<TA, TB, true>();
    dgemm_kernel<TA, TB, true><<<grid, 256, smem, st>>>(p);
  } else {
    set_attr_once<TA, TB, false>();
    dgemm_kernel<TA, TB, false><<<grid, 256, smem, st>>>(p);
  }
}

static cudaError_t dgemm_impl(char ta, char tb, int m, int n, int k, double alpha, const double* A, int lda,
                              const double* B, int ldb, double beta, double* C, int ldc, double* work,
                              size_t work_elems, cudaStream_t st, int symhalf);

cudaError_t dgemm(char ta, char tb, int m, int n, int k, double alpha, const double* A, int lda,
                  const double* B, int ldb, double beta, double* C, int ldc, double* work,
                  size_t work_elems, cudaStream_t st) {
  return dgemm_impl(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work, work_elems, st, 0);
}

// [S1 | S2] = Q^T [AQ | BQ] for symmetric S1, S2 (m x m each, m a multiple of the 64-wide
// tile): the strictly-lower tiles of each half are not computed; symmetrize_tiles fills them
cudaError_t dgemm_tn_sym2(int m, int k, const double* Q, int ldq, const double* AB, int ldab, double* C,
                          double* work, size_t work_elems, cudaStream_t st) {
  if (m % dg::BM != 0 || m % dg::BN != 0) return cudaErrorInvalidValue;
  return dgemm_impl('T', 'N', m, 2 * m, k, 1.0, Q, ldq, AB, ldab, 0.0, C, m, work, work_elems, st, m);
}

static cudaError_t dgemm_impl(char ta, char tb, int m, int n, int k, double alpha, const double* A, int lda,
                              const double* B, int ldb, double beta, double* C, int ldc, double* work,
                              size_t work_elems, cudaStream_t st, int symhalf) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  const bool TA = ta == 'T' || ta == 't', TB = tb == 'T' || tb == 't';
  const int tiles = ((m + dg::BM - 1) / dg::BM) * ((n + dg::BN - 1) / dg::BN);
  // split K until ~2 waves of CTAs, keeping >= 256 of K per slice
  int slices = 1;
  while (tiles * slices < 2 * 148 && k / (slices * 2) >= 256) slices *= 2;
  if ((size_t)slices * m * n > work_elems) slices = 1;
  int kslice = (k + slices - 1) / slices;
  kslice = (kslice + dg::BK - 1) / dg::BK * dg::BK;
  slices = (k + kslice - 1) / kslice;
  if (slices < 1) slices = 1;
  DgemmArgs p{m, n, k, kslice, A, lda, B, ldb, C, ldc, 0, alpha, beta, 0, 0, 0, symhalf};
  if (slices > 1) {
    p.c = work;
    p.ldc = m;
    p.sc = (int64_t)m * n;
    p.alpha = 1.0;
    p.beta = 0.0;
  }
  dim3 grid((n + dg::BN - 1) / dg::BN, (m + dg::BM - 1) / dg::BM, slices);
  const int smem = dg::NS * dg::STAGE * (int)sizeof(double);
  // 16-byte copies need even contiguous dimensions (A: K if transposed else M; B: N if transposed
  // else K; split-K slices are multiples of BK), even leading dimensions and 16-byte bases
  const bool v16 = ((TA ? k : m) % 2 == 0) && ((TB ? n : k) % 2 == 0) && lda % 2 == 0 && ldb % 2 == 0 &&
                   ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  if (!TA && !TB) launch_dgemm<false, false>(v16, grid, smem, st, p);
  if (TA && !TB) launch_dgemm<true, false>(v16, grid, smem, st, p);
  if (!TA && TB) launch_dgemm<false, true>(v16, grid, smem, st, p);
  if (TA && TB) launch_dgemm<true, true>(v16, grid, smem, st, p);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || slices == 1) return e;
  const int64_t total = (int64_t)m * n;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(work, slices, (int64_t)m * n, m, n, alpha, beta, C, ldc);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t dgemm_batched(bool TA, int m, int n, int k, double alpha, const double* A, int lda,
                          int64_t sa, const double* B, int ldb, int64_t sb, double beta, double* C,
                          int ldc, int64_t sc, int batch, cudaStream_t st) {
  if (m <= 0 || n <= 0 || batch <= 0) return cudaSuccess;
  DgemmArgs p{m, n, k, k, A, lda, B, ldb, C, ldc, sc, alpha, beta, 1, sa, sb};
  const int smem = dg::NS * dg::STAGE * (int)sizeof(double);
  for (int z0 = 0; z0 < batch; z0 += 65535) {
    const int nz = std::min(batch - z0, 65535);
    DgemmArgs q = p;
    q.a += z0 * sa;
    q.b += z0 * sb;
    q.c += z0 * sc;
    dim3 grid((n + dg::BN - 1) / dg::BN, (m + dg::BM - 1) / dg::BM, nz);
    // 16-byte copies when every operand pair stays 16-byte aligned (as in dgemm_impl)
    const bool v16 = ((TA ? k : m) % 2 == 0) && (k % 2 == 0) && lda % 2 == 0 && ldb % 2 == 0 && sa % 2 == 0 &&
                     sb % 2 == 0 && (reinterpret_cast<uintptr_t>(q.a) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(q.b) & 15) == 0;
    if (TA) launch_dgemm<true, false>(v16, grid, smem, st, q);
    else launch_dgemm<false, false>(v16, grid, smem, st, q);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t bt_apply(int L, int b, const double* diag, const double* low, const double* x, int ldx,
                     double* y, int ldy, int m, cudaStream_t st, int l0, int l1) {
  // (b <= 32 goes through band_apply on band-row copies, band_apply.cu); layers [l0, l1) of y:
  // y_l = D_l x_l + C_{l-1} x_{l-1} + C_l^T x_{l+1}
  if (l1 < 0) l1 = L;
  if (l1 <= l0) return cudaSuccess;
  const int64_t bb = (int64_t)b * b;
  cudaError_t e = dgemm_batched(false, b, m, b, 1.0, diag + l0 * bb, b, bb, x + (int64_t)l0 * b, ldx, b, 0.0,
                                y + (int64_t)l0 * b, ldy, b, l1 - l0, st);
  if (e != cudaSuccess) return e;
  const int a0 = std::max(l0, 1);  // y_l += C_{l-1} x_{l-1}, l in [a0, l1)
  if (l1 > a0) {
    e = dgemm_batched(false, b, m, b, 1.0, low + (a0 - 1) * bb, b, bb, x + (int64_t)(a0 - 1) * b, ldx, b, 1.0,
                      y + (int64_t)a0 * b, ldy, b, l1 - a0, st);
    if (e != cudaSuccess) return e;
  }
  const int u1 = std::min(l1, L - 1);  // y_l += C_l^T x_{l+1}, l in [l0, u1)
  if (u1 > l0)
    e = dgemm_batched(true, b, m, b, 1.0, low + l0 * bb, b, bb, x + (int64_t)(l0 + 1) * b, ldx, b, 1.0,
                      y + (int64_t)l0 * b, ldy, b, u1 - l0, st);
  return e;
}

__global__ void symmetrize_kernel(double* c, int m, int ld) {
  const int64_t total = (int64_t)m * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    if (i < j) {
      // hermitian_part (dense.hpp:127-134): (M(i,j) + M(j,i)) * 0.5 on both sides
      const double v = (c[i + (int64_t)j * ld] + c[j + (int64_t)i * ld]) * 0.5;
      c[i + (int64_t)j * ld] = v;
      c[j + (int64_t)i * ld] = v;
    }
  }
}

// hermitian_part (dense.hpp:127-134) of a matrix whose strictly-lower 64-wide tiles were not
// computed (dgemm_tn_sym2): inside a diagonal tile average the pair, elsewhere mirror the upper
__global__ void symmetrize_tiles_kernel(double* c, int m, int ld, int tile) {
  const int64_t total = (int64_t)m * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    if (i < j) {
      const double u = c[i + (int64_t)j * ld];
      const double v = (i / tile == j / tile) ? (u + c[j + (int64_t)i * ld]) * 0.5 : u;
      c[i + (int64_t)j * ld] = v;
      c[j + (int64_t)i * ld] = v;
    }
  }
}

cudaError_t symmetrize_tiles(double* c, int m, int ld, cudaStream_t st) {
  const int64_t total = (int64_t)m * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  symmetrize_tiles_kernel<<<blocks, 256, 0, st>>>(c, m, ld, dg::BM);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t symmetrize(double* c, int m, int ld, cudaStream_t st) {
  const int64_t total = (int64_t)m * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  symmetrize_kernel<<<blocks, 256, 0, st>>>(c, m, ld);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
