// misc.cu — residual reductions (residual.hpp:29-68) and small data-movement kernels.

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

// One CTA per eigenpair column; fixed-order block reductions (run-to-run deterministic).
// pairs: the rows are interleaved complex entries (Hermitian pencils), summed as complex moduli
__global__ void __launch_bounds__(256) residual_sums_kernel(int n, const double* __restrict__ ax,
                                                            const double* __restrict__ bx,
                                                            const double* __restrict__ x, int ld,
                                                            const double* __restrict__ lam,
                                                            double* __restrict__ out, int pairs) {
  const int j = blockIdx.x;
  const double l = lam[j];
  const double* a = ax + (int64_t)j * ld;
  const double* b = bx + (int64_t)j * ld;
  const double* xc = x + (int64_t)j * ld;
  double num = 0.0, den = 0.0, xn = 0.0;
  if (pairs) {
    for (int i = threadIdx.x; 2 * i + 1 < n; i += blockDim.x) {
      num += hypot(a[2 * i] - l * b[2 * i], a[2 * i + 1] - l * b[2 * i + 1]);
      den += hypot(a[2 * i], a[2 * i + 1]);
      xn += hypot(xc[2 * i], xc[2 * i + 1]);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      num += fabs(a[i] - l * b[i]);
      den += fabs(a[i]);
      xn += fabs(xc[i]);
    }
  }
  __shared__ double red[3][8];
  num = warp_sum(num);
  den = warp_sum(den);
  xn = warp_sum(xn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = num; red[1][warp] = den; red[2][warp] = xn; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
    out[3 * j + threadIdx.x] = s;
  }
}

cudaError_t residual_sums(int n, int m, const double* ax, const double* bx, const double* x, int ld,
                          const double* lam, double* out, cudaStream_t st, bool pairs) {
  if (m <= 0) return cudaSuccess;
  residual_sums_kernel<<<m, 256, 0, st>>>(n, ax, bx, x, ld, lam, out, pairs ? 1 : 0);
  ++g_launches;
  return cudaGetLastError();
}

// Cancellation factor of the Ritz block X = Q Phi (m x mo Phi, ld m), the look-ahead contour
// pass's admission test (feast_gpu.cpp, lookahead): K = max_i sum_j ||q_j||_B |Phi_ji| with
// ||q_j||_B = sqrt(B_Q(j, j)). Every X column has unit B-norm, so K = 1 means no cancellation in
// forming X; K measures how much the per-column rounding of solves on B Q grows when they are
// recombined by Phi afterwards. One CTA per column i; the max over columns is order-independent
// (atomicMax on the bits of non-negative doubles).
__global__ void __launch_bounds__(128) cancellation_factor_kernel(int m, const double* __restrict__ bq, int ldb,
                                                                  const double* __restrict__ phi, int ldp,
                                                                  unsigned long long* __restrict__ out) {
  const int i = blockIdx.x;
  double s = 0.0;
  for (int j = threadIdx.x; j < m; j += blockDim.x)
    s += sqrt(fmax(bq[j + (int64_t)j * ldb], 0.0)) * fabs(phi[j + (int64_t)i * ldp]);
  s = warp_sum(s);
  __shared__ double red[4];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double k = red[0] + red[1] + red[2] + red[3];
    atomicMax(out, __double_as_longlong(k));
  }
}

cudaError_t cancellation_factor(int m, int mo, const double* bq, int ldb, const double* phi, int ldp,
                                double* out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(double), st);
  if (mo <= 0) return cudaGetLastError();
  cancellation_factor_kernel<<<mo, 128, 0, st>>>(m, bq, ldb, phi, ldp, reinterpret_cast<unsigned long long*>(out));
  ++g_launches;
  return cudaGetLastError();
}

// dst[i] = sum_{r < slices} src[r * stride + i], summed in slice order (the loopback group's
// allreduce: every rank adds the same slots in the same order, so all get the same bits)
__global__ void sum_slices_kernel(const double* __restrict__ src, int slices, int64_t stride, size_t count,
                                  double* __restrict__ dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double acc = src[i];
    for (int r = 1; r < slices; ++r) acc += src[r * stride + i];
    dst[i] = acc;
  }
}

cudaError_t sum_slices(const double* src, int slices, int64_t stride, size_t count, double* dst, cudaStream_t st) {
  if (!count) return cudaSuccess;
  sum_slices_kernel<<<(unsigned)std::min<size_t>((count + 255) / 256, 4096), 256, 0, st>>>(src, slices, stride,
                                                                                         count, dst);
  ++g_launches;
  return cudaGetLastError();
}

// out = x + t y (add_scaled, operator.hpp:282-304, on the device storage of A0 and S)
__global__ void axpby_kernel(const double* __restrict__ x, const double* __restrict__ y, double t, size_t n,
                             double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = x[i] + y[i] * t;
}

cudaError_t axpby(const double* x, const double* y, double t, size_t n, double* out, cudaStream_t st) {
  if (!n) return cudaSuccess;
  axpby_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, st>>>(x, y, t, n, out);
  ++g_launches;
  return cudaGetLastError();
}

// ||A||_1 = max absolute row sum of a symmetric operator (operator.hpp:195-212): block-tridiagonal
// storage (L > 0: row i of layer l = [C_{l-1} | D_l | C_l^T](i, :)) or dense n x n (L = 0, b = n);
// one thread per row, max by atomicMax on the bits of non-negative doubles
__global__ void operator_norm1_kernel(int L, int b, const double* __restrict__ a, unsigned long long* out) {
  const int64_t rows = L > 0 ? (int64_t)L * b : b;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    if (L > 0) {
      const int l = (int)(r / b), i = (int)(r % b);
      const int64_t bb = (int64_t)b * b, nd = (int64_t)L * bb;
      for (int j = 0; j < b; ++j) s += fabs(a[l * bb + i + (int64_t)j * b]);
      if (l > 0) for (int j = 0; j < b; ++j) s += fabs(a[nd + (l - 1) * bb + i + (int64_t)j * b]);
      if (l + 1 < L) for (int j = 0; j < b; ++j) s += fabs(a[nd + l * bb + j + (int64_t)i * b]);
    } else {
      for (int j = 0; j < b; ++j) s += fabs(a[r + (int64_t)j * b]);
    }
    atomicMax(out, __double_as_longlong(s));
  }
}

cudaError_t operator_norm1(int L, int b, const double* a, double* out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(double), st);
  const int64_t rows = L > 0 ? (int64_t)L * b : b;
  operator_norm1_kernel<<<(unsigned)std::min<int64_t>((rows + 255) / 256, 4096), 256, 0, st>>>(
      L, b, a, reinterpret_cast<unsigned long long*>(out));
  ++g_launches;
  return cudaGetLastError();
}

// out(:, j) = J in(:, j): (re, im) -> (-im, re) per interleaved pair (multiplication by i of a
// complex column carried as a real one); rows [n, ld) zero
__global__ void rotate_pairs_kernel(const double* __restrict__ in, int n, int64_t ld, int m, double* __restrict__ out) {
  const int64_t total = ld * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % ld, j = e / ld;
    const double* c = in + j * ld;
    out[i + j * ld] = i >= n ? 0.0 : ((i & 1) ? c[i - 1] : -c[i + 1]);
  }
}

cudaError_t rotate_pairs(const double* in, int n, int64_t ld, int m, double* out, cudaStream_t st) {
  const int64_t total = ld * m;
  if (!total) return cudaSuccess;
  rotate_pairs_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(in, n, ld, m, out);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void fill_zero_kernel(double* p, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

cudaError_t fill_zero(double* p, size_t count, cudaStream_t st) {
  if (!count) return cudaSuccess;
  fill_zero_kernel<<<(unsigned)std::min<size_t>((count + 255) / 256, 4096), 256, 0, st>>>(p, count);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void gather_columns_kernel(const double* src, int ld, int n, const int* idx, int m,
                                      double* dst, int ldd) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)n * m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k % n), j = (int)(k / n);
    dst[i + (int64_t)j * ldd] = src[i + (int64_t)idx[j] * ld];
  }
}

cudaError_t gather_columns(const double* src, int ld, int n, const int* idx, int m, double* dst,
                           int ldd, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const int64_t total = (int64_t)n * m;
  gather_columns_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(
      src, ld, n, idx, m, dst, ldd);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void conj_kernel(double2* p, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    p[i].y = -p[i].y;
}

cudaError_t conj_inplace(double2* p, size_t count, cudaStream_t st) {
  if (!count) return cudaSuccess;
  conj_kernel<<<(unsigned)std::min<size_t>((count + 255) / 256, 4096), 256, 0, st>>>(p, count);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void split_complex_kernel(const double2* w, double* y, int n, int64_t ld, int m) {
  const int64_t total = (int64_t)n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e - j * n;
    const double2 v = w[i + j * ld];
    y[i + j * ld] = v.x;
    y[i + (j + m) * ld] = v.y;
  }
}

__global__ void merge_complex_kernel(double2* w, int n, int64_t ld, int m) {
  const int64_t total = (int64_t)n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e - j * n;
    const double2 re = w[i + j * ld], im = w[i + (j + m) * ld];
    w[i + j * ld] = make_double2(re.x - im.y, re.y + im.x);
  }
}

cudaError_t split_complex(const double2* w, double* y, int n, int64_t ld, int m, cudaStream_t st) {
  const int64_t total = (int64_t)n * m;
  if (!total) return cudaSuccess;
  split_complex_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(w, y, n, ld, m);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t merge_complex(double2* w, int n, int64_t ld, int m, cudaStream_t st) {
  const int64_t total = (int64_t)n * m;
  if (!total) return cudaSuccess;
  merge_complex_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(w, n, ld, m);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu

namespace feastgpu {

// ---------------------------------------------------------------------------
// random_block<double> (core.hpp:84-106) on the device, bit-identical to the host's
// std::mt19937_64(seed): Y(i, j) = 2 * ((w >> 11) * 2^-53) - 1 for the column-major stream of
// words w. MT19937-64 is one sequential recurrence, but each 312-word twist splits into two
// data-parallel halves (words 0..155 read only old state; words 156..311 read old state and
// the new words 0..155), so one CTA runs the whole stream with three barriers per 312 words.
// ---------------------------------------------------------------------------
namespace {
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;
FEAST_DEV uint64_t mt_mix(uint64_t hi, uint64_t lo) {
  const uint64_t y = (hi & kMtUpper) | (lo & kMtLower);
  return (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}
FEAST_DEV uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}
}  // namespace

__global__ void __launch_bounds__(320) mt64_block_kernel(uint64_t seed, int n, int m, double* __restrict__ out,
                                                         int ld) {
  __shared__ uint64_t x[kMtN];
  const int i = threadIdx.x;
  if (i == 0) {
    x[0] = seed;
    for (int k = 1; k < kMtN; ++k) x[k] = 6364136223846793005ull * (x[k - 1] ^ (x[k - 1] >> 62)) + (uint64_t)k;
  }
  const int64_t total = (int64_t)n * m;
  int row = i % n, col = i / n;           // position of word o = round * 312 + i
  const int step_col = kMtN / n, step_row = kMtN % n;
  for (int64_t base = 0; base < total; base += kMtN) {
    __syncthreads();
    uint64_t a = 0, b = 0, c = 0;
    if (i < kMtN) {
      a = x[i];
      if (i + 1 < kMtN) b = x[i + 1];
      if (i < kMtM) c = x[i + kMtM];
    }
    __syncthreads();
    uint64_t w = 0;
    if (i < kMtM) {
      w = c ^ mt_mix(a, b);
      x[i] = w;
    }
    __syncthreads();
    if (i >= kMtM && i < kMtN) {
      w = x[i - kMtM] ^ mt_mix(a, i + 1 < kMtN ? b : x[0]);
      x[i] = w;
    }
    if (i < kMtN && base + i < total)
      out[row + (int64_t)col * ld] = 2.0 * ((double)(mt_temper(w) >> 11) * 0x1p-53) - 1.0;
    row += step_row;
    col += step_col;
    if (row >= n) {
      row -= n;
      ++col;
    }
  }
}

__global__ void interleave_pairs_kernel(const double* __restrict__ a, const double* __restrict__ b, size_t n,
                                        double2* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_double2(a[i], b[i]);
}

cudaError_t interleave_pairs(const double* a, const double* b, size_t n, double2* out, cudaStream_t st) {
  if (!n) return cudaSuccess;
  interleave_pairs_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(a, b, n, out);
  ++g_launches;
  return cudaGetLastError();
}

// W_s(i, j) = (Y(i, j), 0) for every node slot s < nodes, i < n (ld ld), j < m
__global__ void real_to_complex_slots_kernel(const double* __restrict__ y, int64_t n, int64_t m, int64_t ld,
                                             int nodes, double2* __restrict__ w) {
  const int64_t per = ld * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < per * nodes;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx % per;
    w[idx] = make_double2(y[k], 0.0);
  }
}

cudaError_t real_to_complex_slots(const double* y, int64_t ld, int64_t m, int nodes, double2* w, cudaStream_t st) {
  const int64_t total = ld * m * nodes;
  if (!total) return cudaSuccess;
  real_to_complex_slots_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
      y, ld, m, ld, nodes, w);
  ++g_launches;
  return cudaGetLastError();
}

// accumulate_subspace_hermitian's reduction (core.hpp:198-214) for real symmetric pencils: node
// slot s holds W_s = G_s [Yr | Yi] (ld x 2m complex). With W1 = W_s(:, j), W2 = W_s(:, m + j):
//   s1 = G Y = W1 + i W2,  s2 = G^H Y = conj(G conj Y) = conj(W1) + i conj(W2)
//   Q -= c1 s1 + c2 s2,    c1 = coeff_s / 2, c2 = conj(coeff_s) / 2   (coeff = w r e^{i theta} / 2)
// summed over s in ascending order (accumulate: continue Q from an earlier node batch)
__global__ void hermitian_terms_kernel(const double2* __restrict__ w, int nodes, int64_t ld, int n, int m,
                                       const double2* __restrict__ coeff, double2* __restrict__ q,
                                       int accumulate) {
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    double2 acc = accumulate ? q[i + j * ld] : make_double2(0.0, 0.0);
    for (int s = 0; s < nodes; ++s) {
      const double2* ws = w + (int64_t)s * ld * 2 * m;
      const double2 w1 = ws[i + j * ld], w2 = ws[i + (j + m) * ld];
      const double2 s1 = make_double2(w1.x - w2.y, w1.y + w2.x);   // W1 + i W2
      const double2 s2 = make_double2(w1.x + w2.y, -w1.y + w2.x);  // conj(W1) + i conj(W2)
      const double2 cf = coeff[s];
      const double2 c1 = make_double2(0.5 * cf.x, 0.5 * cf.y), c2 = make_double2(0.5 * cf.x, -0.5 * cf.y);
      const double2 t1 = cmul(c1, s1), t2 = cmul(c2, s2);
      const double2 term = make_double2(t1.x + t2.x, t1.y + t2.y);
      acc.x -= term.x;
      acc.y -= term.y;
    }
    q[i + j * ld] = acc;
  }
}

cudaError_t hermitian_terms(const double2* w, int nodes, int64_t ld, int n, int m, const double2* coeff,
                            double2* q, int accumulate, cudaStream_t st) {
  const int64_t total = (int64_t)n * m;
  if (!total) return cudaSuccess;
  hermitian_terms_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
      w, nodes, ld, n, m, coeff, q, accumulate);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t random_block_device(uint64_t seed, int n, int m, double* out, int ld, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  mt64_block_kernel<<<1, 320, 0, st>>>(seed, n, m, out, ld);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
