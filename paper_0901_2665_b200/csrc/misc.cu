// misc.cu — residual reductions (residual.hpp:29-68) and small data-movement kernels.

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

// One CTA per eigenpair column; fixed-order block reductions (run-to-run deterministic).
__global__ void __launch_bounds__(256) residual_sums_kernel(int n, const double* __restrict__ ax,
                                                            const double* __restrict__ bx,
                                                            const double* __restrict__ x, int ld,
                                                            const double* __restrict__ lam,
                                                            double* __restrict__ out) {
  const int j = blockIdx.x;
  const double l = lam[j];
  const double* a = ax + (int64_t)j * ld;
  const double* b = bx + (int64_t)j * ld;
  const double* xc = x + (int64_t)j * ld;
  double num = 0.0, den = 0.0, xn = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    num += fabs(a[i] - l * b[i]);
    den += fabs(a[i]);
    xn += fabs(xc[i]);
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
                          const double* lam, double* out, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  residual_sums_kernel<<<m, 256, 0, st>>>(n, ax, bx, x, ld, lam, out);
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
