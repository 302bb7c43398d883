// csr_ingest.cu — CSR operators taken in on the device (set_pencil's block-tridiagonal route).
//
// The reference validates a CSR SymmetricOperator on the host (operator.hpp:237-268: index
// range, a mirror entry with the same value for every off-diagonal entry), takes its 1-norm
// (operator.hpp:195-212), picks the banded route from the bandwidth (inner_solver.hpp:84-92)
// and assembles the band (assemble.hpp:12-57). Here the CSR arrays are uploaded once and all of
// that runs as two passes over the nonzeros on the device; the host reads back one small
// record (first error, bandwidth, which block sizes hold the pattern, the 1-norm) and makes the
// same decisions and raises the same errors as the host path (feast_gpu.cpp: validate_csr,
// csr_bandwidth, csr_fits_blocktri, norm_one, to_blocktri), which remains for the other
// storage kinds.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kernels.h"

namespace feastgpu {

namespace {

// std::lower_bound as libstdc++ implements it (the host check calls it on rows that may be
// unsorted, so the probe sequence itself must match for the error reported to be the same)
__device__ __forceinline__ int lower_bound_idx(const int* __restrict__ col, int lo, int hi, int v) {
  int first = lo, len = hi - lo;
  while (len > 0) {
    const int half = len >> 1;
    const int mid = first + half;
    if (col[mid] < v) {
      first = mid + 1;
      len = len - half - 1;
    } else {
      len = half;
    }
  }
  return first;
}

// one warp per row: lanes take the row's entries, lane 0 sums |values| in entry order (the
// host's order, so the 1-norm is bit-identical)
__global__ void __launch_bounds__(256) csr_scan_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const double* __restrict__ val, CsrStats* __restrict__ st) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int k0 = rp[i], k1 = rp[i + 1];
    unsigned long long err = ~0ull;
    int bw = 0;
    unsigned bad = 0;
    for (int k = k0 + lane; k < k1; k += 32) {
      const int j = ci[k];
      if (j < 0 || j >= n) {
        err = min(err, (unsigned long long)k * 4 + kCsrOutOfRange);
        continue;
      }
      const int d = i > j ? i - j : j - i;
      bw = max(bw, d);
#pragma unroll
      for (int s = 0; s < kCsrBlockCandidates; ++s) {
        const int li = i >> (4 + s), lj = j >> (4 + s);
        if (li - lj > 1 || lj - li > 1) bad |= 1u << s;
      }
      if (j <= i) continue;
      // mirror (j, i) with the same value (operator.hpp:237-261)
      const int b = rp[j], e = rp[j + 1];
      const int f = lower_bound_idx(ci, b, e, i);
      const double v = val[k];
      if (f == e || ci[f] != i) {
        bool found = false, differ = false;
        for (int q = b; q < e && !differ; ++q)
          if (ci[q] == i) {
            found = true;
            differ = val[q] != v;
          }
        if (differ) err = min(err, (unsigned long long)k * 4 + kCsrMirrorDiffers);
        else if (!found) err = min(err, (unsigned long long)k * 4 + kCsrMirrorMissing);
      } else if (val[f] != v) {
        err = min(err, (unsigned long long)k * 4 + kCsrMirrorDiffers);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      err = min(err, __shfl_xor_sync(0xffffffffu, err, o));
      bw = max(bw, __shfl_xor_sync(0xffffffffu, bw, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
      double s = 0.0;
      for (int k = k0; k < k1; ++k) s += fabs(val[k]);
      // non-negative doubles order like their bit patterns (a NaN sum is skipped, as std::max
      // skips it on the host)
      if (!(s != s)) atomicMax(&st->norm1_bits, (unsigned long long)__double_as_longlong(s));
      if (err != ~0ull) atomicMin(&st->first_error, err);
      if (bw) atomicMax(&st->bandwidth, bw);
      if (bad) atomicOr(&st->misfit_mask, bad);
    }
  }
}

__global__ void csr_stats_init_kernel(CsrStats* st, int count) {
  const int t = threadIdx.x;
  if (t < count) {
    st[t].first_error = ~0ull;
    st[t].norm1_bits = 0ull;
    st[t].bandwidth = 0;
    st[t].misfit_mask = 0u;
  }
}

// one thread per row: row i only ever writes row i of its layer's diagonal block and of the
// coupling below it, so the scatter is race-free and sums duplicates in entry order (as
// to_blocktri does); rows of the padding get B = I
__global__ void csr_to_blocktri_kernel(int n, int npad, int sh, const int* __restrict__ rp, const int* __restrict__ ci,
                                       const double* __restrict__ val, double* __restrict__ diag,
                                       double* __restrict__ low, int unit_padding) {
  const int msk = (1 << sh) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x) {
    const int li = i >> sh, ii = i & msk;
    if (i >= n) {
      if (unit_padding) diag[((size_t)li << (2 * sh)) + ii + ((size_t)ii << sh)] = 1.0;
      continue;
    }
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k], lj = j >> sh, jj = j & msk;
      if (li == lj) diag[((size_t)li << (2 * sh)) + ii + ((size_t)jj << sh)] += val[k];
      else if (li == lj + 1) low[((size_t)lj << (2 * sh)) + ii + ((size_t)jj << sh)] += val[k];
    }
  }
}

}  // namespace

cudaError_t csr_scan(int n, const int* row_ptr, const int* col_idx, const double* values, CsrStats* stats,
                     bool init, cudaStream_t st) {
  if (init) {
    csr_stats_init_kernel<<<1, 32, 0, st>>>(stats, 1);
    ++g_launches;
  }
  const int warps = n;
  const int blocks = (int)std::min<int64_t>(((int64_t)warps * 32 + 255) / 256, 148 * 8);
  csr_scan_kernel<<<blocks, 256, 0, st>>>(n, row_ptr, col_idx, values, stats);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t csr_to_blocktri(int n, int b, int L, const int* row_ptr, const int* col_idx, const double* values,
                            double* diag, double* low, bool unit_padding, cudaStream_t st) {
  int sh = 0;
  while ((1 << sh) < b) ++sh;
  const size_t nd = (size_t)L * b * b, nl = (size_t)(L > 1 ? L - 1 : 0) * b * b;
  cudaError_t err = cudaMemsetAsync(diag, 0, sizeof(double) * nd, st);
  if (err != cudaSuccess) return err;
  if (nl && (err = cudaMemsetAsync(low, 0, sizeof(double) * nl, st)) != cudaSuccess) return err;
  const int npad = L * b;
  csr_to_blocktri_kernel<<<(npad + 127) / 128, 128, 0, st>>>(n, npad, sh, row_ptr, col_idx, values, diag, low,
                                                            unit_padding ? 1 : 0);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
