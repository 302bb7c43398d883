// common.cuh — shared device helpers for libfeastgpu (sm_100a only).
//
// FP64 on sm_100a: tcgen05.mma has no .kind::f64 and wgmma does not exist, so the
// FP64 tensor path is the warp-level DMMA (mma.sync.aligned.m8n8k4 .f64), measured at
// 37.1 TFLOP/s on this pool's B200 (tools/microbench/fp64_peak.cu) vs 33 TFLOP/s for DFMA.
// Complex products are 4 real DMMAs (no 3M trick, for accuracy).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define FEAST_DEV __device__ __forceinline__

namespace feastgpu {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// complex helpers on double2 (x = re, y = im), interleaved like std::complex<double>
// ---------------------------------------------------------------------------
FEAST_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
FEAST_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
FEAST_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
FEAST_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// Complex division in Smith's scaled form (overflow-safe, ~1 ulp).
FEAST_DEV double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    const double r = b.x / b.y, d = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}
FEAST_DEV double cabs_(double2 a) { return hypot(a.x, a.y); }

// ---------------------------------------------------------------------------
// DMMA: D(8x8) += A(8x4, row) * B(4x8, col), fp64. Lane l: g = l>>2, t = l&3.
//   a = A[g][t], b = B[t][g], c0 = C[g][2t], c1 = C[g][2t+1].
// ---------------------------------------------------------------------------
FEAST_DEV void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// complex tile accumulate: (cr + i ci) += (a) * (b), all 8x8 / 8x4 / 4x8 fragments
struct CAcc {
  double r0, r1, i0, i1;
  FEAST_DEV void zero() { r0 = r1 = i0 = i1 = 0.0; }
};
FEAST_DEV void cmma(CAcc& c, double2 a, double2 b) {
  dmma884(c.r0, c.r1, a.x, b.x);
  dmma884(c.r0, c.r1, -a.y, b.y);
  dmma884(c.i0, c.i1, a.x, b.y);
  dmma884(c.i0, c.i1, a.y, b.x);
}
// real matrix times complex vector fragment
FEAST_DEV void rcmma(CAcc& c, double a, double2 b) {
  dmma884(c.r0, c.r1, a, b.x);
  dmma884(c.i0, c.i1, a, b.y);
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers
// ---------------------------------------------------------------------------
FEAST_DEV void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
FEAST_DEV void cp_async8(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// 8-byte copy that writes 0.0 instead when !valid (src-size 0): tile fills issue every
// element back to back instead of serialising one global latency per loop iteration
FEAST_DEV void cp_async8z(double* smem, const double* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}
FEAST_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
FEAST_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
template <int N>
FEAST_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

FEAST_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
FEAST_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace feastgpu
