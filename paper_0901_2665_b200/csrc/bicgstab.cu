// bicgstab.cu — the iterative inner solver of the reference (IterativeSolver /
// BicgstabShiftSystem, inner_solver.hpp:115-240): unpreconditioned BiCGStab on x -> z B x - A x,
// every right-hand side to its own relative residual target, with the reference's stagnation
// restart and failure rule, batched over every (node, column) pair on the device.
//
// The reference runs the columns one after another; here all C = nodes * m columns iterate
// together. Each column keeps its own scalars (rho, alpha, omega, iteration count) and freezes
// once it meets ||r|| <= tol ||b|| or reaches max_iter, so every column follows the reference's
// recurrence; only the dot products are summed in a fixed tree order instead of sequentially.
//
// Per iteration: the two operator applies of all columns at once (A and B are real, so the
// complex operands go through the real apply kernels as [Re | Im] column blocks: band_apply /
// bt_apply / dgemm on 2C columns) and two column kernels (one CTA per column, fixed-order block
// reductions): bicg_a forms v = z B p - A p, alpha and s; bicg_b forms t, omega, the x and r
// updates, ||r||, and the next iteration's head (rho, beta, p, or a restart).

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

namespace {

constexpr int kNT = 256;

// (cadd, csub, cmul, cdiv: common.cuh)
FEAST_DEV double2 cconjmul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
FEAST_DEV double cabs2(double2 a) { return hypot(a.x, a.y); }  // std::abs of a complex

// fixed-order block reduction of a complex partial; every thread gets the total
FEAST_DEV double2 block_sum2(double2 v, double2* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double2 s = red[0];
  for (int w = 1; w < kNT / 32; ++w) s = cadd(s, red[w]);
  return s;
}

// the loop head of inner_solver.hpp:150-167 for column c: rho_next = <r0, r>; a stagnation
// restart (it counts as an iteration) or beta and p = r + beta (p - omega v), packed for the apply
FEAST_DEV void head(const BicgArgs& a, int c, double2* red) {
  BicgCol& st = a.col[c];
  const int64_t o = (int64_t)c * a.ld;
  while (st.active) {
    double2 part = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < a.n; i += kNT) part = cadd(part, cconjmul(a.R0[o + i], a.R[o + i]));
    const double2 rho_next = block_sum2(part, red);
    if (cabs2(rho_next) < 1e-290 || cabs2(st.omega) < 1e-290) {
      for (int i = threadIdx.x; i < a.n; i += kNT) {
        a.R0[o + i] = a.R[o + i];
        a.P[o + i] = make_double2(0.0, 0.0);
        a.V[o + i] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        st.rho = st.alpha = st.omega = make_double2(1.0, 0.0);
        st.it += 1;
        st.active = st.it < a.max_iter && st.rnorm > a.tol * st.bnorm;
      }
      __syncthreads();
      continue;
    }
    const double2 beta = cmul(cdiv(rho_next, st.rho), cdiv(st.alpha, st.omega));
    const double2 om = st.omega;
    for (int i = threadIdx.x; i < a.n; i += kNT) {
      const double2 p = cadd(a.R[o + i], cmul(beta, csub(a.P[o + i], cmul(om, a.V[o + i]))));
      a.P[o + i] = p;
      a.PR[o + i] = p.x;
      a.PR[(int64_t)a.C * a.ld + o + i] = p.y;
    }
    __syncthreads();
    if (threadIdx.x == 0) st.rho = rho_next;
    __syncthreads();
    break;
  }
}

}  // namespace

// x = 0, r = r0 = b (real y column or complex b), p = v = 0, scalars 1; then the first head
__global__ void __launch_bounds__(kNT) bicg_init_kernel(BicgArgs a, const double* __restrict__ y, int ldy,
                                                        const double2* __restrict__ bc, int ldb) {
  __shared__ double2 red[kNT / 32];
  const int c = blockIdx.x, j = c % a.m;
  const int64_t o = (int64_t)c * a.ld;
  double2 part = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < a.n; i += kNT) {
    const double2 b = bc ? bc[i + (int64_t)j * ldb] : make_double2(y[i + (int64_t)j * ldy], 0.0);
    a.X[o + i] = make_double2(0.0, 0.0);
    a.R[o + i] = b;
    a.R0[o + i] = b;
    a.P[o + i] = make_double2(0.0, 0.0);
    a.V[o + i] = make_double2(0.0, 0.0);
    part.x += b.x * b.x + b.y * b.y;
  }
  const double bn = sqrt(block_sum2(part, red).x);
  BicgCol& st = a.col[c];
  if (threadIdx.x == 0) {
    st.rho = st.alpha = st.omega = make_double2(1.0, 0.0);
    st.bnorm = bn;
    st.rnorm = bn;
    st.it = 0;
    st.active = bn != 0.0 && 0 < a.max_iter && bn > a.tol * bn;
  }
  __syncthreads();
  head(a, c, red);
  if (threadIdx.x == 0 && st.active) atomicOr(a.any_active, 1);
}

// v = z B p - A p, alpha = rho / <r0, v>, s = r - alpha v (packed for the next apply)
__global__ void __launch_bounds__(kNT) bicg_a_kernel(BicgArgs a) {
  __shared__ double2 red[kNT / 32];
  const int c = blockIdx.x;
  BicgCol& st = a.col[c];
  if (!st.active) return;
  const double2 z = a.z[c / a.m];
  const int64_t o = (int64_t)c * a.ld, oi = (int64_t)a.C * a.ld + o;
  double2 part = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < a.n; i += kNT) {
    const double2 bp = make_double2(a.BR[o + i], a.BR[oi + i]), ap = make_double2(a.AR[o + i], a.AR[oi + i]);
    const double2 v = csub(cmul(z, bp), ap);
    a.V[o + i] = v;
    part = cadd(part, cconjmul(a.R0[o + i], v));
  }
  const double2 alpha = cdiv(st.rho, block_sum2(part, red));
  for (int i = threadIdx.x; i < a.n; i += kNT) {
    const double2 s = csub(a.R[o + i], cmul(alpha, a.V[o + i]));
    a.S[o + i] = s;
    a.PR[o + i] = s.x;
    a.PR[oi + i] = s.y;
  }
  __syncthreads();
  if (threadIdx.x == 0) st.alpha = alpha;
}

// t = z B s - A s, omega = <t, s> / ||t||^2, x += alpha p + omega s, r = s - omega t, the loop
// condition, then the next head
__global__ void __launch_bounds__(kNT) bicg_b_kernel(BicgArgs a) {
  __shared__ double2 red[kNT / 32];
  const int c = blockIdx.x;
  BicgCol& st = a.col[c];
  if (!st.active) return;
  const double2 z = a.z[c / a.m];
  const int64_t o = (int64_t)c * a.ld, oi = (int64_t)a.C * a.ld + o;
  double2 pts = make_double2(0.0, 0.0), ptt = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < a.n; i += kNT) {
    const double2 bs = make_double2(a.BR[o + i], a.BR[oi + i]), as = make_double2(a.AR[o + i], a.AR[oi + i]);
    const double2 t = csub(cmul(z, bs), as);
    a.T[o + i] = t;
    ptt.x += t.x * t.x + t.y * t.y;
    pts = cadd(pts, cconjmul(t, a.S[o + i]));
  }
  const double tt = block_sum2(ptt, red).x;
  const double2 ts = block_sum2(pts, red);
  const double2 omega = tt > 0.0 ? make_double2(ts.x / tt, ts.y / tt) : make_double2(0.0, 0.0);
  const double2 alpha = st.alpha;
  double2 prr = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < a.n; i += kNT) {
    const double2 s = a.S[o + i];
    a.X[o + i] = cadd(a.X[o + i], cadd(cmul(alpha, a.P[o + i]), cmul(omega, s)));
    const double2 r = csub(s, cmul(omega, a.T[o + i]));
    a.R[o + i] = r;
    prr.x += r.x * r.x + r.y * r.y;
  }
  const double rn = sqrt(block_sum2(prr, red).x);
  if (threadIdx.x == 0) {
    st.omega = omega;
    st.rnorm = rn;
    st.it += 1;
    st.active = st.it < a.max_iter && rn > a.tol * st.bnorm;
  }
  __syncthreads();
  head(a, c, red);
  if (threadIdx.x == 0 && st.active) atomicOr(a.any_active, 1);
}

// failed columns: the reference's "inner solve did not reach tolerance" (inner_solver.hpp:181-182)
__global__ void bicg_check_kernel(BicgArgs a, int* failed) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.C; c += gridDim.x * blockDim.x) {
    const BicgCol& st = a.col[c];
    if (st.bnorm != 0.0 && st.rnorm > a.tol * st.bnorm) atomicOr(failed, 1);
  }
}

// q (ld x m) = [q] - sum_e Re(coeff_e x_e) over the batch's nodes in ascending order
__global__ void bicg_terms_kernel(const double2* __restrict__ x, int nodes, int n, int m, int64_t ld,
                                  const double2* __restrict__ coeff, double* __restrict__ q, int accumulate) {
  const int64_t total = (int64_t)n * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    double acc = accumulate ? q[i + j * ld] : 0.0;
    for (int e = 0; e < nodes; ++e) {
      const double2 v = x[i + ((int64_t)e * m + j) * ld], cf = coeff[e];
      acc -= cf.x * v.x - cf.y * v.y;
    }
    q[i + j * ld] = acc;
  }
}

cudaError_t bicg_init(const BicgArgs& a, const double* y, int ldy, const double2* bc, int ldb, cudaStream_t st) {
  bicg_init_kernel<<<a.C, kNT, 0, st>>>(a, y, ldy, bc, ldb);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t bicg_a(const BicgArgs& a, cudaStream_t st) {
  bicg_a_kernel<<<a.C, kNT, 0, st>>>(a);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t bicg_b(const BicgArgs& a, cudaStream_t st) {
  bicg_b_kernel<<<a.C, kNT, 0, st>>>(a);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t bicg_check(const BicgArgs& a, int* failed, cudaStream_t st) {
  bicg_check_kernel<<<(a.C + 255) / 256, 256, 0, st>>>(a, failed);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t bicg_terms(const double2* x, int nodes, int n, int m, int64_t ld, const double2* coeff, double* q,
                       int accumulate, cudaStream_t st) {
  const int64_t total = (int64_t)n * m;
  bicg_terms_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, st>>>(x, nodes, n, m, ld, coeff,
                                                                                           q, accumulate);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
