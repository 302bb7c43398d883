// spike.cu — SPIKE partitioning of the block-Thomas chain (b <= 32).
//
// A node's L layers are cut into P chunks of Lc = L / P layers. Each chunk is factored and swept as
// its own block-tridiagonal system (bt_factor / bt_sweep with `chunks`): P times more independent
// chains, each P times shorter, so one node's solve fills the GPU and the factorisation's serial
// chain shrinks by P. The couplings between chunks are restored exactly:
//   chunk c:  M_c x_c + E_last C_{e_c}^T x_{c+1,first} + E_first C_{f_c - 1} x_{c-1,last} = f_c
//   =>        x_c = g_c - V_c x_{c+1,first} - W_c x_{c-1,last},   g_c = M_c^{-1} f_c,
//   V_c = M_c^{-1} E_last C_{e_c}^T,  W_c = M_c^{-1} E_first C_{f_c - 1}  (the spikes, b columns each,
//   computed once per factorisation by a complex sweep of the chunks),
// and the boundary values u_j = x_{j,last}, v_j = x_{j+1,first} (j < P - 1) solve the reduced
// system of 2 (P - 1) b unknowns per node
//   u_j + V_{j,last} v_j + W_{j,last} u_{j-1} = g_{j,last}
//   v_j + V_{j+1,first} v_{j+1} + W_{j+1,first} u_j = g_{j+1,first}
// (dense complex LU, zgetrf_batched, once per factorisation). The quadrature term of the chunk,
// Re(c x_c) = Re(c g_c) - Re(c V_c v_c) - Re(c W_c u_{c-1}), is corrected as ONE real GEMM per
// chunk: T_c -= [Re cV | -Im cV | Re cW | -Im cW] [Re v; Im v; Re u; Im u]. Same algebra as the
// reference's BandedLU solve (lu.hpp:162-201) up to rounding; the parity tests hold it to the
// reference's pivoted band solves.

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace feastgpu {

FEAST_DEV double2 zb_pair(double2 e, double2 z) { return make_double2(z.x * e.y - e.x, z.y * e.y); }

// spike right-hand sides per node slot (npad x 2b complex, ld npad): columns [0, b) hold
// C_{e_c}^T at chunk c's last layer rows (c < P-1), columns [b, 2b) hold C_{f_c - 1} at chunk c's
// first layer rows (c > 0); zero elsewhere. ablow = the (A, B) pairs of C_l = M(l+1, l).
__global__ void spike_rhs_kernel(int L, int b, int P, const double2* __restrict__ ablow, const double2* __restrict__ z,
                                 double2* __restrict__ spk, int64_t ld) {
  const int e = blockIdx.y;
  const int Lc = L / P;
  const int64_t bb = (int64_t)b * b, total = ld * 2 * b;
  const double2 ze = z[e];
  double2* S = spk + (int64_t)e * total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx % ld;
    const int col = (int)(idx / ld);
    const int l = (int)(row / b), i = (int)(row % b), c = l / Lc, li = l % Lc;
    double2 v = make_double2(0.0, 0.0);
    if (col < b) {  // V: at the last layer of chunk c < P-1: (C_l^T)(i, col) = C_l(col, i), l = e_c
      if (li == Lc - 1 && c < P - 1) v = zb_pair(ablow[(int64_t)l * bb + col + (int64_t)i * b], ze);
    } else {        // W: at the first layer of chunk c > 0: C_{l-1}(i, j), l = f_c
      const int j = col - b;
      if (li == 0 && c > 0) v = zb_pair(ablow[(int64_t)(l - 1) * bb + i + (int64_t)j * b], ze);
    }
    S[idx] = v;
  }
}

// the reduced matrix R (nr = 2 (P-1) b, column-major, nr x nr per node) from the spikes
__global__ void spike_reduced_kernel(int L, int b, int P, const double2* __restrict__ spk, int64_t ld,
                                     double2* __restrict__ R) {
  const int e = blockIdx.y;
  const int Lc = L / P, nr = 2 * (P - 1) * b;
  const int64_t nn = (int64_t)nr * nr;
  const double2* S = spk + (int64_t)e * ld * 2 * b;
  double2* Re = R + (int64_t)e * nn;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nn; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % nr), cidx = (int)(idx / nr);
    const int rb = r / b, ri = r % b, cb = cidx / b, ci = cidx % b;
    const int j = rb / 2;
    double2 v = make_double2(rb == cb && ri == ci ? 1.0 : 0.0, 0.0);
    if ((rb & 1) == 0) {  // u_j: chunk j's last layer rows; V_j -> v_j (block 2j+1), W_j -> u_{j-1} (2j-2)
      const int64_t row = (int64_t)(j * Lc + Lc - 1) * b + ri;
      if (cb == 2 * j + 1) v = S[row + (int64_t)ci * ld];
      if (j >= 1 && cb == 2 * j - 2) v = S[row + (int64_t)(b + ci) * ld];
    } else {              // v_j: chunk j+1's first layer rows; V_{j+1} -> v_{j+1} (2j+3), W_{j+1} -> u_j (2j)
      const int64_t row = (int64_t)((j + 1) * Lc) * b + ri;
      if (j + 1 <= P - 2 && cb == 2 * j + 3) v = S[row + (int64_t)ci * ld];
      if (cb == 2 * j) v = S[row + (int64_t)(b + ci) * ld];
    }
    Re[idx] = v;
  }
}

// correction operand per node slot (npad x 4b real, ld npad): [Re cV | -Im cV | Re cW | -Im cW]
__global__ void spike_coef_kernel(int b, const double2* __restrict__ spk, int64_t ld, const double2* __restrict__ coeff,
                                  double* __restrict__ ra) {
  const int e = blockIdx.y;
  const double2 cf = coeff[e];
  const int64_t total = ld * 2 * b;
  const double2* S = spk + (int64_t)e * total;
  double* A = ra + (int64_t)e * ld * 4 * b;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx % ld;
    const int col = (int)(idx / ld);            // 0 .. 2b-1 (V then W)
    const double2 v = cmul(cf, S[idx]);
    const int base = col < b ? col : 2 * b + (col - b);
    A[row + (int64_t)base * ld] = v.x;
    A[row + (int64_t)(base + b) * ld] = -v.y;
  }
}

// reduced right-hand sides per node (nr x m complex, ld nr): block 2j <- chunk j's last layer of
// the boundary x the sweep left in W, block 2j+1 <- chunk j+1's first layer
__global__ void spike_gather_kernel(int L, int b, int P, const double2* __restrict__ w, int64_t ld, int m,
                                    double2* __restrict__ rz) {
  const int e = blockIdx.y;
  const int Lc = L / P, nr = 2 * (P - 1) * b;
  const int64_t total = (int64_t)nr * m;
  const double2* W = w + (int64_t)e * ld * m;
  double2* Z = rz + (int64_t)e * total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % nr), col = (int)(idx / nr);
    const int rb = r / b, ri = r % b, j = rb / 2;
    const int64_t row = (rb & 1) == 0 ? (int64_t)(j * Lc + Lc - 1) * b + ri : (int64_t)((j + 1) * Lc) * b + ri;
    Z[idx] = W[row + (int64_t)col * ld];
  }
}

// per node and chunk c the real B-operand of the correction (4b x m, ld 4b):
// [Re v_c; Im v_c; Re u_{c-1}; Im u_{c-1}] with zeros where the chunk has no such neighbour
__global__ void spike_zops_kernel(int b, int P, const double2* __restrict__ rz, int m, double* __restrict__ zr) {
  const int e = blockIdx.y;
  const int nr = 2 * (P - 1) * b, k4 = 4 * b;
  const int64_t per_chunk = (int64_t)k4 * m, total = per_chunk * P;
  const double2* Z = rz + (int64_t)e * nr * m;
  double* O = zr + (int64_t)e * total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / per_chunk);
    const int64_t rem = idx % per_chunk;
    const int r = (int)(rem % k4), col = (int)(rem / k4);
    const int part = r / b, i = r % b;  // 0: Re v, 1: Im v, 2: Re u, 3: Im u
    double v = 0.0;
    if (part < 2 && c <= P - 2) {
      const double2 x = Z[(int64_t)(2 * c + 1) * b + i + (int64_t)col * nr];
      v = part == 0 ? x.x : x.y;
    } else if (part >= 2 && c >= 1) {
      const double2 x = Z[(int64_t)(2 * (c - 1)) * b + i + (int64_t)col * nr];
      v = part == 2 ? x.x : x.y;
    }
    O[idx] = v;
  }
}

static unsigned grid_for(int64_t total) { return (unsigned)std::min<int64_t>((total + 255) / 256, 2048); }

cudaError_t spike_rhs(int L, int b, int P, int nodes, const double2* ablow, const double2* z, double2* spk, int64_t ld,
                      cudaStream_t st) {
  spike_rhs_kernel<<<dim3(grid_for(ld * 2 * b), nodes), 256, 0, st>>>(L, b, P, ablow, z, spk, ld);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t spike_reduced(int L, int b, int P, int nodes, const double2* spk, int64_t ld, double2* R, cudaStream_t st) {
  const int64_t nr = 2 * (int64_t)(P - 1) * b;
  spike_reduced_kernel<<<dim3(grid_for(nr * nr), nodes), 256, 0, st>>>(L, b, P, spk, ld, R);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t spike_coef(int b, int nodes, const double2* spk, int64_t ld, const double2* coeff, double* ra,
                       cudaStream_t st) {
  spike_coef_kernel<<<dim3(grid_for(ld * 2 * b), nodes), 256, 0, st>>>(b, spk, ld, coeff, ra);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t spike_gather(int L, int b, int P, int nodes, const double2* w, int64_t ld, int m, double2* rz,
                         cudaStream_t st) {
  const int64_t nr = 2 * (int64_t)(P - 1) * b;
  spike_gather_kernel<<<dim3(grid_for(nr * m), nodes), 256, 0, st>>>(L, b, P, w, ld, m, rz);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t spike_zops(int b, int P, int nodes, const double2* rz, int m, double* zr, cudaStream_t st) {
  spike_zops_kernel<<<dim3(grid_for((int64_t)4 * b * m * P), nodes), 256, 0, st>>>(b, P, rz, m, zr);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace feastgpu
