// kernels.h — host-side launchers for the sm_100a kernels of libfeastgpu.
// Every launcher enqueues on `st` and returns cudaGetLastError() of its launch(es).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace feastgpu {

struct cplx_t {
  double re, im;
};

// Launch counter (evidence that the native path ran; read via feast_gpu_launch_count).
extern int64_t g_launches;

// ---------------- block-tridiagonal shifted solves (block Thomas) -------------
// A/B in block-tridiagonal storage packed as double2 (x = A entry, y = B entry):
//   abdiag: L blocks b*b col-major, ablow: (L-1) blocks, C_l = M(l+1, l).
// For node slot s (0..nodes-1): shift z[s]; factors Sinv[s] (L*b*b), G[s] ((L-1)*b*b).
struct BtFactorArgs {
  int L, b, nodes;
  const double2* abdiag;
  const double2* ablow;
  const double2* z;       // [nodes]
  double2* sinv;          // nodes * L*b*b
  double2* g;             // nodes * (L-1)*b*b: G_l = S_l^{-1} C_l^T
  double2* h;             // nodes * (L-1)*b*b: H_l = S_l^{-1} C_{l-1}, l >= 1
  double2* scratch;       // unused (kept for the launcher signature)
  int* status;            // set to 1 on a singular block pivot
  double2* work;          // b >= 128: bt_factor_work_elems(b, nodes) double2
  int kmid = -1;          // >= 0: twisted recursion meeting at layer kmid (bt_twist_layer)
  // SPIKE chunks (b <= 32): `nodes` counts (node, chunk) pairs, chunk c of node e at slot
  // e * chunks + c holds layers [c L, (c + 1) L) of the pencil (L = layers per chunk), factored as
  // its own block-tridiagonal system (the couplings between chunks are left to the spikes)
  int chunks = 1;
};
cudaError_t bt_factor(const BtFactorArgs& a, cudaStream_t st);
// Meeting layer of the twisted (two-ended) block-Thomas recursion for b <= 64 and L >= 4
// (L / 2), else -1 (plain top-down chain; also when !enable, feast_gpu_set_twist).
int bt_twist_layer(int L, int b, bool enable);
size_t bt_factor_work_elems(int b, int nodes);

// Panel layout of the factors for b >= 128 (the bulk-copy sweep): each b x b factor is stored
// as P = b / RB row panels, panel p holding rows [p*RB, (p+1)*RB) column by column (RB
// contiguous entries per column), row r of column k at position r ^ (2*(k & 3)) — a bank
// swizzle for the sweep's shared-memory reads. RB = bt_panel_rows(b); 0 = plain col-major.
int bt_panel_rows(int b);

// Sweeps: for every node slot s and column j < m:
//   real mode (0)    : T_s = Re(coeff[s] * (z_s B - A)^{-1} Y)  (Y real, T real, ld = ldv)
//   complex mode (1) : W_s <- (z_s B - A)^{-1} W_s              (complex in place; b < 128)
//   complex out (2)  : W_s = (z_s B - A)^{-1} Y                 (Y real, W complex; b >= 128)
struct BtSweepArgs {
  int L, b, nodes, m, ldv;
  const double2* ablow;
  const double2* z;
  const double2* coeff;
  const double2* sinv;
  const double2* g;
  const double2* h;
  const double* y;        // real mode input (n*m, shared by nodes)
  double* t;              // real mode output: nodes * ldv*m
  double2* w;             // workspace / complex in-out: nodes * ldv*m
  int complex_mode;
  int kmid = -1;          // the factors' twisted meeting layer (must match bt_factor's)
  // SPIKE chunks (b <= 32, bt_factor's): slot s = node * chunks + c solves chunk c's rows
  // [c L b, (c + 1) L b) of node s / chunks's blocks (y, t, w at that row offset of the node's
  // slot); in real mode the complex x of each chunk's first and last layer also go to w
  int chunks = 1;
};
cudaError_t bt_sweep(const BtSweepArgs& a, cudaStream_t st);
cudaError_t bt_sweep_pipe16(const BtSweepArgs& a, cudaStream_t st);   // sweep_pipe.cu (b = 16)

// SPIKE partitioning of the chain (spike.cu): spike right-hand sides, the reduced matrix
// (nr = 2 (P-1) b per node), the correction operand [Re cV | -Im cV | Re cW | -Im cW], the reduced
// right-hand sides gathered from the sweep's boundary x, and the per-chunk correction B-operands
cudaError_t spike_rhs(int L, int b, int P, int nodes, const double2* ablow, const double2* z, double2* spk, int64_t ld,
                      cudaStream_t st);
cudaError_t spike_reduced(int L, int b, int P, int nodes, const double2* spk, int64_t ld, double2* R, cudaStream_t st);
cudaError_t spike_coef(int b, int nodes, const double2* spk, int64_t ld, const double2* coeff, double* ra,
                       cudaStream_t st);
cudaError_t spike_gather(int L, int b, int P, int nodes, const double2* w, int64_t ld, int m, double2* rz,
                         cudaStream_t st);
cudaError_t spike_zops(int b, int P, int nodes, const double2* rz, int m, double* zr, cudaStream_t st);
// batched complex GEMM (gemm.cu): C_z = alpha A_z B_z + beta C_z
cudaError_t zgemm_batched(int m, int n, int k, double2 alpha, const double2* a, int lda, int64_t sa,
                          const double2* b, int ldb, int64_t sb, double2 beta, double2* c, int ldc,
                          int64_t sc, int batch, cudaStream_t st);
// batched dense complex LU / solves (dense.cu), the reduced systems' factorisation
struct LuLookahead;
cudaError_t zgetrf_batched(int n, int nodes, double2* lu, int64_t stride, int* ipiv, int* perm, double2* dinv,
                           int* status, cudaStream_t st, const LuLookahead* la = nullptr);
cudaError_t zgetrs_batched(int n, int nodes, int m, const double2* lu, int64_t stride, const int* perm,
                           const double2* dinv, double2* w, int ldv, double2* scratch, cudaStream_t st);

// Q = -sum_{s} T_s (ascending s), n rows (ld) x m; accumulate: Q -= sum (the next node batch)
cudaError_t reduce_terms(const double* t, int nodes, int64_t slice, int n, int m, int ld,
                         double* q, cudaStream_t st, int accumulate = 0);

// block-tridiagonal real operator apply: Y = Op * X (layer-batched DMMA GEMMs), layers [l0, l1)
// of Y (l1 < 0: all)
cudaError_t bt_apply(int L, int b, const double* diag, const double* low, const double* x, int ldx,
                     double* y, int ldy, int m, cudaStream_t st, int l0 = 0, int l1 = -1);

// ---------------- dense shifted solves (batched complex LU) -------------------
// look-ahead resources of zgetrf_batched: a (high-priority) side stream and two events
struct LuLookahead {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_cols = nullptr, ev_panel = nullptr;
};
struct DenseFactorArgs {
  int n, nodes;
  const double* a;        // n*n real
  const double* bm;       // n*n real
  const double2* z;
  double2* lu;            // nodes * n*n complex
  int* ipiv;              // nodes * n
  int* perm;              // nodes * n (row permutation applied to the RHS)
  double2* dinv;          // nodes * (n/nb) * 2 * nb*nb : inverses of unit-L and U diagonal blocks
  int* status;
  LuLookahead la;         // side == nullptr: panels on the main stream
};
cudaError_t dense_factor(const DenseFactorArgs& a, cudaStream_t st);
constexpr int kDenseNb = 64;

struct DenseSolveArgs {
  int n, nodes, m, ldv;
  const double2* lu;
  const int* perm;
  const double2* dinv;
  const double2* coeff;
  const double* y;
  double* t;
  double2* w;
  int complex_mode;
};
cudaError_t dense_solve(const DenseSolveArgs& a, cudaStream_t st);

// ---------------- iterative inner solver (bicgstab.cu) -------------------------
// BiCGStab (inner_solver.hpp:115-240) on z B - A for C = nodes * m columns at once.
struct BicgCol {
  double2 rho, alpha, omega;
  double bnorm, rnorm;
  int it, active;
};
struct BicgArgs {
  int n, ld, C, m;          // rows, leading dimension, columns, columns per node
  const double2* z;         // per node: the shift (conjugated for ConjTranspose solves)
  double2 *X, *R, *R0, *P, *V, *S, *T;  // ld x C complex each
  double *PR, *AR, *BR;     // ld x 2C real: the packed [Re | Im] apply operand, A and B times it
  BicgCol* col;             // C
  double tol;
  int max_iter;
  int* any_active;          // set by columns still iterating after a kernel
};
// rhs: y (real, ld ldy, column j of every node) or bc (complex, ld ldb, column j of every node)
cudaError_t bicg_init(const BicgArgs& a, const double* y, int ldy, const double2* bc, int ldb, cudaStream_t st);
cudaError_t bicg_a(const BicgArgs& a, cudaStream_t st);   // after PR -> AR, BR: v, alpha, s -> PR
cudaError_t bicg_b(const BicgArgs& a, cudaStream_t st);   // after PR -> AR, BR: t, omega, x, r, next p -> PR
cudaError_t bicg_check(const BicgArgs& a, int* failed, cudaStream_t st);
// q = [q] - sum_e Re(coeff_e x_e), nodes ascending (x: ld x nodes*m complex)
cudaError_t bicg_terms(const double2* x, int nodes, int n, int m, int64_t ld, const double2* coeff, double* q,
                       int accumulate, cudaStream_t st);

// ---------------- real GEMM (DMMA) -------------------------------------------
// C(m x n) = alpha * op(A) * op(B) + beta * C, column-major; op = 'N' or 'T'.
// Split-K with a deterministic reduction when k is large relative to m*n.
cudaError_t dgemm(char ta, char tb, int m, int n, int k, double alpha, const double* A, int lda,
                  const double* B, int ldb, double beta, double* C, int ldc, double* work,
                  size_t work_elems, cudaStream_t st);

// batched C_z = alpha op(A_z) B_z + beta C_z (op = T when TA), z < batch, strides sa, sb, sc
cudaError_t dgemm_batched(bool TA, int m, int n, int k, double alpha, const double* A, int lda, int64_t sa,
                          const double* B, int ldb, int64_t sb, double beta, double* C, int ldc, int64_t sc,
                          int batch, cudaStream_t st);

// [S1 | S2] = Q^T [AQ | BQ] (m x 2m, ld m) with S1, S2 symmetric and m a multiple of 64: only
// the upper tiles of each half are computed; follow with symmetrize_tiles on each half
cudaError_t dgemm_tn_sym2(int m, int k, const double* Q, int ldq, const double* AB, int ldab, double* C,
                          double* work, size_t work_elems, cudaStream_t st);
cudaError_t symmetrize_tiles(double* c, int m, int ld, cudaStream_t st);
// C = (M + M^T)/2 in place (square m x m, ld)
cudaError_t symmetrize(double* c, int m, int ld, cudaStream_t st);

// band-row copy of a block-tridiagonal operator (b = 16, 32): row l b + i = [C_{l-1} | D_l | C_l^T](i, :)
cudaError_t band_rows(int L, int b, const double* diag, const double* low, double* ab, cudaStream_t st);
// y1 = A x, and y2 = B x in the same pass when ab2 != nullptr (band rows from band_rows), layers
// [l0, l1) of y (l1 < 0: all)
cudaError_t band_apply(int L, int b, const double* ab1, const double* ab2, const double* x, int ldx, double* y1,
                       double* y2, int ldy, int m, cudaStream_t st, int l0 = 0, int l1 = -1);

// ---------------- reduced generalized eigensolver ----------------------------
struct EigWork;  // opaque, sized for mmax
EigWork* eig_create(int mmax);
void eig_destroy(EigWork* w);
// Symmetric eigen-decomposition of W (m x m, ld m, overwritten): eigenvalues ascending
// into `evals` (device), vectors into `v` (device, m x m), stable order. vfloor > 0: the
// tridiagonal route computes vectors only for evals > vfloor * max(evals) (others zero).
// ev_tridiag (may be null): recorded on `st` right behind the tridiagonalisation kernel.
cudaError_t sym_eig(EigWork* w, int m, double* a, double* evals, double* v, cudaStream_t st,
                    double vfloor = 0.0, bool low_smem = false, cudaEvent_t ev_tridiag = nullptr);
// Householder tridiagonalisation of a symmetric m x m matrix (3 <= m <= tri_tiles_max_dim())
// on one SM with the matrix in registers: d[m], e[m-1], tau[m], reflectors in hv (m x m)
int tri_tiles_max_dim();
cudaError_t tridiag_tiles(int m, const double* a, double* d, double* e, double* hv, double* tau,
                          cudaStream_t st);
// V = H_0 ... H_{m-3} Z with block reflectors (tri_back.cu); tw: tri_back_wy_ws(m) doubles
size_t tri_back_wy_ws(int m);
cudaError_t tri_back_wy(int m, const double* hv, const double* tau, const double* z, double* v, double* tw,
                        cudaStream_t st);
// one-CTA tiled Cholesky (chol_tiles.cu) for m <= chol_tiles_max_dim(): same contract as cholesky()
int chol_tiles_max_dim();
cudaError_t chol_tiles(int m, double* a, double rel_tol, int* status, double* dinv, cudaStream_t st);
// Cholesky with relative pivot floor: L (lower, in place in `a`), status[0] = 1 on failure
// (status must be zero on entry). dinv receives the inverses of the 32x32 diagonal tiles of
// L (ceil(m/32) * 1024 doubles), consumed by the triangular solves.
cudaError_t cholesky(int m, double* a, double rel_tol, int* status, double* dinv, cudaStream_t st);
// X <- L^{-1} X   (L lower m x m from cholesky(), X m x ncols); low_smem: a route that leaves
// room on each SM for a concurrent kernel (the look-ahead contour pass)
cudaError_t trsm_lower(int m, const double* l, const double* dinv, double* x, int ldx, int ncols,
                       cudaStream_t st, bool low_smem = false);
// X <- L^{-T} X
cudaError_t trsm_lower_t(int m, const double* l, const double* dinv, double* x, int ldx, int ncols,
                         cudaStream_t st, bool low_smem = false);
// transpose copy: dst(n x m) = src(m x n)^T
cudaError_t transpose(const double* src, int m, int n, int lds, double* dst, int ldd,
                      cudaStream_t st);
// S(:, j) = V(:, keep[j]) / sqrt(d[keep[j]])
cudaError_t scale_columns(const double* v, int m, const int* keep, const double* d, int nk,
                          double* s, cudaStream_t st);

// ---------------- residuals ---------------------------------------------------
// per column j: num = sum|AX - lam_j BX|, den = sum|AX|, xn = sum|X|  -> out[3*j + {0,1,2}]
// pairs: rows are interleaved complex entries, summed as complex moduli (Hermitian pencils)
cudaError_t residual_sums(int n, int m, const double* ax, const double* bx, const double* x,
                          int ld, const double* lam, double* out, cudaStream_t st, bool pairs = false);
// out(:, j) = J in(:, j), J (re, im) = (-im, re) on interleaved pairs; n rows, ld, m columns
cudaError_t rotate_pairs(const double* in, int n, int64_t ld, int m, double* out, cudaStream_t st);

// random_block<double> (core.hpp:84-106) on the device: out(i, j) for i < n, j < m (ld), the
// mt19937_64(seed) stream mapped to [-1, 1) column by column, bit-identical to the host
cudaError_t random_block_device(uint64_t seed, int n, int m, double* out, int ld, cudaStream_t st);

// out[i] = (a[i], b[i]): the interleaved (A, B) pairs of the block-tridiagonal factorisation
// ---------------- CSR operators taken in on the device (csr_ingest.cu) ----------
// Result of csr_scan over one operator: first_error = 4 * (entry index) + code of the first
// failing entry in row-major order (~0: none), the bandwidth max |i - j|, bit s of misfit_mask
// set when the pattern is not block-tridiagonal at block size 16 << s, and the 1-norm (max
// absolute row sum = column sum for a symmetric pattern) as the bits of a non-negative double.
constexpr int kCsrOutOfRange = 0, kCsrMirrorMissing = 1, kCsrMirrorDiffers = 2;
constexpr int kCsrBlockCandidates = 6;  // 16 .. 512
struct CsrStats {
  unsigned long long first_error;
  unsigned long long norm1_bits;
  int bandwidth;
  unsigned misfit_mask;
};
cudaError_t csr_scan(int n, const int* row_ptr, const int* col_idx, const double* values, CsrStats* stats,
                     bool init, cudaStream_t st);
// block-tridiagonal storage (L diagonal blocks, L-1 couplings C_l = M(l+1, l), b x b col-major,
// b a power of two) from device CSR arrays; unit_padding: rows n..L*b-1 get a unit diagonal
cudaError_t csr_to_blocktri(int n, int b, int L, const int* row_ptr, const int* col_idx, const double* values,
                            double* diag, double* low, bool unit_padding, cudaStream_t st);
cudaError_t interleave_pairs(const double* a, const double* b, size_t n, double2* out, cudaStream_t st);

// accumulate_subspace_hermitian for real symmetric pencils (misc.cu): complex right-hand
// sides [Yr | Yi] into every node slot, then Q -= sum_s c1 G Y + c2 G^H Y in ascending s
cudaError_t real_to_complex_slots(const double* y, int64_t ld, int64_t m, int nodes, double2* w, cudaStream_t st);
cudaError_t hermitian_terms(const double2* w, int nodes, int64_t ld, int n, int m, const double2* coeff,
                            double2* q, int accumulate, cudaStream_t st);

// look-ahead admission test: *out = max_i sum_j sqrt(bq(j,j)) |phi(j,i)|, i < mo, j < m
cudaError_t cancellation_factor(int m, int mo, const double* bq, int ldb, const double* phi, int ldp,
                                double* out, cudaStream_t st);

// dst = sum of `slices` blocks of `count` doubles at src + r * stride, in slice order
cudaError_t sum_slices(const double* src, int slices, int64_t stride, size_t count, double* dst, cudaStream_t st);

// out = x + t y
cudaError_t axpby(const double* x, const double* y, double t, size_t n, double* out, cudaStream_t st);
// *out = ||A||_1 of block-tridiagonal storage [diag | lower] (L layers of b) or dense (L = 0, n = b)
cudaError_t operator_norm1(int L, int b, const double* a, double* out, cudaStream_t st);

// misc
cudaError_t fill_zero(double* p, size_t count, cudaStream_t st);
cudaError_t gather_columns(const double* src, int ld, int n, const int* idx, int m, double* dst,
                           int ldd, cudaStream_t st);
cudaError_t conj_inplace(double2* p, size_t count, cudaStream_t st);
// complex right-hand sides through the real-input sweep: y[:, j] = Re w[:, j],
// y[:, m + j] = Im w[:, j] (n rows, ld both); then w[:, j] <- w[:, j] + i w[:, m + j]
cudaError_t split_complex(const double2* w, double* y, int n, int64_t ld, int m, cudaStream_t st);
cudaError_t merge_complex(double2* w, int n, int64_t ld, int m, cudaStream_t st);

}  // namespace feastgpu
