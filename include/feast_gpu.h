/*
 * feast_gpu.h — C-ABI of libfeastgpu.so, the B200-native FEAST inner loop.
 *
 * Drop-in boundary for the reference's solver plugin + loop
 * (reference: /root/reference/proj/include/feast/...):
 *
 *   feast_gpu_solve        replaces feast::feast_solve<double>            core.hpp:264-391
 *   feast_gpu_prepare      replaces the ensure_factors() lambda           core.hpp:304-311
 *                          (InnerSolver<T>::prepare(z) per node,          inner_solver.hpp:32-39)
 *   feast_gpu_solve_shift  replaces ShiftSystem::solve_in_place           inner_solver.hpp:24-28
 *   feast_gpu_contour_pass replaces accumulate_subspace_real              core.hpp:163-185
 *   feast_gpu_rayleigh_ritz replaces rayleigh_ritz + trace_of_in_interval core.hpp:228-240,114-124
 *   feast_gpu_reduced_gevp replaces linalg::reduced_gevp                  eigh.hpp:178-225
 *   feast_gpu_residuals    replaces linalg::residual_norms                residual.hpp:29-68
 *
 * Conventions (same as the reference, dense.hpp:15-17, types.hpp:12):
 *   - all arithmetic is IEEE fp64; dense blocks are column-major, (i,j) at i + j*ld;
 *   - complex values are interleaved (re, im) pairs, byte-compatible with std::complex<double>;
 *   - every pointer argument is a HOST pointer unless its name ends in _dev;
 *   - return codes map 1:1 onto the reference exception classes (types.hpp:15-38):
 *       FEAST_EINPUT     <-> feast::InputError          (CLI exit 4)
 *       FEAST_ENUMERICAL <-> feast::NumericalError      (CLI exit 5)
 *       FEAST_EBREAKDOWN <-> feast::SubspaceBreakdown   (a status, not a throw, out of feast_solve)
 *     plus FEAST_ECUDA / FEAST_ENCCL for device / collective failures (NumericalError class).
 *   - one host thread per context at a time (the InnerSolver threading contract of
 *     inner_solver.hpp:30-31 is met by serialising on the context's stream).
 */
#ifndef FEAST_GPU_H_
#define FEAST_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FEAST_GPU_ABI_VERSION 1

typedef enum {
  FEAST_OK = 0,
  FEAST_EINPUT = 4,
  FEAST_ENUMERICAL = 5,
  FEAST_EBREAKDOWN = 6,
  FEAST_ECUDA = 7,
  FEAST_ENCCL = 8,
  FEAST_EINTERNAL = 9
} feast_code_t;

/* Storage of one symmetric operator (operator.hpp:37-40 plus the block-tridiagonal
 * layout the BASELINE configs 3 and 5 need). */
typedef enum {
  FEAST_STORAGE_DENSE = 0,    /* n*n column-major, exactly symmetric            */
  FEAST_STORAGE_CSR = 1,      /* symmetric-complete CSR, int32 indices          */
  FEAST_STORAGE_BLOCKTRI = 2, /* nblocks diagonal b*b blocks + (nblocks-1) lower
                                 couplings C_l = M(l+1, l); M(l, l+1) = C_l^T   */
  /* complex Hermitian operators (feast_gpu_set_pencil_hermitian): `dense` / `values` hold
     interleaved (re, im) pairs, std::complex<double> layout (types.hpp:12)          */
  FEAST_STORAGE_DENSE_Z = 16, /* n*n complex column-major, exactly Hermitian      */
  FEAST_STORAGE_CSR_Z = 17    /* Hermitian-complete CSR, nnz complex values       */
} feast_storage_t;

typedef struct {
  int32_t kind;            /* feast_storage_t */
  int32_t n;               /* dimension (BLOCKTRI: nblocks * bsize)           */
  const double* dense;     /* DENSE: n*n                                      */
  const int32_t* row_ptr;  /* CSR: n+1                                        */
  const int32_t* col_idx;  /* CSR: nnz                                        */
  const double* values;    /* CSR: nnz                                        */
  int32_t nblocks;         /* BLOCKTRI                                        */
  int32_t bsize;           /* BLOCKTRI                                        */
  const double* diag;      /* BLOCKTRI: nblocks * b*b, block l at l*b*b       */
  const double* lower;     /* BLOCKTRI: (nblocks-1) * b*b, C_l at l*b*b       */
} feast_operator_t;

/* Mirrors feast::FeastConfig (core.hpp:25-33). `threads` is accepted for API
 * parity; on the GPU it has no effect on results (SPEC determinism rule). */
typedef struct {
  int32_t m0;
  int32_t n_e;
  double trace_tol;
  int32_t max_loops;
  uint64_t seed;
  int32_t threads;
  int32_t low_memory;
} feast_config_t;

/* Mirrors feast::FeastStatus (core.hpp:35-41), same order. */
typedef enum {
  FEAST_STATUS_CONVERGED = 0,
  FEAST_STATUS_MAX_LOOPS = 1,
  FEAST_STATUS_NO_EIGENVALUES = 2,
  FEAST_STATUS_SATURATED = 3,
  FEAST_STATUS_BREAKDOWN = 4
} feast_run_status_t;

/* Mirrors feast::FeastResult<double> (core.hpp:61-78). The caller allocates the
 * arrays: eigenvalues/residuals/residual_absolute_only hold m0 entries,
 * eigenvectors/subspace hold n*m0 doubles, trace_history/in_interval_counts hold
 * max_loops+1 entries. Any array pointer may be NULL to skip that output. */
typedef struct {
  double* eigenvalues;
  double* eigenvectors;
  double* residuals;
  int32_t* residual_absolute_only;
  double* trace_history;
  int32_t* in_interval_counts;
  double* subspace;
  /* scalar outputs */
  int32_t m;               /* eigenpairs found inside the interval          */
  int32_t subspace_cols;   /* columns of the last Ritz block (<= m0)        */
  int32_t loops_used;
  int32_t status;          /* feast_run_status_t                            */
  double max_residual;
  double factorize_s, solve_s, reduce_s, total_s; /* FeastTimings core.hpp:54-59 */
} feast_result_t;

/* ------------------------------------------------------------------------- */
/* Context                                                                   */
/* ------------------------------------------------------------------------- */
typedef struct feast_gpu_ctx feast_gpu_ctx;

int feast_gpu_abi_version(void);

/* Creates a context on CUDA device `device`. `stream` may be NULL (the context
 * creates its own) or an existing cudaStream_t the caller owns. */
int feast_gpu_create(int device, void* stream, feast_gpu_ctx** out);
void feast_gpu_destroy(feast_gpu_ctx* ctx);
const char* feast_gpu_last_error(const feast_gpu_ctx* ctx);

/* Multi-GPU: contour nodes are sharded over `nranks` ranks (contiguous blocks,
 * ascending e); one NCCL allreduce(sum) of the N*M0 partial Q per pass.
 * `nccl_unique_id` is the 128-byte ncclUniqueId rank 0 created
 * (feast_gpu_nccl_unique_id) and broadcast out of band. */
int feast_gpu_nccl_unique_id(void* id_out_128_bytes);
int feast_gpu_set_comm(feast_gpu_ctx* ctx, const void* nccl_unique_id, int rank, int nranks);

/* Loopback rank group: several contexts of ONE process (one host thread each, any devices)
 * joined as ranks 0..nranks-1 with the same collectives as the NCCL group (device copies and
 * host barriers). It runs the sharded loop and the row-distributed Rayleigh-Ritz step on a
 * single GPU, which is how they are tested here; production runs one process per GPU with
 * feast_gpu_set_comm. With nranks = 1 and a non-zero id, feast_gpu_set_comm builds a one-rank
 * NCCL communicator, so the NCCL calls themselves also run on one GPU. */
typedef struct feast_gpu_group feast_gpu_group;
int feast_gpu_group_create(int nranks, feast_gpu_group** out);
void feast_gpu_group_destroy(feast_gpu_group* group);
int feast_gpu_set_group(feast_gpu_ctx* ctx, feast_gpu_group* group, int rank);

/* Rayleigh-Ritz across the ranks of a group (default 1): each rank applies A, B and projects on
 * its row slab (whole layers for block-tridiagonal pencils), one allreduce of the 2 M0^2 reduced
 * values, the reduced eigensolve replicated, the N x M0 blocks the solves need allgathered by
 * slabs. 0 = replicated Rayleigh-Ritz on every rank (rayleigh_ritz, core.hpp:228-240). */
int feast_gpu_set_row_distribution(feast_gpu_ctx* ctx, int enable);

/* Uploads the pencil (A symmetric, B symmetric positive definite). CSR inputs
 * whose pattern is block-tridiagonal are stored block-tridiagonal; other CSR
 * inputs are densified (the reference's Dense policy, inner_solver.hpp:88-92). */
int feast_gpu_set_pencil(feast_gpu_ctx* ctx, const feast_operator_t* a, const feast_operator_t* b);

/* Complex Hermitian pencils (feast_solve<cplx>, core.hpp:264-391 with T = std::complex<double>;
 * SymmetricOperator<cplx>, operator.hpp:33-268): A Hermitian, B Hermitian positive definite, both
 * FEAST_STORAGE_DENSE_Z or FEAST_STORAGE_CSR_Z. Validation messages as the reference's
 * (conjugate symmetry, real diagonal). The pencil is carried as the real symmetric pencil of
 * twice the size (each entry x + iy as the block [[x, -y], [y, x]]), on which every solver
 * path of this library runs; feast_gpu_solve_hermitian reads it back as the complex pencil. */
int feast_gpu_set_pencil_hermitian(feast_gpu_ctx* ctx, const feast_operator_t* a, const feast_operator_t* b);

/* feast_solve<cplx> on a Hermitian pencil: m0 complex subspace columns (m0 <= 512), the start
 * block random_block<cplx>(n, m0, seed) (real then imaginary part per entry, core.hpp:84-106) or
 * initial_y (n*y_cols complex, interleaved). Results as feast_gpu_solve's, except that
 * eigenvectors (n*m0) and subspace (n*m0) hold COMPLEX entries (2 doubles each, interleaved);
 * residuals use complex moduli (residual.hpp:29-68). */
int feast_gpu_solve_hermitian(feast_gpu_ctx* ctx, double emin, double emax, const feast_config_t* config,
                              const double* initial_y, int y_cols, feast_result_t* result);

/* Contour on the upper half circle over [emin, emax] with n_e Gauss-Legendre
 * nodes (quadrature.cpp:69-87), then factors every node this rank owns
 * (ensure_factors, core.hpp:304-311). */
int feast_gpu_prepare(feast_gpu_ctx* ctx, double emin, double emax, int n_e);

/* Memory plan for the factors (ensure_factors vs low_memory, core.hpp:302-311,335-336):
 * nodes = 0 keeps every owned node's factors resident when they fit 80% of the free HBM
 * and otherwise streams them in the largest batches that do; nodes > 0 forces batches of
 * that many nodes. Streamed factors are recomputed every pass, batch by batch, and the
 * quadrature sum continues in ascending e across batches (results are bit-identical to the
 * resident plan). Takes effect at the next feast_gpu_prepare / feast_gpu_solve. */
int feast_gpu_set_node_batch(feast_gpu_ctx* ctx, int nodes);

/* Inner solver, the InnerSolver the reference's feast_solve takes (inner_solver.hpp:32-39):
 *   kind 0: DirectSolver (default) — factors of z_e B - A per node, solves on the factors;
 *   kind 1: IterativeSolver(a, b, tol, max_iter) (inner_solver.hpp:209-240) — unpreconditioned
 *           BiCGStab per right-hand side to ||r|| <= tol ||b|| with the reference's restart and
 *           failure rules (FEAST_ENUMERICAL "BicgstabShiftSystem: inner solve did not reach
 *           tolerance"); max_iter <= 0 means max(1000, 20 n); the loop's trace tolerance is
 *           floored at tol^2 (core.hpp:296-297). tol outside (0, 1) is FEAST_EINPUT.
 * Takes effect at the next factorisation / solve. */
int feast_gpu_set_inner_solver(feast_gpu_ctx* ctx, int kind, double tol, int max_iter);

/* FactorPolicy of the DirectSolver (inner_solver.hpp:40-47, 80-95), applied at the next
 * feast_gpu_set_pencil: 0 Auto (block-tridiagonal factors when both operators are sparse and
 * (3 bw + 1) 2 <= n, dense otherwise), 1 Dense (dense LU for any storage), 2 Banded (sparse
 * operands required, FEAST_EINPUT "DirectSolver: banded policy requires sparse operands"
 * otherwise; block-tridiagonal factors, or dense when no block size up to 512 holds the band). */
int feast_gpu_set_factor_policy(feast_gpu_ctx* ctx, int policy);

/* Block-Thomas recursion for block-tridiagonal pencils with b <= 64: enable = 1 (default) runs
 * the two-ended (twisted) elimination that meets at layer L/2, enable = 0 the plain top-down
 * chain of BandedLU (lu.hpp:127-206). Both give the same solves to rounding; takes effect at the
 * next factorisation. */
int feast_gpu_set_twist(feast_gpu_ctx* ctx, int enable);

/* SPIKE partitioning of the block-Thomas chain (b <= 32): chunks = P cuts each node's L layers
 * into P independently factored and swept chunks (P times more parallel chains, P times shorter),
 * with the couplings restored through spikes, a reduced system of 2 (P - 1) b unknowns per node
 * and a GEMM correction (spike.cu). 0 = automatic, 1 = off; P must be a power of two; it is
 * reduced until it divides L with at least 8 layers per chunk. Takes effect at the next
 * factorisation; the solves agree with the unpartitioned ones to rounding. */
int feast_gpu_set_spike(feast_gpu_ctx* ctx, int chunks);

/* random_block<double> (core.hpp:84-106) generated on the device: out (host, n*m column-major)
 * = 2 * ((w >> 11) * 2^-53) - 1 over the std::mt19937_64(seed) words w, bit-identical to the
 * reference's host generator. feast_gpu_solve draws its initial block this way. */
int feast_gpu_random_block(feast_gpu_ctx* ctx, int n, int m, uint64_t seed, double* out);

/* Storage chosen for the pencil at feast_gpu_set_pencil: block size b and layer count L of the
 * block-tridiagonal re-blocking (b = 0, L = 0 for the dense path), and twist = the meeting
 * layer of the two-ended block-Thomas recursion used by the factors (-1: plain chain; valid
 * after feast_gpu_prepare). Introspection for tests and benchmarks; any pointer may be NULL. */
int feast_gpu_storage(const feast_gpu_ctx* ctx, int* b, int* layers, int* twist);

/* Contour points actually used (host copies): z (2*n_e interleaved) and the
 * quadrature coefficients c_e = 0.5 * w_e * r * e^{i theta_e} (2*n_e). */
int feast_gpu_contour(const feast_gpu_ctx* ctx, double* z, double* coeff);

/* ShiftSystem::solve_in_place for node e on the prepared factors:
 * rhs (n*m complex, interleaved) <- (z_e B - A)^{-1} rhs   (mode 0 = Normal)
 *                                   (z_e B - A)^{-H} rhs   (mode 1 = ConjTranspose) */
int feast_gpu_solve_shift(feast_gpu_ctx* ctx, int e, double* rhs, int m, int mode);

/* accumulate_subspace_real: Q = -sum_e Re(c_e (z_e B - A)^{-1} Y), Y and Q n*m real. */
int feast_gpu_contour_pass(feast_gpu_ctx* ctx, const double* y, int m, double* q);

/* accumulate_subspace_hermitian (core.hpp:190-215): q (n*m complex) = -sum_e (w_e r / 4)
 * (e^{i theta_e} G_e + e^{-i theta_e} G_e^H) y for a complex block y (n*m, interleaved), on the
 * prepared factors, nodes summed in ascending e (+ allreduce across ranks). For the real
 * symmetric pencils this path holds, G^H y = conj(G conj(y)): one complex solve of [Re y | Im y]
 * per node gives both terms. */
int feast_gpu_contour_pass_hermitian(feast_gpu_ctx* ctx, const double* y, int m, double* q);

/* rayleigh_ritz on Q (n*m real): Ritz values (ascending, m_out of them) and Ritz
 * vectors X (n*m_out). truncated = spectral-truncation fallback was used. */
int feast_gpu_rayleigh_ritz(feast_gpu_ctx* ctx, const double* q, int m, double* eigenvalues,
                            double* x, int* m_out, int* truncated);

/* reduced_gevp on host blocks a_q, b_q (m*m): eigenvalues (m_out, ascending) and
 * phi (m*m_out), B_Q-orthonormal. Returns FEAST_EBREAKDOWN like SubspaceBreakdown. */
int feast_gpu_reduced_gevp(feast_gpu_ctx* ctx, int m, const double* a_q, const double* b_q,
                           double* eigenvalues, double* phi, int* m_out, int* truncated);

/* residual_norms (residual.hpp:29-68) for m pairs on the uploaded pencil. */
int feast_gpu_residuals(feast_gpu_ctx* ctx, int m, const double* lambdas, const double* x,
                        double* residuals, int32_t* absolute_only, double* max_residual);

/* The whole FEAST loop (core.hpp:264-391) with Q, Y, X and the factors resident
 * on the device. initial_y (n*y_cols) may be NULL (seeded random_block). The
 * pencil must have been set; the contour/factors are (re)built for [emin, emax]. */
int feast_gpu_solve(feast_gpu_ctx* ctx, double emin, double emax, const feast_config_t* config,
                    const double* initial_y, int y_cols, feast_result_t* result);

/* Look-ahead contour pass (default on): during each Rayleigh-Ritz step the next pass's Ne solves
 * run on B Q, concurrently with the reduced eigensolve, and the next subspace is formed as
 * (that result) Phi — the same iteration as core.hpp:356-388 by linearity of the filter. Used from
 * pass 1 on, when the Ritz block's cancellation factor max_i sum_j ||q_j||_B |Phi_ji| is <= the bound (otherwise the
 * pass is redone in the reference order), never with streamed factors. enable = 0 runs every
 * pass in the reference order; max_cancellation > 0 replaces the admission bound 1e3. */
int feast_gpu_set_lookahead(feast_gpu_ctx* ctx, int enable, double max_cancellation);

/* Warm-started parameter sweep, run_sweep (run.cpp:63-125): for each step k the pencil
 * (A0 + steps[k] S, B) (add_scaled, operator.hpp:282-304) is solved over [emin, emax]; a
 * converged step's Ritz block, topped up with random_block(n, m0 - cols, seed + 1000003 (k + 1))
 * columns when truncation shrank it, times B starts the next step. Operators, factors and the
 * warm block stay on the device (A = A0 + t S is formed there). results[k] is filled like
 * feast_gpu_solve's (caller-allocated arrays); step_codes[k] = FEAST_OK, or FEAST_ENUMERICAL for
 * a step whose solve raised NumericalError (the next step then starts cold, as in the
 * reference); any other error ends the sweep with that code. The storage is chosen for the
 * union of the A0, S and B patterns; the pencil stays set afterwards (at the last step's A). */
int feast_gpu_sweep(feast_gpu_ctx* ctx, const feast_operator_t* a0, const feast_operator_t* b,
                    const feast_operator_t* s, const double* steps, int nsteps, double emin, double emax,
                    const feast_config_t* config, feast_result_t* results, int* step_codes);

/* Benchmark hook: runs `passes` loop bodies (contour pass + Rayleigh-Ritz + trace/count
 * + Y = B X) on the device-resident state set up by feast_gpu_bench_init (after
 * feast_gpu_prepare), with no stopping rule. Each pass is bracketed by CUDA events on the
 * context stream, the passes pipelined as in feast_gpu_solve (look-ahead included); when
 * flush_bytes > 0 a buffer of that size is overwritten once before the passes (outside the
 * events). Outputs: device milliseconds of the whole sequence and phase_ms[4] summed over the
 * passes = {contour-solve kernel(s), Q reduction + allreduce, Rayleigh-Ritz (projection +
 * reduced eigensolve), dominant kernel alone}; with look-ahead the phases overlap. */
int feast_gpu_bench_init(feast_gpu_ctx* ctx, int m0, uint64_t seed);
int feast_gpu_bench_passes(feast_gpu_ctx* ctx, int passes, size_t flush_bytes, double* total_ms,
                           double* phase_ms);

/* Passes of this context (solves and bench) whose look-ahead result was admitted. */
int feast_gpu_lookahead_count(const feast_gpu_ctx* ctx);

/* Number of kernel launches this context issued since creation (evidence counter). */
int64_t feast_gpu_launch_count(const feast_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FEAST_GPU_H_ */
