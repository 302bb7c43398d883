// feast_gpu.cpp — host side of libfeastgpu: the C-ABI of include/feast_gpu.h.
//
// This is the C++ host driver the north star asks for. It keeps the reference solver's
// API and status semantics (feast::feast_solve<double>, core.hpp:264-391) and drives the
// sm_100a kernels: contour solves + fused quadrature epilogue (blocktri.cu / dense.cu),
// the ordered reduction of Q and the NCCL allreduce across ranks, Rayleigh-Ritz with
// the reduced eigensolve on device (gemm.cu, eig.cu), residuals (misc.cu).
// Nothing here computes on the CPU except scalars: the contour constants (once per
// solve), the start block (mt19937_64, as the reference), the trace/count/status logic.

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <exception>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/feast_gpu.h"
#include "kernels.h"

using namespace feastgpu;

namespace {

// ----------------------------------------------------------------------------
// error plumbing: C++ exceptions inside, integer codes at the C-ABI
// ----------------------------------------------------------------------------
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw Failure(code, m); }

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      fail(FEAST_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x);      \
  } while (0)

// ----------------------------------------------------------------------------
// NCCL, resolved at run time (no link-time dependency; torch's copy is reused if loaded)
// ----------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, const void* /*by value 128B*/, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
};
struct NcclUid {
  char internal[128];
};
typedef int (*nccl_init_fn)(void**, int, NcclUid, int);
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (api.h) {
      api.getUniqueId = (int (*)(void*))dlsym(api.h, "ncclGetUniqueId");
      api.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
          api.h, "ncclAllReduce");
      api.allGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(api.h, "ncclAllGather");
      api.commDestroy = (int (*)(void*))dlsym(api.h, "ncclCommDestroy");
      api.getErrorString = (const char* (*)(int))dlsym(api.h, "ncclGetErrorString");
    }
  }
  return api;
}
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

// ----------------------------------------------------------------------------
// Collectives of one context's rank group. NcclComm is the product path (one process per GPU,
// NVLink / NVSwitch; NCCL picks NVLS on NVSwitch systems). LocalComm is a loopback group of
// contexts inside ONE process (one host thread per context, any devices): the same collective
// semantics through device copies and host barriers — no kernel ever waits on another rank's
// kernel — so the sharded loop and the row-distributed Rayleigh-Ritz run, and are tested, on a
// single GPU (tests/test_gpu_sharding.py).
// ----------------------------------------------------------------------------
struct Comm {
  virtual ~Comm() = default;
  // p <- sum over ranks of p (count doubles, in place), identical on every rank
  virtual void allreduce(double* p, size_t count, cudaStream_t st) = 0;
  // recv[r * count .. (r + 1) * count) <- rank r's send (count doubles)
  virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  // this rank failed: release the others (a loopback group's barriers; NCCL ranks see the abort
  // of the process)
  virtual void abort() {}
};

struct NcclComm : Comm {
  void* comm = nullptr;
  ~NcclComm() override {
    if (comm && nccl().commDestroy) nccl().commDestroy(comm);
  }
  static void check(int r, const char* what) {
    if (r != 0) fail(FEAST_ENCCL, std::string(what) + ": " + (nccl().getErrorString ? nccl().getErrorString(r) : "?"));
  }
  void allreduce(double* p, size_t count, cudaStream_t st) override {
    if (!nccl().allReduce) fail(FEAST_ENCCL, "NCCL not available");
    check(nccl().allReduce(p, p, count, kNcclFloat64, kNcclSum, comm, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (!nccl().allGather) fail(FEAST_ENCCL, "NCCL not available");
    check(nccl().allGather(send, recv, count, kNcclFloat64, comm, st), "ncclAllGather");
  }
};

}  // namespace

struct feast_gpu_group {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  double* stage = nullptr;  // nranks slots (device memory of the first rank's device)
  size_t slot = 0;          // doubles per slot
  // all ranks meet here; a rank that fails breaks the group so the others fail instead of hanging
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) fail(FEAST_ENCCL, "local group: another rank failed");
    const uint64_t g = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      fail(FEAST_ENCCL, "local group: barrier timed out or another rank failed");
    }
  }
  void breakup() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

namespace {

struct LocalComm : Comm {
  feast_gpu_group* g;
  int rank;
  LocalComm(feast_gpu_group* grp, int r) : g(grp), rank(r) {}
  void abort() override { g->breakup(); }
  void stage_ready(size_t count) {  // every rank enters; rank 0 sizes the slots
    g->barrier();
    if (rank == 0 && g->slot < count) {
      if (g->stage) CK(cudaFree(g->stage));
      g->stage = nullptr;
      g->slot = 0;
      CK(cudaMalloc(reinterpret_cast<void**>(&g->stage), sizeof(double) * count * g->nranks));
      g->slot = count;
    }
    g->barrier();
  }
  void allreduce(double* p, size_t count, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    stage_ready(count);
    CK(cudaMemcpyAsync(g->stage + rank * g->slot, p, sizeof(double) * count, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
    CK(sum_slices(g->stage, g->nranks, (int64_t)g->slot, count, p, st));  // rank order: same bits everywhere
    CK(cudaStreamSynchronize(st));
    g->barrier();
  }
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    stage_ready(count);
    CK(cudaMemcpyAsync(g->stage + rank * g->slot, send, sizeof(double) * count, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
    for (int r = 0; r < g->nranks; ++r)
      CK(cudaMemcpyAsync(recv + r * count, g->stage + r * g->slot, sizeof(double) * count, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
  }
};

// ----------------------------------------------------------------------------
// Gauss-Legendre + half-circle contour (restates quadrature.cpp:14-87): Newton on the
// three-term Legendre recurrence in extended precision, positive half mirrored.
// ----------------------------------------------------------------------------
void legendre(int n, long double x, long double& p, long double& dp) {
  long double a = 1.0L, b = x;
  for (int k = 2; k <= n; ++k) {
    const long double c = ((2.0L * k - 1.0L) * x * b - (k - 1.0L) * a) / k;
    a = b;
    b = c;
  }
  p = b;
  dp = n * (x * b - a) / (x * x - 1.0L);
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  if (n < 1 || n > 64) fail(FEAST_EINPUT, "gauss_legendre: point count out of supported range");
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const long double pi = 3.14159265358979323846264338327950288L;
  for (int i = 0; i < n / 2; ++i) {
    long double r = std::cos(static_cast<double>(pi * (i + 0.75L) / (n + 0.5L)));
    long double p = 0, dp = 1;
    for (int it = 0; it < 100; ++it) {
      legendre(n, r, p, dp);
      const long double d = p / dp;
      r -= d;
      if (std::fabs(static_cast<double>(d)) <= 1e-15) {
        legendre(n, r, p, dp);
        r -= p / dp;
        break;
      }
    }
    legendre(n, r, p, dp);
    const long double wt = 2.0L / ((1.0L - r * r) * dp * dp);
    x[n - 1 - i] = static_cast<double>(r);
    x[i] = -static_cast<double>(r);
    w[n - 1 - i] = w[i] = static_cast<double>(wt);
  }
  if (n % 2) {
    long double p, dp;
    legendre(n, 0.0L, p, dp);
    x[n / 2] = 0.0;
    w[n / 2] = static_cast<double>(2.0L / (dp * dp));
  }
}

// Device buffers come from the device's stream-ordered memory pool on the calling context's
// stream (set by guarded()): freed memory stays in the pool (release threshold = max, set at
// feast_gpu_create), so a fresh context in the same process (a second solve, the bench's e2e
// leg) reuses it without cudaMalloc/cudaFree round trips, and no free synchronises the device.
thread_local cudaStream_t g_alloc_stream = nullptr;
struct AllocStream {
  cudaStream_t prev;
  explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocStream() { g_alloc_stream = prev; }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void ensure(size_t count) {
    if (count <= n) return;
    if (p && n) cudaFreeAsync(p, g_alloc_stream);
    p = nullptr;
    n = 0;
    if (count) {
      CK(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, g_alloc_stream));
      n = count;
    }
  }
  void release() {
    if (p && n) cudaFreeAsync(p, g_alloc_stream);  // n == 0: a non-owning view into another buffer
    p = nullptr;
    n = 0;
  }
};

// bytes the pool holds in reserve (freed by earlier contexts, reusable by this one)
size_t pool_spare(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return 0;
  uint64_t reserved = 0, used = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  return reserved > used ? (size_t)(reserved - used) : 0;
}

}  // namespace

struct feast_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t aux = nullptr;     // side stream: the initial block's generator runs beside the factor
  cudaEvent_t y_ready = nullptr;  // recorded on aux; the main stream waits on it before the first pass
  bool y_pending = false;
  std::string err;
  // multi-GPU: rank group (NCCL, or a loopback group of contexts in one process)
  std::unique_ptr<Comm> comm;
  int rank = 0, nranks = 1;
  bool row_dist = true;  // row-distributed Rayleigh-Ritz across the ranks (feast_gpu_set_row_distribution)
  DevBuf<double> G;      // allgather staging (row-distributed)
  // pencil
  bool have_pencil = false;
  int n = 0, npad = 0;
  bool blocktri = false;
  int L = 0, b = 0;
  DevBuf<double> A, Bm;            // dense n*n
  DevBuf<double2> abdiag, ablow;  // block-tridiagonal (A, B) pairs
  double norm_a1 = 0.0;
  // contour
  bool have_contour = false;
  double emin = 0, emax = 0, radius = 0;
  int ne = 0, e0 = 0, e1 = 0;
  std::vector<double2> z, coeff;  // all nodes
  DevBuf<double2> dz, dcoeff;     // owned nodes
  // factors: all owned nodes resident (batch == 0 or batch >= owned), or streamed in node
  // batches of `batch` (factors recomputed every pass: the memory plan for pencils whose
  // factors exceed HBM, e.g. BASELINE config 5 at 1-2 GPUs); res0/rescnt = resident range
  bool factored = false;
  int batch_req = 0, batch = 0, res0 = -1, rescnt = 0;
  DevBuf<double2> sinv, gfac, hfac, lu, dinv, scratch, fwork;
  DevBuf<double> A0, Sop;       // feast_gpu_sweep: the unperturbed A and the perturbation S (A's layout)
  DevBuf<double> Aband, Bband;  // band-row copies of A, B for the applies (b <= 32; band_apply.cu)
  int kmid = -1;  // twisted block-Thomas meeting layer of the current factors (bt_twist_layer)
  DevBuf<int> ipiv, perm, status, fstatus;  // status: reduced Cholesky; fstatus: factorisation
  bool chol_failed_prev = false;  // the last reduced_gevp took the truncation path
  bool gevp_enqueued = false;     // reduced_gevp_start enqueued the whole Cholesky path
  // look-ahead contour pass (rayleigh_ritz_la): setting, and whether the last eigensolve's
  // cancellation factor admitted it (the predictor for launching the next one)
  bool lookahead = true, lookahead_ok = true;
  double la_kmax = 1e3;  // admission bound of the look-ahead pass (kLookaheadMaxK)
  cudaStream_t eigs = nullptr;  // high-priority stream of the reduced eigensolve
  cudaEvent_t ev_proj = nullptr, ev_eig = nullptr, ev_pre_eig = nullptr;
  cudaEvent_t ev_lu_cols = nullptr, ev_lu_panel = nullptr;  // LU look-ahead (dense factorisation)
  double* hpin = nullptr;       // pinned: status, cancellation factor, eigenvalues
  size_t hpin_n = 0;
  DevBuf<double> kfac;
  // inner solver (inner_solver.hpp): 0 = DirectSolver, 1 = IterativeSolver (BiCGStab, bicgstab.cu)
  int inner_kind = 0;
  double inner_tol = 0.0;
  int inner_max_iter = 0;
  int factor_policy = 0;  // FactorPolicy at set_pencil: 0 Auto, 1 Dense, 2 Banded (inner_solver.hpp:40-47)
  DevBuf<double2> bvec;   // BiCGStab: X R R0 P V S T, npad x C each
  DevBuf<double> breal;   // BiCGStab: PR AR BR, npad x 2C each
  DevBuf<BicgCol> bcol;
  DevBuf<int> bflag;
  DevBuf<double2> bz;
  // SPIKE partitioning of the block-Thomas chain (spike.cu, b <= 32): requested chunk count
  // (feast_gpu_set_spike; 0 = automatic) and the one the current factors use
  int spike_req = 0, spike = 1;
  DevBuf<double2> spk, rlu, rdinv, rz, rzs;  // spikes [V | W], reduced LU, its block inverses, reduced RHS
  DevBuf<double> sra, rzr;                  // correction operands [Re cV | -Im cV | Re cW | -Im cW], z parts
  DevBuf<int> ripiv, rperm;
  bool hermitian = false;  // set_pencil_hermitian: the doubled real pencil of a complex one
  int nz = 0;              // its complex dimension
  bool twist = true;  // two-ended block-Thomas recursion where it applies (feast_gpu_set_twist)
  // workspaces
  int mcap = 0;
  DevBuf<double> Y, Q, X, AQ, BQ, T, gw;
  DevBuf<double2> W;
  DevBuf<double> Aq, Bq, Cm, Lm, Phi, Ev, Vm, S, Tm, Dv;
  DevBuf<int> keep;
  DevBuf<double> csr;        // CSR operators as uploaded (set_pencil's device route)
  DevBuf<CsrStats> csrstats;
  EigWork* eig = nullptr;
  int eig_cap = 0;
  // host phase tracing (FEAST_TRACE=1: host wall clock per phase to stderr; =2: with a stream
  // sync before each mark, so device work is attributed to the phase that enqueued it)
  int trace = 0;
  std::chrono::steady_clock::time_point tmark;
  // bench state
  int bench_m = 0;
  bool bench_have_q = false;  // the bench loop's next pass already has its Q (look-ahead)
  int bench_pass = 0;
  int lookahead_count = 0;    // passes (solve or bench) whose look-ahead result was admitted
  bool timing = false;
  cudaEvent_t ev[8] = {};
  cudaEvent_t pev[2][4] = {};  // phase timing per pass parity: contour start, contour end, RR start, solves end

  int owned() const { return e1 - e0; }
  bool streamed() const { return batch > 0 && batch < owned(); }
  int wnodes() const { return streamed() ? batch : owned(); }  // node slots in the workspaces
};

namespace {

// Small page-locked buffers (the per-pass status / eigenvalue read-back) from a process-wide pool:
// cudaMallocHost / cudaFreeHost cost milliseconds and synchronise, and an end-to-end solve opens
// a fresh context every time.
std::mutex g_pin_mu;
std::vector<std::pair<double*, size_t>> g_pin_free;
double* pinned_small_get(size_t count, size_t& got) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_pin_free.size(); ++i)
      if (g_pin_free[i].second >= count) {
        double* p = g_pin_free[i].first;
        got = g_pin_free[i].second;
        g_pin_free.erase(g_pin_free.begin() + i);
        return p;
      }
  }
  double* p = nullptr;
  const size_t n = std::max<size_t>(count, 1026);  // (M0 up to 1024 + 2 scalars)
  CK(cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(double) * n));
  got = n;
  return p;
}
void pinned_small_release(double*& p, size_t& n) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace_back(p, n);
  p = nullptr;
  n = 0;
}

void ensure_eig(feast_gpu_ctx* c, int m) {
  if (c->eig && c->eig_cap >= m) return;
  if (c->eig) {
    CK(cudaStreamSynchronize(c->stream));  // a released workspace may go to another context
    if (c->eigs) CK(cudaStreamSynchronize(c->eigs));
    eig_destroy(c->eig);
  }
  c->eig = eig_create(std::max(m, 16));
  if (!c->eig) fail(FEAST_ECUDA, "CUDA: out of memory for the reduced eigensolver workspace");
  c->eig_cap = std::max(m, 16);
}

// reduced blocks: Aq and Bq adjacent (the m x 2m output of Q^T [AQ | BQ], ld m)
void ensure_reduced(feast_gpu_ctx* c, int m) {
  const size_t mm = (size_t)m * m;
  c->Aq.ensure(2 * mm);
  c->Bq.p = c->Aq.p + mm;
  c->Bq.n = 0;
  for (DevBuf<double>* d : {&c->Cm, &c->Lm, &c->Phi, &c->Vm, &c->S, &c->Tm}) d->ensure(mm);
  c->Ev.ensure(m);
  c->keep.ensure(m);
  c->kfac.ensure(1);
  c->status.ensure(1);
  c->Dv.ensure((size_t)((m + 31) / 32) * 1024);
  if (c->hpin_n < (size_t)m + 2) {
    pinned_small_release(c->hpin, c->hpin_n);
    c->hpin = pinned_small_get((size_t)m + 2, c->hpin_n);
  }
}

void plan_batch(feast_gpu_ctx* c, int m);

void ensure_workspace(feast_gpu_ctx* c, int m) {
  if (m <= c->mcap) return;
  // the node batch decides how many W/T slots there are: plan it for this m first (a plan made
  // for the owned nodes before the workspaces existed would size W/T for every node)
  if (c->have_pencil) plan_batch(c, m);
  const size_t nv = (size_t)c->npad * m;
  const int own = std::max(c->wnodes(), 1);
  c->Y.ensure(nv);
  c->Q.ensure(nv);
  c->X.ensure(nv);
  c->AQ.ensure(2 * nv);  // [AQ | BQ] adjacent: one Q^T [AQ | BQ] GEMM forms both projections
  c->BQ.p = c->AQ.p + nv;
  c->BQ.n = 0;
  // doubles; the dense path's complex-mode shim reuses it as double2 (2 nv per slot), the
  // block-tridiagonal path needs the real terms only (nv per slot: 6.4 GB saved per node slot
  // at config 5, the difference between one and two resident node slots on 180 GB)
  c->T.ensure((c->blocktri ? 1 : 2) * nv * own);
  c->W.ensure(nv * own);
  const size_t mm = (size_t)m * m;
  ensure_reduced(c, m);
  c->gw.ensure(std::max<size_t>(mm * 64, nv));
  ensure_eig(c, m);
  c->mcap = m;
}

void sync(feast_gpu_ctx* c) { CK(cudaStreamSynchronize(c->stream)); }

// Y = random_block(n, m, seed) (core.hpp:84-106) generated on the device into c->Y on the side
// stream (zero padding rows); the main stream joins it before its first use (join_aux)
void device_random_block(feast_gpu_ctx* c, int m, uint64_t seed) {
  if (!c->aux) {
    CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->y_ready, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(c->y_ready, c->stream));  // Y's previous readers on the main stream
  CK(cudaStreamWaitEvent(c->aux, c->y_ready, 0));
  if (c->npad != c->n) CK(fill_zero(c->Y.p, (size_t)c->npad * m, c->aux));
  CK(random_block_device(seed, c->n, m, c->Y.p, c->npad, c->aux));
  CK(cudaEventRecord(c->y_ready, c->aux));
  c->y_pending = true;
}
void join_aux(feast_gpu_ctx* c) {
  if (!c->y_pending) return;
  CK(cudaStreamWaitEvent(c->stream, c->y_ready, 0));
  c->y_pending = false;
}

void trace_mark(feast_gpu_ctx* c, const char* what) {
  if (!c->trace) return;
  if (c->trace >= 2) sync(c);
  const auto now = std::chrono::steady_clock::now();
  if (what)
    std::fprintf(stderr, "[feast_gpu] %-34s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - c->tmark).count());
  c->tmark = now;
}

// ------------------------------- pencil -------------------------------------
// Host-side pencil preparation runs over row ranges on up to 8 threads (the C-ABI call is the
// user's; its validation and re-blocking were ~11 ms of a 70 ms end-to-end solve at config 2).
// fn(lo, hi) must only write state owned by rows [lo, hi); a Failure thrown by any range is
// rethrown (the one from the lowest range, so the message is deterministic).
template <typename F>
void parallel_rows(int n, int align, F&& fn) {
  const int hw = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const int nt = n < 4096 ? 1 : hw;
  if (nt == 1) {
    fn(0, n);
    return;
  }
  std::vector<int> cut(nt + 1);
  for (int t = 0; t <= nt; ++t) cut[t] = std::min(n, (int)(((int64_t)n * t / nt + align - 1) / align * align));
  cut[nt] = n;
  std::vector<std::exception_ptr> errs(nt);
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        if (cut[t] < cut[t + 1]) fn(cut[t], cut[t + 1]);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void validate_dense_symmetric(const double* m, int n) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < j; ++i)
      if (m[i + (size_t)j * n] != m[j + (size_t)i * n])
        fail(FEAST_EINPUT, "SymmetricOperator: matrix is not symmetric");
}

int csr_bandwidth(const feast_operator_t* o) {
  std::atomic<int> bw{0};
  parallel_rows(o->n, 1, [&](int r0, int r1) {
    int b = 0;
    for (int i = r0; i < r1; ++i)
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) b = std::max(b, std::abs(i - o->col_idx[k]));
    int cur = bw.load();
    while (b > cur && !bw.compare_exchange_weak(cur, b)) {
    }
  });
  return bw;
}

void validate_csr(const feast_operator_t* o) {
  const int n = o->n;
  if (o->row_ptr[0] != 0) fail(FEAST_EINPUT, "SymmetricOperator: bad row_ptr");
  for (int i = 0; i < n; ++i)
    if (o->row_ptr[i + 1] < o->row_ptr[i]) fail(FEAST_EINPUT, "SymmetricOperator: bad row_ptr");
  parallel_rows(n, 1, [&](int r0, int r1) {
    for (int i = r0; i < r1; ++i) {
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) {
        const int j = o->col_idx[k];
        if (j < 0 || j >= n) fail(FEAST_EINPUT, "SymmetricOperator: triplet index out of range");
        if (j <= i) continue;
        // mirror (j, i) must exist with the same value (operator.hpp:237-261)
        const int* b = o->col_idx + o->row_ptr[j];
        const int* e = o->col_idx + o->row_ptr[j + 1];
        const int* f = std::lower_bound(b, e, i);
        if (f == e || *f != i) {
          bool found = false;  // unsorted rows: linear scan
          for (const int* q = b; q != e; ++q)
            if (*q == i) {
              found = true;
              if (o->values[o->row_ptr[j] + (q - b)] != o->values[k])
                fail(FEAST_EINPUT, "SymmetricOperator: mirror entries disagree");
            }
          if (!found) fail(FEAST_EINPUT, "SymmetricOperator: missing mirror entry");
        } else if (o->values[o->row_ptr[j] + (f - b)] != o->values[k]) {
          fail(FEAST_EINPUT, "SymmetricOperator: mirror entries disagree");
        }
      }
    }
  });
}

// smallest block size (multiple of 16; of 32 above 128) for which the CSR pattern is
// block-tridiagonal
int log2_exact(int b) {  // b is a power of two (round_block)
  int s = 0;
  while ((1 << s) < b) ++s;
  return s;
}
bool csr_fits_blocktri(const feast_operator_t* o, int b) {
  const int sh = log2_exact(b);
  std::atomic<bool> ok{true};
  parallel_rows(o->n, 1, [&](int r0, int r1) {
    for (int i = r0; i < r1 && ok.load(std::memory_order_relaxed); ++i) {
      const int li = i >> sh;
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k)
        if (std::abs(li - (o->col_idx[k] >> sh)) > 1) {
          ok = false;
          break;
        }
    }
  });
  return ok;
}
// block sizes the sweep kernels are specialised for (sweep.cu)
int round_block(int b) {
  int r = 16;
  while (r < b) r *= 2;
  return r;
}
constexpr int kMaxBlock = 512;

// dense view (host) of any operator
std::vector<double> to_dense(const feast_operator_t* o) {
  const int n = o->n;
  std::vector<double> m((size_t)n * n, 0.0);
  if (o->kind == FEAST_STORAGE_DENSE) {
    std::memcpy(m.data(), o->dense, sizeof(double) * m.size());
  } else if (o->kind == FEAST_STORAGE_CSR) {
    for (int i = 0; i < n; ++i)
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) m[i + (size_t)o->col_idx[k] * n] += o->values[k];
  } else {
    const int b = o->bsize;
    for (int l = 0; l < o->nblocks; ++l) {
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) m[(l * b + i) + (size_t)(l * b + j) * n] = o->diag[(size_t)l * b * b + i + j * b];
      if (l + 1 < o->nblocks)
        for (int j = 0; j < b; ++j)
          for (int i = 0; i < b; ++i) {
            const double v = o->lower[(size_t)l * b * b + i + j * b];
            m[((l + 1) * b + i) + (size_t)(l * b + j) * n] = v;
            m[(l * b + j) + (size_t)((l + 1) * b + i) * n] = v;
          }
    }
  }
  return m;
}

// block-tridiagonal host view with block size b and L = ceil(n/b) blocks; padding rows
// get A = 0, B = 1 (decoupled, never reached by a zero-padded right-hand side)
void to_blocktri(const feast_operator_t* o, int b, int L, bool is_b, std::vector<double>& diag,
                 std::vector<double>& low) {
  const int n = o->n;
  diag.assign((size_t)L * b * b, 0.0);
  low.assign((size_t)(L > 1 ? L - 1 : 0) * b * b, 0.0);
  if (is_b)
    for (int r = n; r < L * b; ++r) diag[(size_t)(r / b) * b * b + (r % b) * (b + 1)] = 1.0;
  if (o->kind == FEAST_STORAGE_BLOCKTRI && o->bsize == b) {
    std::memcpy(diag.data(), o->diag, sizeof(double) * (size_t)o->nblocks * b * b);
    if (o->nblocks > 1) std::memcpy(low.data(), o->lower, sizeof(double) * (size_t)(o->nblocks - 1) * b * b);
    return;
  }
  const int sh = log2_exact(b), msk = b - 1;
  auto put = [&](int i, int j, double v) {
    const int li = i >> sh, lj = j >> sh, ii = i & msk, jj = j & msk;
    if (li == lj) diag[((size_t)li << (2 * sh)) + ii + ((size_t)jj << sh)] += v;
    else if (li == lj + 1) low[((size_t)lj << (2 * sh)) + ii + ((size_t)jj << sh)] += v;
  };
  if (o->kind == FEAST_STORAGE_CSR) {  // row i writes only layer i/b's diagonal and lower blocks
    parallel_rows(n, b, [&](int r0, int r1) {
      for (int i = r0; i < r1; ++i)
        for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) put(i, o->col_idx[k], o->values[k]);
    });
  } else if (o->kind == FEAST_STORAGE_BLOCKTRI) {  // re-block (lower triangle suffices)
    const int bo = o->bsize;
    for (int l = 0; l < o->nblocks; ++l) {
      for (int j = 0; j < bo; ++j)
        for (int i = 0; i < bo; ++i) {
          const double v = o->diag[(size_t)l * bo * bo + i + (size_t)j * bo];
          if (v != 0.0) put(l * bo + i, l * bo + j, v);
        }
      if (l + 1 < o->nblocks)
        for (int j = 0; j < bo; ++j)
          for (int i = 0; i < bo; ++i) {
            const double v = o->lower[(size_t)l * bo * bo + i + (size_t)j * bo];
            if (v != 0.0) put((l + 1) * bo + i, l * bo + j, v);
          }
    }
  } else {
    fail(FEAST_EINPUT, "set_pencil: cannot re-block this operator");
  }
}

double norm_one(const feast_operator_t* o) {  // operator.hpp:195-212
  const int n = o->n;
  std::vector<double> cs(n, 0.0);
  if (o->kind == FEAST_STORAGE_DENSE) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) cs[j] += std::fabs(o->dense[i + (size_t)j * n]);
  } else if (o->kind == FEAST_STORAGE_CSR) {
    for (int i = 0; i < n; ++i)
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) cs[i] += std::fabs(o->values[k]);
  } else {
    const int b = o->bsize;
    for (int l = 0; l < o->nblocks; ++l) {
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) cs[l * b + j] += std::fabs(o->diag[(size_t)l * b * b + i + j * b]);
      if (l + 1 < o->nblocks)
        for (int j = 0; j < b; ++j)
          for (int i = 0; i < b; ++i) {
            const double v = std::fabs(o->lower[(size_t)l * b * b + i + j * b]);
            cs[l * b + j] += v;        // column l*b+j gets C_l entries
            cs[(l + 1) * b + i] += v;  // column (l+1)*b+i gets C_l^T entries
          }
    }
  }
  double best = 0.0;
  for (double v : cs) best = std::max(best, v);
  return best;
}

void check_operator(const feast_operator_t* o) {
  if (!o) fail(FEAST_EINPUT, "set_pencil: null operator");
  if (o->n < 1) fail(FEAST_EINPUT, "feast_solve: empty operator");
  switch (o->kind) {
    case FEAST_STORAGE_DENSE:
      if (!o->dense) fail(FEAST_EINPUT, "set_pencil: dense data missing");
      validate_dense_symmetric(o->dense, o->n);
      break;
    case FEAST_STORAGE_CSR:
      if (!o->row_ptr || !o->col_idx || !o->values) fail(FEAST_EINPUT, "set_pencil: CSR data missing");
      validate_csr(o);
      break;
    case FEAST_STORAGE_BLOCKTRI: {
      if (!o->diag || (o->nblocks > 1 && !o->lower) || o->bsize < 1 ||
          (int64_t)o->nblocks * o->bsize != o->n)
        fail(FEAST_EINPUT, "set_pencil: bad block-tridiagonal descriptor");
      const int b = o->bsize;
      for (int l = 0; l < o->nblocks; ++l)
        for (int j = 0; j < b; ++j)
          for (int i = 0; i < j; ++i)
            if (o->diag[(size_t)l * b * b + i + j * b] != o->diag[(size_t)l * b * b + j + i * b])
              fail(FEAST_EINPUT, "SymmetricOperator: matrix is not symmetric");
      break;
    }
    default:
      fail(FEAST_EINPUT, "set_pencil: unknown storage kind");
  }
}

// ---- Hermitian pencils -------------------------------------
// A complex Hermitian operator (kinds FEAST_STORAGE_DENSE_Z / FEAST_STORAGE_CSR_Z: complex
// entries interleaved) is carried as the real symmetric operator of twice the size whose entry
// a_ij = x + iy is the 2 x 2 block [[x, -y], [y, x]] at rows (2i, 2i+1), columns (2j, 2j+1). An
// interleaved complex vector IS a real vector of that operator, multiplication by i is the
// rotation J (re, im) -> (-im, re) that commutes with both operators, and a complex eigenpair
// (lambda, phi) is the pair of real ones (lambda, phi), (lambda, J phi). The FEAST loop of the
// complex pencil (core.hpp:264-391 with T = cplx) is then the real loop on the doubled pencil,
// started from [Y | J Y] and read through one representative per Ritz pair (feast_solve's pair
// mode) — every kernel, the look-ahead pass and the multi-rank path carry over unchanged.
void validate_hermitian(const feast_operator_t* o) {
  if (!o) fail(FEAST_EINPUT, "set_pencil: null operator");
  if (o->n < 1) fail(FEAST_EINPUT, "feast_solve: empty operator");
  const int n = o->n;
  if (o->kind == FEAST_STORAGE_DENSE_Z) {  // from_dense (operator.hpp:45-62)
    if (!o->dense) fail(FEAST_EINPUT, "set_pencil: dense data missing");
    const double* m = o->dense;
    for (int j = 0; j < n; ++j) {
      for (int i = 0; i <= j; ++i) {
        const size_t ij = 2 * ((size_t)i + (size_t)j * n), ji = 2 * ((size_t)j + (size_t)i * n);
        if (m[ij] != m[ji] || m[ij + 1] != -m[ji + 1]) fail(FEAST_EINPUT, "SymmetricOperator: matrix is not symmetric");
      }
      if (m[2 * ((size_t)j + (size_t)j * n) + 1] != 0.0) fail(FEAST_EINPUT, "SymmetricOperator: diagonal must be real");
    }
    return;
  }
  if (o->kind != FEAST_STORAGE_CSR_Z) fail(FEAST_EINPUT, "set_pencil_hermitian: operators must be DENSE_Z or CSR_Z");
  if (!o->row_ptr || !o->col_idx || !o->values) fail(FEAST_EINPUT, "set_pencil: CSR data missing");
  if (o->row_ptr[0] != 0) fail(FEAST_EINPUT, "SymmetricOperator: bad row_ptr");
  for (int i = 0; i < n; ++i)
    if (o->row_ptr[i + 1] < o->row_ptr[i]) fail(FEAST_EINPUT, "SymmetricOperator: bad row_ptr");
  const double* v = o->values;
  for (int i = 0; i < n; ++i)  // validate_sparse_symmetry (operator.hpp:237-262)
    for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) {
      const int j = o->col_idx[k];
      if (j < 0 || j >= n) fail(FEAST_EINPUT, "SymmetricOperator: triplet index out of range");
      if (i == j) {
        if (v[2 * (size_t)k + 1] != 0.0) fail(FEAST_EINPUT, "SymmetricOperator: diagonal must be real");
        continue;
      }
      if (j < i) continue;
      bool found = false;
      for (int k2 = o->row_ptr[j]; k2 < o->row_ptr[j + 1]; ++k2)
        if (o->col_idx[k2] == i) {
          if (v[2 * (size_t)k2] != v[2 * (size_t)k] || v[2 * (size_t)k2 + 1] != -v[2 * (size_t)k + 1])
            fail(FEAST_EINPUT, "SymmetricOperator: mirror entries disagree");
          found = true;
          break;
        }
      if (!found) fail(FEAST_EINPUT, "SymmetricOperator: missing mirror entry");
    }
}

double norm_one_hermitian(const feast_operator_t* o) {  // norm_one (operator.hpp:195-212), |complex|
  const int n = o->n;
  double best = 0.0;
  if (o->kind == FEAST_STORAGE_DENSE_Z) {
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) {
        const size_t q = 2 * ((size_t)i + (size_t)j * n);
        s += std::hypot(o->dense[q], o->dense[q + 1]);
      }
      best = std::max(best, s);
    }
  } else {
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) s += std::hypot(o->values[2 * (size_t)k], o->values[2 * (size_t)k + 1]);
      best = std::max(best, s);
    }
  }
  return best;
}

struct EmbeddedOp {
  std::vector<int> rp, ci;
  std::vector<double> val, dense;
  feast_operator_t op{};
};

// the real symmetric operator of twice the size (2 x 2 blocks [[x, -y], [y, x]])
void embed_hermitian(const feast_operator_t* o, EmbeddedOp& e) {
  const int n = o->n, n2 = 2 * n;
  e.op = feast_operator_t{};
  e.op.n = n2;
  if (o->kind == FEAST_STORAGE_DENSE_Z) {
    e.dense.assign((size_t)n2 * n2, 0.0);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const size_t q = 2 * ((size_t)i + (size_t)j * n);
        const double x = o->dense[q], y = o->dense[q + 1];
        double* d = e.dense.data();
        d[(2 * i) + (size_t)(2 * j) * n2] = x;
        d[(2 * i + 1) + (size_t)(2 * j) * n2] = y;
        d[(2 * i) + (size_t)(2 * j + 1) * n2] = -y;
        d[(2 * i + 1) + (size_t)(2 * j + 1) * n2] = x;
      }
    e.op.kind = FEAST_STORAGE_DENSE;
    e.op.dense = e.dense.data();
    return;
  }
  // CSR: rows sorted by column; exact-zero parts are dropped, and since an entry and its mirror
  // carry the same value the pattern stays symmetric-complete
  e.rp.assign(n2 + 1, 0);
  std::vector<std::pair<int, double>> row;
  for (int i = 0; i < n; ++i) {
    for (int half = 0; half < 2; ++half) {  // rows 2i (re) and 2i + 1 (im)
      row.clear();
      for (int k = o->row_ptr[i]; k < o->row_ptr[i + 1]; ++k) {
        const int j = o->col_idx[k];
        const double x = o->values[2 * (size_t)k], y = o->values[2 * (size_t)k + 1];
        const double c0 = half ? y : x, c1 = half ? x : -y;  // columns 2j, 2j + 1
        if (c0 != 0.0) row.emplace_back(2 * j, c0);  // (the mirror entry has the same value)
        if (c1 != 0.0) row.emplace_back(2 * j + 1, c1);
      }
      std::sort(row.begin(), row.end(), [](const std::pair<int, double>& a, const std::pair<int, double>& b) {
        return a.first < b.first;
      });
      for (auto& [col, val] : row) {
        e.ci.push_back(col);
        e.val.push_back(val);
      }
      e.rp[2 * i + half + 1] = (int)e.ci.size();
    }
  }
  e.op.kind = FEAST_STORAGE_CSR;
  e.op.row_ptr = e.rp.data();
  e.op.col_idx = e.ci.data();
  e.op.values = e.val.data();
}

// ---- CSR operators taken in on the device (csr_ingest.cu) ----------------------
// The route for the common case (A and B both CSR, row pointers well formed): the CSR arrays
// go up once through the pinned stage, csr_scan validates them and measures bandwidth, block
// fit and 1-norm in one pass, csr_to_blocktri assembles the blocks. Errors, messages and
// storage decisions are those of the host path above (validate_csr, csr_bandwidth,
// csr_fits_blocktri, norm_one, to_blocktri), which serves every other combination.
bool csr_rowptr_ok(const feast_operator_t* o) {
  if (!o || o->kind != FEAST_STORAGE_CSR || o->n < 1 || !o->row_ptr || !o->col_idx || !o->values) return false;
  if (o->row_ptr[0] != 0) return false;
  for (int i = 0; i < o->n; ++i)
    if (o->row_ptr[i + 1] < o->row_ptr[i]) return false;
  return true;
}

struct PinnedStage;
constexpr size_t kPinnedStageMax = (size_t)256 << 20;  // bytes (PinnedStage)
PinnedStage& pinned_stage();
double* pinned_stage_lock_get(size_t count, std::unique_lock<std::mutex>& lk);

// copies (dst, src, bytes) pieces on up to 8 host threads
void parallel_copies(const std::vector<std::tuple<char*, const char*, size_t>>& segs) {
  constexpr size_t piece = 1u << 20;
  std::vector<std::tuple<char*, const char*, size_t>> work;
  for (auto& [d, s, nb] : segs)
    for (size_t off = 0; off < nb; off += piece) work.emplace_back(d + off, s + off, std::min(piece, nb - off));
  const int nt = (int)std::min<size_t>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())), work.size());
  if (nt <= 1) {
    for (auto& [d, s, nb] : work) std::memcpy(d, s, nb);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t w = t; w < work.size(); w += nt) std::memcpy(std::get<0>(work[w]), std::get<1>(work[w]), std::get<2>(work[w]));
    });
  for (auto& x : th) x.join();
}

struct DeviceCsr {
  const int* rp[2];
  const int* ci[2];
  const double* val[2];
  CsrStats stats[2];
};

// upload A and B, scan both; throws the host path's InputError for the first bad entry of A,
// then of B
DeviceCsr csr_upload_scan(feast_gpu_ctx* c, const feast_operator_t* a, const feast_operator_t* b) {
  const int n = a->n;
  const size_t nnz[2] = {(size_t)a->row_ptr[n], (size_t)b->row_ptr[n]};
  const size_t ints = 2 * ((size_t)n + 1) + nnz[0] + nnz[1];
  const size_t idoubles = (ints + 1) / 2, total = idoubles + nnz[0] + nnz[1];
  c->csr.ensure(total);
  c->csrstats.ensure(2);
  DeviceCsr d;
  int* ip = reinterpret_cast<int*>(c->csr.p);
  double* vp = c->csr.p + idoubles;
  const feast_operator_t* ops[2] = {a, b};
  {
    std::unique_lock<std::mutex> lk;
    double* st = pinned_stage_lock_get(total, lk);
    std::vector<std::tuple<char*, const char*, size_t>> segs;
    int* sip = st ? reinterpret_cast<int*>(st) : nullptr;
    size_t io = 0, vo = 0;
    for (int t = 0; t < 2; ++t) {
      const feast_operator_t* o = ops[t];
      d.rp[t] = ip + io;
      if (st) segs.emplace_back(reinterpret_cast<char*>(sip + io), reinterpret_cast<const char*>(o->row_ptr), sizeof(int) * (n + 1));
      else CK(cudaMemcpyAsync(ip + io, o->row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, c->stream));
      io += n + 1;
      d.ci[t] = ip + io;
      if (st) segs.emplace_back(reinterpret_cast<char*>(sip + io), reinterpret_cast<const char*>(o->col_idx), sizeof(int) * nnz[t]);
      else if (nnz[t]) CK(cudaMemcpyAsync(ip + io, o->col_idx, sizeof(int) * nnz[t], cudaMemcpyHostToDevice, c->stream));
      io += nnz[t];
      d.val[t] = vp + vo;
      if (st) segs.emplace_back(reinterpret_cast<char*>(st + idoubles + vo), reinterpret_cast<const char*>(o->values), sizeof(double) * nnz[t]);
      else if (nnz[t]) CK(cudaMemcpyAsync(vp + vo, o->values, sizeof(double) * nnz[t], cudaMemcpyHostToDevice, c->stream));
      vo += nnz[t];
    }
    if (st) {
      parallel_copies(segs);
      CK(cudaMemcpyAsync(c->csr.p, st, sizeof(double) * total, cudaMemcpyHostToDevice, c->stream));
    }
    for (int t = 0; t < 2; ++t) CK(csr_scan(n, d.rp[t], d.ci[t], d.val[t], c->csrstats.p + t, true, c->stream));
    CK(cudaMemcpyAsync(d.stats, c->csrstats.p, sizeof(d.stats), cudaMemcpyDeviceToHost, c->stream));
    sync(c);  // (also the end of the stage's use)
  }
  static const char* msg[3] = {"SymmetricOperator: triplet index out of range",
                               "SymmetricOperator: missing mirror entry",
                               "SymmetricOperator: mirror entries disagree"};
  for (int t = 0; t < 2; ++t)
    if (d.stats[t].first_error != ~0ull) fail(FEAST_EINPUT, msg[d.stats[t].first_error & 3]);
  return d;
}

// host -> device copy of `bytes` from pageable memory through the pinned stage: two halves
// alternate, host threads fill one while the DMA drains the other (synchronous on return)
void upload_chunked(feast_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  const size_t half = std::min<size_t>(kPinnedStageMax / 2, ((bytes + 1) / 2 + 63) / 64 * 64);
  std::unique_lock<std::mutex> lk;
  double* st = pinned_stage_lock_get(2 * half / sizeof(double), lk);
  if (!st) {
    lk.unlock();
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    sync(c);
    return;
  }
  cudaEvent_t ev[2];
  CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  bool used[2] = {false, false};
  char* stage[2] = {reinterpret_cast<char*>(st), reinterpret_cast<char*>(st) + half};
  size_t off = 0;
  for (int k = 0; off < bytes; ++k, off += half) {
    const int h = k & 1;
    const size_t len = std::min(half, bytes - off);
    if (used[h]) CK(cudaEventSynchronize(ev[h]));
    parallel_copies({{stage[h], reinterpret_cast<const char*>(src) + off, len}});
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, stage[h], len, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(ev[h], c->stream));
    used[h] = true;
  }
  sync(c);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
}

// s (may be null): a perturbation A + t S will be formed on the device (feast_gpu_sweep); the
// storage is chosen for the union of the three patterns and S is stored like A (c->Sop), with a
// copy of A (c->A0)
void set_pencil(feast_gpu_ctx* c, const feast_operator_t* a, const feast_operator_t* b,
                const feast_operator_t* s = nullptr) {
  trace_mark(c, nullptr);
  c->hermitian = false;
  if (s) {
    check_operator(s);
    if (s->n != a->n) fail(FEAST_EINPUT, "run_sweep: perturbation dimension mismatch");
  }
  const bool dev_csr = !s && csr_rowptr_ok(a) && csr_rowptr_ok(b) && a->n == b->n;
  DeviceCsr dcsr{};
  if (dev_csr) {
    dcsr = csr_upload_scan(c, a, b);
    trace_mark(c, "set_pencil: CSR upload + device validation");
  } else {
    check_operator(a);
    check_operator(b);
    trace_mark(c, "set_pencil: validate operators");
  }
  if (a->n != b->n) fail(FEAST_EINPUT, "feast_solve: operator dimensions differ");
  const int n = a->n;
  // storage policy (the reference's Auto policy, inner_solver.hpp:84-92, with the banded
  // factorisation replaced by block-tridiagonal block Thomas)
  int bsz = 0;
  const bool a_bt = a->kind == FEAST_STORAGE_BLOCKTRI, b_bt = b->kind == FEAST_STORAGE_BLOCKTRI;
  const bool a_sp = (a->kind == FEAST_STORAGE_CSR || a_bt) && (!s || s->kind != FEAST_STORAGE_DENSE),
             b_sp = b->kind == FEAST_STORAGE_CSR || b_bt;
  std::vector<const feast_operator_t*> ops{a, b};
  if (s) ops.push_back(s);
  // FactorPolicy (inner_solver.hpp:80-95): Dense keeps dense factors for any storage, Banded
  // requires sparse operands, Auto chooses by bandwidth as below
  if (c->factor_policy == 2 && !(a_sp && b_sp)) fail(FEAST_EINPUT, "DirectSolver: banded policy requires sparse operands");
  if (a_sp && b_sp && c->factor_policy != 1) {
    if (a_bt && b_bt && a->bsize == b->bsize && round_block(a->bsize) == a->bsize && a->bsize <= kMaxBlock &&
        (!s || (s->kind == FEAST_STORAGE_BLOCKTRI && s->bsize == a->bsize))) {
      bsz = a->bsize;
    } else {
      int bw = 0;
      for (const feast_operator_t* o : ops) {
        if (dev_csr) bw = std::max({bw, dcsr.stats[0].bandwidth, dcsr.stats[1].bandwidth});
        else if (o->kind == FEAST_STORAGE_CSR) bw = std::max(bw, csr_bandwidth(o));
        else bw = std::max(bw, 2 * o->bsize - 1);
      }
      if ((3 * bw + 1) * 2 <= n || c->factor_policy == 2) {
        // smallest supported block size whose block-tridiagonal pattern holds both operators
        const int lo = round_block(std::max(1, (bw + 2) / 2));
        const int hi = std::min(std::max(round_block(std::max(bw, 1)), lo), kMaxBlock);
        for (int cand = lo; cand <= hi && !bsz; cand *= 2) {
          bool ok = true;
          for (const feast_operator_t* o : ops) {
            if (dev_csr) ok = ok && !(((dcsr.stats[0].misfit_mask | dcsr.stats[1].misfit_mask) >> (log2_exact(cand) - 4)) & 1u);
            else if (o->kind == FEAST_STORAGE_CSR) ok = ok && csr_fits_blocktri(o, cand);
            else ok = ok && cand >= o->bsize && cand % o->bsize == 0;
          }
          if (ok) bsz = cand;
        }
        if (!bsz && round_block(std::max(bw, 1)) <= kMaxBlock) bsz = round_block(std::max(bw, 1));
      }
    }
  }
  c->have_pencil = false;
  c->have_contour = false;
  c->factored = false;
  c->mcap = 0;
  c->n = n;
  trace_mark(c, "set_pencil: storage choice");
  if (dev_csr) {
    double nrm;
    std::memcpy(&nrm, &dcsr.stats[0].norm1_bits, sizeof(double));
    c->norm_a1 = nrm;
  } else {
    c->norm_a1 = norm_one(a);
  }
  trace_mark(c, "set_pencil: norm_1(A)");
  if (bsz) {
    c->blocktri = true;
    c->b = bsz;
    c->L = (n + bsz - 1) / bsz;
    c->npad = c->L * bsz;
    // plain real copies [diag blocks | lower blocks] for the operator applies (bt_apply); the
    // interleaved (A, B) pairs of the factorisation are packed from them on the device
    const size_t nd = (size_t)c->L * bsz * bsz, nl = (size_t)(c->L > 1 ? c->L - 1 : 0) * bsz * bsz;
    c->A.ensure(nd + nl);
    c->Bm.ensure(nd + nl);
    if (dev_csr) {
      CK(csr_to_blocktri(n, bsz, c->L, dcsr.rp[0], dcsr.ci[0], dcsr.val[0], c->A.p, c->A.p + nd, false, c->stream));
      CK(csr_to_blocktri(n, bsz, c->L, dcsr.rp[1], dcsr.ci[1], dcsr.val[1], c->Bm.p, c->Bm.p + nd, true, c->stream));
    } else if (!s && a->kind == FEAST_STORAGE_BLOCKTRI && b->kind == FEAST_STORAGE_BLOCKTRI && a->bsize == bsz &&
               b->bsize == bsz && a->nblocks == c->L) {
      // already in this storage (e.g. a memory-mapped FEASTOP1 file, pencil_io.py): stream the
      // blocks up through the pinned stage, no host-side copy of the operator
      upload_chunked(c, c->A.p, a->diag, sizeof(double) * nd);
      upload_chunked(c, c->Bm.p, b->diag, sizeof(double) * nd);
      if (nl) {
        upload_chunked(c, c->A.p + nd, a->lower, sizeof(double) * nl);
        upload_chunked(c, c->Bm.p + nd, b->lower, sizeof(double) * nl);
      }
      trace_mark(c, "set_pencil: block upload");
    } else {
      std::vector<double> ad, al, bd, bl;
      to_blocktri(a, bsz, c->L, false, ad, al);
      to_blocktri(b, bsz, c->L, true, bd, bl);
      if (s) {
        std::vector<double> sd, sl;
        to_blocktri(s, bsz, c->L, false, sd, sl);
        c->Sop.ensure(nd + nl);
        CK(cudaMemcpyAsync(c->Sop.p, sd.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, c->stream));
        if (nl) CK(cudaMemcpyAsync(c->Sop.p + nd, sl.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, c->stream));
        sync(c);
      }
      trace_mark(c, "set_pencil: re-block A, B");
      CK(cudaMemcpyAsync(c->A.p, ad.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->Bm.p, bd.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, c->stream));
      if (nl) {
        CK(cudaMemcpyAsync(c->A.p + nd, al.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->Bm.p + nd, bl.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, c->stream));
      }
      sync(c);  // the host vectors die here
    }
    c->abdiag.ensure(nd);
    c->ablow.ensure(std::max<size_t>(nl, 1));
    CK(interleave_pairs(c->A.p, c->Bm.p, nd, c->abdiag.p, c->stream));
    if (nl) CK(interleave_pairs(c->A.p + nd, c->Bm.p + nd, nl, c->ablow.p, c->stream));
    if (bsz <= 32) {
      const size_t nb3 = (size_t)c->L * bsz * 3 * bsz;
      c->Aband.ensure(nb3);
      c->Bband.ensure(nb3);
      CK(band_rows(c->L, bsz, c->A.p, c->A.p + nd, c->Aband.p, c->stream));
      CK(band_rows(c->L, bsz, c->Bm.p, c->Bm.p + nd, c->Bband.p, c->stream));
    } else {
      c->Aband.release();
      c->Bband.release();
    }
    sync(c);
    c->csr.release();  // back to the stream-ordered pool (reused by the next set_pencil)
    trace_mark(c, "set_pencil: alloc + H2D");
  } else {
    c->blocktri = false;
    c->b = 0;
    c->L = 0;
    c->npad = n;
    c->A.ensure((size_t)n * n);
    c->Bm.ensure((size_t)n * n);
    if (a->kind == FEAST_STORAGE_DENSE) {
      CK(cudaMemcpyAsync(c->A.p, a->dense, sizeof(double) * n * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    } else {
      auto d = to_dense(a);
      CK(cudaMemcpyAsync(c->A.p, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice, c->stream));
      sync(c);
    }
    if (b->kind == FEAST_STORAGE_DENSE) {
      CK(cudaMemcpyAsync(c->Bm.p, b->dense, sizeof(double) * n * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    } else {
      auto d = to_dense(b);
      CK(cudaMemcpyAsync(c->Bm.p, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice, c->stream));
      sync(c);
    }
    if (s) {
      c->Sop.ensure((size_t)n * n);
      auto d = to_dense(s);
      CK(cudaMemcpyAsync(c->Sop.p, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice, c->stream));
      sync(c);
    }
    sync(c);
  }
  if (s) {  // the unperturbed A, kept for A0 + t S
    c->A0.ensure(c->A.n);
    CK(cudaMemcpyAsync(c->A0.p, c->A.p, sizeof(double) * c->A.n, cudaMemcpyDeviceToDevice, c->stream));
    sync(c);
  } else {
    c->A0.release();
    c->Sop.release();
  }
  c->have_pencil = true;
}

// A = A0 + t S on the device (add_scaled, operator.hpp:282-304), with the derived copies (the
// (A, B) pairs of the factorisation, the band rows) and ||A||_1 brought up to date
void perturb_pencil(feast_gpu_ctx* c, double t) {
  const size_t cnt = c->A.n;
  CK(axpby(c->A0.p, c->Sop.p, t, cnt, c->A.p, c->stream));
  if (c->blocktri) {
    const size_t nd = (size_t)c->L * c->b * c->b, nl = (size_t)(c->L > 1 ? c->L - 1 : 0) * c->b * c->b;
    CK(interleave_pairs(c->A.p, c->Bm.p, nd, c->abdiag.p, c->stream));
    if (nl) CK(interleave_pairs(c->A.p + nd, c->Bm.p + nd, nl, c->ablow.p, c->stream));
    if (c->b <= 32) CK(band_rows(c->L, c->b, c->A.p, c->A.p + nd, c->Aband.p, c->stream));
  }
  c->kfac.ensure(1);
  CK(operator_norm1(c->blocktri ? c->L : 0, c->blocktri ? c->b : c->n, c->A.p, c->kfac.p, c->stream));
  CK(cudaMemcpyAsync(&c->norm_a1, c->kfac.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  c->factored = false;
}

// ------------------------------- contour + factors ---------------------------
void build_contour(feast_gpu_ctx* c, double emin, double emax, int ne) {
  if (!(emin < emax)) fail(FEAST_EINPUT, "SearchInterval: lambda_min must be strictly below lambda_max");
  const double scale = std::max({1.0, std::fabs(emin), std::fabs(emax)});
  if (emax - emin < 1e-12 * scale) fail(FEAST_EINPUT, "build_contour: interval is degenerate at round-off scale");
  std::vector<double> x, w;
  gauss_legendre(ne, x, w);
  c->emin = emin;
  c->emax = emax;
  c->ne = ne;
  c->radius = 0.5 * (emax - emin);
  const double mid = 0.5 * (emin + emax);
  c->z.resize(ne);
  c->coeff.resize(ne);
  for (int e = 0; e < ne; ++e) {
    const double th = -(M_PI / 2.0) * (x[e] - 1.0);
    c->z[e] = make_double2(mid + c->radius * std::cos(th), c->radius * std::sin(th));
    const double f = 0.5 * w[e] * c->radius;  // coeff = 0.5 w r e^{i theta} (core.hpp:174-175)
    c->coeff[e] = make_double2(f * std::cos(th), f * std::sin(th));
  }
  // contiguous node blocks per rank, ascending e
  c->e0 = (int)((int64_t)ne * c->rank / c->nranks);
  c->e1 = (int)((int64_t)ne * (c->rank + 1) / c->nranks);
  const int own = c->owned();
  c->dz.ensure(std::max(own, 1));
  c->dcoeff.ensure(std::max(own, 1));
  if (own) {
    CK(cudaMemcpyAsync(c->dz.p, c->z.data() + c->e0, sizeof(double2) * own, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->dcoeff.p, c->coeff.data() + c->e0, sizeof(double2) * own, cudaMemcpyHostToDevice, c->stream));
  }
  c->have_contour = true;
  c->factored = false;
  c->mcap = 0;  // per-node workspaces depend on the owned node count
}

size_t factor_bytes_per_node(const feast_gpu_ctx* c) {
  if (c->blocktri) return sizeof(double2) * (size_t)(3 * c->L - 2) * c->b * c->b;
  return sizeof(double2) * (size_t)c->n * c->n;
}

// node batch for this context: forced (feast_gpu_set_node_batch), else all owned nodes if their
// factors plus their per-slot solve workspaces (W complex, T real; sized for m right-hand sides)
// fit 80% of the HBM left after the m-column vector blocks, else as many as do (at least one).
// Planned before the workspaces are sized (ensure_workspace) and again at each factorisation.
void plan_batch(feast_gpu_ctx* c, int m) {
  const int own = c->owned();
  if (c->batch_req > 0) {
    c->batch = std::min(c->batch_req, std::max(own, 1));
    return;
  }
  const size_t have = sizeof(double2) * (c->sinv.n + c->gfac.n + c->hfac.n + c->lu.n + c->W.n) +
                      sizeof(double) * (c->T.n + c->Y.n + c->Q.n + c->X.n + c->AQ.n + c->gw.n);  // already ours
  const size_t nv = (size_t)c->npad * m, mm = (size_t)m * m;
  const size_t fixed = m > 0 ? sizeof(double) * (5 * nv + std::max<size_t>(mm * 64, nv)) : 0;  // Y Q X AQ|BQ gw
  const size_t per = factor_bytes_per_node(c) + (m > 0 ? sizeof(double2) * nv + sizeof(double) * nv * (c->blocktri ? 1 : 2) : 0);
  // memory freed by earlier contexts stays in the pool: when it (and what this context already
  // holds) covers every node, skip cudaMemGetInfo (a driver query of ~1 ms on the end-to-end path)
  size_t fr = pool_spare(c->device);
  if (0.8 * (double)(fr + have) - (double)fixed < (double)own * (double)per) {
    size_t dev_free = 0, tot = 0;
    CK(cudaMemGetInfo(&dev_free, &tot));
    fr += dev_free;
  }
  const double budget = 0.8 * (double)(fr + have) - (double)fixed;
  const size_t avail = budget > 0.0 ? (size_t)budget : 0;
  c->batch = (size_t)own * per <= avail ? own : (int)std::max<size_t>(1, avail / per);
}

// SPIKE chunk count for the current pencil: requested (feast_gpu_set_spike), or automatic: the
// smallest power of two P <= 8 with owned nodes x P >= 8, i.e. the chunking that gives a rank
// with few nodes (8-GPU sharding: one node per GPU) as many independent chains as eight nodes.
// Measured on config 2 (tools/spike_sweep.py, profiles/r02_spike_sweep.log): with 8 nodes on one
// GPU the unpartitioned sweep already has 384 CTAs and its register-heavy CTAs cap residency at
// ~3 per SM, so P = 4 shortened the sweep only 12 % while its correction cost more; with one node
// per GPU the sweep has 48 CTAs and P = 8 is what fills the GPU. The rule depends on the node
// count only (not on M0, unknown at feast_gpu_prepare, nor on the node batch, so every memory plan
// factors alike). Always a power of two dividing L with at least 8 layers per chunk (b <= 32).
int spike_chunks(const feast_gpu_ctx* c) {
  if (!c->blocktri || c->b > 32 || c->inner_kind != 0) return 1;
  int P = c->spike_req;
  if (P == 0) {
    P = 1;
    while (P < 8 && (int64_t)std::max(c->owned(), 1) * P < 8) P *= 2;
  }
  while (P > 1 && (c->L % P != 0 || c->L / P < 8)) P /= 2;
  return std::max(P, 1);
}

// the SPIKE data of owned nodes [s0, s0 + cnt) (factor slots 0..cnt-1): spikes V, W by one complex
// sweep of the chunks, the reduced matrix and its LU, the correction operand (spike.cu)
void spike_factor(feast_gpu_ctx* c, int s0, int cnt) {
  const int P = c->spike, Lc = c->L / P, b = c->b, slots = c->wnodes();
  const int nr = 2 * (P - 1) * b, nblk = (nr + kDenseNb - 1) / kDenseNb;
  const int64_t ld = c->npad;
  c->spk.ensure((size_t)slots * ld * 2 * b);
  CK(spike_rhs(c->L, b, P, cnt, c->ablow.p, c->dz.p + s0, c->spk.p, ld, c->stream));
  BtSweepArgs sa{Lc, b, cnt * P, 2 * b, (int)ld, c->ablow.p, c->dz.p + s0, c->dcoeff.p + s0, c->sinv.p, c->gfac.p,
                 c->hfac.p, nullptr, nullptr, c->spk.p, 1, c->kmid};
  sa.chunks = P;
  CK(bt_sweep(sa, c->stream));
  c->rlu.ensure((size_t)slots * nr * nr);
  c->rdinv.ensure((size_t)slots * nblk * 2 * kDenseNb * kDenseNb);
  c->ripiv.ensure((size_t)slots * nr);
  c->rperm.ensure((size_t)slots * nr);
  CK(spike_reduced(c->L, b, P, cnt, c->spk.p, ld, c->rlu.p, c->stream));
  CK(zgetrf_batched(nr, cnt, c->rlu.p, (int64_t)nr * nr, c->ripiv.p, c->rperm.p, c->rdinv.p, c->fstatus.p, c->stream));
  c->sra.ensure((size_t)slots * ld * 4 * b);
  CK(spike_coef(b, cnt, c->spk.p, ld, c->dcoeff.p + s0, c->sra.p, c->stream));
}

// block-Thomas solves (b <= 32) of owned nodes [sn, sn + cnt) held in factor slots [slot, slot + cnt)
// for m right-hand sides: real mode (y -> T = Re(c x)) or complex mode (W in place), with the SPIKE
// reduced system and correction when the factors are chunked. w / t are the first node's blocks
// (ld npad, node stride npad m).
void bt_solve(feast_gpu_ctx* c, int sn, int slot, int cnt, int m, const double* y, double* t, double2* w,
              int complex_mode) {
  const int P = c->spike, Lc = c->L / P, b = c->b;
  const size_t bb = (size_t)b * b;
  const size_t cs0 = (size_t)slot * P;  // first chunk slot
  BtSweepArgs a{Lc, b, cnt * P, m, c->npad, c->ablow.p, c->dz.p + sn, c->dcoeff.p + sn, c->sinv.p + cs0 * Lc * bb,
                c->gfac.p + cs0 * (Lc > 1 ? Lc - 1 : 0) * bb, c->hfac.p + cs0 * (Lc > 1 ? Lc - 1 : 0) * bb, y, t, w,
                complex_mode, c->kmid};
  a.chunks = P;
  CK(bt_sweep(a, c->stream));
  if (P == 1) return;
  const int nr = 2 * (P - 1) * b, nblk = (nr + kDenseNb - 1) / kDenseNb;
  const int64_t ld = c->npad;
  const double2* rlu = c->rlu.p + (size_t)slot * nr * nr;
  c->rz.ensure((size_t)cnt * nr * m);
  c->rzs.ensure((size_t)cnt * nr * m);
  CK(spike_gather(c->L, b, P, cnt, w, ld, m, c->rz.p, c->stream));
  CK(zgetrs_batched(nr, cnt, m, rlu, (int64_t)nr * nr, c->rperm.p + (size_t)slot * nr,
                    c->rdinv.p + (size_t)slot * nblk * 2 * kDenseNb * kDenseNb, c->rz.p, nr, c->rzs.p, c->stream));
  if (!complex_mode) {  // T_c -= [Re cV | -Im cV | Re cW | -Im cW] [Re v; Im v; Re u; Im u]
    c->rzr.ensure((size_t)cnt * 4 * b * m * P);
    CK(spike_zops(b, P, cnt, c->rz.p, m, c->rzr.p, c->stream));
    const double* ra = c->sra.p + (size_t)slot * ld * 4 * b;
    for (int cc = 0; cc < P; ++cc)
      CK(dgemm_batched(false, Lc * b, m, 4 * b, -1.0, ra + (size_t)cc * Lc * b, (int)ld, ld * 4 * b,
                       c->rzr.p + (size_t)cc * 4 * b * m, 4 * b, (int64_t)P * 4 * b * m, 1.0, t + (size_t)cc * Lc * b,
                       (int)ld, ld * m, cnt, c->stream));
    return;
  }
  // complex: W_c -= V_c v_c + W_c u_{c-1}
  const double2 one = make_double2(1.0, 0.0), mone = make_double2(-1.0, 0.0);
  const double2* spk = c->spk.p + (size_t)slot * ld * 2 * b;
  for (int cc = 0; cc < P; ++cc) {
    double2* wc = w + (size_t)cc * Lc * b;
    const double2* sv = spk + (size_t)cc * Lc * b;
    if (cc <= P - 2)
      CK(zgemm_batched(Lc * b, m, b, mone, sv, (int)ld, ld * 2 * b, c->rz.p + (size_t)(2 * cc + 1) * b, nr,
                       (int64_t)nr * m, one, wc, (int)ld, ld * m, cnt, c->stream));
    if (cc >= 1)
      CK(zgemm_batched(Lc * b, m, b, mone, sv + ld * b, (int)ld, ld * 2 * b, c->rz.p + (size_t)(2 * cc - 2) * b, nr,
                       (int64_t)nr * m, one, wc, (int)ld, ld * m, cnt, c->stream));
  }
}

// factors of owned nodes [s0, s0 + cnt) into factor slots 0..cnt-1
void factor_range(feast_gpu_ctx* c, int s0, int cnt) {
  c->fstatus.ensure(1);
  CK(cudaMemsetAsync(c->fstatus.p, 0, sizeof(int), c->stream));
  if (c->blocktri) {
    const size_t bb = (size_t)c->b * c->b;
    const int slots = c->wnodes();
    c->sinv.ensure(slots * c->L * bb);
    c->gfac.ensure(std::max<size_t>(slots * (c->L - 1) * bb, 1));
    c->hfac.ensure(std::max<size_t>(slots * (c->L - 1) * bb, 1));
    if (c->b >= 128) c->fwork.ensure(bt_factor_work_elems(c->b, cnt));
    const int P = c->spike = spike_chunks(c);
    const int Lc = c->L / P;
    BtFactorArgs a{Lc, c->b, cnt * P, c->abdiag.p, c->ablow.p, c->dz.p + s0, c->sinv.p, c->gfac.p, c->hfac.p,
                   c->scratch.p, c->fstatus.p, c->fwork.p, c->kmid = bt_twist_layer(Lc, c->b, c->twist)};
    a.chunks = P;
    CK(bt_factor(a, c->stream));
    if (P > 1) spike_factor(c, s0, cnt);
    if (!c->streamed()) c->fwork.release();  // transient unless it is reused every pass
  } else {
    const int n = c->n, nb = kDenseNb, nblk = (n + nb - 1) / nb, slots = c->wnodes();
    c->lu.ensure((size_t)slots * n * n);
    c->ipiv.ensure((size_t)slots * n);
    c->perm.ensure((size_t)slots * n);
    c->dinv.ensure((size_t)slots * nblk * 2 * nb * nb);
    DenseFactorArgs a{n, cnt, c->A.p, c->Bm.p, c->dz.p + s0, c->lu.p, c->ipiv.p, c->perm.p, c->dinv.p, c->fstatus.p};
    a.la = LuLookahead{c->eigs, c->ev_lu_cols, c->ev_lu_panel};  // panels beside the trailing updates
    CK(dense_factor(a, c->stream));
  }
  int st = 0;
  CK(cudaMemcpyAsync(&st, c->fstatus.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (st) fail(FEAST_ENUMERICAL, c->blocktri ? "BlockThomas: block pivot is numerically singular"
                                             : "DenseLU: matrix is numerically singular");
  c->res0 = s0;
  c->rescnt = cnt;
}

void factor(feast_gpu_ctx* c) {
  if (!c->have_pencil) fail(FEAST_EINPUT, "feast_gpu: pencil not set");
  if (!c->have_contour) fail(FEAST_EINPUT, "feast_gpu: contour not prepared");
  if (c->inner_kind == 1) {  // IterativeSolver::prepare keeps only the shift (inner_solver.hpp:229-231)
    c->res0 = 0;
    c->rescnt = c->owned();
    c->factored = true;
    return;
  }
  const int own = c->owned();
  c->fstatus.ensure(1);
  c->res0 = -1;
  c->rescnt = 0;
  if (own == 0) {
    c->factored = true;
    return;
  }
  const int prev = c->wnodes();
  plan_batch(c, c->mcap);
  if (c->wnodes() != prev) {  // per-node workspaces follow the node slots
    const int m = c->mcap;
    c->mcap = 0;
    if (m > 0) ensure_workspace(c, m);
  }
  factor_range(c, 0, c->wnodes());
  c->factored = true;
}

// make owned node s resident (streamed mode), returns its factor slot
int resident_slot(feast_gpu_ctx* c, int s) {
  if (s >= c->res0 && s < c->res0 + c->rescnt) return s - c->res0;
  const int s0 = (s / c->wnodes()) * c->wnodes();
  factor_range(c, s0, std::min(c->wnodes(), c->owned() - s0));
  return s - s0;
}

// ------------------------------- passes --------------------------------------
// sum over ranks of a device block (in place on `st`); a no-op without a rank group
void allreduce_sum(feast_gpu_ctx* c, double* p, size_t count, cudaStream_t st) {
  if (c->comm) c->comm->allreduce(p, count, st);
}

// q = -sum_e Re(c_e (z_e B - A)^{-1} y) over ALL nodes (allreduce across ranks); y, q npad x m.
// ev_start / ev_solved (may be null) are recorded before the first solve and after the last one.
void bicg_solve(feast_gpu_ctx* c, int s0, int cnt, int m, const double* y, const double2* bc, int ldb, bool conj_z);

void contour_pass(feast_gpu_ctx* c, int m, const double* y, double* q, cudaEvent_t ev_start = nullptr,
                  cudaEvent_t ev_solved = nullptr) {
  join_aux(c);
  if (c->inner_kind == 1) {  // IterativeSolver: BiCGStab per (node, column), node batches that fit
    const int own = c->owned();
    const size_t nv = (size_t)c->npad * m;
    if (ev_start) CK(cudaEventRecord(ev_start, c->stream));
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t per = (sizeof(double2) * 7 + sizeof(double) * 6) * nv;  // BiCGStab vectors per node
    const int nb = std::max(1, std::min(own, (int)(0.5 * (double)(fr + c->bvec.n * sizeof(double2) +
                                                               c->breal.n * sizeof(double)) / per)));
    for (int s0 = 0; s0 < own; s0 += nb) {
      const int cnt = std::min(nb, own - s0);
      bicg_solve(c, s0, cnt, m, y, nullptr, 0, false);
      CK(bicg_terms(c->bvec.p, cnt, c->npad, m, c->npad, c->dcoeff.p + s0, q, s0 > 0, c->stream));
    }
    if (own == 0) CK(fill_zero(q, nv, c->stream));
    if (ev_solved) CK(cudaEventRecord(ev_solved, c->stream));
    allreduce_sum(c, q, nv, c->stream);
    return;
  }
  const int own = c->owned();
  const size_t nv = (size_t)c->npad * m;
  if (ev_start) CK(cudaEventRecord(ev_start, c->stream));
  if (own > 0) {
    // node batches in ascending order (one batch = every owned node unless streamed); the
    // reduction continues the same ascending-e sum across batches, so the result is
    // bit-identical to the resident path
    const int nbt = c->wnodes();
    for (int s0 = 0; s0 < own; s0 += nbt) {
      const int cnt = std::min(nbt, own - s0);
      if (c->res0 != s0 || c->rescnt != cnt) factor_range(c, s0, cnt);
      if (c->blocktri && c->b <= 32) {
        bt_solve(c, s0, 0, cnt, m, y, c->T.p, c->W.p, 0);
      } else if (c->blocktri) {
        BtSweepArgs a{c->L, c->b, cnt, m, c->npad, c->ablow.p, c->dz.p + s0, c->dcoeff.p + s0, c->sinv.p,
                      c->gfac.p, c->hfac.p, y, c->T.p, c->W.p, 0, c->kmid};
        CK(bt_sweep(a, c->stream));
      } else {
        DenseSolveArgs a{c->n, cnt, m, c->npad, c->lu.p, c->perm.p, c->dinv.p, c->dcoeff.p + s0, y, c->T.p,
                         c->W.p, 0};
        CK(dense_solve(a, c->stream));
      }
      if (ev_solved && s0 + cnt >= own) CK(cudaEventRecord(ev_solved, c->stream));
      CK(reduce_terms(c->T.p, cnt, (int64_t)nv, c->npad, m, c->npad, q, c->stream, s0 > 0));
    }
  } else {
    if (ev_solved) CK(cudaEventRecord(ev_solved, c->stream));
    CK(fill_zero(q, nv, c->stream));
  }
  allreduce_sum(c, q, nv, c->stream);
}

void apply_both(feast_gpu_ctx* c, const double* x, double* ya, double* yb, int m);

// BiCGStab (inner_solver.hpp:124-184) for owned nodes [s0, s0 + cnt), m right-hand sides each (y
// real, ld npad, or bc complex, ld ldb, shared by the nodes); solutions in c->bvec (X block,
// npad x cnt*m complex). conj_z: the ConjTranspose solves (inner_solver.hpp:129).
void bicg_solve(feast_gpu_ctx* c, int s0, int cnt, int m, const double* y, const double2* bc, int ldb, bool conj_z) {
  const int C = cnt * m;
  const size_t nv = (size_t)c->npad * C;
  c->bvec.ensure(7 * nv);
  c->breal.ensure(6 * nv);
  c->bcol.ensure(C);
  c->bflag.ensure(2);
  c->bz.ensure(cnt);
  std::vector<double2> zs(cnt);
  for (int e = 0; e < cnt; ++e) {
    zs[e] = c->z[c->e0 + s0 + e];
    if (conj_z) zs[e].y = -zs[e].y;
  }
  CK(cudaMemcpyAsync(c->bz.p, zs.data(), sizeof(double2) * cnt, cudaMemcpyHostToDevice, c->stream));
  BicgArgs a;
  a.n = c->npad;
  a.ld = c->npad;
  a.C = C;
  a.m = m;
  a.z = c->bz.p;
  double2* v = c->bvec.p;
  a.X = v;
  a.R = v + nv;
  a.R0 = v + 2 * nv;
  a.P = v + 3 * nv;
  a.V = v + 4 * nv;
  a.S = v + 5 * nv;
  a.T = v + 6 * nv;
  a.PR = c->breal.p;
  a.AR = a.PR + 2 * nv;
  a.BR = a.AR + 2 * nv;
  a.col = c->bcol.p;
  a.tol = c->inner_tol;
  a.max_iter = c->inner_max_iter > 0 ? c->inner_max_iter : std::max(1000, 20 * c->n);
  a.any_active = c->bflag.p;
  CK(cudaMemsetAsync(c->bflag.p, 0, 2 * sizeof(int), c->stream));
  CK(bicg_init(a, y, c->npad, bc, ldb, c->stream));
  int active = 0;
  CK(cudaMemcpyAsync(&active, c->bflag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  constexpr int kChunk = 8;  // iterations between host checks of the any-active flag
  while (active) {
    for (int k = 0; k < kChunk; ++k) {
      apply_both(c, a.PR, a.AR, a.BR, 2 * C);
      CK(bicg_a(a, c->stream));
      apply_both(c, a.PR, a.AR, a.BR, 2 * C);
      if (k == kChunk - 1) CK(cudaMemsetAsync(c->bflag.p, 0, sizeof(int), c->stream));
      CK(bicg_b(a, c->stream));
    }
    CK(cudaMemcpyAsync(&active, c->bflag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  }
  CK(bicg_check(a, c->bflag.p + 1, c->stream));
  int failed = 0;
  CK(cudaMemcpyAsync(&failed, c->bflag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (failed) fail(FEAST_ENUMERICAL, "BicgstabShiftSystem: inner solve did not reach tolerance");
}

// accumulate_subspace_hermitian (core.hpp:190-215) for the real symmetric pencils this path
// holds: (z B - A)^H = conj(z B - A), so the ConjTranspose solve is conj(G conj(Y)) and ONE
// complex-mode solve of the 2m columns [Yr | Yi] per node gives both (hermitian_terms). Input
// c->Y = [Yr | Yi] (npad x 2m real); output Q complex (npad x m) in c->AQ. Same node order,
// node batches and allreduce as contour_pass.
void contour_pass_hermitian(feast_gpu_ctx* c, int m) {
  join_aux(c);
  if (c->inner_kind == 1) fail(FEAST_EINPUT, "contour_pass_hermitian: needs the direct inner solver");
  const int own = c->owned();
  const int m2 = 2 * m;
  double2* qc = reinterpret_cast<double2*>(c->AQ.p);
  if (own > 0) {
    const int nbt = c->wnodes();
    for (int s0 = 0; s0 < own; s0 += nbt) {
      const int cnt = std::min(nbt, own - s0);
      if (c->res0 != s0 || c->rescnt != cnt) factor_range(c, s0, cnt);
      if (c->blocktri && bt_panel_rows(c->b) > 0) {  // real input, complex output (mode 2)
        BtSweepArgs a{c->L, c->b, cnt, m2, c->npad, c->ablow.p, c->dz.p + s0, c->dcoeff.p + s0, c->sinv.p,
                      c->gfac.p, c->hfac.p, c->Y.p, nullptr, c->W.p, 2, c->kmid};
        CK(bt_sweep(a, c->stream));
      } else {
        CK(real_to_complex_slots(c->Y.p, c->npad, m2, cnt, c->W.p, c->stream));
        if (c->blocktri) {
          bt_solve(c, s0, 0, cnt, m2, nullptr, nullptr, c->W.p, 1);
        } else {
          DenseSolveArgs a{c->n, cnt, m2, c->npad, c->lu.p, c->perm.p, c->dinv.p, c->dcoeff.p + s0, nullptr, c->T.p,
                           c->W.p, 1};
          CK(dense_solve(a, c->stream));
        }
      }
      CK(hermitian_terms(c->W.p, cnt, c->npad, c->npad, m, c->dcoeff.p + s0, qc, s0 > 0, c->stream));
    }
  } else {
    CK(fill_zero(c->AQ.p, 2 * (size_t)c->npad * m, c->stream));
  }
  allreduce_sum(c, c->AQ.p, 2 * (size_t)c->npad * m, c->stream);
}

// ------------------------------- row slabs -------------------------------------
// Row-distributed Rayleigh-Ritz: with R ranks, rank r owns a row slab of the
// N x M0 blocks (block-tridiagonal: whole layers [l0, l1); dense: an equal row range). It forms
// A Q and B Q on its slab only (the block-tridiagonal applies read one layer of Q on each side,
// the halo; dense applies read all of Q), the partial projections of its slab, and ONE allreduce
// of the 2 M0^2 values gives every rank [A_Q | B_Q]; the reduced eigensolve is replicated. The
// N x M0 blocks that the solves need in full (B Q for the look-ahead pass, Y = B X otherwise) are
// allgathered by slabs. The N-proportional Rayleigh-Ritz work (applies, projections, Q Phi) so
// divides by R.
struct Slab {
  int r0 = 0, r1 = 0;  // owned rows
  int h0 = 0, h1 = 0;  // rows of Q this rank keeps valid (owned + halo)
  int l0 = 0, l1 = -1; // owned layers (block-tridiagonal)
};

bool row_distributed(const feast_gpu_ctx* c) { return c->comm && c->nranks > 1 && c->row_dist; }

Slab slab_of(const feast_gpu_ctx* c, int rank) {
  Slab s;
  if (!row_distributed(c)) {
    s.r1 = s.h1 = c->npad;
    s.l1 = c->blocktri ? c->L : -1;
    return s;
  }
  if (c->blocktri) {
    s.l0 = (int)((int64_t)c->L * rank / c->nranks);
    s.l1 = (int)((int64_t)c->L * (rank + 1) / c->nranks);
    s.r0 = s.l0 * c->b;
    s.r1 = s.l1 * c->b;
    s.h0 = std::max(s.l0 - 1, 0) * c->b;
    s.h1 = std::min(s.l1 + 1, c->L) * c->b;
  } else {
    s.r0 = (int)((int64_t)c->npad * rank / c->nranks);
    s.r1 = (int)((int64_t)c->npad * (rank + 1) / c->nranks);
    s.h0 = 0;
    s.h1 = c->npad;
  }
  return s;
}

int slab_max_rows(const feast_gpu_ctx* c) {
  int mx = 0;
  for (int r = 0; r < c->nranks; ++r) {
    const Slab s = slab_of(c, r);
    mx = std::max(mx, s.r1 - s.r0);
  }
  return mx;
}

// rows [s.r0, s.r1) of y = Op x (x valid on [s.h0, s.h1))
void apply_op(feast_gpu_ctx* c, int which, const double* x, double* y, int m, const Slab& s) {
  if (s.r1 <= s.r0 || m <= 0) return;
  if (c->blocktri && c->b <= 32) {
    CK(band_apply(c->L, c->b, which ? c->Bband.p : c->Aband.p, nullptr, x, c->npad, y, nullptr, c->npad, m,
                  c->stream, s.l0, s.l1));
  } else if (c->blocktri) {
    const double* base = which ? c->Bm.p : c->A.p;
    CK(bt_apply(c->L, c->b, base, base + (size_t)c->L * c->b * c->b, x, c->npad, y, c->npad, m, c->stream, s.l0,
                s.l1));
  } else {
    CK(dgemm('N', 'N', s.r1 - s.r0, m, c->n, 1.0, (which ? c->Bm.p : c->A.p) + s.r0, c->n, x, c->npad, 0.0,
             y + s.r0, c->npad, c->gw.p, c->gw.n, c->stream));
  }
}
void apply_op(feast_gpu_ctx* c, int which, const double* x, double* y, int m) {
  Slab all;
  all.r1 = all.h1 = c->npad;
  all.l1 = c->blocktri ? c->L : -1;
  apply_op(c, which, x, y, m, all);
}

// y = B x on all rows (m columns)
cudaError_t apply_op_cols(feast_gpu_ctx* c, const double* x, double* y, int m) {
  apply_op(c, 1, x, y, m);
  return cudaSuccess;
}

// A x and B x on rows of s (one pass over x for small blocks)
void apply_both(feast_gpu_ctx* c, const double* x, double* ya, double* yb, int m, const Slab& s) {
  if (c->blocktri && c->b <= 32) {
    if (s.r1 > s.r0 && m > 0)
      CK(band_apply(c->L, c->b, c->Aband.p, c->Bband.p, x, c->npad, ya, yb, c->npad, m, c->stream, s.l0, s.l1));
    return;
  }
  apply_op(c, 0, x, ya, m, s);
  apply_op(c, 1, x, yb, m, s);
}
void apply_both(feast_gpu_ctx* c, const double* x, double* ya, double* yb, int m) {
  Slab all;
  all.r1 = all.h1 = c->npad;
  all.l1 = c->blocktri ? c->L : -1;
  apply_both(c, x, ya, yb, m, all);
}

// every rank's slab of M (npad x m) into every rank's M: pack, allgather, unpack
void allgather_rows(feast_gpu_ctx* c, double* M, int m) {
  if (!row_distributed(c) || m <= 0) return;
  const int sm = slab_max_rows(c);
  const size_t cnt = (size_t)sm * m;
  c->G.ensure(cnt * (c->nranks + 1));
  double* send = c->G.p;
  double* recv = send + cnt;
  const Slab me = slab_of(c, c->rank);
  const size_t ld = sizeof(double) * c->npad;
  if (me.r1 > me.r0)
    CK(cudaMemcpy2DAsync(send, sizeof(double) * sm, M + me.r0, ld, sizeof(double) * (me.r1 - me.r0), m,
                         cudaMemcpyDeviceToDevice, c->stream));
  c->comm->allgather(send, recv, cnt, c->stream);
  for (int r = 0; r < c->nranks; ++r) {
    const Slab o = slab_of(c, r);
    if (r == c->rank || o.r1 <= o.r0) continue;
    CK(cudaMemcpy2DAsync(M + o.r0, ld, recv + r * cnt, sizeof(double) * sm, sizeof(double) * (o.r1 - o.r0), m,
                         cudaMemcpyDeviceToDevice, c->stream));
  }
}

struct Reduced {
  std::vector<double> evals;
  int mo = 0;
  bool truncated = false;
  double kfactor = 0.0;  // cancellation factor of X = Q Phi (cancellation_factor, misc.cu)
  bool lookahead = false;  // c->X holds the look-ahead contour pass on B Q, admitted for use
};

// ---------------------------------------------------------------------------------------------
// Look-ahead contour pass. The FEAST filter is linear and Phi is real, so the next pass's
// subspace -sum_e Re(c_e (z_e B - A)^{-1} B X) with X = Q Phi equals
// (-sum_e Re(c_e (z_e B - A)^{-1} B Q)) Phi. The solves on B Q need only the projections, not the
// reduced eigensolve, so they run on the main stream WHILE the eigensolve runs on a
// high-priority stream (it is a chain of latency-bound few-CTA kernels, ~1 ms at m = 192, that
// leaves most SMs idle); afterwards one GEMM forms the next Q. In exact arithmetic the iteration
// is the reference's (core.hpp:356-388). In floating point each solved column carries its own
// relative rounding, which Phi recombines: the error grows by at most the cancellation factor
// K = max_i sum_j ||q_j||_B |Phi_ji| (1 when forming X cancels nothing; a few in the converged
// regime where Q is close to X diag(rho); 1e4-1e6 after the random start block of pass 0, ~50-100
// after pass 1). The look-ahead result is used only when K <= kLookaheadMaxK; otherwise the pass
// is redone in the reference order (X = Q Phi, Y = B X, solves on Y). It is not launched during
// pass 0 (K is always large there) nor after a pass whose K exceeded the bound. Measured
// (tools/lookahead_study.py, profiles/r02_lookahead_study.log): even admitting every pass (bound
// 1e6) the solves end with the same status and loop count as the reference order and eigenvalues
// within 5e-12 relative. Disabled for streamed node batches (the factors would be recomputed for
// a pass that may be discarded).
constexpr double kLookaheadMaxK = 1e3;  // default admission bound (feast_gpu_set_lookahead)

// [Aq | Bq] = Q^T [AQ | BQ] (rayleigh_ritz core.hpp:228-236) on the main stream; row-distributed:
// each rank projects its slab and one allreduce of the 2 m^2 partial sums completes it
void rr_project(feast_gpu_ctx* c, int m) {
  const int n = c->npad;
  // the one-GEMM projection needs BQ right after AQ and Bq right after Aq AT THIS m: the
  // buffers are sized for mcap columns, and m shrinks after a truncated pass (core.hpp:387)
  c->BQ.p = c->AQ.p + (size_t)n * m;
  c->Bq.p = c->Aq.p + (size_t)m * m;
  const Slab s = slab_of(c, c->rank);
  const int k = s.r1 - s.r0;
  apply_both(c, c->Q.p, c->AQ.p, c->BQ.p, m, s);
  const bool sym = m % 64 == 0;  // symmetric halves: upper tiles only (2/3 of the flops at m = 192)
  if (k == 0)
    CK(fill_zero(c->Aq.p, 2 * (size_t)m * m, c->stream));
  else if (sym)
    CK(dgemm_tn_sym2(m, k, c->Q.p + s.r0, n, c->AQ.p + s.r0, n, c->Aq.p, c->gw.p, c->gw.n, c->stream));
  else
    CK(dgemm('T', 'N', m, 2 * m, k, 1.0, c->Q.p + s.r0, n, c->AQ.p + s.r0, n, 0.0, c->Aq.p, m, c->gw.p, c->gw.n,
             c->stream));
  if (row_distributed(c)) c->comm->allreduce(c->Aq.p, 2 * (size_t)m * m, c->stream);
  if (sym) {
    CK(symmetrize_tiles(c->Aq.p, m, m, c->stream));
    CK(symmetrize_tiles(c->Bq.p, m, m, c->stream));
  } else {
    CK(symmetrize(c->Aq.p, m, m, c->stream));
    CK(symmetrize(c->Bq.p, m, m, c->stream));
  }
}

// the look-ahead pass solves on B Q, which a row-distributed step holds by slabs
void lookahead_input(feast_gpu_ctx* c, int m) { allgather_rows(c, c->BQ.p, m); }

// reduced_gevp (eigh.hpp:178-225) on device blocks Aq, Bq (m x m) on stream `st`: Phi (m x mo)
// -> c->Phi, eigenvalues + status + cancellation factor back to the host. The Cholesky path is
// enqueued by reduced_gevp_start; reduced_gevp_finish waits for it and runs the truncation
// fallback when the factorisation failed. (The main stream may run the look-ahead contour pass
// in between.)
// concurrent: the look-ahead contour pass will run beside the eigensolve. It is held back until
// the eigensolve reaches the tridiagonalisation (event c->ev_pre_eig): that kernel keeps the matrix
// in registers and needs a whole SM, which the solves' CTAs would otherwise occupy for their entire
// chains; the kernels after it take the routes that leave room on shared SMs (low_smem).
void reduced_gevp_start(feast_gpu_ctx* c, int m, cudaStream_t st, bool concurrent = false) {
  const size_t mm = (size_t)m * m;
  double* h = c->hpin;
  CK(cudaMemcpyAsync(c->Lm.p, c->Bq.p, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(c->status.p, 0, sizeof(int), st));
  CK(cholesky(m, c->Lm.p, 1e-13, c->status.p, c->Dv.p, st));
  // While the Cholesky factorisations succeed, the rest of the path is enqueued without waiting
  // for the pivot check: status and eigenvalues come back with ONE synchronisation. After a
  // failed one (the subspace is in the truncation regime, where it usually stays) the status is
  // read first (reduced_gevp_finish), so a failing pass does not pay a full eigensolve on a
  // partial factor.
  c->gevp_enqueued = !c->chol_failed_prev;
  if (c->gevp_enqueued) {
    // C = L^-1 A L^-T  via two lower solves and transposes (eigh.hpp:192-196)
    CK(cudaMemcpyAsync(c->Cm.p, c->Aq.p, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
    CK(trsm_lower(m, c->Lm.p, c->Dv.p, c->Cm.p, m, m, st));
    CK(transpose(c->Cm.p, m, m, m, c->Tm.p, m, st));
    CK(trsm_lower(m, c->Lm.p, c->Dv.p, c->Tm.p, m, m, st));
    CK(transpose(c->Tm.p, m, m, m, c->Cm.p, m, st));
    CK(symmetrize(c->Cm.p, m, m, st));
    // The look-ahead solves are released when the tridiagonalisation STARTS for m <= 192 (the
    // register-tile kernel occupies one SM for ~0.5 ms) and when it ENDS beyond (the 16-CTA cluster /
    // cooperative routes): with the solves running beside the cluster tridiagonalisation, full-size
    // config 3 (m = 300) returned results that differed from run to run in the 11th digit (6 distinct
    // eigenvalue sums in 10 solves; one in 10, bit-identical to the look-ahead-free order of kernels,
    // with the release behind it). Each kernel alone is bit-reproducible beside the other
    // (tools/contention_probe.py), so the cause is not pinned down; the later release costs the
    // overlap of a ~1.5 ms kernel with a 40 ms sweep.
    const bool release_early = m <= tri_tiles_max_dim();
    if (concurrent && release_early) CK(cudaEventRecord(c->ev_pre_eig, st));
    CK(sym_eig(c->eig, m, c->Cm.p, c->Ev.p, c->Phi.p, st, 0.0, concurrent,
               concurrent && !release_early ? c->ev_pre_eig : nullptr));
    CK(trsm_lower_t(m, c->Lm.p, c->Dv.p, c->Phi.p, m, m, st, concurrent));  // Phi = L^-T W
    CK(cancellation_factor(m, m, c->Bq.p, m, c->Phi.p, m, c->kfac.p, st));
    CK(cudaMemcpyAsync(h + 1, c->kfac.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h + 2, c->Ev.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  } else if (concurrent) {
    CK(cudaEventRecord(c->ev_pre_eig, st));
  }
  CK(cudaMemcpyAsync(h, c->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(c->ev_eig, st));
}

Reduced reduced_gevp_finish(feast_gpu_ctx* c, int m, cudaStream_t st) {
  Reduced r;
  const size_t mm = (size_t)m * m;
  double* h = c->hpin;
  CK(cudaEventSynchronize(c->ev_eig));
  int chol_status = 0;
  std::memcpy(&chol_status, h, sizeof(int));
  if (c->gevp_enqueued && chol_status == 0) {
    c->chol_failed_prev = false;
    r.evals.assign(h + 2, h + 2 + m);
    r.kfactor = h[1];
    r.mo = m;
    return r;
  }
  c->chol_failed_prev = chol_status != 0;
  if (chol_status == 0) {  // (the status was read first: finish the Cholesky path now)
    c->chol_failed_prev = false;
    c->gevp_enqueued = false;
    CK(cudaMemcpyAsync(c->Cm.p, c->Aq.p, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
    CK(trsm_lower(m, c->Lm.p, c->Dv.p, c->Cm.p, m, m, st));
    CK(transpose(c->Cm.p, m, m, m, c->Tm.p, m, st));
    CK(trsm_lower(m, c->Lm.p, c->Dv.p, c->Tm.p, m, m, st));
    CK(transpose(c->Tm.p, m, m, m, c->Cm.p, m, st));
    CK(symmetrize(c->Cm.p, m, m, st));
    CK(sym_eig(c->eig, m, c->Cm.p, c->Ev.p, c->Phi.p, st));
    CK(trsm_lower_t(m, c->Lm.p, c->Dv.p, c->Phi.p, m, m, st));
    CK(cancellation_factor(m, m, c->Bq.p, m, c->Phi.p, m, c->kfac.p, st));
    CK(cudaMemcpyAsync(h + 1, c->kfac.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h + 2, c->Ev.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(c->ev_eig, st));
    CK(cudaEventSynchronize(c->ev_eig));
    r.evals.assign(h + 2, h + 2 + m);
    r.kfactor = h[1];
    r.mo = m;
    return r;
  }
  // spectral truncation fallback (eigh.hpp:204-224)
  CK(cudaMemcpyAsync(c->Cm.p, c->Bq.p, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
  CK(symmetrize(c->Cm.p, m, m, st));
  // mass-matrix modes at or below the 1e-14 truncation floor are discarded below, so their
  // vectors are not computed (the near-null cluster of a filtered subspace is large)
  CK(sym_eig(c->eig, m, c->Cm.p, c->Ev.p, c->Vm.p, st, 1e-14));
  std::vector<double> d(m);
  CK(cudaMemcpyAsync(d.data(), c->Ev.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double dmax = d.back();
  if (!(dmax > 0.0)) fail(FEAST_EBREAKDOWN, "reduced_gevp: projected mass matrix has no positive modes");
  std::vector<int> keep;
  for (int i = 0; i < m; ++i)
    if (d[i] > 1e-14 * dmax) keep.push_back(i);
  if (keep.empty()) fail(FEAST_EBREAKDOWN, "reduced_gevp: projected mass matrix has no usable modes");
  const int k = (int)keep.size();
  CK(cudaMemcpyAsync(c->keep.p, keep.data(), sizeof(int) * k, cudaMemcpyHostToDevice, st));
  CK(scale_columns(c->Vm.p, m, c->keep.p, c->Ev.p, k, c->S.p, st));   // S = V_keep diag(d^-1/2)
  CK(dgemm('N', 'N', m, k, m, 1.0, c->Aq.p, m, c->S.p, m, 0.0, c->Tm.p, m, c->gw.p, c->gw.n, st));
  CK(dgemm('T', 'N', k, k, m, 1.0, c->S.p, m, c->Tm.p, m, 0.0, c->Cm.p, k, c->gw.p, c->gw.n, st));
  CK(symmetrize(c->Cm.p, k, k, st));
  CK(sym_eig(c->eig, k, c->Cm.p, c->Ev.p, c->Vm.p, st));
  CK(dgemm('N', 'N', m, k, k, 1.0, c->S.p, m, c->Vm.p, k, 0.0, c->Phi.p, m, c->gw.p, c->gw.n, st));
  CK(cancellation_factor(m, k, c->Bq.p, m, c->Phi.p, m, c->kfac.p, st));
  CK(cudaMemcpyAsync(h + 1, c->kfac.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h + 2, c->Ev.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(c->ev_eig, st));
  CK(cudaEventSynchronize(c->ev_eig));
  r.evals.assign(h + 2, h + 2 + k);
  r.kfactor = h[1];
  r.mo = k;
  r.truncated = true;
  return r;
}

// reduced_gevp on the main stream (the C-ABI's feast_gpu_reduced_gevp)
Reduced reduced_gevp(feast_gpu_ctx* c, int m) {
  reduced_gevp_start(c, m, c->stream);
  return reduced_gevp_finish(c, m, c->stream);
}

// rayleigh_ritz (core.hpp:228-240) on c->Q (m columns) with the reduced eigensolve on the
// high-priority stream. lookahead: the main stream also runs the look-ahead contour pass on B Q
// into c->X meanwhile (r.lookahead then says whether it is admitted). ev_* (may be null): RR
// start / eigensolve end / look-ahead contour start and solved (timing).
Reduced rayleigh_ritz_la(feast_gpu_ctx* c, int m, bool lookahead, cudaEvent_t ev_rr0 = nullptr,
                         cudaEvent_t ev_c0 = nullptr, cudaEvent_t ev_c1 = nullptr) {
  if (ev_rr0) CK(cudaEventRecord(ev_rr0, c->stream));
  rr_project(c, m);
  CK(cudaEventRecord(c->ev_proj, c->stream));
  CK(cudaStreamWaitEvent(c->eigs, c->ev_proj, 0));
  reduced_gevp_start(c, m, c->eigs, lookahead);
  if (lookahead) {
    lookahead_input(c, m);
    CK(cudaStreamWaitEvent(c->stream, c->ev_pre_eig, 0));
    contour_pass(c, m, c->BQ.p, c->X.p, ev_c0, ev_c1);
  }
  Reduced r = reduced_gevp_finish(c, m, c->eigs);
  r.lookahead = lookahead && r.kfactor <= c->la_kmax;
  c->lookahead_ok = r.kfactor <= c->la_kmax;
  CK(cudaStreamWaitEvent(c->stream, c->ev_eig, 0));  // Phi is read on the main stream from here on
  return r;
}

// X = Q Phi (the Ritz block; rayleigh_ritz's last step), all rows on every rank
void ritz_vectors(feast_gpu_ctx* c, int m, const Reduced& r) {
  const int n = c->npad;
  const Slab s = slab_of(c, c->rank);
  if (s.r1 > s.r0)
    CK(dgemm('N', 'N', s.r1 - s.r0, r.mo, m, 1.0, c->Q.p + s.r0, n, c->Phi.p, m, 0.0, c->X.p + s.r0, n, c->gw.p,
             c->gw.n, c->stream));
  allgather_rows(c, c->X.p, r.mo);
}

// rayleigh_ritz without look-ahead, X = Q Phi formed (the C-ABI's feast_gpu_rayleigh_ritz)
Reduced rayleigh_ritz(feast_gpu_ctx* c, int m) {
  Reduced r = rayleigh_ritz_la(c, m, false);
  ritz_vectors(c, m, r);
  return r;
}

// after a Rayleigh-Ritz step that continues the loop: with an admitted look-ahead pass the next
// Q = (look-ahead result) Phi (returns true: the next pass's contour solves are done); else the
// reference order's Y = B X with X = Q Phi over all retained Ritz vectors (core.hpp:387), and
// the next pass solves on Y (returns false)
bool next_subspace(feast_gpu_ctx* c, int m, const Reduced& r) {
  const int n = c->npad;
  const Slab s = slab_of(c, c->rank);  // row-distributed: only the rows the next projection reads
  if (r.lookahead) {
    CK(dgemm('N', 'N', s.h1 - s.h0, r.mo, m, 1.0, c->X.p + s.h0, n, c->Phi.p, m, 0.0, c->Q.p + s.h0, n, c->gw.p,
             c->gw.n, c->stream));
    return true;
  }
  if (s.h1 > s.h0)
    CK(dgemm('N', 'N', s.h1 - s.h0, r.mo, m, 1.0, c->Q.p + s.h0, n, c->Phi.p, m, 0.0, c->X.p + s.h0, n, c->gw.p,
             c->gw.n, c->stream));
  apply_op(c, 1, c->X.p, c->Y.p, r.mo, s);
  allgather_rows(c, c->Y.p, r.mo);
  return false;
}

void upload_block(feast_gpu_ctx* c, const double* host, int m, double* dev) {
  // rows [0, n) from host (ld n), zero padding rows [n, npad)
  if (c->npad != c->n) CK(fill_zero(dev, (size_t)c->npad * m, c->stream));
  CK(cudaMemcpy2DAsync(dev, sizeof(double) * c->npad, host, sizeof(double) * c->n, sizeof(double) * c->n, m,
                       cudaMemcpyHostToDevice, c->stream));
}
// Process-wide pinned staging buffer for large transfers: the DMA into page-locked memory runs
// at link speed and the copy into the caller's pageable block is spread over host threads
// (pageable cudaMemcpy measured 4 GB/s on the result blocks; pinning the caller's memory per
// call with cudaHostRegister was slower still). Grown on demand up to kPinnedStageMax and kept
// for reuse; larger transfers go through it in rounds (downloads) or take the pageable path
// (uploads), so a config-5-sized result does not leave gigabytes page-locked.
struct PinnedStage {
  std::mutex mu;
  double* p = nullptr;
  size_t n = 0;
  double* get(size_t count) {
    if (count * sizeof(double) > kPinnedStageMax) return nullptr;
    if (count > n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      if (cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(double) * count) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return nullptr;
      }
      n = count;
    }
    return p;
  }
};
PinnedStage& pinned_stage() {
  static PinnedStage* s = new PinnedStage();  // never destroyed: may be used until exit
  return *s;
}
// the stage for `count` doubles with its lock held in lk (nullptr: pinned memory unavailable)
double* pinned_stage_lock_get(size_t count, std::unique_lock<std::mutex>& lk) {
  PinnedStage& ps = pinned_stage();
  lk = std::unique_lock<std::mutex>(ps.mu);
  return ps.get(count);
}

void download_block(feast_gpu_ctx* c, const double* dev, int m, double* host) {
  const size_t cnt = (size_t)c->n * m;
  if (cnt * sizeof(double) >= (8u << 20)) {
    PinnedStage& ps = pinned_stage();
    std::lock_guard<std::mutex> lk(ps.mu);
    if (double* st = ps.get(cnt)) {
      CK(cudaMemcpy2DAsync(st, sizeof(double) * c->n, dev, sizeof(double) * c->npad, sizeof(double) * c->n, m,
                           cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      const size_t chunk = (cnt + 7) / 8;
      std::vector<std::thread> th;
      for (size_t off = 0; off < cnt; off += chunk)
        th.emplace_back([=] { std::memcpy(host + off, st + off, sizeof(double) * std::min(chunk, cnt - off)); });
      for (auto& t : th) t.join();
      return;
    }
  }
  CK(cudaMemcpy2DAsync(host, sizeof(double) * c->n, dev, sizeof(double) * c->npad, sizeof(double) * c->n, m,
                       cudaMemcpyDeviceToHost, c->stream));
}

// Several result blocks at once, pipelined: column chunks of ~4 MB are DMA'd into the pinned
// stage back to back, each followed by an event, and host threads copy chunk i into the
// caller's block as soon as its event fires, while the later chunks are still in flight.
struct Download {
  const double* dev;
  int m;
  double* host;
};
void download_blocks(feast_gpu_ctx* c, const std::vector<Download>& dl) {
  const size_t n = c->n;
  size_t total = 0;
  for (auto& d : dl) total += n * d.m;
  if (total * sizeof(double) < (8u << 20)) {
    for (auto& d : dl) download_block(c, d.dev, d.m, d.host);
    return;
  }
  const int per = std::max<int>(1, (int)((4u << 20) / (sizeof(double) * n)));  // columns per chunk
  const size_t chunk_max = n * per;
  const size_t round_max = std::max(chunk_max, std::min(total, kPinnedStageMax / sizeof(double)));
  std::unique_lock<std::mutex> lk;
  double* st = pinned_stage_lock_get(round_max, lk);
  if (!st) {
    lk.unlock();
    for (auto& d : dl) {
      CK(cudaMemcpy2DAsync(d.host, sizeof(double) * n, d.dev, sizeof(double) * c->npad, sizeof(double) * n, d.m,
                           cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
    return;
  }
  struct Chunk {
    const double* dev;
    double* host;
    int w;
  };
  std::vector<Chunk> all;
  for (auto& d : dl)
    for (int j = 0; j < d.m; j += per) all.push_back({d.dev + (size_t)c->npad * j, d.host + n * j, std::min(per, d.m - j)});
  // chunk events, per device (an event belongs to the device current at its creation); guarded
  // by the stage lock
  static std::vector<std::pair<int, std::vector<cudaEvent_t>>> dev_events;
  std::vector<cudaEvent_t>* evs = nullptr;
  for (auto& de : dev_events)
    if (de.first == c->device) evs = &de.second;
  if (!evs) {
    dev_events.emplace_back(c->device, std::vector<cudaEvent_t>());
    evs = &dev_events.back().second;
  }
  // rounds of chunks that fit the stage: DMA chunk i into the stage with an event behind it,
  // host threads copy chunk i out as soon as its event fires while later chunks are in flight
  for (size_t c0 = 0; c0 < all.size();) {
    size_t c1 = c0, used = 0;
    while (c1 < all.size() && used + n * all[c1].w <= round_max) used += n * all[c1++].w;
    std::vector<size_t> off(c1 - c0);
    size_t o = 0;
    for (size_t i = c0; i < c1; ++i) {
      if (evs->size() <= i - c0) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs->push_back(e);
      }
      off[i - c0] = o;
      CK(cudaMemcpy2DAsync(st + o, sizeof(double) * n, all[i].dev, sizeof(double) * c->npad, sizeof(double) * n,
                           all[i].w, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaEventRecord((*evs)[i - c0], c->stream));
      o += n * all[i].w;
    }
    const int cnt = (int)(c1 - c0);
    const int nt = std::min(cnt, (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency())));
    std::atomic<bool> bad{false};
    auto work = [&](int t) {
      for (int i = t; i < cnt; i += nt) {
        if (cudaEventSynchronize((*evs)[i]) != cudaSuccess) {
          bad = true;
          return;
        }
        std::memcpy(all[c0 + i].host, st + off[i], sizeof(double) * n * all[c0 + i].w);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    if (bad) CK(cudaStreamSynchronize(c->stream));  // raises the stream's error
    c0 = c1;
  }
}

// residual_norms (residual.hpp:29-68) of the first m columns of X (device, ld npad)
void residuals(feast_gpu_ctx* c, int m, const double* lam_host, const double* xdev, double* res,
               int32_t* absonly, double* maxres) {
  *maxres = 0.0;
  if (m == 0) return;
  DevBuf<double> lam, sums;
  lam.ensure(m);
  sums.ensure(3 * (size_t)m);
  CK(cudaMemcpyAsync(lam.p, lam_host, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  apply_both(c, xdev, c->AQ.p, c->BQ.p, m);
  CK(residual_sums(c->n, m, c->AQ.p, c->BQ.p, xdev, c->npad, lam.p, sums.p, c->stream, c->hermitian));
  std::vector<double> h(3 * (size_t)m);
  CK(cudaMemcpyAsync(h.data(), sums.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  lam.release();
  sums.release();
  const double eps = 2.220446049250313e-16;
  for (int j = 0; j < m; ++j) {
    const double num = h[3 * j], den = h[3 * j + 1], xn = h[3 * j + 2];
    const double floor = 4.0 * (c->hermitian ? c->nz : c->n) * eps * c->norm_a1 * xn;
    if (den <= std::max(1e-300, floor)) {
      res[j] = num;
      if (absonly) absonly[j] = 1;
    } else {
      res[j] = num / den;
      if (absonly) absonly[j] = 0;
    }
    *maxres = std::max(*maxres, res[j]);
  }
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Pair mode, degenerate eigenvalues: a complex eigenvalue of multiplicity s is a real one of
// multiplicity 2s, and one representative per real pair need not span the complex eigenspace.
// For each cluster of in-interval representatives (relative gap <= 1e-10) the 2s real Ritz
// vectors of the cluster are read as complex vectors and B-orthonormalised by modified
// Gram-Schmidt in the complex inner product, accepting a candidate only while it keeps half its
// B-norm (a J-partner of an accepted vector keeps none); the s accepted vectors replace the
// cluster's columns of c->Q (eigenvectors of the result, keep order). Clusters are rare (exact
// multiplicities); the small host computation touches only their columns.
void hermitian_clusters(feast_gpu_ctx* c, const std::vector<double>& lam, const std::vector<int>& keep,
                        const Reduced& rr) {
  const int k = (int)keep.size();
  std::vector<std::pair<int, int>> cl;  // [first, last] positions in keep
  for (int j = 0; j < k;) {
    int e = j;
    while (e + 1 < k && lam[e + 1] - lam[e] <= 1e-10 * std::max(1.0, std::fabs(lam[e]))) ++e;
    if (e > j) cl.emplace_back(j, e);
    j = e + 1;
  }
  if (cl.empty()) return;
  const size_t n2 = c->n, ld = c->npad;
  for (auto [j0, j1] : cl) {
    const int s = j1 - j0 + 1;
    const int r0 = keep[j0], r1 = std::min(keep[j1] + 1, rr.mo - 1);  // real Ritz columns r0 .. r1
    const int nc = r1 - r0 + 1;
    std::vector<double> x(n2 * nc), bx(n2 * nc);
    CK(apply_op_cols(c, c->X.p + ld * r0, c->AQ.p, nc));  // B x (AQ is free in finalize)
    CK(cudaMemcpy2DAsync(x.data(), sizeof(double) * n2, c->X.p + ld * r0, sizeof(double) * ld, sizeof(double) * n2, nc,
                         cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpy2DAsync(bx.data(), sizeof(double) * n2, c->AQ.p, sizeof(double) * ld, sizeof(double) * n2, nc,
                         cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    auto dot = [&](const double* a, const double* b) {  // a^H b over interleaved complex entries
      double re = 0.0, im = 0.0;
      for (size_t i = 0; i + 1 < n2; i += 2) {
        re += a[i] * b[i] + a[i + 1] * b[i + 1];
        im += a[i] * b[i + 1] - a[i + 1] * b[i];
      }
      return std::make_pair(re, im);
    };
    std::vector<int> acc;
    for (int q = 0; q < nc && (int)acc.size() < s; ++q) {
      double* u = x.data() + n2 * q;
      double* bu = bx.data() + n2 * q;
      for (int a : acc) {
        const double* v = x.data() + n2 * a;
        const double* bv = bx.data() + n2 * a;
        const auto al = dot(v, bu);  // <v, u>_B
        for (size_t i = 0; i + 1 < n2; i += 2) {
          const double ur = u[i] - (al.first * v[i] - al.second * v[i + 1]);
          const double ui = u[i + 1] - (al.first * v[i + 1] + al.second * v[i]);
          u[i] = ur;
          u[i + 1] = ui;
          const double br = bu[i] - (al.first * bv[i] - al.second * bv[i + 1]);
          const double bi = bu[i + 1] - (al.first * bv[i + 1] + al.second * bv[i]);
          bu[i] = br;
          bu[i + 1] = bi;
        }
      }
      const double nrm2 = dot(u, bu).first;
      if (!(nrm2 > 0.25)) continue;
      const double inv = 1.0 / std::sqrt(nrm2);
      for (size_t i = 0; i < n2; ++i) {
        u[i] *= inv;
        bu[i] *= inv;
      }
      acc.push_back(q);
    }
    for (int t = 0; t < (int)acc.size(); ++t)
      CK(cudaMemcpyAsync(c->Q.p + ld * (j0 + t), x.data() + n2 * acc[t], sizeof(double) * n2, cudaMemcpyHostToDevice,
                         c->stream));
    sync(c);
  }
}

// The FEAST loop (core.hpp:264-391), state resident on the device.
// y_dev: the initial block (y_cols columns) is already in c->Y (feast_gpu_sweep's warm start)
void feast_solve(feast_gpu_ctx* c, double emin, double emax, const feast_config_t* cfg,
                 const double* initial_y, int y_cols, feast_result_t* out, bool y_dev = false) {
  const auto t_start = std::chrono::steady_clock::now();
  trace_mark(c, nullptr);
  if (!c->have_pencil) fail(FEAST_EINPUT, "feast_gpu: pencil not set");
  if (!cfg || !out) fail(FEAST_EINPUT, "feast_gpu_solve: null argument");
  const int n = c->n;
  // Hermitian pencils (pair mode): the real loop on the doubled pencil with 2 m0 columns, read
  // through one representative per Ritz pair (set_pencil_hermitian)
  const bool pair = c->hermitian;
  const int step = pair ? 2 : 1;
  if (cfg->m0 < 1 || cfg->m0 > (pair ? c->nz : n)) fail(FEAST_EINPUT, "feast_solve: m0 must be in [1, n]");
  if (cfg->m0 * step > 1024) fail(FEAST_EINPUT, "feast_solve: m0 exceeds the supported reduced size");
  if (pair && y_dev) fail(FEAST_EINPUT, "run_sweep: sweeps are defined for real pencils");
  if (cfg->max_loops < 1) fail(FEAST_EINPUT, "feast_solve: max_loops must be positive");
  if (!(cfg->trace_tol > 0.0)) fail(FEAST_EINPUT, "feast_solve: trace_tol must be positive");
  if (cfg->threads < 1) fail(FEAST_EINPUT, "feast_solve: threads must be positive");
  if ((initial_y || y_dev) && (y_cols < 1 || y_cols > cfg->m0))
    fail(FEAST_EINPUT, "feast_solve: initial block shape mismatch");
  if (!(emin < emax)) fail(FEAST_EINPUT, "SearchInterval: lambda_min must be strictly below lambda_max");

  c->chol_failed_prev = false;
  const bool same_contour = c->have_contour && c->emin == emin && c->emax == emax && c->ne == cfg->n_e;
  if (!same_contour) build_contour(c, emin, emax, cfg->n_e);
  // max(trace_tol, residual_target^2) (core.hpp:296-297): 0 for direct solves, tol for BiCGStab
  const double inner = c->inner_kind == 1 ? c->inner_tol : 0.0;
  const double effective_tol = std::max(cfg->trace_tol, inner * inner);
  ensure_workspace(c, cfg->m0 * step);
  trace_mark(c, "solve: contour + workspaces");

  *out = feast_result_t{out->eigenvalues, out->eigenvectors, out->residuals, out->residual_absolute_only,
                        out->trace_history, out->in_interval_counts, out->subspace};
  int m = (initial_y || y_dev) ? y_cols : cfg->m0;
  if (y_dev) {
    trace_mark(c, "solve: initial block resident");
  } else {
    std::vector<double> y(initial_y ? (size_t)n * m : 0);
    if (initial_y) std::memcpy(y.data(), initial_y, sizeof(double) * y.size());
    if (initial_y) {
      upload_block(c, y.data(), m, c->Y.p);
      sync(c);
      trace_mark(c, "solve: initial block H2D");
    } else {
      // (pair mode: random_block<cplx>(n, m0) is the real stream random_block(2n, m0), interleaved)
      device_random_block(c, m, cfg->seed);  // overlaps the factorisation (side stream)
      trace_mark(c, "solve: initial block (device mt19937_64)");
    }
    if (pair) {  // [Y | J Y]: the complex block as the real columns of the doubled pencil
      join_aux(c);
      CK(rotate_pairs(c->Y.p, c->n, c->npad, m, c->Y.p + (size_t)c->npad * m, c->stream));
      m *= 2;
    }
  }
  if (!same_contour || !c->factored) c->factored = false;

  double prev_trace = 0.0;
  int prev_count = -1;
  std::vector<double> history;
  std::vector<int> counts;

  auto finalize = [&](int status, const Reduced& rr, int pass, int mq) {
    ritz_vectors(c, mq, rr);  // X = Q Phi (rayleigh_ritz, core.hpp:238)
    sync(c);
    out->status = status;
    out->loops_used = pass;
    std::vector<int> keep;
    for (int i = 0; i < rr.mo; i += step)
      if (emin <= rr.evals[i] && rr.evals[i] <= emax) keep.push_back(i);
    const int k = (int)keep.size();
    out->m = k;
    out->subspace_cols = pair ? (rr.mo + 1) / 2 : rr.mo;
    std::vector<double> lam(k);
    for (int j = 0; j < k; ++j) lam[j] = rr.evals[keep[j]];
    if (out->eigenvalues) std::memcpy(out->eigenvalues, lam.data(), sizeof(double) * k);
    // eigenvectors = X[:, keep] -> Q buffer (free at this point)
    if (k) {
      CK(cudaMemcpyAsync(c->keep.p, keep.data(), sizeof(int) * k, cudaMemcpyHostToDevice, c->stream));
      CK(gather_columns(c->X.p, c->npad, c->npad, c->keep.p, k, c->Q.p, c->npad, c->stream));
    }
    trace_mark(c, "finalize: gather");
    // (pinning the caller's blocks with cudaHostRegister for these copies measured slower:
    // 13.4 vs 10.2 ms for 41 MB at config 2, the registration costs more than it saves)
    if (pair) {
      if (k) hermitian_clusters(c, lam, keep, rr);  // complex-orthonormal degenerate eigenvectors
      // the subspace: one representative per Ritz pair, into the free AQ buffer
      std::vector<int> rep;
      for (int i = 0; i < rr.mo; i += 2) rep.push_back(i);
      CK(cudaMemcpyAsync(c->keep.p, rep.data(), sizeof(int) * rep.size(), cudaMemcpyHostToDevice, c->stream));
      CK(gather_columns(c->X.p, c->npad, c->npad, c->keep.p, (int)rep.size(), c->AQ.p, c->npad, c->stream));
    }
    std::vector<Download> dl;
    if (out->eigenvectors && k) dl.push_back({c->Q.p, k, out->eigenvectors});
    if (out->subspace) dl.push_back({pair ? c->AQ.p : c->X.p, out->subspace_cols, out->subspace});
    download_blocks(c, dl);
    trace_mark(c, "finalize: D2H eigenvectors + subspace");
    std::vector<double> res(k);
    std::vector<int32_t> ab(k);
    residuals(c, k, lam.data(), c->Q.p, res.data(), ab.data(), &out->max_residual);
    if (out->residuals && k) std::memcpy(out->residuals, res.data(), sizeof(double) * k);
    if (out->residual_absolute_only && k) std::memcpy(out->residual_absolute_only, ab.data(), sizeof(int32_t) * k);
    if (out->trace_history) std::memcpy(out->trace_history, history.data(), sizeof(double) * history.size());
    if (out->in_interval_counts) std::memcpy(out->in_interval_counts, counts.data(), sizeof(int) * counts.size());
    sync(c);
    trace_mark(c, "finalize: residuals");
    out->total_s = secs(t_start);
  };

  // the look-ahead contour pass overlaps each reduced eigensolve with the next pass's solves
  // (rayleigh_ritz_la); not with streamed factors (a discarded look-ahead would have refactored
  // every batch). low_memory keeps it and refactors before it, so results stay bit-identical to
  // the default (test_core.cpp:341-376)
  const bool la_allowed = c->lookahead && c->inner_kind == 0;  // (an inexact solve is not linear)
  c->lookahead_ok = true;
  bool have_q = false;  // this pass's Q is already formed (admitted look-ahead)
  for (int pass = 0; pass <= cfg->max_loops; ++pass) {
    // phase times from device events (FeastTimings, core.hpp:54-59): the only host
    // synchronisation per pass is the one the trace check needs (the Ritz values, in
    // reduced_gevp_finish); event set pass & 1 = {contour start, contour end, RR start}
    cudaEvent_t* pe = c->pev[pass & 1];
    if (!have_q) {
      if (cfg->low_memory) c->factored = false;
      if (!c->factored) {
        const auto t0 = std::chrono::steady_clock::now();
        factor(c);
        out->factorize_s += secs(t0);
        trace_mark(c, "solve: factor");
      }
      CK(cudaEventRecord(pe[0], c->stream));
      contour_pass(c, m, c->Y.p, c->Q.p);
      CK(cudaEventRecord(pe[1], c->stream));
      trace_mark(c, "solve: contour pass");
    }
    const bool la = la_allowed && pass >= 1 && (pass == 1 || c->lookahead_ok) && !c->streamed() &&
                    pass < cfg->max_loops;
    Reduced rr;
    try {
      cudaEvent_t* pn = c->pev[(pass + 1) & 1];
      CK(cudaEventRecord(pe[2], c->stream));
      rr_project(c, m);
      CK(cudaEventRecord(c->ev_proj, c->stream));
      CK(cudaStreamWaitEvent(c->eigs, c->ev_proj, 0));
      reduced_gevp_start(c, m, c->eigs, la);
      if (la) {
        lookahead_input(c, m);
        if (cfg->low_memory) {
          const auto t0 = std::chrono::steady_clock::now();
          c->factored = false;
          factor(c);
          out->factorize_s += secs(t0);
        }
        CK(cudaStreamWaitEvent(c->stream, c->ev_pre_eig, 0));
        CK(cudaEventRecord(pn[0], c->stream));
        contour_pass(c, m, c->BQ.p, c->X.p);
        CK(cudaEventRecord(pn[1], c->stream));
      }
      rr = reduced_gevp_finish(c, m, c->eigs);
      if (c->trace)
        std::fprintf(stderr, "[feast_gpu] pass %d: m=%d mo=%d truncated=%d K=%.3e lookahead=%d\n", pass, m, rr.mo,
                     (int)rr.truncated, rr.kfactor, (int)la);
      rr.lookahead = la && rr.kfactor <= c->la_kmax;
      c->lookahead_ok = rr.kfactor <= c->la_kmax;
      if (rr.lookahead) ++c->lookahead_count;
      CK(cudaStreamWaitEvent(c->stream, c->ev_eig, 0));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, pe[0], pe[1]));  // this pass's contour solves (complete)
      out->solve_s += 1e-3 * ms;
      CK(cudaEventElapsedTime(&ms, pe[2], c->ev_eig));
      out->reduce_s += 1e-3 * ms;
    } catch (const Failure& f) {
      if (f.code != FEAST_EBREAKDOWN) throw;
      CK(cudaStreamSynchronize(c->stream));
      out->status = FEAST_STATUS_BREAKDOWN;
      out->loops_used = pass;
      if (out->trace_history) std::memcpy(out->trace_history, history.data(), sizeof(double) * history.size());
      if (out->in_interval_counts) std::memcpy(out->in_interval_counts, counts.data(), sizeof(int) * counts.size());
      out->total_s = secs(t_start);
      return;
    }
    trace_mark(c, "solve: rayleigh-ritz");

    double tr = 0.0;
    int cnt = 0;
    for (int i = 0; i < rr.mo; i += step)  // (pair mode: one representative per Ritz pair)
      if (emin <= rr.evals[i] && rr.evals[i] <= emax) {
        tr += rr.evals[i];
        ++cnt;
      }
    history.push_back(tr);
    counts.push_back(cnt);

    if (cnt == cfg->m0) {
      finalize(FEAST_STATUS_SATURATED, rr, pass, m);
      return;
    }
    if (pass >= 1) {
      if (cnt == 0 && prev_count == 0) {
        finalize(FEAST_STATUS_NO_EIGENVALUES, rr, pass, m);
        return;
      }
      const double denom = std::max(std::fabs(tr), emax - emin);
      if (cnt == prev_count && std::fabs(tr - prev_trace) <= effective_tol * denom) {
        finalize(FEAST_STATUS_CONVERGED, rr, pass, m);
        return;
      }
    }
    if (pass == cfg->max_loops) {
      finalize(FEAST_STATUS_MAX_LOOPS, rr, pass, m);
      return;
    }
    prev_trace = tr;
    prev_count = cnt;
    have_q = next_subspace(c, m, rr);
    m = rr.mo;
  }
  fail(FEAST_EINTERNAL, "feast_solve: unreachable");
}

// run_sweep (run.cpp:63-125) with the operators and the warm-start block resident on the device:
// step k solves (A0 + steps[k] S, B) after A = A0 + t S is formed in place; a converged step's
// Ritz block (c->X, still on the device after finalize), topped up with seeded random columns when
// truncation shrank it (seed + 1000003 (k + 1)), times B is the next step's start block. A step
// that fails with NumericalError is reported (codes[k]) and the next one starts cold, as in the
// reference; other errors end the sweep.
void sweep(feast_gpu_ctx* c, const feast_operator_t* a0, const feast_operator_t* b, const feast_operator_t* s,
           const double* steps, int nsteps, double emin, double emax, const feast_config_t* cfg,
           feast_result_t* results, int* codes) {
  if (!a0 || !b || !s || !cfg || !results || !codes) fail(FEAST_EINPUT, "feast_gpu_sweep: null argument");
  if (nsteps < 1 || !steps) fail(FEAST_EINPUT, "run_sweep: no steps given");
  set_pencil(c, a0, b, s);
  bool have_warm = false;
  int warm_cols = 0;
  for (int k = 0; k < nsteps; ++k) {
    perturb_pencil(c, steps[k]);
    codes[k] = FEAST_OK;
    try {
      feast_solve(c, emin, emax, cfg, nullptr, have_warm ? warm_cols : 0, &results[k], have_warm);
    } catch (const Failure& f) {
      if (f.code != FEAST_ENUMERICAL) throw;
      codes[k] = FEAST_ENUMERICAL;
      c->err = f.what();
      have_warm = false;
      continue;
    }
    const feast_result_t& r = results[k];
    if (r.status == FEAST_STATUS_CONVERGED && r.subspace_cols > 0) {
      const int cols = r.subspace_cols, m0 = cfg->m0;
      if (cols < m0) {  // X (npad x m0 buffer) gets the seeded columns after the Ritz block
        if (c->npad != c->n) CK(fill_zero(c->X.p + (size_t)c->npad * cols, (size_t)c->npad * (m0 - cols), c->stream));
        CK(random_block_device(cfg->seed + 1000003ull * (uint64_t)(k + 1), c->n, m0 - cols,
                               c->X.p + (size_t)c->npad * cols, c->npad, c->stream));
      }
      apply_op(c, 1, c->X.p, c->Y.p, m0);  // warm = B * block
      have_warm = true;
      warm_cols = m0;
    } else {
      have_warm = false;
    }
  }
  sync(c);
}

template <typename F>
int guarded(feast_gpu_ctx* c, F&& f) {
  AllocStream as(c ? c->stream : nullptr);
  try {
    if (c) CK(cudaSetDevice(c->device));
    f();
    return FEAST_OK;
  } catch (const Failure& e) {
    if (c) c->err = e.what();
    if (c && c->comm) c->comm->abort();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    if (c && c->comm) c->comm->abort();
    return FEAST_EINTERNAL;
  }
}

}  // namespace

// =============================================================================
// C-ABI
// =============================================================================
extern "C" {

int feast_gpu_abi_version(void) { return FEAST_GPU_ABI_VERSION; }

int feast_gpu_create(int device, void* stream, feast_gpu_ctx** out) {
  if (!out) return FEAST_EINPUT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FEAST_ECUDA;
  if (device < 0 || device >= ndev) return FEAST_EINPUT;
  auto* c = new feast_gpu_ctx();
  c->device = device;
  {
    cudaMemPool_t pool;
    if (cudaSetDevice(device) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (const char* t = std::getenv("FEAST_TRACE")) c->trace = std::atoi(t);
  const int rc = guarded(c, [&] {
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->eigs, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&c->ev_proj, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_pre_eig, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_lu_cols, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_lu_panel, cudaEventDisableTiming));
    CK(cudaEventCreate(&c->ev_eig));
    for (auto& pe : c->pev)
      for (auto& e : pe) CK(cudaEventCreate(&e));
  });
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return FEAST_OK;
}

void feast_gpu_destroy(feast_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->aux) cudaStreamSynchronize(c->aux);
  if (c->eigs) cudaStreamSynchronize(c->eigs);
  cudaStreamSynchronize(c->stream);
  AllocStream as(c->stream);
  for (DevBuf<double>* d : {&c->A, &c->Bm, &c->Y, &c->Q, &c->X, &c->AQ, &c->BQ, &c->T, &c->gw, &c->Aq, &c->Bq,
                            &c->Cm, &c->Lm, &c->Phi, &c->Ev, &c->Vm, &c->S, &c->Tm, &c->Dv, &c->Aband, &c->Bband, &c->csr, &c->G, &c->breal, &c->A0, &c->Sop, &c->sra, &c->rzr})
    d->release();
  c->csrstats.release();  // every buffer, before the stream goes (the destructor would free on a dead stream)
  c->kfac.release();
  for (DevBuf<double2>* d : {&c->abdiag, &c->ablow, &c->dz, &c->dcoeff, &c->sinv, &c->gfac, &c->hfac, &c->lu, &c->dinv,
                             &c->scratch, &c->W, &c->fwork})
    d->release();
  for (DevBuf<int>* d : {&c->ipiv, &c->perm, &c->status, &c->fstatus, &c->keep, &c->bflag}) d->release();
  c->bvec.release();
  c->bz.release();
  c->bcol.release();
  for (DevBuf<double2>* d : {&c->spk, &c->rlu, &c->rdinv, &c->rz, &c->rzs}) d->release();
  c->ripiv.release();
  c->rperm.release();
  cudaStreamSynchronize(c->stream);  // the frees above are stream-ordered
  if (c->eig) eig_destroy(c->eig);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& pe : c->pev)
    for (auto& e : pe)
      if (e) cudaEventDestroy(e);
  c->comm.reset();
  if (c->eigs) {
    cudaStreamSynchronize(c->eigs);
    cudaStreamDestroy(c->eigs);
  }
  if (c->ev_proj) cudaEventDestroy(c->ev_proj);
  if (c->ev_pre_eig) cudaEventDestroy(c->ev_pre_eig);
  if (c->ev_lu_cols) cudaEventDestroy(c->ev_lu_cols);
  if (c->ev_lu_panel) cudaEventDestroy(c->ev_lu_panel);
  if (c->ev_eig) cudaEventDestroy(c->ev_eig);
  pinned_small_release(c->hpin, c->hpin_n);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->y_ready) cudaEventDestroy(c->y_ready);
  delete c;
}

const char* feast_gpu_last_error(const feast_gpu_ctx* c) { return c ? c->err.c_str() : "null context"; }

int feast_gpu_nccl_unique_id(void* id_out) {
  NcclApi& api = nccl();
  if (!api.getUniqueId) return FEAST_ENCCL;
  return api.getUniqueId(id_out) == 0 ? FEAST_OK : FEAST_ENCCL;
}

int feast_gpu_set_comm(feast_gpu_ctx* c, const void* uid, int rank, int nranks) {
  return guarded(c, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(FEAST_EINPUT, "set_comm: bad rank/nranks");
    c->comm.reset();
    c->rank = rank;
    c->nranks = nranks;
    c->have_contour = false;
    c->factored = false;
    c->mcap = 0;
    // a communicator whenever an id is given: with nranks = 1 the NCCL path runs on one GPU
    if (uid && (nranks > 1 || std::any_of((const char*)uid, (const char*)uid + 128, [](char x) { return x != 0; }))) {
      NcclApi& api = nccl();
      auto init = api.h ? (nccl_init_fn)dlsym(api.h, "ncclCommInitRank") : nullptr;
      if (!init) fail(FEAST_ENCCL, "NCCL not available");
      NcclUid id;
      std::memcpy(id.internal, uid, 128);
      auto nc = std::make_unique<NcclComm>();
      const int r = init(&nc->comm, nranks, id, rank);
      if (r != 0) fail(FEAST_ENCCL, "ncclCommInitRank failed");
      c->comm = std::move(nc);
    } else if (nranks > 1) {
      fail(FEAST_EINPUT, "set_comm: an NCCL unique id is required for nranks > 1");
    }
  });
}

int feast_gpu_group_create(int nranks, feast_gpu_group** out) {
  if (!out || nranks < 1) return FEAST_EINPUT;
  *out = new feast_gpu_group();
  (*out)->nranks = nranks;
  return FEAST_OK;
}

void feast_gpu_group_destroy(feast_gpu_group* g) {
  if (!g) return;
  if (g->stage) cudaFree(g->stage);
  delete g;
}

int feast_gpu_set_group(feast_gpu_ctx* c, feast_gpu_group* g, int rank) {
  return guarded(c, [&] {
    if (!g || rank < 0 || rank >= g->nranks) fail(FEAST_EINPUT, "set_group: bad group/rank");
    c->comm = std::make_unique<LocalComm>(g, rank);
    c->rank = rank;
    c->nranks = g->nranks;
    c->have_contour = false;
    c->factored = false;
    c->mcap = 0;
  });
}

int feast_gpu_set_pencil(feast_gpu_ctx* c, const feast_operator_t* a, const feast_operator_t* b) {
  return guarded(c, [&] { set_pencil(c, a, b); });
}

int feast_gpu_prepare(feast_gpu_ctx* c, double emin, double emax, int n_e) {
  return guarded(c, [&] {
    if (!c->have_pencil) fail(FEAST_EINPUT, "feast_gpu: pencil not set");
    build_contour(c, emin, emax, n_e);
    factor(c);
  });
}

int feast_gpu_set_node_batch(feast_gpu_ctx* c, int nodes) {
  return guarded(c, [&] {
    if (nodes < 0) fail(FEAST_EINPUT, "set_node_batch: negative batch");
    c->batch_req = nodes;
    c->factored = false;  // re-plan at the next factorisation
  });
}

int feast_gpu_set_twist(feast_gpu_ctx* c, int enable) {
  return guarded(c, [&] {
    c->twist = enable != 0;
    c->factored = false;  // the factors' layout follows the recursion
  });
}

int feast_gpu_random_block(feast_gpu_ctx* c, int n, int m, uint64_t seed, double* out) {
  return guarded(c, [&] {
    if (n < 1 || m < 1 || !out) fail(FEAST_EINPUT, "random_block: bad shape");
    DevBuf<double> d;
    d.ensure((size_t)n * m);
    CK(random_block_device(seed, n, m, d.p, n, c->stream));
    CK(cudaMemcpyAsync(out, d.p, sizeof(double) * n * (size_t)m, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int feast_gpu_storage(const feast_gpu_ctx* c, int* b, int* layers, int* twist) {
  if (!c || !c->have_pencil) return FEAST_EINPUT;
  if (b) *b = c->blocktri ? c->b : 0;
  if (layers) *layers = c->blocktri ? c->L : 0;
  if (twist) *twist = c->blocktri ? c->kmid : -1;
  return FEAST_OK;
}

int feast_gpu_contour(const feast_gpu_ctx* c, double* z, double* coeff) {
  if (!c || !c->have_contour) return FEAST_EINPUT;
  for (int e = 0; e < c->ne; ++e) {
    if (z) { z[2 * e] = c->z[e].x; z[2 * e + 1] = c->z[e].y; }
    if (coeff) { coeff[2 * e] = c->coeff[e].x; coeff[2 * e + 1] = c->coeff[e].y; }
  }
  return FEAST_OK;
}

int feast_gpu_solve_shift(feast_gpu_ctx* c, int e, double* rhs, int m, int mode) {
  return guarded(c, [&] {
    if (!c->factored) fail(FEAST_EINPUT, "feast_gpu: factors not prepared");
    if (e < c->e0 || e >= c->e1) fail(FEAST_EINPUT, "solve_shift: node not owned by this rank");
    if (m < 1) fail(FEAST_EINPUT, "solve_shift: no right-hand sides");
    // panel-layout factors (b >= 128): the sweep takes real right-hand sides, so the complex
    // ones go through as 2m real columns [Re | Im] and are recombined afterwards
    if (c->inner_kind == 1) {  // BicgstabShiftSystem::solve_in_place (inner_solver.hpp:124-184)
      ensure_workspace(c, m);
      DevBuf<double2> b;
      b.ensure((size_t)c->npad * m);
      CK(cudaMemsetAsync(b.p, 0, sizeof(double2) * c->npad * m, c->stream));
      CK(cudaMemcpy2DAsync(b.p, sizeof(double2) * c->npad, rhs, sizeof(double2) * c->n, sizeof(double2) * c->n, m,
                           cudaMemcpyHostToDevice, c->stream));
      bicg_solve(c, e - c->e0, 1, m, nullptr, b.p, c->npad, mode != 0);
      CK(cudaMemcpy2DAsync(rhs, sizeof(double2) * c->n, c->bvec.p, sizeof(double2) * c->npad, sizeof(double2) * c->n,
                           m, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      return;
    }
    const bool split = c->blocktri && bt_panel_rows(c->b) > 0;
    ensure_workspace(c, split ? 2 * m : m);
    const int sn = e - c->e0;                 // owned node index (shift, coefficient)
    const int s = resident_slot(c, sn);       // its factor / workspace slot
    const size_t nv = (size_t)c->npad * m;
    double2* w = c->W.p + s * (split ? 2 : 1) * nv;
    CK(cudaMemsetAsync(w, 0, sizeof(double2) * nv, c->stream));
    CK(cudaMemcpy2DAsync(w, sizeof(double2) * c->npad, rhs, sizeof(double2) * c->n, sizeof(double2) * c->n, m,
                         cudaMemcpyHostToDevice, c->stream));
    // (zB - A)^H = conj(zB - A) for real symmetric A, B: solve at conj by conjugating in/out
    if (mode) CK(conj_inplace(w, nv, c->stream));
    if (c->blocktri && !split) {
      bt_solve(c, sn, s, 1, m, nullptr, nullptr, w, 1);
    } else if (c->blocktri) {
      const size_t bb = (size_t)c->b * c->b;
      if (split) CK(split_complex(w, c->AQ.p, c->npad, c->npad, m, c->stream));
      BtSweepArgs a{c->L, c->b, 1, split ? 2 * m : m, c->npad, c->ablow.p, c->dz.p + sn, c->dcoeff.p + sn,
                    c->sinv.p + s * c->L * bb, c->gfac.p + s * (c->L - 1) * bb,
                    c->hfac.p + s * (c->L - 1) * bb, split ? c->AQ.p : nullptr, nullptr, w, split ? 2 : 1,
                    c->kmid};
      CK(bt_sweep(a, c->stream));
      if (split) CK(merge_complex(w, c->npad, c->npad, m, c->stream));
    } else {
      const int n = c->n, nb = kDenseNb, nblk = (n + nb - 1) / nb;
      DenseSolveArgs a{n, 1, m, c->npad, c->lu.p + (size_t)s * n * n, c->perm.p + (size_t)s * n,
                       c->dinv.p + (size_t)s * nblk * 2 * nb * nb, c->dcoeff.p + sn, nullptr, c->T.p, w, 1};
      CK(dense_solve(a, c->stream));
    }
    if (mode) CK(conj_inplace(w, nv, c->stream));
    CK(cudaMemcpy2DAsync(rhs, sizeof(double2) * c->n, w, sizeof(double2) * c->npad, sizeof(double2) * c->n, m,
                         cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int feast_gpu_contour_pass(feast_gpu_ctx* c, const double* y, int m, double* q) {
  return guarded(c, [&] {
    if (!c->factored) fail(FEAST_EINPUT, "feast_gpu: factors not prepared");
    ensure_workspace(c, m);
    upload_block(c, y, m, c->Y.p);
    contour_pass(c, m, c->Y.p, c->Q.p);
    download_block(c, c->Q.p, m, q);
    sync(c);
  });
}

int feast_gpu_contour_pass_hermitian(feast_gpu_ctx* c, const double* y, int m, double* q) {
  return guarded(c, [&] {
    if (!c->factored) fail(FEAST_EINPUT, "feast_gpu: factors not prepared");
    if (m < 1) fail(FEAST_EINPUT, "contour_pass_hermitian: no columns");
    ensure_workspace(c, 2 * m);
    const int n = c->n;
    std::vector<double> ri((size_t)n * 2 * m);  // [Re Y | Im Y]
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < n; ++i) {
        const size_t k = (size_t)i + (size_t)j * n;
        ri[k] = y[2 * k];
        ri[k + (size_t)n * m] = y[2 * k + 1];
      }
    upload_block(c, ri.data(), 2 * m, c->Y.p);
    contour_pass_hermitian(c, m);
    CK(cudaMemcpy2DAsync(q, sizeof(double2) * n, c->AQ.p, sizeof(double2) * c->npad, sizeof(double2) * n, m,
                         cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int feast_gpu_rayleigh_ritz(feast_gpu_ctx* c, const double* q, int m, double* eigenvalues, double* x, int* m_out,
                            int* truncated) {
  return guarded(c, [&] {
    if (!c->have_pencil) fail(FEAST_EINPUT, "feast_gpu: pencil not set");
    if (m < 1 || m > 1024) fail(FEAST_EINPUT, "rayleigh_ritz: bad block width");
    ensure_workspace(c, m);
    upload_block(c, q, m, c->Q.p);
    Reduced r = rayleigh_ritz(c, m);
    if (eigenvalues) std::memcpy(eigenvalues, r.evals.data(), sizeof(double) * r.mo);
    if (x) download_block(c, c->X.p, r.mo, x);
    sync(c);
    if (m_out) *m_out = r.mo;
    if (truncated) *truncated = r.truncated;
  });
}

int feast_gpu_reduced_gevp(feast_gpu_ctx* c, int m, const double* a_q, const double* b_q, double* eigenvalues,
                           double* phi, int* m_out, int* truncated) {
  return guarded(c, [&] {
    if (m < 1 || m > 1024) fail(FEAST_EINPUT, "reduced_gevp: blocks must be square with equal size");
    if (c->mcap < m) {
      const size_t mm = (size_t)m * m;
      ensure_reduced(c, m);
      c->gw.ensure(mm * 64);
      ensure_eig(c, m);
    }
    c->status.ensure(1);
    CK(cudaMemcpyAsync(c->Aq.p, a_q, sizeof(double) * m * m, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->Bq.p, b_q, sizeof(double) * m * m, cudaMemcpyHostToDevice, c->stream));
    Reduced r = reduced_gevp(c, m);
    if (eigenvalues) std::memcpy(eigenvalues, r.evals.data(), sizeof(double) * r.mo);
    if (phi) CK(cudaMemcpyAsync(phi, c->Phi.p, sizeof(double) * m * r.mo, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (m_out) *m_out = r.mo;
    if (truncated) *truncated = r.truncated;
  });
}

int feast_gpu_residuals(feast_gpu_ctx* c, int m, const double* lambdas, const double* x, double* res,
                        int32_t* absonly, double* maxres) {
  return guarded(c, [&] {
    if (!c->have_pencil) fail(FEAST_EINPUT, "feast_gpu: pencil not set");
    ensure_workspace(c, std::max(m, 1));
    upload_block(c, x, m, c->X.p);
    double mx = 0.0;
    std::vector<double> r(m);
    std::vector<int32_t> ab(m);
    residuals(c, m, lambdas, c->X.p, r.data(), ab.data(), &mx);
    if (res) std::memcpy(res, r.data(), sizeof(double) * m);
    if (absonly) std::memcpy(absonly, ab.data(), sizeof(int32_t) * m);
    if (maxres) *maxres = mx;
  });
}

int feast_gpu_solve(feast_gpu_ctx* c, double emin, double emax, const feast_config_t* config,
                    const double* initial_y, int y_cols, feast_result_t* result) {
  return guarded(c, [&] {
    if (c->hermitian) fail(FEAST_EINPUT, "feast_gpu_solve: the pencil is Hermitian (feast_gpu_solve_hermitian)");
    feast_solve(c, emin, emax, config, initial_y, y_cols, result);
  });
}

int feast_gpu_bench_init(feast_gpu_ctx* c, int m0, uint64_t seed) {
  return guarded(c, [&] {
    if (!c->factored) fail(FEAST_EINPUT, "feast_gpu: factors not prepared");
    ensure_workspace(c, m0);
    device_random_block(c, m0, seed);
    join_aux(c);
    sync(c);
    c->bench_m = m0;
    c->bench_have_q = false;
    c->lookahead_ok = true;
  });
}

int feast_gpu_bench_passes(feast_gpu_ctx* c, int passes, size_t flush_bytes, double* total_ms,
                           double* phase_ms) {
  return guarded(c, [&] {
    if (!c->factored || c->bench_m < 1) fail(FEAST_EINPUT, "bench: call feast_gpu_bench_init first");
    double ph[4] = {0, 0, 0, 0};
    DevBuf<char> flush;
    if (flush_bytes) {  // L2 flushed once before the region; inside, the passes run back to back
      flush.ensure(flush_bytes);
      CK(cudaMemsetAsync(flush.p, 0x5a, flush_bytes, c->stream));
    }
    const bool la_allowed = c->lookahead && !c->streamed() && c->inner_kind == 0;
    int m = c->bench_m;
    bool have_q = c->bench_have_q;
    float ms = 0.f;
    CK(cudaEventRecord(c->ev[0], c->stream));
    for (int p = 0; p < passes; ++p) {
      cudaEvent_t* pe = c->pev[(c->bench_pass + p) & 1];  // (the ring continues across calls)
      cudaEvent_t* pn = c->pev[(c->bench_pass + p + 1) & 1];
      if (!have_q) {
        CK(cudaEventRecord(pe[0], c->stream));
        contour_pass(c, m, c->Y.p, c->Q.p, nullptr, pe[3]);
        CK(cudaEventRecord(pe[1], c->stream));
      }
      const bool la = la_allowed && c->lookahead_ok;
      CK(cudaEventRecord(pe[2], c->stream));
      rr_project(c, m);
      CK(cudaEventRecord(c->ev_proj, c->stream));
      CK(cudaStreamWaitEvent(c->eigs, c->ev_proj, 0));
      reduced_gevp_start(c, m, c->eigs, la);
      if (la) {
        lookahead_input(c, m);
        CK(cudaStreamWaitEvent(c->stream, c->ev_pre_eig, 0));
        CK(cudaEventRecord(pn[0], c->stream));
        contour_pass(c, m, c->BQ.p, c->X.p, nullptr, pn[3]);
        CK(cudaEventRecord(pn[1], c->stream));
      }
      Reduced r = reduced_gevp_finish(c, m, c->eigs);
      r.lookahead = la && r.kfactor <= c->la_kmax;
      c->lookahead_ok = r.kfactor <= c->la_kmax;
      CK(cudaStreamWaitEvent(c->stream, c->ev_eig, 0));
      // this pass's contour solves are complete (they precede the projection)
      CK(cudaEventElapsedTime(&ms, pe[0], pe[3]));
      ph[0] += ms;
      ph[3] += ms;
      CK(cudaEventElapsedTime(&ms, pe[3], pe[1]));
      ph[1] += ms;
      CK(cudaEventElapsedTime(&ms, pe[2], c->ev_eig));
      ph[2] += ms;
      have_q = next_subspace(c, m, r);
      m = r.mo;
      if (r.lookahead) ++c->lookahead_count;
    }
    CK(cudaEventRecord(c->ev[1], c->stream));
    CK(cudaEventSynchronize(c->ev[1]));
    CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    c->bench_m = m;
    c->bench_have_q = have_q;
    c->bench_pass += passes;
    flush.release();
    if (total_ms) *total_ms = ms;
    if (phase_ms)
      for (int i = 0; i < 4; ++i) phase_ms[i] = ph[i];
  });
}

int feast_gpu_sweep(feast_gpu_ctx* c, const feast_operator_t* a0, const feast_operator_t* b,
                    const feast_operator_t* s, const double* steps, int nsteps, double emin, double emax,
                    const feast_config_t* config, feast_result_t* results, int* step_codes) {
  return guarded(c, [&] { sweep(c, a0, b, s, steps, nsteps, emin, emax, config, results, step_codes); });
}

int feast_gpu_set_pencil_hermitian(feast_gpu_ctx* c, const feast_operator_t* a, const feast_operator_t* b) {
  return guarded(c, [&] {
    validate_hermitian(a);
    validate_hermitian(b);
    if (a->n != b->n) fail(FEAST_EINPUT, "feast_solve: operator dimensions differ");
    EmbeddedOp ea, eb;
    embed_hermitian(a, ea);
    embed_hermitian(b, eb);
    set_pencil(c, &ea.op, &eb.op);
    c->hermitian = true;
    c->nz = a->n;
    c->norm_a1 = norm_one_hermitian(a);
  });
}

int feast_gpu_solve_hermitian(feast_gpu_ctx* c, double emin, double emax, const feast_config_t* config,
                              const double* initial_y, int y_cols, feast_result_t* result) {
  return guarded(c, [&] {
    if (!c->hermitian) fail(FEAST_EINPUT, "feast_gpu_solve_hermitian: set a Hermitian pencil first");
    feast_solve(c, emin, emax, config, initial_y, y_cols, result);
  });
}

int feast_gpu_set_inner_solver(feast_gpu_ctx* c, int kind, double tol, int max_iter) {
  return guarded(c, [&] {
    if (kind != 0 && kind != 1) fail(FEAST_EINPUT, "set_inner_solver: kind must be 0 (direct) or 1 (iterative)");
    if (kind == 1 && (!(tol > 0.0) || tol >= 1.0)) fail(FEAST_EINPUT, "IterativeSolver: tolerance must be in (0, 1)");
    c->inner_kind = kind;
    c->inner_tol = kind == 1 ? tol : 0.0;
    c->inner_max_iter = kind == 1 ? max_iter : 0;
    c->factored = false;
  });
}

int feast_gpu_set_factor_policy(feast_gpu_ctx* c, int policy) {
  return guarded(c, [&] {
    if (policy < 0 || policy > 2) fail(FEAST_EINPUT, "set_factor_policy: policy must be 0 (Auto), 1 (Dense) or 2 (Banded)");
    c->factor_policy = policy;
  });
}

int feast_gpu_set_spike(feast_gpu_ctx* c, int chunks) {
  return guarded(c, [&] {
    if (chunks < 0 || chunks > 64 || (chunks & (chunks - 1))) fail(FEAST_EINPUT, "set_spike: chunks must be 0 or a power of two <= 64");
    c->spike_req = chunks;
    c->factored = false;
  });
}

int feast_gpu_set_row_distribution(feast_gpu_ctx* c, int enable) {
  return guarded(c, [&] { c->row_dist = enable != 0; });
}

int feast_gpu_set_lookahead(feast_gpu_ctx* c, int enable, double max_cancellation) {
  return guarded(c, [&] {
    c->lookahead = enable != 0;
    c->la_kmax = max_cancellation > 0.0 ? max_cancellation : kLookaheadMaxK;
  });
}

int feast_gpu_lookahead_count(const feast_gpu_ctx* c) { return c ? c->lookahead_count : 0; }

int64_t feast_gpu_launch_count(const feast_gpu_ctx*) { return g_launches; }

}  // extern "C"
