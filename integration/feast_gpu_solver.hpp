// integration/feast_gpu_solver.hpp — the reference-side binding a feastlite maintainer adds to
// drive the B200 path through feastlite's own plugin API.
//
//   * feast::gpu::GpuDirectSolver : feast::InnerSolver<double>   (inner_solver.hpp:32-39)
//       prepare(z) hands out a ShiftSystem whose solve_in_place runs on the GPU factors
//       (feast_gpu_solve_shift); the reference's own feast_solve (core.hpp:264) keeps the loop.
//   * feast::gpu::feast_solve(a, b, interval, config, initial_y)  (same signature as
//       core.hpp:264-268): the whole loop on the device through feast_gpu_solve.
//
// Header-only; needs the feastlite headers and links against libfeastgpu.so.
#pragma once

#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "feast/core.hpp"
#include "feast_gpu.h"

namespace feast::gpu {

[[noreturn]] inline void rethrow(int code, const feast_gpu_ctx* ctx) {
  const std::string msg = ctx ? feast_gpu_last_error(ctx) : "feast_gpu: no context";
  if (code == FEAST_EINPUT) throw InputError(msg);
  if (code == FEAST_EBREAKDOWN) throw SubspaceBreakdown(msg);
  throw NumericalError(msg);
}

// feast_operator_t view of a SymmetricOperator<double> (dense col-major or CSR; the vectors
// it points into must outlive the upload)
struct OperatorView {
  feast_operator_t op{};
  DenseMatrix<double> dense;
  explicit OperatorView(const SymmetricOperator<double>& a) {
    op.n = a.n();
    if (a.storage() == SymmetricOperator<double>::Storage::Dense) {
      dense = a.to_dense();
      op.kind = FEAST_STORAGE_DENSE;
      op.dense = dense.data().data();
    } else {
      op.kind = FEAST_STORAGE_CSR;
      op.row_ptr = a.row_ptr().data();
      op.col_idx = a.col_idx().data();
      op.values = a.values().data();
    }
  }
};

class Context {
 public:
  explicit Context(int device = 0) {
    const int rc = feast_gpu_create(device, nullptr, &ctx_);
    if (rc) rethrow(rc, nullptr);
  }
  ~Context() { feast_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  feast_gpu_ctx* get() const { return ctx_; }
  std::mutex& lock() const { return mu_; }

 private:
  feast_gpu_ctx* ctx_ = nullptr;
  mutable std::mutex mu_;
};

class GpuShiftSystem final : public ShiftSystem {
 public:
  GpuShiftSystem(std::shared_ptr<Context> ctx, int e) : ctx_(std::move(ctx)), e_(e) {}
  void solve_in_place(DenseMatrix<cplx>& rhs, SolveMode mode) const override {
    std::lock_guard<std::mutex> g(ctx_->lock());  // InnerSolver threading contract
    const int rc = feast_gpu_solve_shift(ctx_->get(), e_, reinterpret_cast<double*>(rhs.data().data()),
                                         rhs.cols(), mode == SolveMode::ConjTranspose ? 1 : 0);
    if (rc) rethrow(rc, ctx_->get());
  }

 private:
  std::shared_ptr<Context> ctx_;
  int e_;
};

// Factors every contour node of (interval, n_e) on the GPU up front; prepare(z) returns the
// node whose shift is z (the reference calls it with exactly build_contour's points).
class GpuDirectSolver final : public InnerSolver<double> {
 public:
  GpuDirectSolver(const SymmetricOperator<double>& a, const SymmetricOperator<double>& b,
                  const SearchInterval& interval, int n_e, int device = 0)
      : ctx_(std::make_shared<Context>(device)) {
    OperatorView va(a), vb(b);
    int rc = feast_gpu_set_pencil(ctx_->get(), &va.op, &vb.op);
    if (!rc) rc = feast_gpu_prepare(ctx_->get(), interval.lambda_min(), interval.lambda_max(), n_e);
    if (rc) rethrow(rc, ctx_->get());
    std::vector<double> z(2 * n_e);
    feast_gpu_contour(ctx_->get(), z.data(), nullptr);
    for (int e = 0; e < n_e; ++e) z_.emplace_back(z[2 * e], z[2 * e + 1]);
  }
  std::unique_ptr<ShiftSystem> prepare(cplx z) const override {
    for (std::size_t e = 0; e < z_.size(); ++e)
      if (std::abs(z - z_[e]) <= 1e-13 * (1.0 + std::abs(z)))
        return std::make_unique<GpuShiftSystem>(ctx_, static_cast<int>(e));
    throw InputError("GpuDirectSolver: shift is not a node of the prepared contour");
  }
  double residual_target() const override { return 0.0; }

 private:
  std::shared_ptr<Context> ctx_;
  std::vector<cplx> z_;
};

// The whole FEAST loop on the device (drop-in for feast::feast_solve<double>).
inline FeastResult<double> feast_solve(const SymmetricOperator<double>& a, const SymmetricOperator<double>& b,
                                       const SearchInterval& interval, const FeastConfig& config,
                                       const DenseMatrix<double>* initial_y = nullptr, int device = 0) {
  Context ctx(device);
  OperatorView va(a), vb(b);
  int rc = feast_gpu_set_pencil(ctx.get(), &va.op, &vb.op);
  if (rc) rethrow(rc, ctx.get());
  const int n = a.n(), m0 = config.m0 > 0 ? config.m0 : 1;
  FeastResult<double> r;
  std::vector<double> ev(m0), vec((size_t)n * m0), res(m0), tr(config.max_loops + 1), sub((size_t)n * m0);
  std::vector<int32_t> ab(m0), cnt(config.max_loops + 1);
  feast_result_t out{ev.data(), vec.data(), res.data(), ab.data(), tr.data(), cnt.data(), sub.data()};
  const feast_config_t c{config.m0, config.n_e, config.trace_tol, config.max_loops, config.seed,
                         config.threads, config.low_memory ? 1 : 0};
  rc = feast_gpu_solve(ctx.get(), interval.lambda_min(), interval.lambda_max(), &c,
                       initial_y ? initial_y->data().data() : nullptr, initial_y ? initial_y->cols() : 0, &out);
  if (rc) rethrow(rc, ctx.get());
  const int m = out.m, k = out.subspace_cols;
  const int nh = out.status == FEAST_STATUS_BREAKDOWN ? out.loops_used : out.loops_used + 1;
  r.eigenvalues.assign(ev.begin(), ev.begin() + m);
  r.eigenvectors = DenseMatrix<double>(n, m);
  std::copy(vec.begin(), vec.begin() + (size_t)n * m, r.eigenvectors.data().begin());
  r.residuals.assign(res.begin(), res.begin() + m);
  for (int j = 0; j < m; ++j) r.residual_absolute_only.push_back(ab[j] != 0);
  r.max_residual = out.max_residual;
  r.loops_used = out.loops_used;
  r.trace_history.assign(tr.begin(), tr.begin() + nh);
  r.in_interval_counts.assign(cnt.begin(), cnt.begin() + nh);
  r.status = static_cast<FeastStatus>(out.status);
  r.subspace = DenseMatrix<double>(n, k);
  std::copy(sub.begin(), sub.begin() + (size_t)n * k, r.subspace.data().begin());
  r.timings = {out.factorize_s, out.solve_s, out.reduce_s, out.total_s};
  return r;
}

}  // namespace feast::gpu
