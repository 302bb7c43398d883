// oracle/ref_gpu_shim.cpp — TEST INFRASTRUCTURE: exercises the reference-side binding of
// integration/feast_gpu_solver.hpp. The REFERENCE's own feast_solve (core.hpp:264) runs with
// feast::gpu::GpuDirectSolver plugged in as its InnerSolver, so every shifted solve goes
// through the C-ABI to the GPU (plugin-level drop-in); and feast::gpu::feast_solve (the
// loop-level drop-in) is called with the reference's own types. Built into
// oracle/_ref/libfeastref_gpu.so together with ref_driver.cpp (oracle/Makefile).

#include <cstring>
#include <exception>

#include "../integration/feast_gpu_solver.hpp"
#include "feast/core.hpp"
#include "feast_gpu.h"

using feast::linalg::DenseMatrix;
using feast::linalg::SymmetricOperator;

namespace refdrv {
SymmetricOperator<double> to_ref(const feast_operator_t* op);
feast::FeastConfig to_ref(const feast_config_t* c);
int code_of(const std::exception& e);
}  // namespace refdrv

namespace {
void pack(const feast::FeastResult<double>& r, feast_result_t* out) {
  const int m = (int)r.eigenvalues.size();
  out->m = m;
  out->subspace_cols = r.subspace.cols();
  out->loops_used = r.loops_used;
  out->status = (int)r.status;
  out->max_residual = r.max_residual;
  out->factorize_s = r.timings.factorize_s;
  out->solve_s = r.timings.solve_s;
  out->reduce_s = r.timings.reduce_s;
  out->total_s = r.timings.total_s;
  if (out->eigenvalues) std::memcpy(out->eigenvalues, r.eigenvalues.data(), sizeof(double) * m);
  if (out->eigenvectors)
    std::memcpy(out->eigenvectors, r.eigenvectors.data().data(), sizeof(double) * r.eigenvectors.data().size());
  if (out->residuals) std::memcpy(out->residuals, r.residuals.data(), sizeof(double) * m);
  if (out->residual_absolute_only)
    for (int j = 0; j < m; ++j) out->residual_absolute_only[j] = r.residual_absolute_only[j];
  if (out->trace_history)
    std::memcpy(out->trace_history, r.trace_history.data(), sizeof(double) * r.trace_history.size());
  if (out->in_interval_counts)
    for (size_t k = 0; k < r.in_interval_counts.size(); ++k) out->in_interval_counts[k] = r.in_interval_counts[k];
  if (out->subspace) std::memcpy(out->subspace, r.subspace.data().data(), sizeof(double) * r.subspace.data().size());
}
}  // namespace

extern "C" {

// mode 0: reference feast_solve + GpuDirectSolver plugin; mode 1: feast::gpu::feast_solve
int shim_feast_solve(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                     const feast_config_t* config, int mode, feast_result_t* out) {
  try {
    const auto ra = refdrv::to_ref(a);
    const auto rb = refdrv::to_ref(b);
    const feast::SearchInterval iv(emin, emax);
    const feast::FeastConfig cfg = refdrv::to_ref(config);
    if (mode == 0) {
      feast::gpu::GpuDirectSolver solver(ra, rb, iv, cfg.n_e, 0);
      pack(feast::feast_solve<double>(ra, rb, iv, cfg, &solver, nullptr), out);
    } else {
      pack(feast::gpu::feast_solve(ra, rb, iv, cfg, nullptr, 0), out);
    }
    return 0;
  } catch (const std::exception& e) {
    return refdrv::code_of(e);
  }
}

}  // extern "C"
