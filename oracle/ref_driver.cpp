// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" driver around the UNMODIFIED reference library compiled from
// /root/reference/proj (see oracle/Makefile; the only change is kMaxReducedDimension
// raised from 128 to 4096 in a generated overlay of eigh.hpp). It lets
// the Python tests and bench.py's cpu_baseline leg call the reference's own code
// path: feast::feast_solve<double> (core.hpp:264), accumulate_subspace_real
// (core.hpp:163), reduced_gevp (eigh.hpp:178), residual_norms (residual.hpp:29),
// gauss_legendre / build_contour (quadrature.cpp:28,69), random_block (core.hpp:84),
// oracle::scalar_filter / reference_gevp (oracle.cpp:162,200).
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
// may load the library built from this file.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "feast/core.hpp"
#include "feast/oracle.hpp"
#include "feast/quadrature.hpp"
#include "feast_gpu.h"

using feast::cplx;
using feast::linalg::DenseMatrix;
using feast::linalg::SymmetricOperator;
using feast::linalg::Triplet;
using feast::linalg::TripletLayout;

namespace refdrv {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const feast::SubspaceBreakdown*>(&e)) return FEAST_EBREAKDOWN;
  if (dynamic_cast<const feast::InputError*>(&e)) return FEAST_EINPUT;
  if (dynamic_cast<const feast::NumericalError*>(&e)) return FEAST_ENUMERICAL;
  return FEAST_EINTERNAL;
}

// feast_operator_t -> the reference's SymmetricOperator (operator.hpp:45,66).
SymmetricOperator<double> to_ref(const feast_operator_t* op) {
  const int n = op->n;
  if (op->kind == FEAST_STORAGE_DENSE) {
    DenseMatrix<double> m(n, n);
    std::memcpy(m.data().data(), op->dense, sizeof(double) * (size_t)n * n);
    return SymmetricOperator<double>::from_dense(std::move(m));
  }
  std::vector<Triplet<double>> t;
  if (op->kind == FEAST_STORAGE_CSR) {
    t.reserve(op->row_ptr[n]);
    for (int i = 0; i < n; ++i)
      for (int k = op->row_ptr[i]; k < op->row_ptr[i + 1]; ++k)
        t.push_back({i, op->col_idx[k], op->values[k]});
    return SymmetricOperator<double>::from_triplets(n, std::move(t), TripletLayout::Full);
  }
  if (op->kind == FEAST_STORAGE_BLOCKTRI) {
    const int L = op->nblocks, b = op->bsize;
    if ((int64_t)L * b != n) throw feast::InputError("ref_driver: blocktri shape mismatch");
    for (int l = 0; l < L; ++l) {
      const double* d = op->diag + (size_t)l * b * b;
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i)
          if (d[i + (size_t)j * b] != 0.0) t.push_back({l * b + i, l * b + j, d[i + (size_t)j * b]});
      if (l + 1 < L) {
        const double* c = op->lower + (size_t)l * b * b;  // C_l = M(l+1, l)
        for (int j = 0; j < b; ++j)
          for (int i = 0; i < b; ++i) {
            const double v = c[i + (size_t)j * b];
            if (v == 0.0) continue;
            t.push_back({(l + 1) * b + i, l * b + j, v});
            t.push_back({l * b + j, (l + 1) * b + i, v});
          }
      }
    }
    return SymmetricOperator<double>::from_triplets(n, std::move(t), TripletLayout::Full);
  }
  throw feast::InputError("ref_driver: unknown storage kind");
}

feast::FeastConfig to_ref(const feast_config_t* c) {
  feast::FeastConfig f;
  f.m0 = c->m0;
  f.n_e = c->n_e;
  f.trace_tol = c->trace_tol;
  f.max_loops = c->max_loops;
  f.seed = c->seed;
  f.threads = c->threads;
  f.low_memory = c->low_memory != 0;
  return f;
}

}  // namespace refdrv
using namespace refdrv;

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_max_reduced_dimension(void) { return feast::linalg::kMaxReducedDimension; }

int ref_gauss_legendre(int n, double* nodes, double* weights) {
  try {
    const auto r = feast::quadrature::gauss_legendre(n);
    std::memcpy(nodes, r.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, r.weights.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Per node: node, weight, theta, z (re, im). radius_out gets the contour radius.
int ref_build_contour(double emin, double emax, int ne, double* node, double* weight,
                      double* theta, double* z, double* radius_out) {
  try {
    const auto c = feast::quadrature::build_contour(feast::SearchInterval(emin, emax), ne);
    for (int e = 0; e < ne; ++e) {
      node[e] = c.points[e].node;
      weight[e] = c.points[e].weight;
      theta[e] = c.points[e].theta;
      z[2 * e] = c.points[e].z.real();
      z[2 * e + 1] = c.points[e].z.imag();
    }
    *radius_out = c.radius;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_random_block(int n, int m, uint64_t seed, double* out) {
  try {
    const auto y = feast::random_block<double>(n, m, seed);
    std::memcpy(out, y.data().data(), sizeof(double) * (size_t)n * m);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

double ref_scalar_filter(double lambda, double emin, double emax, int ne) {
  return feast::oracle::scalar_filter(lambda, feast::SearchInterval(emin, emax), ne);
}

int ref_reference_gevp(const feast_operator_t* a, const feast_operator_t* b, double* evals,
                       double* evecs) {
  try {
    const auto s = feast::oracle::reference_gevp(to_ref(a), to_ref(b));
    std::memcpy(evals, s.eigenvalues.data(), sizeof(double) * s.eigenvalues.size());
    if (evecs)
      std::memcpy(evecs, s.eigenvectors.data().data(),
                  sizeof(double) * s.eigenvectors.data().size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// accumulate_subspace_real with the default DirectSolver (policy Auto).
int ref_accumulate_real(const feast_operator_t* a, const feast_operator_t* b, double emin,
                        double emax, int ne, const double* y, int m, double* q, int threads) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    const auto contour = feast::quadrature::build_contour(feast::SearchInterval(emin, emax), ne);
    feast::DirectSolver<double> solver(ra, rb);
    std::vector<std::unique_ptr<feast::ShiftSystem>> keep(ne);
    std::vector<const feast::ShiftSystem*> sys(ne);
    for (int e = 0; e < ne; ++e) {
      keep[e] = solver.prepare(contour.points[e].z);
      sys[e] = keep[e].get();
    }
    DenseMatrix<double> yy(ra.n(), m);
    std::memcpy(yy.data().data(), y, sizeof(double) * (size_t)ra.n() * m);
    const auto qq = feast::accumulate_subspace_real(yy, contour, sys, threads);
    std::memcpy(q, qq.data().data(), sizeof(double) * (size_t)ra.n() * m);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// accumulate_subspace_hermitian (core.hpp:190-215) with the default DirectSolver; y, q complex.
int ref_accumulate_hermitian(const feast_operator_t* a, const feast_operator_t* b, double emin,
                             double emax, int ne, const double* y, int m, double* q, int threads) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    const auto contour = feast::quadrature::build_contour(feast::SearchInterval(emin, emax), ne);
    feast::DirectSolver<double> solver(ra, rb);
    std::vector<std::unique_ptr<feast::ShiftSystem>> keep(ne);
    std::vector<const feast::ShiftSystem*> sys(ne);
    for (int e = 0; e < ne; ++e) {
      keep[e] = solver.prepare(contour.points[e].z);
      sys[e] = keep[e].get();
    }
    DenseMatrix<cplx> yy(ra.n(), m);
    std::memcpy(yy.data().data(), y, sizeof(cplx) * (size_t)ra.n() * m);
    const auto qq = feast::accumulate_subspace_hermitian(yy, contour, sys, threads);
    std::memcpy(q, qq.data().data(), sizeof(cplx) * (size_t)ra.n() * m);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ShiftSystem::solve_in_place at shift z for the DirectSolver of (A, B).
int ref_shift_solve(const feast_operator_t* a, const feast_operator_t* b, double zr, double zi,
                    double* rhs, int m, int mode) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    feast::DirectSolver<double> solver(ra, rb);
    auto sys = solver.prepare(cplx(zr, zi));
    DenseMatrix<cplx> r(ra.n(), m);
    std::memcpy(r.data().data(), rhs, sizeof(cplx) * (size_t)ra.n() * m);
    sys->solve_in_place(r, mode ? feast::linalg::SolveMode::ConjTranspose
                                : feast::linalg::SolveMode::Normal);
    std::memcpy(rhs, r.data().data(), sizeof(cplx) * (size_t)ra.n() * m);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_reduced_gevp(int m, const double* aq, const double* bq, double* evals, double* phi,
                     int* m_out, int* truncated) {
  try {
    DenseMatrix<double> A(m, m), B(m, m);
    std::memcpy(A.data().data(), aq, sizeof(double) * (size_t)m * m);
    std::memcpy(B.data().data(), bq, sizeof(double) * (size_t)m * m);
    const auto r = feast::linalg::reduced_gevp(A, B);
    *m_out = (int)r.eigenvalues.size();
    *truncated = r.truncated ? 1 : 0;
    std::memcpy(evals, r.eigenvalues.data(), sizeof(double) * r.eigenvalues.size());
    std::memcpy(phi, r.phi.data().data(), sizeof(double) * r.phi.data().size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_rayleigh_ritz(const feast_operator_t* a, const feast_operator_t* b, const double* q,
                      int m, double* evals, double* x, int* m_out, int* truncated) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    DenseMatrix<double> qq(ra.n(), m);
    std::memcpy(qq.data().data(), q, sizeof(double) * (size_t)ra.n() * m);
    const auto r = feast::rayleigh_ritz(ra, rb, qq);
    *m_out = (int)r.eigenvalues.size();
    *truncated = r.truncated ? 1 : 0;
    std::memcpy(evals, r.eigenvalues.data(), sizeof(double) * r.eigenvalues.size());
    std::memcpy(x, r.x.data().data(), sizeof(double) * r.x.data().size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_residual_norms(const feast_operator_t* a, const feast_operator_t* b, int m,
                       const double* lambdas, const double* x, double* res, int32_t* absonly,
                       double* maxres) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    DenseMatrix<double> xx(ra.n(), m);
    std::memcpy(xx.data().data(), x, sizeof(double) * (size_t)ra.n() * m);
    std::vector<double> lam(lambdas, lambdas + m);
    const auto rep = feast::linalg::residual_norms(ra, rb, lam, xx);
    for (int j = 0; j < m; ++j) {
      res[j] = rep.values[j];
      absonly[j] = rep.absolute_only[j] ? 1 : 0;
    }
    *maxres = rep.max_value;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Pass-level timing of the reference's own loop body (core.hpp:304-311 factors, then per
// pass accumulate_subspace_real + rayleigh_ritz + y = B X, core.hpp:340-387), with no
// stopping rule. out[0] = factorize seconds, out[1] = summed solve seconds, out[2] = summed
// reduce seconds, out[3] = in-interval count of the last pass.
int ref_bench_passes(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                     int m0, int ne, uint64_t seed, int threads, int passes, double* out) {
  try {
    using clk = std::chrono::steady_clock;
    auto since = [](clk::time_point t0) {
      return std::chrono::duration<double>(clk::now() - t0).count();
    };
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    const feast::SearchInterval iv(emin, emax);
    const auto contour = feast::quadrature::build_contour(iv, ne);
    feast::DirectSolver<double> solver(ra, rb);
    std::vector<std::unique_ptr<feast::ShiftSystem>> keep(ne);
    std::vector<const feast::ShiftSystem*> sys(ne);
    auto t0 = clk::now();
    feast::detail::parallel_points(ne, threads, [&](int e) { keep[e] = solver.prepare(contour.points[e].z); });
    for (int e = 0; e < ne; ++e) sys[e] = keep[e].get();
    out[0] = since(t0);
    out[1] = out[2] = 0.0;
    DenseMatrix<double> y = feast::random_block<double>(ra.n(), m0, seed);
    for (int p = 0; p < passes; ++p) {
      t0 = clk::now();
      const DenseMatrix<double> q = feast::accumulate_subspace_real(y, contour, sys, threads);
      out[1] += since(t0);
      t0 = clk::now();
      const auto rr = feast::rayleigh_ritz(ra, rb, q);
      out[2] += since(t0);
      out[3] = feast::trace_of_in_interval(rr.eigenvalues, iv).count;
      y = rb.apply(rr.x);
    }
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// complex Hermitian operator (FEAST_STORAGE_DENSE_Z / CSR_Z, interleaved) -> SymmetricOperator<cplx>
SymmetricOperator<cplx> to_ref_z(const feast_operator_t* op) {
  const int n = op->n;
  if (op->kind == FEAST_STORAGE_DENSE_Z) {
    DenseMatrix<cplx> m(n, n);
    std::memcpy(m.data().data(), op->dense, sizeof(cplx) * (size_t)n * n);
    return SymmetricOperator<cplx>::from_dense(std::move(m));
  }
  if (op->kind != FEAST_STORAGE_CSR_Z) throw feast::InputError("ref_driver: not a Hermitian operator");
  std::vector<Triplet<cplx>> t;
  t.reserve(op->row_ptr[n]);
  for (int i = 0; i < n; ++i)
    for (int k = op->row_ptr[i]; k < op->row_ptr[i + 1]; ++k)
      t.push_back({i, op->col_idx[k], cplx(op->values[2 * (size_t)k], op->values[2 * (size_t)k + 1])});
  return SymmetricOperator<cplx>::from_triplets(n, std::move(t), TripletLayout::Full);
}

// solver_kind 0: DirectSolver(a, b, FactorPolicy(policy)); 1: IterativeSolver(a, b, tol, max_iter)
// (inner_solver.hpp:77-113, 209-240); -1: the default (nullptr, core.hpp:264-268)
std::unique_ptr<feast::InnerSolver<double>> make_solver(const SymmetricOperator<double>& ra,
                                                        const SymmetricOperator<double>& rb, int solver_kind,
                                                        int policy, double tol, int max_iter) {
  if (solver_kind == 1) return std::make_unique<feast::IterativeSolver<double>>(ra, rb, tol, max_iter);
  if (solver_kind == 0)
    return std::make_unique<feast::DirectSolver<double>>(ra, rb, static_cast<feast::FactorPolicy>(policy));
  return nullptr;
}

int ref_feast_solve_with(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                         const feast_config_t* config, const double* initial_y, int y_cols, int solver_kind,
                         int policy, double tol, int max_iter, feast_result_t* out) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    const int n = ra.n();
    DenseMatrix<double> y0;
    if (initial_y) {
      y0 = DenseMatrix<double>(n, y_cols);
      std::memcpy(y0.data().data(), initial_y, sizeof(double) * (size_t)n * y_cols);
    }
    const auto solver = make_solver(ra, rb, solver_kind, policy, tol, max_iter);
    const auto r = feast::feast_solve<double>(ra, rb, feast::SearchInterval(emin, emax),
                                              to_ref(config), solver.get(),
                                              initial_y ? &y0 : nullptr);
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
      std::memcpy(out->eigenvectors, r.eigenvectors.data().data(),
                  sizeof(double) * r.eigenvectors.data().size());
    if (out->residuals) std::memcpy(out->residuals, r.residuals.data(), sizeof(double) * m);
    if (out->residual_absolute_only)
      for (int j = 0; j < m; ++j) out->residual_absolute_only[j] = r.residual_absolute_only[j];
    if (out->trace_history)
      std::memcpy(out->trace_history, r.trace_history.data(),
                  sizeof(double) * r.trace_history.size());
    if (out->in_interval_counts)
      for (size_t k = 0; k < r.in_interval_counts.size(); ++k)
        out->in_interval_counts[k] = r.in_interval_counts[k];
    if (out->subspace)
      std::memcpy(out->subspace, r.subspace.data().data(),
                  sizeof(double) * r.subspace.data().size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_feast_solve(const feast_operator_t* a, const feast_operator_t* b, double emin,
                    double emax, const feast_config_t* config, const double* initial_y,
                    int y_cols, feast_result_t* out) {
  return ref_feast_solve_with(a, b, emin, emax, config, initial_y, y_cols, -1, 0, 0.0, 0, out);
}

// feast_solve<cplx> (core.hpp:264-391) on a Hermitian pencil; eigenvectors / subspace complex
// (interleaved), initial_y complex n x y_cols or null
int ref_feast_solve_hermitian(const feast_operator_t* a, const feast_operator_t* b, double emin, double emax,
                              const feast_config_t* config, const double* initial_y, int y_cols,
                              feast_result_t* out) {
  try {
    const auto ra = to_ref_z(a);
    const auto rb = to_ref_z(b);
    const int n = ra.n();
    DenseMatrix<cplx> y0;
    if (initial_y) {
      y0 = DenseMatrix<cplx>(n, y_cols);
      std::memcpy(y0.data().data(), initial_y, sizeof(cplx) * (size_t)n * y_cols);
    }
    const auto r = feast::feast_solve<cplx>(ra, rb, feast::SearchInterval(emin, emax), to_ref(config), nullptr,
                                            initial_y ? &y0 : nullptr);
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
      std::memcpy(out->eigenvectors, r.eigenvectors.data().data(), sizeof(cplx) * r.eigenvectors.data().size());
    if (out->residuals) std::memcpy(out->residuals, r.residuals.data(), sizeof(double) * m);
    if (out->residual_absolute_only)
      for (int j = 0; j < m; ++j) out->residual_absolute_only[j] = r.residual_absolute_only[j];
    if (out->trace_history)
      std::memcpy(out->trace_history, r.trace_history.data(), sizeof(double) * r.trace_history.size());
    if (out->in_interval_counts)
      for (size_t k = 0; k < r.in_interval_counts.size(); ++k) out->in_interval_counts[k] = r.in_interval_counts[k];
    if (out->subspace)
      std::memcpy(out->subspace, r.subspace.data().data(), sizeof(cplx) * r.subspace.data().size());
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ShiftSystem::solve_in_place at shift z for a DirectSolver with FactorPolicy `policy` or an
// IterativeSolver (solver_kind as in ref_feast_solve_with)
int ref_shift_solve_with(const feast_operator_t* a, const feast_operator_t* b, double zr, double zi,
                         double* rhs, int m, int mode, int solver_kind, int policy, double tol, int max_iter) {
  try {
    const auto ra = to_ref(a);
    const auto rb = to_ref(b);
    const auto solver = make_solver(ra, rb, solver_kind, policy, tol, max_iter);
    auto sys = solver->prepare(cplx(zr, zi));
    DenseMatrix<cplx> r(ra.n(), m);
    std::memcpy(r.data().data(), rhs, sizeof(cplx) * (size_t)ra.n() * m);
    sys->solve_in_place(r, mode ? feast::linalg::SolveMode::ConjTranspose
                                : feast::linalg::SolveMode::Normal);
    std::memcpy(rhs, r.data().data(), sizeof(cplx) * (size_t)ra.n() * m);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

}  // extern "C"
