"""oracle/oracle.py — TEST INFRASTRUCTURE: Python loaders for the CPU checkers.

Two checkers with one API:
  * kind="reference": oracle/_ref/libfeastref.so — the reference feastlite C++ library
    compiled from /root/reference/proj (oracle/Makefile) behind ref_driver.cpp.
  * kind="port":      oracle/libfeastoracle.so — feast_oracle.c, the plain-C restatement
    of the same algorithm (each function cites the reference file:line it follows).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module. It is the checker, never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_0901_2665_b200 import abi  # noqa: E402

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_op = C.POINTER(abi.FeastOperatorT)

LIBS = {
    "reference": os.path.join(_HERE, "_ref", "libfeastref.so"),
    "port": os.path.join(_HERE, "libfeastoracle.so"),
}
_cache = {}


def available(kind="reference"):
    if kind == "mm":
        return os.path.exists(os.path.join(_HERE, "_ref", "ref_mm_dump"))
    return os.path.exists(LIBS[kind])


def lib(kind="reference"):
    if kind in _cache:
        return _cache[kind]
    path = LIBS[kind]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (make -C oracle)")
    L = C.CDLL(path)
    L.ref_last_error.restype = C.c_char_p
    L.ref_scalar_filter.restype = C.c_double
    L.ref_scalar_filter.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
    L.ref_random_block.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp]
    L.ref_build_contour.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp]
    L.ref_gauss_legendre.argtypes = [C.c_int, _dp, _dp]
    L.ref_accumulate_hermitian.argtypes = [_op, _op, C.c_double, C.c_double, C.c_int, _dp, C.c_int, _dp,
                                           C.c_int]
    L.ref_accumulate_real.argtypes = [_op, _op, C.c_double, C.c_double, C.c_int, _dp, C.c_int,
                                      _dp, C.c_int]
    L.ref_shift_solve.argtypes = [_op, _op, C.c_double, C.c_double, _dp, C.c_int, C.c_int]
    L.ref_reduced_gevp.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _ip, _ip]
    L.ref_rayleigh_ritz.argtypes = [_op, _op, _dp, C.c_int, _dp, _dp, _ip, _ip]
    L.ref_residual_norms.argtypes = [_op, _op, C.c_int, _dp, _dp, _dp, _ip, _dp]
    L.ref_reference_gevp.argtypes = [_op, _op, _dp, _dp]
    L.ref_feast_solve.argtypes = [_op, _op, C.c_double, C.c_double,
                                  C.POINTER(abi.FeastConfigT), _dp, C.c_int,
                                  C.POINTER(abi.FeastResultT)]
    if hasattr(L, "ref_feast_solve_with"):  # the reference build only (explicit InnerSolver)
        L.ref_feast_solve_with.argtypes = [_op, _op, C.c_double, C.c_double, C.POINTER(abi.FeastConfigT), _dp,
                                           C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                           C.POINTER(abi.FeastResultT)]
        L.ref_shift_solve_with.argtypes = [_op, _op, C.c_double, C.c_double, _dp, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_double, C.c_int]
    if hasattr(L, "ref_feast_solve_hermitian"):
        L.ref_feast_solve_hermitian.argtypes = [_op, _op, C.c_double, C.c_double, C.POINTER(abi.FeastConfigT), _dp,
                                                C.c_int, C.POINTER(abi.FeastResultT)]
    if hasattr(L, "ref_bench_passes"):
        L.ref_bench_passes.argtypes = [_op, _op, C.c_double, C.c_double, C.c_int, C.c_int,
                                       C.c_uint64, C.c_int, C.c_int, _dp]
    _cache[kind] = L
    return L


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(L, rc):
    if rc != 0:
        raise OracleError(rc, L.ref_last_error().decode())


def _F(a):
    return np.asfortranarray(a, dtype=np.float64)


def gauss_legendre(n, kind="reference"):
    L = lib(kind)
    x, w = np.zeros(n), np.zeros(n)
    _check(L, L.ref_gauss_legendre(n, abi.dptr(x), abi.dptr(w)))
    return x, w


def build_contour(emin, emax, ne, kind="reference"):
    L = lib(kind)
    node, weight, theta = np.zeros(ne), np.zeros(ne), np.zeros(ne)
    z = np.zeros(2 * ne)
    r = np.zeros(1)
    _check(L, L.ref_build_contour(emin, emax, ne, abi.dptr(node), abi.dptr(weight),
                                  abi.dptr(theta), abi.dptr(z), abi.dptr(r)))
    return dict(node=node, weight=weight, theta=theta, z=z[0::2] + 1j * z[1::2], radius=r[0])


def random_block(n, m, seed, kind="reference"):
    L = lib(kind)
    y = np.zeros((n, m), order="F")
    _check(L, L.ref_random_block(n, m, seed, abi.dptr(y)))
    return y


def scalar_filter(lam, emin, emax, ne, kind="reference"):
    return lib(kind).ref_scalar_filter(lam, emin, emax, ne)


def accumulate_real(a, b, emin, emax, ne, y, threads=1, kind="reference"):
    L = lib(kind)
    y = _F(y)
    q = np.zeros_like(y, order="F")
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_accumulate_real(C.byref(ca), C.byref(cb), emin, emax, ne, abi.dptr(y),
                                    y.shape[1], abi.dptr(q), threads))
    return q


def accumulate_hermitian(a, b, emin, emax, ne, y, threads=1, kind="reference"):
    """accumulate_subspace_hermitian (core.hpp:190-215): y, Q complex n x m."""
    L = lib(kind)
    y = np.asfortranarray(y, dtype=np.complex128)
    q = np.zeros_like(y, order="F")
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_accumulate_hermitian(C.byref(ca), C.byref(cb), emin, emax, ne, y.ctypes.data_as(_dp),
                                         y.shape[1], q.ctypes.data_as(_dp), threads))
    return q


def shift_solve(a, b, z, rhs, mode=0, kind="reference"):
    L = lib(kind)
    r = np.asfortranarray(rhs, dtype=np.complex128).copy(order="F")
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_shift_solve(C.byref(ca), C.byref(cb), z.real, z.imag,
                                r.ctypes.data_as(_dp), r.shape[1], mode))
    return r


def shift_solve_with(a, b, z, rhs, mode=0, solver="direct", policy=0, tol=0.0, max_iter=0, kind="reference"):
    """ShiftSystem::solve_in_place of DirectSolver(policy) or IterativeSolver(tol, max_iter)."""
    L = lib(kind)
    r = np.asfortranarray(rhs, dtype=np.complex128).copy(order="F")
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_shift_solve_with(C.byref(ca), C.byref(cb), z.real, z.imag, r.ctypes.data_as(_dp), r.shape[1],
                                     mode, 1 if solver == "iterative" else 0, policy, tol, max_iter))
    return r


def reduced_gevp(aq, bq, kind="reference"):
    L = lib(kind)
    m = aq.shape[0]
    aq, bq = _F(aq), _F(bq)
    ev = np.zeros(m)
    phi = np.zeros((m, m), order="F")
    mo, tr = C.c_int32(0), C.c_int32(0)
    _check(L, L.ref_reduced_gevp(m, abi.dptr(aq), abi.dptr(bq), abi.dptr(ev), abi.dptr(phi),
                                 C.byref(mo), C.byref(tr)))
    k = mo.value
    return ev[:k], np.asfortranarray(phi.reshape(-1, order="F")[: m * k].reshape((m, k), order="F")), bool(tr.value)


def rayleigh_ritz(a, b, q, kind="reference"):
    L = lib(kind)
    q = _F(q)
    n, m = q.shape
    ev = np.zeros(m)
    x = np.zeros((n, m), order="F")
    mo, tr = C.c_int32(0), C.c_int32(0)
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_rayleigh_ritz(C.byref(ca), C.byref(cb), abi.dptr(q), m, abi.dptr(ev),
                                  abi.dptr(x), C.byref(mo), C.byref(tr)))
    k = mo.value
    return ev[:k], x.reshape(-1, order="F")[: n * k].reshape((n, k), order="F"), bool(tr.value)


def residual_norms(a, b, lambdas, x, kind="reference"):
    L = lib(kind)
    x = _F(x)
    lam = np.ascontiguousarray(lambdas, dtype=np.float64)
    m = len(lam)
    res = np.zeros(m)
    ab = np.zeros(m, dtype=np.int32)
    mx = C.c_double(0)
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_residual_norms(C.byref(ca), C.byref(cb), m, abi.dptr(lam), abi.dptr(x),
                                   abi.dptr(res), abi.iptr(ab), C.byref(mx)))
    return res, ab.astype(bool), mx.value


def reference_gevp(a, b, kind="reference"):
    L = lib(kind)
    n = a.n
    ev = np.zeros(n)
    vec = np.zeros((n, n), order="F")
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_reference_gevp(C.byref(ca), C.byref(cb), abi.dptr(ev), abi.dptr(vec)))
    return ev, vec


def bench_passes(problem, passes, threads=1, kind="reference"):
    """Times the reference loop body (factor once, then `passes` passes of
    accumulate + Rayleigh-Ritz + Y = B X). Returns dict(factorize_s, solve_s, reduce_s, count)."""
    L = lib(kind)
    p = problem
    out = np.zeros(4)
    ca, cb = p.a.to_c(), p.b.to_c()
    _check(L, L.ref_bench_passes(C.byref(ca), C.byref(cb), p.emin, p.emax, p.m0, p.n_e, p.seed,
                                 threads, passes, abi.dptr(out)))
    return dict(factorize_s=out[0], solve_s=out[1], reduce_s=out[2], count=int(out[3]))


SHIM = os.path.join(_HERE, "_ref", "libfeastref_gpu.so")


def shim_feast_solve(problem, mode=0):
    """mode 0: the REFERENCE's feast_solve with feast::gpu::GpuDirectSolver as its InnerSolver
    (every shifted solve on the GPU through the C-ABI); mode 1: feast::gpu::feast_solve."""
    if "shim" not in _cache:
        L = C.CDLL(SHIM)
        L.ref_last_error.restype = C.c_char_p
        L.shim_feast_solve.argtypes = [_op, _op, C.c_double, C.c_double, C.POINTER(abi.FeastConfigT),
                                       C.c_int, C.POINTER(abi.FeastResultT)]
        _cache["shim"] = L
    L = _cache["shim"]
    p = problem
    cfg = abi.FeastConfigT(m0=p.m0, n_e=p.n_e, trace_tol=p.trace_tol, max_loops=p.max_loops,
                           seed=p.seed, threads=1, low_memory=0)
    n = p.n
    out = dict(eigenvalues=np.zeros(p.m0), eigenvectors=np.zeros((n, p.m0), order="F"),
               residuals=np.zeros(p.m0), residual_absolute_only=np.zeros(p.m0, dtype=np.int32),
               trace_history=np.zeros(p.max_loops + 1),
               in_interval_counts=np.zeros(p.max_loops + 1, dtype=np.int32),
               subspace=np.zeros((n, p.m0), order="F"))
    r = abi.FeastResultT()
    r.eigenvalues = abi.dptr(out["eigenvalues"])
    r.eigenvectors = abi.dptr(out["eigenvectors"])
    r.residuals = abi.dptr(out["residuals"])
    r.residual_absolute_only = abi.iptr(out["residual_absolute_only"])
    r.trace_history = abi.dptr(out["trace_history"])
    r.in_interval_counts = abi.iptr(out["in_interval_counts"])
    r.subspace = abi.dptr(out["subspace"])
    ca, cb = p.a.to_c(), p.b.to_c()
    _check(L, L.shim_feast_solve(C.byref(ca), C.byref(cb), p.emin, p.emax, C.byref(cfg), mode, C.byref(r)))
    return unpack_result(out, r, n)


def feast_solve(problem, threads=1, low_memory=False, initial_y=None, kind="reference",
                m0=None, n_e=None, trace_tol=None, max_loops=None, seed=None):
    """Runs the CPU feast_solve (core.hpp:264) on a problems.Problem; returns a dict
    mirroring FeastResult<double>."""
    L = lib(kind)
    p = problem
    n = p.n
    cfg = abi.FeastConfigT(m0=m0 or p.m0, n_e=n_e or p.n_e,
                           trace_tol=trace_tol or p.trace_tol,
                           max_loops=max_loops or p.max_loops,
                           seed=p.seed if seed is None else seed,
                           threads=threads, low_memory=int(low_memory))
    return _run_solve(L, p.a, p.b, p.emin, p.emax, cfg, initial_y, n)


def feast_solve_with(problem, solver="direct", policy=0, tol=0.0, max_iter=0, threads=1, kind="reference"):
    """feast_solve with an explicit InnerSolver: DirectSolver(policy) or IterativeSolver(tol, max_iter)."""
    L = lib(kind)
    p = problem
    cfg = abi.FeastConfigT(m0=p.m0, n_e=p.n_e, trace_tol=p.trace_tol, max_loops=p.max_loops, seed=p.seed,
                           threads=threads, low_memory=0)
    return _run_solve(L, p.a, p.b, p.emin, p.emax, cfg, None, p.n,
                      solver=(1 if solver == "iterative" else 0, policy, tol, max_iter))


def feast_solve_hermitian(a, b, emin, emax, m0, n_e=8, trace_tol=1e-13, max_loops=20, seed=42, initial_y=None,
                          threads=1, kind="reference"):
    """feast_solve<cplx> of the reference on a Hermitian pencil (Operator kinds DENSE_Z / CSR_Z):
    dict like feast_solve's, eigenvectors / subspace complex."""
    L = lib(kind)
    n = a.n
    cfg = abi.FeastConfigT(m0=m0, n_e=n_e, trace_tol=trace_tol, max_loops=max_loops, seed=seed, threads=threads,
                           low_memory=0)
    out = dict(eigenvalues=np.zeros(m0), eigenvectors=np.zeros((n, m0), dtype=np.complex128, order="F"),
               residuals=np.zeros(m0), residual_absolute_only=np.zeros(m0, dtype=np.int32),
               trace_history=np.zeros(max_loops + 1), in_interval_counts=np.zeros(max_loops + 1, dtype=np.int32),
               subspace=np.zeros((n, m0), dtype=np.complex128, order="F"))
    r = abi.FeastResultT()
    r.eigenvalues = abi.dptr(out["eigenvalues"])
    r.eigenvectors = abi.zptr(out["eigenvectors"])
    r.residuals = abi.dptr(out["residuals"])
    r.residual_absolute_only = abi.iptr(out["residual_absolute_only"])
    r.trace_history = abi.dptr(out["trace_history"])
    r.in_interval_counts = abi.iptr(out["in_interval_counts"])
    r.subspace = abi.zptr(out["subspace"])
    y0 = None if initial_y is None else np.asfortranarray(initial_y, dtype=np.complex128)
    ca, cb = a.to_c(), b.to_c()
    _check(L, L.ref_feast_solve_hermitian(C.byref(ca), C.byref(cb), emin, emax, C.byref(cfg), abi.zptr(y0),
                                          0 if y0 is None else y0.shape[1], C.byref(r)))
    m, k, loops = r.m, r.subspace_cols, r.loops_used
    return dict(status=abi.STATUS_NAMES[r.status], m=m, loops_used=loops,
                eigenvalues=out["eigenvalues"][:m].copy(), eigenvectors=out["eigenvectors"][:, :m].copy(),
                residuals=out["residuals"][:m].copy(), max_residual=r.max_residual,
                trace_history=out["trace_history"][: loops + 1].copy(),
                in_interval_counts=out["in_interval_counts"][: loops + 1].copy(),
                subspace=out["subspace"][:, :k].copy())


def _run_solve(L, a, b, emin, emax, cfg, initial_y, n, solver=None):
    m0 = cfg.m0
    out = dict(eigenvalues=np.zeros(m0), eigenvectors=np.zeros((n, m0), order="F"),
               residuals=np.zeros(m0), residual_absolute_only=np.zeros(m0, dtype=np.int32),
               trace_history=np.zeros(cfg.max_loops + 1),
               in_interval_counts=np.zeros(cfg.max_loops + 1, dtype=np.int32),
               subspace=np.zeros((n, m0), order="F"))
    r = abi.FeastResultT()
    r.eigenvalues = abi.dptr(out["eigenvalues"])
    r.eigenvectors = abi.dptr(out["eigenvectors"])
    r.residuals = abi.dptr(out["residuals"])
    r.residual_absolute_only = abi.iptr(out["residual_absolute_only"])
    r.trace_history = abi.dptr(out["trace_history"])
    r.in_interval_counts = abi.iptr(out["in_interval_counts"])
    r.subspace = abi.dptr(out["subspace"])
    y0 = None if initial_y is None else _F(initial_y)
    ca, cb = a.to_c(), b.to_c()
    if solver is None:
        _check(L, L.ref_feast_solve(C.byref(ca), C.byref(cb), emin, emax, C.byref(cfg),
                                    abi.dptr(y0), 0 if y0 is None else y0.shape[1], C.byref(r)))
    else:
        _check(L, L.ref_feast_solve_with(C.byref(ca), C.byref(cb), emin, emax, C.byref(cfg),
                                         abi.dptr(y0), 0 if y0 is None else y0.shape[1], *solver, C.byref(r)))
    return unpack_result(out, r, n)


def unpack_result(out, r, n):
    m, k, loops = r.m, r.subspace_cols, r.loops_used
    return dict(
        status=abi.STATUS_NAMES[r.status], m=m, loops_used=loops,
        eigenvalues=out["eigenvalues"][:m].copy(),
        eigenvectors=out["eigenvectors"].reshape(-1, order="F")[: n * m].reshape((n, m), order="F").copy(),
        residuals=out["residuals"][:m].copy(),
        residual_absolute_only=out["residual_absolute_only"][:m].astype(bool),
        max_residual=r.max_residual,
        trace_history=out["trace_history"][: loops + 1].copy(),
        in_interval_counts=out["in_interval_counts"][: loops + 1].copy(),
        subspace=out["subspace"].reshape(-1, order="F")[: n * k].reshape((n, k), order="F").copy(),
        timings=dict(factorize_s=r.factorize_s, solve_s=r.solve_s, reduce_s=r.reduce_s,
                     total_s=r.total_s),
    )


class ReferenceInputError(Exception):
    """InputError raised inside the reference library (message = what())."""


def mm_load_reference(path):
    """load_matrix_market_real (matrix_market.cpp:106-116) of the reference itself, run as
    oracle/_ref/ref_mm_dump: (n, row_ptr, col_idx, values) of the symmetric-complete CSR operator."""
    import subprocess
    exe = os.path.join(_HERE, "_ref", "ref_mm_dump")
    out = subprocess.run([exe, str(path)], capture_output=True, text=True, check=True).stdout
    head, _, rest = out.partition("\n")
    if head.startswith("ERR "):
        raise ReferenceInputError(head[4:])
    _, n, nnz = head.split()
    n, nnz = int(n), int(nnz)
    lines = rest.split("\n")
    rp = np.array([int(x) for x in lines[:n + 1]], np.int32)
    ci = np.array([int(x.split()[0]) for x in lines[n + 1:n + 1 + nnz]], np.int32)
    v = np.array([float.fromhex(x.split()[1]) for x in lines[n + 1:n + 1 + nnz]], np.float64)
    return n, rp, ci, v
