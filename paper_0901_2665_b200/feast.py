"""Python mirror of the reference solver API over the C-ABI of libfeastgpu.so.

Names, argument meaning and error behaviour follow the reference (feastlite):
  FeastConfig / FeastStatus / FeastResult / SearchInterval   core.hpp:25-78, types.hpp:60-80
  feast_solve(a, b, interval, config, initial_y=None)         core.hpp:264-268
  Error / InputError / NumericalError / SubspaceBreakdown      types.hpp:15-38
and the per-stage entry points of the boundary (GpuContext) mirror the reference
functions they replace (see include/feast_gpu.h).

There is NO CPU fallback: if libfeastgpu.so is missing or no GPU is visible, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfeastgpu.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_op = C.POINTER(abi.FeastOperatorT)


class Error(RuntimeError):
    """feast::Error"""


class InputError(Error):
    """feast::InputError (CLI exit 4)"""


class NumericalError(Error):
    """feast::NumericalError (CLI exit 5)"""


class NotPositiveDefinite(NumericalError):
    pass


class SubspaceBreakdown(NumericalError):
    pass


class DeviceError(NumericalError):
    """CUDA / NCCL failure (NumericalError class at the boundary)."""


_CODES = {abi.FEAST_EINPUT: InputError, abi.FEAST_ENUMERICAL: NumericalError,
          abi.FEAST_EBREAKDOWN: SubspaceBreakdown, abi.FEAST_ECUDA: DeviceError,
          abi.FEAST_ENCCL: DeviceError, abi.FEAST_EINTERNAL: Error}

_lib = None


def _retain_host_heap():
    """Result blocks (eigenvectors, subspace: n x m doubles, 25 MB each at config 2) are fresh
    numpy arrays per solve. With glibc's defaults the previous solve's blocks go back to the OS
    and every download page-faults its destination again (measured: 37 ms cold vs 4 ms warm
    for the config-2 result download, and a 185..307 passes/s spread in the end-to-end number).
    Keep freed heap memory in the process instead: allocations up to 32 MB come from the heap
    (M_MMAP_THRESHOLD) and the heap top is not trimmed (M_TRIM_THRESHOLD)."""
    try:
        libc = C.CDLL("libc.so.6")
        libc.mallopt(-3, 32 << 20)   # M_MMAP_THRESHOLD (the glibc maximum on 64-bit)
        libc.mallopt(-1, 1 << 30)    # M_TRIM_THRESHOLD
    except (OSError, AttributeError):
        pass


def load_library(path: str = LIB_PATH):
    """Loads libfeastgpu.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback)")
    _retain_host_heap()
    L = C.CDLL(path)
    L.feast_gpu_last_error.restype = C.c_char_p
    L.feast_gpu_last_error.argtypes = [C.c_void_p]
    L.feast_gpu_create.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    L.feast_gpu_destroy.argtypes = [C.c_void_p]
    L.feast_gpu_destroy.restype = None
    L.feast_gpu_set_comm.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    L.feast_gpu_nccl_unique_id.argtypes = [C.c_void_p]
    L.feast_gpu_set_pencil.argtypes = [C.c_void_p, _op, _op]
    L.feast_gpu_prepare.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int]
    L.feast_gpu_contour.argtypes = [C.c_void_p, _dp, _dp]
    L.feast_gpu_storage.argtypes = [C.c_void_p, _ip, _ip, _ip]
    L.feast_gpu_random_block.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, _dp]
    L.feast_gpu_set_node_batch.argtypes = [C.c_void_p, C.c_int]
    L.feast_gpu_set_twist.argtypes = [C.c_void_p, C.c_int]
    L.feast_gpu_set_spike.argtypes = [C.c_void_p, C.c_int]
    L.feast_gpu_set_lookahead.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.feast_gpu_set_row_distribution.argtypes = [C.c_void_p, C.c_int]
    L.feast_gpu_set_inner_solver.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int]
    L.feast_gpu_set_factor_policy.argtypes = [C.c_void_p, C.c_int]
    L.feast_gpu_set_pencil_hermitian.argtypes = [C.c_void_p, _op, _op]
    L.feast_gpu_solve_hermitian.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(abi.FeastConfigT), _dp,
                                            C.c_int, C.POINTER(abi.FeastResultT)]
    L.feast_gpu_sweep.argtypes = [C.c_void_p, _op, _op, _op, _dp, C.c_int, C.c_double, C.c_double,
                                  C.POINTER(abi.FeastConfigT), C.c_void_p, _ip]
    L.feast_gpu_group_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.feast_gpu_group_destroy.argtypes = [C.c_void_p]
    L.feast_gpu_set_group.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.feast_gpu_lookahead_count.argtypes = [C.c_void_p]
    L.feast_gpu_solve_shift.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_int]
    L.feast_gpu_contour_pass.argtypes = [C.c_void_p, _dp, C.c_int, _dp]
    L.feast_gpu_contour_pass_hermitian.argtypes = [C.c_void_p, _dp, C.c_int, _dp]
    L.feast_gpu_rayleigh_ritz.argtypes = [C.c_void_p, _dp, C.c_int, _dp, _dp, _ip, _ip]
    L.feast_gpu_reduced_gevp.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _ip, _ip]
    L.feast_gpu_residuals.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _ip, _dp]
    L.feast_gpu_solve.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(abi.FeastConfigT),
                                  _dp, C.c_int, C.POINTER(abi.FeastResultT)]
    L.feast_gpu_bench_init.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
    L.feast_gpu_bench_passes.argtypes = [C.c_void_p, C.c_int, C.c_size_t, _dp, _dp]
    L.feast_gpu_launch_count.argtypes = [C.c_void_p]
    L.feast_gpu_launch_count.restype = C.c_int64
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "feast_gpu_abi_version", "feast_gpu_create", "feast_gpu_destroy", "feast_gpu_last_error",
    "feast_gpu_nccl_unique_id", "feast_gpu_set_comm", "feast_gpu_set_pencil", "feast_gpu_prepare",
    "feast_gpu_contour", "feast_gpu_solve_shift", "feast_gpu_contour_pass",
    "feast_gpu_rayleigh_ritz", "feast_gpu_reduced_gevp", "feast_gpu_residuals", "feast_gpu_solve",
    "feast_gpu_bench_init", "feast_gpu_bench_passes", "feast_gpu_launch_count",
    "feast_gpu_set_node_batch", "feast_gpu_storage", "feast_gpu_random_block",
    "feast_gpu_contour_pass_hermitian", "feast_gpu_set_twist", "feast_gpu_set_lookahead",
    "feast_gpu_lookahead_count", "feast_gpu_set_row_distribution", "feast_gpu_group_create",
    "feast_gpu_group_destroy", "feast_gpu_set_group", "feast_gpu_set_inner_solver",
    "feast_gpu_set_factor_policy", "feast_gpu_sweep", "feast_gpu_set_pencil_hermitian",
    "feast_gpu_solve_hermitian", "feast_gpu_set_spike",
]


# ---------------------------------------------------------------------------
# reference value types
# ---------------------------------------------------------------------------
class SearchInterval:
    """Closed interval [lambda_min, lambda_max] (types.hpp:60-80)."""

    def __init__(self, lambda_min: float, lambda_max: float):
        if not (lambda_min < lambda_max):
            raise InputError("SearchInterval: lambda_min must be strictly below lambda_max")
        self.lo, self.hi = float(lambda_min), float(lambda_max)

    lambda_min = property(lambda s: s.lo)
    lambda_max = property(lambda s: s.hi)
    width = property(lambda s: s.hi - s.lo)
    center = property(lambda s: 0.5 * (s.lo + s.hi))
    radius = property(lambda s: 0.5 * (s.hi - s.lo))

    def contains(self, x):
        return self.lo <= x <= self.hi


@dataclass
class FeastConfig:
    """core.hpp:25-33"""
    m0: int = 0
    n_e: int = 8
    trace_tol: float = 1e-13
    max_loops: int = 20
    seed: int = 42
    threads: int = 1
    low_memory: bool = False

    def to_c(self):
        return abi.FeastConfigT(m0=self.m0, n_e=self.n_e, trace_tol=self.trace_tol,
                                max_loops=self.max_loops, seed=self.seed, threads=self.threads,
                                low_memory=int(self.low_memory))


@dataclass
class FeastTimings:
    factorize_s: float = 0.0
    solve_s: float = 0.0
    reduce_s: float = 0.0
    total_s: float = 0.0


@dataclass
class FeastResult:
    """core.hpp:61-78 (status as the reference's to_string, core.hpp:43-52)"""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    residuals: np.ndarray
    residual_absolute_only: np.ndarray
    max_residual: float
    loops_used: int
    trace_history: np.ndarray
    in_interval_counts: np.ndarray
    status: str
    subspace: np.ndarray
    timings: FeastTimings = field(default_factory=FeastTimings)


def _cols(a, n, k):
    """The first k columns of a Fortran-ordered n x m0 output block, as a view (no copy)."""
    return a[:n, :k]


def _result_buffers(n, config):
    """Caller-allocated arrays of a feast_result_t (include/feast_gpu.h)."""
    m0 = config.m0
    nl = max(config.max_loops, 0) + 1
    out = dict(eigenvalues=np.zeros(max(m0, 1)), eigenvectors=np.empty((n, max(m0, 1)), order="F"),
               residuals=np.zeros(max(m0, 1)), absonly=np.zeros(max(m0, 1), dtype=np.int32),
               trace=np.zeros(nl), counts=np.zeros(nl, dtype=np.int32),
               subspace=np.empty((n, max(m0, 1)), order="F"))
    r = abi.FeastResultT()
    r.eigenvalues = abi.dptr(out["eigenvalues"])
    r.eigenvectors = abi.dptr(out["eigenvectors"])
    r.residuals = abi.dptr(out["residuals"])
    r.residual_absolute_only = abi.iptr(out["absonly"])
    r.trace_history = abi.dptr(out["trace"])
    r.in_interval_counts = abi.iptr(out["counts"])
    r.subspace = abi.dptr(out["subspace"])
    return out, r


def _result_of(out, r, n):
    m, k, loops = r.m, r.subspace_cols, r.loops_used
    nh = loops if r.status == 4 else loops + 1  # breakdown returns before pushing (core.hpp:347-353)
    return FeastResult(
        eigenvalues=out["eigenvalues"][:m].copy(),
        eigenvectors=_cols(out["eigenvectors"], n, m),
        residuals=out["residuals"][:m].copy(),
        residual_absolute_only=out["absonly"][:m].astype(bool),
        max_residual=r.max_residual,
        loops_used=loops,
        trace_history=out["trace"][:nh].copy(),
        in_interval_counts=out["counts"][:nh].copy(),
        status=abi.STATUS_NAMES[r.status],
        subspace=_cols(out["subspace"], n, k) if k else np.zeros((n, 0)),
        timings=FeastTimings(r.factorize_s, r.solve_s, r.reduce_s, r.total_s),
    )


class GpuContext:
    """One device context of the C-ABI (feast_gpu_ctx). Holds A, B, the contour, the
    per-node factors and the device-resident blocks between calls."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.L = load_library()
        h = C.c_void_p()
        rc = self.L.feast_gpu_create(device, C.c_void_p(stream) if stream else None, C.byref(h))
        if rc != 0:
            raise _CODES.get(rc, Error)(f"feast_gpu_create failed with code {rc} (is a GPU visible?)")
        self.h = h
        self.n = None

    def close(self):
        if getattr(self, "h", None):
            self.L.feast_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            msg = self.L.feast_gpu_last_error(self.h).decode()
            raise _CODES.get(rc, Error)(msg)

    # -- boundary entry points -------------------------------------------------
    def set_comm(self, unique_id: bytes, rank: int, nranks: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(self.L.feast_gpu_set_comm(self.h, buf, rank, nranks))

    @staticmethod
    def nccl_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        rc = L.feast_gpu_nccl_unique_id(buf)
        if rc != 0:
            raise DeviceError("ncclGetUniqueId failed")
        return buf.raw

    def set_pencil(self, a, b):
        self._ca, self._cb = a.to_c(), b.to_c()
        self._check(self.L.feast_gpu_set_pencil(self.h, C.byref(self._ca), C.byref(self._cb)))
        self.n = a.n

    def set_node_batch(self, nodes: int):
        """Factor memory plan: 0 = automatic (resident if they fit), k > 0 = stream k nodes."""
        self._check(self.L.feast_gpu_set_node_batch(self.h, int(nodes)))

    def set_inner_solver(self, kind: str = "direct", tol: float = 0.0, max_iter: int = 0):
        """InnerSolver of the loop (inner_solver.hpp): "direct" (DirectSolver, the default) or
        "iterative" (IterativeSolver(tol, max_iter): BiCGStab per right-hand side)."""
        k = {"direct": 0, "iterative": 1}[kind]
        self._check(self.L.feast_gpu_set_inner_solver(self.h, k, float(tol), int(max_iter)))

    def set_factor_policy(self, policy: str = "auto"):
        """FactorPolicy (inner_solver.hpp:40-47) of the DirectSolver, at the next set_pencil."""
        self._check(self.L.feast_gpu_set_factor_policy(self.h, {"auto": 0, "dense": 1, "banded": 2}[policy]))

    def set_group(self, group: "LocalGroup", rank: int):
        """Join a loopback rank group (contexts of this process, one host thread each)."""
        self._check(self.L.feast_gpu_set_group(self.h, group.h, rank))
        self._group = group

    def set_row_distribution(self, enable: bool):
        """Row-distributed Rayleigh-Ritz across the ranks (default on)."""
        self._check(self.L.feast_gpu_set_row_distribution(self.h, int(bool(enable))))

    def set_lookahead(self, enable: bool, max_cancellation: float = 0.0):
        """Look-ahead contour pass overlapping each reduced eigensolve (default on); admitted when
        the Ritz block's cancellation factor is <= max_cancellation (0: the default bound)."""
        self._check(self.L.feast_gpu_set_lookahead(self.h, int(bool(enable)), float(max_cancellation)))

    def lookahead_count(self) -> int:
        return int(self.L.feast_gpu_lookahead_count(self.h))

    def set_spike(self, chunks: int):
        """SPIKE partitioning of the block-Thomas chain into `chunks` (0 auto, 1 off; b <= 32)."""
        self._check(self.L.feast_gpu_set_spike(self.h, int(chunks)))

    def set_twist(self, enable: bool):
        """Two-ended block-Thomas recursion (default on) or the plain top-down chain (b <= 64)."""
        self._check(self.L.feast_gpu_set_twist(self.h, int(bool(enable))))

    def prepare(self, emin, emax, n_e=8):
        self._check(self.L.feast_gpu_prepare(self.h, emin, emax, n_e))
        self.n_e = n_e

    def random_block(self, n: int, m: int, seed: int) -> np.ndarray:
        """random_block<double>(n, m, seed) (core.hpp:84-106), generated on the device."""
        out = np.zeros((n, m), order="F")
        self._check(self.L.feast_gpu_random_block(self.h, n, m, seed, abi.dptr(out)))
        return out

    def storage(self):
        """(b, L, twist): block-tridiagonal block size and layer count (0, 0 when dense), and
        the twisted block-Thomas meeting layer of the current factors (-1: plain chain)."""
        b, lay, tw = C.c_int(0), C.c_int(0), C.c_int(-1)
        self._check(self.L.feast_gpu_storage(self.h, C.pointer(b), C.pointer(lay), C.pointer(tw)))
        return b.value, lay.value, tw.value

    def contour(self):
        z = np.zeros(2 * self.n_e)
        c = np.zeros(2 * self.n_e)
        self._check(self.L.feast_gpu_contour(self.h, abi.dptr(z), abi.dptr(c)))
        return z[0::2] + 1j * z[1::2], c[0::2] + 1j * c[1::2]

    def solve_shift(self, e: int, rhs: np.ndarray, conj_transpose: bool = False) -> np.ndarray:
        """ShiftSystem::solve_in_place (inner_solver.hpp:24-28) for node e."""
        r = np.asfortranarray(rhs, dtype=np.complex128).copy(order="F")
        if r.ndim == 1:
            r = r.reshape(-1, 1, order="F")
        self._check(self.L.feast_gpu_solve_shift(self.h, e, r.ctypes.data_as(_dp), r.shape[1],
                                                 int(conj_transpose)))
        return r

    def contour_pass(self, y: np.ndarray) -> np.ndarray:
        """accumulate_subspace_real (core.hpp:163-185)."""
        y = np.asfortranarray(y, dtype=np.float64)
        q = np.zeros_like(y, order="F")
        self._check(self.L.feast_gpu_contour_pass(self.h, abi.dptr(y), y.shape[1], abi.dptr(q)))
        return q

    def contour_pass_hermitian(self, y: np.ndarray) -> np.ndarray:
        """accumulate_subspace_hermitian (core.hpp:190-215): complex y -> complex Q."""
        y = np.asfortranarray(y, dtype=np.complex128)
        q = np.zeros_like(y, order="F")
        self._check(self.L.feast_gpu_contour_pass_hermitian(self.h, y.ctypes.data_as(_dp), y.shape[1],
                                                            q.ctypes.data_as(_dp)))
        return q

    def rayleigh_ritz(self, q: np.ndarray):
        """rayleigh_ritz (core.hpp:228-240): (eigenvalues, X, truncated)."""
        q = np.asfortranarray(q, dtype=np.float64)
        n, m = q.shape
        ev = np.zeros(m)
        x = np.zeros((n, m), order="F")
        mo, tr = C.c_int32(0), C.c_int32(0)
        self._check(self.L.feast_gpu_rayleigh_ritz(self.h, abi.dptr(q), m, abi.dptr(ev), abi.dptr(x),
                                                   C.byref(mo), C.byref(tr)))
        k = mo.value
        return ev[:k].copy(), _cols(x, n, k), bool(tr.value)

    def reduced_gevp(self, a_q: np.ndarray, b_q: np.ndarray):
        """reduced_gevp (eigh.hpp:178-225): (eigenvalues, phi, truncated)."""
        a_q = np.asfortranarray(a_q, dtype=np.float64)
        b_q = np.asfortranarray(b_q, dtype=np.float64)
        m = a_q.shape[0]
        ev = np.zeros(m)
        phi = np.zeros((m, m), order="F")
        mo, tr = C.c_int32(0), C.c_int32(0)
        self._check(self.L.feast_gpu_reduced_gevp(self.h, m, abi.dptr(a_q), abi.dptr(b_q), abi.dptr(ev),
                                                  abi.dptr(phi), C.byref(mo), C.byref(tr)))
        k = mo.value
        return ev[:k].copy(), _cols(phi, m, k), bool(tr.value)

    def residual_norms(self, lambdas, x):
        """residual_norms (residual.hpp:29-68): (values, absolute_only, max)."""
        x = np.asfortranarray(x, dtype=np.float64)
        lam = np.ascontiguousarray(lambdas, dtype=np.float64)
        m = len(lam)
        res = np.zeros(m)
        ab = np.zeros(m, dtype=np.int32)
        mx = C.c_double(0)
        self._check(self.L.feast_gpu_residuals(self.h, m, abi.dptr(lam), abi.dptr(x), abi.dptr(res),
                                               abi.iptr(ab), C.byref(mx)))
        return res, ab.astype(bool), mx.value

    def solve(self, interval: SearchInterval, config: FeastConfig, initial_y=None) -> FeastResult:
        """feast_solve (core.hpp:264-391) on the uploaded pencil."""
        n = self.n
        self.n_e = config.n_e
        out, r = _result_buffers(n, config)
        y0 = None if initial_y is None else np.asfortranarray(initial_y, dtype=np.float64)
        if y0 is not None and y0.shape[0] != n:
            raise InputError("feast_solve: initial block shape mismatch")
        cfg = config.to_c()
        self._check(self.L.feast_gpu_solve(self.h, interval.lo, interval.hi, C.byref(cfg), abi.dptr(y0),
                                           0 if y0 is None else y0.shape[1], C.byref(r)))
        return _result_of(out, r, n)

    def set_pencil_hermitian(self, a, b):
        """Complex Hermitian pencil (SymmetricOperator<cplx>): operators of kind DENSE_Z / CSR_Z."""
        self._ca, self._cb = a.to_c(), b.to_c()
        self._check(self.L.feast_gpu_set_pencil_hermitian(self.h, C.byref(self._ca), C.byref(self._cb)))
        self.n = a.n

    def solve_hermitian(self, interval: SearchInterval, config: FeastConfig, initial_y=None) -> FeastResult:
        """feast_solve<cplx> (core.hpp:264-391) on the Hermitian pencil: complex eigenvectors and
        subspace, real eigenvalues."""
        n = self.n
        self.n_e = config.n_e
        out, r = _result_buffers(2 * n, config)  # complex n x m0 as interleaved real 2n x m0
        y0 = None if initial_y is None else np.asfortranarray(initial_y, dtype=np.complex128)
        if y0 is not None and y0.shape[0] != n:
            raise InputError("feast_solve: initial block shape mismatch")
        cfg = config.to_c()
        self._check(self.L.feast_gpu_solve_hermitian(self.h, interval.lo, interval.hi, C.byref(cfg), abi.zptr(y0),
                                                     0 if y0 is None else y0.shape[1], C.byref(r)))
        res = _result_of(out, r, 2 * n)
        to_c = lambda a: np.asfortranarray(a).reshape(-1, order="F").view(np.complex128).reshape((n, a.shape[1]), order="F")
        res.eigenvectors = to_c(res.eigenvectors)
        res.subspace = to_c(res.subspace)
        return res

    def sweep(self, a0, b, s, steps, interval: SearchInterval, config: FeastConfig):
        """run_sweep (run.cpp:63-125) on the device: one FeastResult per step, or the
        NumericalError a failed step raised (the next step then starts cold)."""
        steps = np.ascontiguousarray(steps, dtype=np.float64)
        n, k = a0.n, len(steps)
        self._ca, self._cb, self._cs = a0.to_c(), b.to_c(), s.to_c()
        bufs = [_result_buffers(n, config) for _ in range(k)]
        res = (abi.FeastResultT * max(k, 1))()
        for i, (_, r) in enumerate(bufs):
            res[i] = r
        codes = np.zeros(max(k, 1), dtype=np.int32)
        cfg = config.to_c()
        self._check(self.L.feast_gpu_sweep(self.h, C.byref(self._ca), C.byref(self._cb), C.byref(self._cs),
                                           abi.dptr(steps), k, interval.lo, interval.hi, C.byref(cfg), res,
                                           abi.iptr(codes)))
        self.n, self.n_e = n, config.n_e
        out = []
        for i in range(k):
            if codes[i] != 0:
                out.append(_CODES.get(int(codes[i]), Error)(f"step {i}: NumericalError"))
            else:
                out.append(_result_of(bufs[i][0], res[i], n))
        return out

    def bench_init(self, m0: int, seed: int = 42):
        self._check(self.L.feast_gpu_bench_init(self.h, m0, seed))

    def bench_passes(self, passes: int, flush_bytes: int = 0):
        """Device ms over `passes` loop bodies (L2 flushed between passes when flush_bytes)
        and phase ms {solve kernels, Q reduction+allreduce, Rayleigh-Ritz, dominant kernel}."""
        tot = C.c_double(0)
        ph = np.zeros(4)
        self._check(self.L.feast_gpu_bench_passes(self.h, passes, flush_bytes, C.byref(tot), abi.dptr(ph)))
        return tot.value, ph

    def launch_count(self) -> int:
        return int(self.L.feast_gpu_launch_count(self.h))


class LocalGroup:
    """feast_gpu_group: a loopback rank group of contexts inside one process (the collectives of
    the NCCL group through device copies and host barriers; include/feast_gpu.h)."""

    def __init__(self, nranks: int):
        self.L = load_library()
        h = C.c_void_p()
        if self.L.feast_gpu_group_create(int(nranks), C.byref(h)) != 0:
            raise InputError("feast_gpu_group_create failed")
        self.h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "h", None):
            self.L.feast_gpu_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_nodes(n_e: int, rank: int, nranks: int):
    """Contour nodes owned by `rank` (mirror of build_contour's split in feast_gpu.cpp):
    contiguous blocks in ascending e, [floor(n_e*r/R), floor(n_e*(r+1)/R))."""
    return range(n_e * rank // nranks, n_e * (rank + 1) // nranks)


def feast_solve(a, b, interval: SearchInterval, config: FeastConfig, initial_y=None,
                device: int = 0) -> FeastResult:
    """Drop-in for feast::feast_solve<double>(a, b, interval, config, nullptr, initial_y)."""
    ctx = GpuContext(device)
    try:
        ctx.set_pencil(a, b)
        return ctx.solve(interval, config, initial_y)
    finally:
        ctx.close()
