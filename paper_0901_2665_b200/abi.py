"""ctypes mirror of include/feast_gpu.h (the C-ABI boundary).

Shared by the product wrapper (feast.py) and the test-only oracle loader
(oracle/oracle.py): both libraries speak the same structs.
"""
from __future__ import annotations

import ctypes as C

FEAST_OK = 0
FEAST_EINPUT = 4
FEAST_ENUMERICAL = 5
FEAST_EBREAKDOWN = 6
FEAST_ECUDA = 7
FEAST_ENCCL = 8
FEAST_EINTERNAL = 9

STORAGE_DENSE = 0
STORAGE_CSR = 1
STORAGE_BLOCKTRI = 2
STORAGE_DENSE_Z = 16   # complex Hermitian, interleaved (feast_gpu_set_pencil_hermitian)
STORAGE_CSR_Z = 17

# feast_run_status_t == feast::FeastStatus order (core.hpp:35-41)
STATUS_NAMES = ["converged", "max-loops", "no-eigenvalues-in-interval",
                "subspace-saturated", "subspace-breakdown"]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class FeastOperatorT(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("n", C.c_int32),
        ("dense", _dp),
        ("row_ptr", _ip),
        ("col_idx", _ip),
        ("values", _dp),
        ("nblocks", C.c_int32),
        ("bsize", C.c_int32),
        ("diag", _dp),
        ("lower", _dp),
    ]


class FeastConfigT(C.Structure):
    _fields_ = [
        ("m0", C.c_int32),
        ("n_e", C.c_int32),
        ("trace_tol", C.c_double),
        ("max_loops", C.c_int32),
        ("seed", C.c_uint64),
        ("threads", C.c_int32),
        ("low_memory", C.c_int32),
    ]


class FeastResultT(C.Structure):
    _fields_ = [
        ("eigenvalues", _dp),
        ("eigenvectors", _dp),
        ("residuals", _dp),
        ("residual_absolute_only", _ip),
        ("trace_history", _dp),
        ("in_interval_counts", _ip),
        ("subspace", _dp),
        ("m", C.c_int32),
        ("subspace_cols", C.c_int32),
        ("loops_used", C.c_int32),
        ("status", C.c_int32),
        ("max_residual", C.c_double),
        ("factorize_s", C.c_double),
        ("solve_s", C.c_double),
        ("reduce_s", C.c_double),
        ("total_s", C.c_double),
    ]


def dptr(a):
    """double* into a C-contiguous float64 numpy array (or NULL)."""
    if a is None:
        return C.cast(None, _dp)
    assert a.dtype.name == "float64" and a.flags["C_CONTIGUOUS"] or a.flags["F_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def zptr(a):
    """double* over the interleaved (re, im) pairs of a contiguous complex128 array (or NULL)."""
    if a is None:
        return C.cast(None, _dp)
    assert a.dtype.name == "complex128" and (a.flags["C_CONTIGUOUS"] or a.flags["F_CONTIGUOUS"])
    return a.ctypes.data_as(_dp)


def iptr(a):
    if a is None:
        return C.cast(None, _ip)
    assert a.dtype.name == "int32"
    return a.ctypes.data_as(_ip)
