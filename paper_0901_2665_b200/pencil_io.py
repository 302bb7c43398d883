"""Binary pencil files at the boundary: a format for operators too large
for Matrix Market text (config 5: A and B are 8.6 GB each as block-tridiagonal storage, ~20 GB of
text), read back through a memory map so the upload streams straight from the page cache.

Layout (little-endian), one operator per file:

    offset  size  field
    0       8     magic  b"FEASTOP1"
    8       4     kind   (0 dense, 1 CSR, 2 block-tridiagonal: include/feast_gpu.h feast_storage_t)
    12      4     reserved (0)
    16      8     n
    24      8     nnz      (CSR; 0 otherwise)
    32      8     nblocks  (block-tridiagonal; 0 otherwise)
    40      8     bsize    (block-tridiagonal; 0 otherwise)
    48      16    reserved (0)
    64      ...   payload, each array 64-byte aligned:
                    dense: n*n float64, column-major
                    CSR:   row_ptr int32[n+1], col_idx int32[nnz], values float64[nnz]
                    block-tridiagonal: diag float64[nblocks*b*b] (each block column-major),
                                       lower float64[(nblocks-1)*b*b] (C_l = M(l+1, l))

The arrays are the boundary's own storage kinds, so a loaded operator goes to
`GpuContext.set_pencil` unchanged (no conversion, no copy beyond the memory map)."""
from __future__ import annotations

import os
import struct

import numpy as np

from . import abi
from .feast import InputError
from .problems import Operator

MAGIC = b"FEASTOP1"
HEADER = struct.Struct("<8sii4q16x")
ALIGN = 64


def _pad(off):
    return (off + ALIGN - 1) // ALIGN * ALIGN


def _arrays(op):
    if op.kind == abi.STORAGE_DENSE:
        return [np.asfortranarray(op.dense, dtype=np.float64).reshape(-1, order="F")]
    if op.kind == abi.STORAGE_CSR:
        return [np.ascontiguousarray(op.row_ptr, np.int32), np.ascontiguousarray(op.col_idx, np.int32),
                np.ascontiguousarray(op.values, np.float64)]
    return [np.ascontiguousarray(op.diag, np.float64).reshape(-1), np.ascontiguousarray(op.lower, np.float64).reshape(-1)]


def save_operator(path, op: Operator):
    nnz = int(op.row_ptr[op.n]) if op.kind == abi.STORAGE_CSR else 0
    head = HEADER.pack(MAGIC, int(op.kind), 0, int(op.n), nnz, int(op.nblocks), int(op.bsize))
    with open(path, "wb") as f:
        f.write(head)
        f.write(b"\0" * (ALIGN - len(head)))
        for arr in _arrays(op):
            off = f.tell()
            if off % ALIGN:
                f.write(b"\0" * (_pad(off) - off))
            arr.tofile(f)


def load_operator(path, mmap: bool = True) -> Operator:
    """The operator of a FEASTOP1 file; arrays are read-only memory maps unless mmap=False."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(HEADER.size)
    if len(head) < HEADER.size:
        raise InputError(f"{path}: truncated header")
    magic, kind, _, n, nnz, nblocks, bsize = HEADER.unpack(head)
    if magic != MAGIC:
        raise InputError(f"{path}: not a FEASTOP1 operator file")
    if n < 1 or kind not in (abi.STORAGE_DENSE, abi.STORAGE_CSR, abi.STORAGE_BLOCKTRI):
        raise InputError(f"{path}: bad header (kind {kind}, n {n})")
    if kind == abi.STORAGE_DENSE:
        specs = [(np.float64, n * n)]
    elif kind == abi.STORAGE_CSR:
        specs = [(np.int32, n + 1), (np.int32, nnz), (np.float64, nnz)]
    else:
        if nblocks * bsize != n or bsize < 1:
            raise InputError(f"{path}: bad block-tridiagonal shape ({nblocks} x {bsize} != {n})")
        specs = [(np.float64, nblocks * bsize * bsize), (np.float64, max(nblocks - 1, 0) * bsize * bsize)]
    arrays, off = [], ALIGN
    for dt, cnt in specs:
        off = _pad(off)
        nbytes = cnt * np.dtype(dt).itemsize
        if off + nbytes > size:
            raise InputError(f"{path}: truncated payload")
        if mmap:
            arrays.append(np.memmap(path, dtype=dt, mode="r", offset=off, shape=(cnt,)) if cnt else np.zeros(0, dt))
        else:
            arrays.append(np.fromfile(path, dtype=dt, count=cnt, offset=off))
        off += nbytes
    if kind == abi.STORAGE_DENSE:
        return Operator(kind, n, dense=arrays[0].reshape((n, n), order="F"))
    if kind == abi.STORAGE_CSR:
        if arrays[0][0] != 0 or arrays[0][n] != nnz:
            raise InputError(f"{path}: CSR row pointers do not span the entries")
        return Operator(kind, n, row_ptr=arrays[0], col_idx=arrays[1], values=arrays[2])
    return Operator(kind, n, nblocks=nblocks, bsize=bsize, diag=arrays[0].reshape((nblocks, bsize, bsize)),
                    lower=arrays[1].reshape((max(nblocks - 1, 0), bsize, bsize)))
