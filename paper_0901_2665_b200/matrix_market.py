"""Matrix Market input at the boundary: the reference's reader and writer
(`src/matrix_market.cpp:33-166`, declared in `include/feast/matrix_market.hpp:17-25`) and the
triplet assembly they feed (`SymmetricOperator::from_triplets`, `operator.hpp:66-104`), producing
the symmetric-complete CSR `Operator` that `feast.GpuContext.set_pencil` uploads (where the device
ingestion of `csr_ingest.cu` validates and re-blocks it).

Same accepted files and the same `InputError` messages ("<path>:<line>: <what>"): a
`%%MatrixMarket matrix coordinate real symmetric` banner (a `complex hermitian` file is parsed
and then rejected, as by `load_matrix_market_real`), `%` comment and blank lines skipped, a size
line, 1-based entries; the lower-triangle entries are mirrored, duplicates are summed in file
order after a stable (row, col) sort, and the writer emits the lower triangle with `%.17g`.
"""
from __future__ import annotations

import re

import numpy as np

from .feast import InputError
from .problems import Operator


def _fail(path, line, what):
    raise InputError(f"{path}:{line}: {what}")


_WS = " \t\n\v\f\r"  # isspace() in the "C" locale
_INT = re.compile(r"[+-]?[0-9]+")
_FLT = re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]*)(?:[eE][+-]?[0-9]*)?")
_FLT_FULL = re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")
_LL_MAX = (1 << 63) - 1


class _Stream:
    """std::istringstream >> for long long and double (libstdc++ num_get, "C" locale): skip
    isspace(), take the longest prefix the numeric grammar accepts (so '3.0' read as an integer
    yields 3 and leaves '.0', and '1.5d0' read as a double yields 1.5 and leaves 'd0'), then
    convert; no digits, an incomplete exponent ('1e'), 'nan' / 'inf' and out-of-range values set
    the fail bit, and every later extraction fails too."""

    def __init__(self, line):
        self.s, self.pos, self.failed = line, 0, False

    def _skip(self):
        while self.pos < len(self.s) and self.s[self.pos] in _WS:
            self.pos += 1

    def integer(self):
        if self.failed:
            return None
        self._skip()
        m = _INT.match(self.s, self.pos)
        if not m:
            self.failed = True
            return None
        self.pos = m.end()
        v = int(m.group())
        if v > _LL_MAX or v < -_LL_MAX - 1:
            self.failed = True
            return None
        return v

    def real(self):
        if self.failed:
            return None
        self._skip()
        m = _FLT.match(self.s, self.pos)
        if not m or not m.group():
            self.failed = True
            return None
        self.pos = m.end()
        txt = m.group()
        if not _FLT_FULL.fullmatch(txt):  # strtod must consume everything num_get collected
            self.failed = True
            return None
        v = float(txt)
        if v in (float("inf"), float("-inf")):
            self.failed = True
            return None
        return v


def _words(line):
    return [w for w in re.split("[" + _WS + "]+", line) if w]


def _parse(path):
    """matrix_market.cpp:33-102: (n, complex_field, rows0, cols0, re)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise InputError("cannot open matrix file: " + str(path)) from None
    with f:
        # std::getline splits on '\n' only: a '\r' of a CRLF file stays in its line
        lines = f.read().decode("latin-1").split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline: a trailing newline ends the last line, it is not a line
    if not lines:
        _fail(path, 1, "empty file")
    lineno = 1
    head = _words(lines[0])
    banner, obj, fmt, field, sym = (head + [""] * 5)[:5]
    if banner != "%%MatrixMarket":
        _fail(path, lineno, "missing MatrixMarket banner")
    if obj.lower() != "matrix":
        _fail(path, lineno, "unsupported object: " + obj)
    if fmt.lower() != "coordinate":
        _fail(path, lineno, "unsupported format (coordinate required): " + fmt)
    field, sym = field.lower(), sym.lower()
    if field == "real" and sym == "symmetric":
        cplx = False
    elif field == "complex" and sym == "hermitian":
        cplx = True
    else:
        _fail(path, lineno, f"symmetry flag mismatch: need 'real symmetric' or 'complex hermitian', "
                            f"got '{field} {sym}'")
    pos = 1
    rows = cols = count = -1
    while pos < len(lines):
        line = lines[pos]
        pos += 1
        lineno += 1
        if not line or line[0] == "%":
            continue
        ls = _Stream(line)
        rows, cols, count = ls.integer(), ls.integer(), ls.integer()
        if ls.failed:
            _fail(path, lineno, "malformed size line")
        break
    if rows < 0:
        _fail(path, lineno, "missing size line")
    if rows != cols:
        _fail(path, lineno, "matrix is not square")
    if rows < 1:
        _fail(path, lineno, "matrix dimension must be positive")
    if count < 0:
        _fail(path, lineno, "negative entry count")
    ii = np.empty(count, np.int64)
    jj = np.empty(count, np.int64)
    re_ = np.empty(count, np.float64)
    seen = 0
    while seen < count:
        if pos >= len(lines):
            _fail(path, lineno + 1, "unexpected end of file")
        line = lines[pos]
        pos += 1
        lineno += 1
        if not line or line[0] == "%":
            continue
        ls = _Stream(line)
        i, j, v = ls.integer(), ls.integer(), ls.real()
        if ls.failed:
            _fail(path, lineno, "malformed entry")
        if cplx:
            ls.real()
            if ls.failed:
                _fail(path, lineno, "missing imaginary part")
        if i < 1 or i > rows or j < 1 or j > cols:
            _fail(path, lineno, "index out of range")
        ii[seen], jj[seen], re_[seen] = i - 1, j - 1, v
        seen += 1
    return int(rows), cplx, ii, jj, re_


def operator_from_triplets(n, rows, cols, values, mirror_off_diagonal=True) -> Operator:
    """SymmetricOperator::from_triplets (operator.hpp:66-104) for real values: mirror the
    off-diagonal entries (MirrorOffDiagonal), stable (row, col) sort, sum duplicates in order,
    then the symmetry check of validate_sparse_symmetry."""
    if n <= 0:
        raise InputError("SymmetricOperator: dimension must be positive")
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    values = np.asarray(values, np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= n):
        raise InputError("SymmetricOperator: triplet index out of range")
    if mirror_off_diagonal:
        off = rows != cols
        # interleave each entry with its mirror (all.push_back(t); all.push_back(mirror))
        k = np.arange(rows.size)
        order_key = np.concatenate([2 * k, 2 * k[off] + 1])
        r = np.concatenate([rows, cols[off]])
        c = np.concatenate([cols, rows[off]])
        v = np.concatenate([values, values[off]])
        o = np.argsort(order_key, kind="stable")
        r, c, v = r[o], c[o], v[o]
    else:
        r, c, v = rows, cols, values
    o = np.lexsort((c, r))  # stable: ties keep insertion order
    r, c, v = r[o], c[o], v[o]
    if r.size:
        start = np.flatnonzero(np.concatenate([[True], (r[1:] != r[:-1]) | (c[1:] != c[:-1])]))
        end = np.append(start[1:], r.size)
        sums = v[start] + 0.0  # T v{}; v += x: 0.0 + x (turns -0.0 into +0.0, as the reference)
        for q in np.flatnonzero(end - start > 1):  # duplicates: summed in order
            sums[q] = _seq_sum(v[start[q]:end[q]])
        r, c = r[start], c[start]
    else:
        sums = v
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    _check_symmetry(n, row_ptr, c, sums)
    return Operator.from_csr(n, row_ptr, c, sums)


def _seq_sum(x):
    s = 0.0
    for t in x:
        s += float(t)
    return s


def _check_symmetry(n, row_ptr, col, val):
    """validate_sparse_symmetry (operator.hpp:237-261): every off-diagonal entry has a mirror
    with the same value."""
    r = np.repeat(np.arange(n), np.diff(row_ptr))
    up = col > r
    lo = col < r
    key_up = r[up] * n + col[up]
    key_lo = col[lo] * n + r[lo]  # (j, i) stored at row i: mirror of (i, j)
    if key_up.size != key_lo.size:
        raise InputError("SymmetricOperator: missing mirror entry")
    ou, ol = np.argsort(key_up, kind="stable"), np.argsort(key_lo, kind="stable")
    if not np.array_equal(key_up[ou], key_lo[ol]):
        raise InputError("SymmetricOperator: missing mirror entry")
    if not np.array_equal(val[up][ou], val[lo][ol]):
        raise InputError("SymmetricOperator: mirror entries disagree")


def load_matrix_market_real(path) -> Operator:
    """load_matrix_market_real (matrix_market.cpp:106-116)."""
    n, cplx, ii, jj, re = _parse(path)
    if cplx:
        raise InputError(f"{path}: symmetry flag mismatch: real symmetric input required")
    return operator_from_triplets(n, ii, jj, re, mirror_off_diagonal=True)


def save_matrix_market(path, op: Operator) -> None:
    """save_matrix_market (matrix_market.cpp:124-166) for real operators: the stored entries with
    column <= row (all of the lower triangle for dense storage), 1-based, %.17g."""
    try:
        f = open(path, "w")
    except OSError:
        raise InputError("cannot write matrix file: " + str(path)) from None
    with f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        if op.row_ptr is not None:
            n = op.n
            r = np.repeat(np.arange(n), np.diff(op.row_ptr))
            keep = op.col_idx <= r
            rr, cc, vv = r[keep], op.col_idx[keep], op.values[keep]
        else:
            m = op.dense if op.dense is not None else _blocktri_dense(op)
            n = op.n
            rr, cc = np.tril_indices(n)
            vv = m[rr, cc]
        f.write(f"{n} {n} {rr.size}\n")
        f.writelines(f"{i + 1} {j + 1} {v:.17g}\n" for i, j, v in zip(rr.tolist(), cc.tolist(), vv.tolist()))


def _blocktri_dense(op):
    n, b = op.n, op.bsize
    m = np.zeros((n, n))
    for l in range(op.nblocks):
        m[l * b:(l + 1) * b, l * b:(l + 1) * b] = op.diag_block(l)
        if l + 1 < op.nblocks:
            c = op.lower_block(l)
            m[(l + 1) * b:(l + 2) * b, l * b:(l + 1) * b] = c
            m[l * b:(l + 1) * b, (l + 1) * b:(l + 2) * b] = c.T
    return m
