"""Seeded synthetic pencils for the five BASELINE.json configs (and scaled variants).

The reference ships no generator for these shapes (its generators.cpp builds FD/FEM
Laplacians only), so these are the stand-ins BASELINE.json names.
Draws use numpy's PCG64 (`np.random.default_rng(seed)`) in a fixed order; the
matrices are built one triangle at a time and mirrored so they are EXACTLY symmetric
(SymmetricOperator::from_dense / from_triplets reject any asymmetry,
operator.hpp:45-62,237-261). Both the GPU path and the CPU oracle read the same arrays.

Operators are held in the boundary's storage kinds (include/feast_gpu.h):
dense column-major, symmetric-complete CSR (int32), or block-tridiagonal
(diagonal blocks + lower couplings C_l = M(l+1, l)).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass
class Operator:
    kind: int
    n: int
    dense: Optional[np.ndarray] = None      # (n, n) Fortran order
    row_ptr: Optional[np.ndarray] = None
    col_idx: Optional[np.ndarray] = None
    values: Optional[np.ndarray] = None
    nblocks: int = 0
    bsize: int = 0
    diag: Optional[np.ndarray] = None       # (L, b, b): diag[l] is column-major b*b (stored [l, j, i])
    lower: Optional[np.ndarray] = None      # (L-1, b, b)
    _keep: list = field(default_factory=list, repr=False)

    # --- constructors -----------------------------------------------------
    @staticmethod
    def from_dense(m: np.ndarray) -> "Operator":
        m = np.asfortranarray(m, dtype=np.float64)
        assert m.shape[0] == m.shape[1]
        return Operator(abi.STORAGE_DENSE, m.shape[0], dense=m)

    @staticmethod
    def from_csr(n, row_ptr, col_idx, values) -> "Operator":
        return Operator(abi.STORAGE_CSR, n,
                        row_ptr=np.ascontiguousarray(row_ptr, dtype=np.int32),
                        col_idx=np.ascontiguousarray(col_idx, dtype=np.int32),
                        values=np.ascontiguousarray(values, dtype=np.float64))

    @staticmethod
    def from_blocktri(diag: np.ndarray, lower: np.ndarray) -> "Operator":
        """diag[l] / lower[l] given as ordinary (row, col) b*b numpy matrices."""
        L, b, _ = diag.shape
        # store each block column-major: element (i, j) at j*b + i  -> transpose the C-order block
        d = np.ascontiguousarray(np.transpose(diag, (0, 2, 1)), dtype=np.float64)
        lo = np.ascontiguousarray(np.transpose(lower, (0, 2, 1)), dtype=np.float64) if L > 1 \
            else np.zeros((0, b, b))
        return Operator(abi.STORAGE_BLOCKTRI, L * b, nblocks=L, bsize=b, diag=d, lower=lo)

    @staticmethod
    def from_dense_hermitian(m: np.ndarray) -> "Operator":
        """Complex Hermitian dense operator (SymmetricOperator<cplx>::from_dense)."""
        m = np.asfortranarray(m, dtype=np.complex128)
        assert m.shape[0] == m.shape[1]
        return Operator(abi.STORAGE_DENSE_Z, m.shape[0], dense=m)

    @staticmethod
    def from_csr_hermitian(n, row_ptr, col_idx, values) -> "Operator":
        """Complex Hermitian-complete CSR operator (SymmetricOperator<cplx>, Full layout)."""
        return Operator(abi.STORAGE_CSR_Z, n,
                        row_ptr=np.ascontiguousarray(row_ptr, dtype=np.int32),
                        col_idx=np.ascontiguousarray(col_idx, dtype=np.int32),
                        values=np.ascontiguousarray(values, dtype=np.complex128))

    @property
    def is_complex(self) -> bool:
        return self.kind in (abi.STORAGE_DENSE_Z, abi.STORAGE_CSR_Z)

    @staticmethod
    def identity_csr(n: int) -> "Operator":
        return Operator.from_csr(n, np.arange(n + 1), np.arange(n), np.ones(n))

    # --- views ------------------------------------------------------------
    def diag_block(self, l):
        return self.diag[l].T

    def lower_block(self, l):
        return self.lower[l].T

    def to_c(self) -> abi.FeastOperatorT:
        s = abi.FeastOperatorT()
        s.kind, s.n = self.kind, self.n
        s.dense = abi.zptr(self.dense) if self.is_complex else abi.dptr(self.dense)
        s.row_ptr = abi.iptr(self.row_ptr)
        s.col_idx = abi.iptr(self.col_idx)
        s.values = abi.zptr(self.values) if self.is_complex else abi.dptr(self.values)
        s.nblocks, s.bsize = self.nblocks, self.bsize
        s.diag = abi.dptr(self.diag)
        s.lower = abi.dptr(self.lower)
        return s

    def to_dense(self) -> np.ndarray:
        n = self.n
        if self.kind in (abi.STORAGE_DENSE, abi.STORAGE_DENSE_Z):
            return np.array(self.dense)
        m = np.zeros((n, n), dtype=np.complex128 if self.is_complex else np.float64)
        if self.kind in (abi.STORAGE_CSR, abi.STORAGE_CSR_Z):
            rows = np.repeat(np.arange(n), np.diff(self.row_ptr))
            m[rows, self.col_idx] = self.values
            return m
        b = self.bsize
        for l in range(self.nblocks):
            m[l * b:(l + 1) * b, l * b:(l + 1) * b] = self.diag_block(l)
            if l + 1 < self.nblocks:
                c = self.lower_block(l)
                m[(l + 1) * b:(l + 2) * b, l * b:(l + 1) * b] = c
                m[l * b:(l + 1) * b, (l + 1) * b:(l + 2) * b] = c.T
        return m

    def to_scipy(self):
        import scipy.sparse as sp
        if self.kind in (abi.STORAGE_DENSE, abi.STORAGE_DENSE_Z):
            return sp.csr_matrix(self.dense)
        if self.kind in (abi.STORAGE_CSR, abi.STORAGE_CSR_Z):
            return sp.csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.n, self.n))
        L, b = self.nblocks, self.bsize
        blocks = [[None] * L for _ in range(L)]
        for l in range(L):
            blocks[l][l] = sp.csr_matrix(self.diag_block(l))
            if l + 1 < L:
                c = sp.csr_matrix(self.lower_block(l))
                blocks[l + 1][l] = c
                blocks[l][l + 1] = c.T
        return sp.bmat(blocks, format="csr")

    def matmul(self, x: np.ndarray) -> np.ndarray:
        if self.kind in (abi.STORAGE_DENSE, abi.STORAGE_DENSE_Z):
            return self.dense @ x
        return self.to_scipy() @ x


@dataclass
class Problem:
    name: str
    a: Operator
    b: Operator
    emin: float
    emax: float
    m0: int
    n_e: int = 8
    trace_tol: float = 1e-13
    max_loops: int = 20
    seed: int = 42
    expected_count: Optional[int] = None
    note: str = ""

    @property
    def n(self):
        return self.a.n


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def _sym_from_upper(u: np.ndarray) -> np.ndarray:
    """Mirror the upper triangle (incl. diagonal) of u: exactly symmetric."""
    m = np.triu(u)
    return m + np.triu(m, 1).T


def banded_csr(n: int, diag: np.ndarray, offdiag: dict) -> Operator:
    """Symmetric banded CSR from its diagonal and {offset d: values for (i, i+d)}."""
    import scipy.sparse as sp
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    vals = [diag]
    for d, v in offdiag.items():
        i = np.arange(n - d)
        rows += [i, i + d]
        cols += [i + d, i]
        vals += [v, v]
    m = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    m.sort_indices()
    return Operator.from_csr(n, m.indptr, m.indices, m.data)


def csr_bandwidth(op: Operator) -> int:
    rows = np.repeat(np.arange(op.n), np.diff(op.row_ptr))
    return int(np.max(np.abs(rows - op.col_idx))) if len(rows) else 0


# ---------------------------------------------------------------------------
# Inertia (Sylvester) counts: #eigenvalues of (A, B) below sigma
# ---------------------------------------------------------------------------
def _neg_count_sym(m: np.ndarray) -> int:
    return int(np.sum(np.linalg.eigvalsh(m) < 0.0))


def inertia_count(a: Operator, b: Operator, sigma: float) -> int:
    """Number of eigenvalues of A x = lambda B x strictly below sigma (B SPD):
    negative inertia of A - sigma B. Dense: eigvalsh; block-tridiagonal / banded CSR:
    Haynsworth additivity over the block-LDL^T Schur complements."""
    if a.kind == abi.STORAGE_DENSE or b.kind == abi.STORAGE_DENSE:
        return _neg_count_sym(a.to_dense() - sigma * b.to_dense())
    if a.kind == abi.STORAGE_BLOCKTRI and b.kind == abi.STORAGE_BLOCKTRI:
        L, bs = a.nblocks, a.bsize
        get_d = lambda l: a.diag_block(l) - sigma * b.diag_block(l)
        get_c = lambda l: a.lower_block(l) - sigma * b.lower_block(l)
    else:
        bw = max(csr_bandwidth(a), csr_bandwidth(b))
        bs = max(bw, 1)
        sa, sb = a.to_scipy(), b.to_scipy()
        m = (sa - sigma * sb).tocsr()
        n = a.n
        L = (n + bs - 1) // bs

        def dense_block(r0, r1, c0, c1):
            return m[r0:r1, c0:c1].toarray()
        get_d = lambda l: dense_block(l * bs, min(n, (l + 1) * bs), l * bs, min(n, (l + 1) * bs))
        get_c = lambda l: dense_block((l + 1) * bs, min(n, (l + 2) * bs), l * bs, min(n, (l + 1) * bs))
    count = 0
    s = get_d(0)
    for l in range(L):
        w, v = np.linalg.eigh(s)
        count += int(np.sum(w < 0.0))
        if l + 1 < L:
            c = get_c(l)
            # S_{l+1} = D_{l+1} - C_l S_l^{-1} C_l^T via the eigen-decomposition of S_l
            t = c @ v
            s = get_d(l + 1) - (t / w) @ t.T
            s = 0.5 * (s + s.T)
    return count


def interval_with_count(a: Operator, b: Operator, want: int, start: float, span: float,
                        rel_gap: float = 1e-3, max_iter: int = 80):
    """[lo, hi] holding exactly `want` eigenvalues, lo just below the first
    eigenvalue >= start, endpoints at gap midpoints located by bisection on the
    inertia count (the Sturm count the BASELINE configs call for)."""
    c0 = inertia_count(a, b, start)

    def locate(k):  # bracket eigenvalue index k (0-based): count(x) <= k < count(y)
        lo, hi = start - span, start + span
        while inertia_count(a, b, lo) > k:
            lo -= span
        while inertia_count(a, b, hi) <= k:
            hi += span
        for _ in range(max_iter):
            mid = 0.5 * (lo + hi)
            if inertia_count(a, b, mid) <= k:
                lo = mid
            else:
                hi = mid
            if hi - lo < 1e-13 * max(1.0, abs(mid)):
                break
        return 0.5 * (lo + hi)

    lam_prev, lam_first = locate(c0 - 1), locate(c0)
    lam_last, lam_next = locate(c0 + want - 1), locate(c0 + want)
    lo = 0.5 * (lam_prev + lam_first)
    hi = 0.5 * (lam_last + lam_next)
    assert inertia_count(a, b, hi) - inertia_count(a, b, lo) == want
    return lo, hi, dict(lam_prev=lam_prev, lam_first=lam_first, lam_last=lam_last,
                        lam_next=lam_next)


# ---------------------------------------------------------------------------
# The five configs (BASELINE.json "configs"), each with a scale knob for tests
# ---------------------------------------------------------------------------
def config1(n: int = 1024, seed: int = 1, m0: int = 160, emin=-1.0, emax=1.0,
            yseed: int = 42) -> Problem:
    """Dense standard problem: A = U diag(lam) U^T, U from QR of a Gaussian matrix,
    lam ~ U[-10, 10], B = I (identity CSR); interval [-1, 1]; Ne=8, trace_tol=1e-12.
    The reference has only the circle contour (quadrature.cpp:83-84), so
    the config's 'half-ellipse' is the circle (aspect 1)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    u, _ = np.linalg.qr(g)
    lam = rng.uniform(-10.0, 10.0, n)
    a = (u * lam) @ u.T
    a = 0.5 * (a + a.T)
    count = int(np.sum((lam >= emin) & (lam <= emax)))
    return Problem(f"cfg1_dense_n{n}", Operator.from_dense(a), Operator.identity_csr(n),
                   emin, emax, m0, n_e=8, trace_tol=1e-12, max_loops=20, seed=yseed,
                   expected_count=count, note="lam known by construction")


def config2_operators(n: int = 16384, bw: int = 16, seed: int = 2):
    rng = np.random.default_rng(seed)
    ad = rng.uniform(-2.0, 2.0, n)
    aoff = {}
    for d in range(1, bw + 1):
        aoff[d] = -1.0 / (1.0 + d) * rng.uniform(0.5, 1.5, n - d)
    boff = {}
    for d in range(1, bw + 1):
        boff[d] = 0.05 * rng.uniform(-1.0, 1.0, n - d)
    bd = np.ones(n)
    # diagonal shift so lambda_min(B) >= 0.5 (LAPACK band eigensolver on B)
    from scipy.linalg import eigvals_banded
    band = np.zeros((bw + 1, n))
    band[0] = bd
    for d in range(1, bw + 1):
        band[d, : n - d] = boff[d]
    lmin = float(eigvals_banded(band, lower=True, select="i", select_range=(0, 0))[0])
    if lmin < 0.5:
        bd = bd + (0.5 - lmin)
    return banded_csr(n, ad, aoff), banded_csr(n, bd, boff), lmin


def blocktri_operators(L: int, b: int, seed: int, coupling_density: float = 0.10):
    """Block-tridiagonal 'nanotube-like' pencil (configs 3 and 5).
    A: diagonal blocks symmetric, N(0,1)/sqrt(b) entries (upper triangle mirrored) plus
    onsite energies U[-1,1] on the diagonal; couplings sparse, 10% of entries drawn from
    N(0, 0.5) read as VARIANCE 0.5 (std sqrt(0.5)) — BASELINE leaves variance-vs-std open.
    B: I diagonal blocks, dense 0.02 * N(0,1)/sqrt(b) couplings."""
    rng = np.random.default_rng(seed)
    sb = 1.0 / np.sqrt(b)
    diag = np.empty((L, b, b))
    for l in range(L):
        d = _sym_from_upper(rng.standard_normal((b, b)) * sb)
        d[np.diag_indices(b)] += rng.uniform(-1.0, 1.0, b)
        diag[l] = d
    lower = np.empty((max(L - 1, 0), b, b))
    for l in range(L - 1):
        mask = rng.random((b, b)) < coupling_density
        lower[l] = np.where(mask, rng.standard_normal((b, b)) * np.sqrt(0.5), 0.0)
    bdiag = np.broadcast_to(np.eye(b), (L, b, b)).copy()
    blower = np.empty((max(L - 1, 0), b, b))
    for l in range(L - 1):
        blower[l] = 0.02 * sb * rng.standard_normal((b, b))
    return Operator.from_blocktri(diag, lower), Operator.from_blocktri(bdiag, blower)


def _cached_interval(key: str, compute):
    path = os.path.join(_HERE, "intervals.json")
    table = {}
    if os.path.exists(path):
        with open(path) as f:
            table = json.load(f)
    if key in table:
        return table[key]["lo"], table[key]["hi"]
    lo, hi, info = compute()
    table[key] = dict(lo=lo, hi=hi, **info)
    try:
        with open(path, "w") as f:
            json.dump(table, f, indent=1, sort_keys=True)
    except OSError:
        pass
    return lo, hi


def config2(n: int = 16384, bw: int = 16, seed: int = 2, m0: int = 192, want: int = 128,
            yseed: int = 42) -> Problem:
    a, b, _ = config2_operators(n, bw, seed)
    lo, hi = _cached_interval(f"cfg2_n{n}_bw{bw}_s{seed}_k{want}",
                              lambda: interval_with_count(a, b, want, start=0.0, span=0.5))
    return Problem(f"cfg2_band_n{n}", a, b, lo, hi, m0, n_e=8, seed=yseed,
                   expected_count=want)


def config3(L: int = 256, b: int = 256, seed: int = 3, m0: int = 300, want: int = 200,
            n_e: int = 8, yseed: int = 42) -> Problem:
    a, bb = blocktri_operators(L, b, seed)
    lo, hi = _cached_interval(f"blocktri_L{L}_b{b}_s{seed}_k{want}",
                              lambda: interval_with_count(a, bb, want, start=0.0, span=0.25))
    return Problem(f"cfg3_blocktri_L{L}_b{b}", a, bb, lo, hi, m0, n_e=n_e, seed=yseed,
                   expected_count=want)


def config4(n: int = 8192, seed: int = 4, m0: int = 600, want: int = 400,
            yseed: int = 42) -> Problem:
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n)) / np.sqrt(n)
    a = 0.5 * (g + g.T)
    h = rng.standard_normal((n, n))
    bm = np.eye(n) + 0.1 * (h @ h.T) / n
    bm = 0.5 * (bm + bm.T)
    A, B = Operator.from_dense(a), Operator.from_dense(bm)

    def dense_interval():
        # all generalized eigenvalues once (LAPACK sygvd), then gap midpoints around `want`
        # consecutive eigenvalues starting at the first one >= 0
        import scipy.linalg as sl
        ev = sl.eigh(a, bm, eigvals_only=True)
        k0 = int(np.searchsorted(ev, 0.0))
        lo_, hi_ = 0.5 * (ev[k0 - 1] + ev[k0]), 0.5 * (ev[k0 + want - 1] + ev[k0 + want])
        return lo_, hi_, dict(lam_prev=float(ev[k0 - 1]), lam_first=float(ev[k0]),
                              lam_last=float(ev[k0 + want - 1]), lam_next=float(ev[k0 + want]))
    lo, hi = _cached_interval(f"cfg4_n{n}_s{seed}_k{want}", dense_interval)
    return Problem(f"cfg4_dense_n{n}", A, B, lo, hi, m0, n_e=8, seed=yseed,
                   expected_count=want)


def config5(L: int = 2048, b: int = 512, seed: int = 5, m0: int = 768, want: int = 512,
            yseed: int = 42) -> Problem:
    p = config3(L=L, b=b, seed=seed, m0=m0, want=want, n_e=16, yseed=yseed)
    p.name = f"cfg5_blocktri_L{L}_b{b}"
    return p


def small_dense(n: int = 60, seed: int = 7, want: int = 6, m0: int = 10, gen: bool = True,
                yseed: int = 42) -> Problem:
    """Random dense symmetric A and SPD B (generalized), interval at gap midpoints
    around `want` eigenvalues — the shape of test_core.cpp:94-109 / acceptance.cpp:344."""
    rng = np.random.default_rng(seed)
    a = _sym_from_upper(rng.uniform(-1, 1, (n, n)))
    if gen:
        r = rng.uniform(-1, 1, (n, n))
        bm = r.T @ r / n + np.eye(n)
        bm = _sym_from_upper(bm)
    else:
        bm = np.eye(n)
    import scipy.linalg as sl
    ev = sl.eigh(a, bm, eigvals_only=True)
    start = n // 3
    lo = 0.5 * (ev[start - 1] + ev[start])
    hi = 0.5 * (ev[start + want - 1] + ev[start + want])
    return Problem(f"small_dense_n{n}", Operator.from_dense(a), Operator.from_dense(bm),
                   lo, hi, m0, seed=yseed, expected_count=want)
