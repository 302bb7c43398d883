"""Complex Hermitian pencils: feast_gpu_set_pencil_hermitian /
feast_gpu_solve_hermitian against the reference's own feast_solve<cplx> (core.hpp:264-391 with
T = std::complex<double>; SymmetricOperator<cplx>, DenseLU / BandedLU over complex shifted
systems, complex Jacobi for the reduced problem) on the same seeded inputs: same status and count,
eigenvalues within 1e-10 relative, complex principal angles <= 1e-8 in the B inner product,
residuals (complex moduli, residual.hpp:29-68) at the reference's level; plus the reference's
input validation and a multiplicity case (test_core.cpp:242-310 covers the complex path)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_0901_2665_b200 import problems as P

pytestmark = pytest.mark.gpu


def herm(m):
    """exactly Hermitian: upper triangle mirrored with conjugation, real diagonal"""
    u = np.triu(m)
    h = u + np.triu(u, 1).conj().T
    h[np.diag_indices(len(h))] = h[np.diag_indices(len(h))].real
    return np.asfortranarray(h)


def dense_pencil(n=60, seed=3):
    rng = np.random.default_rng(seed)
    a = herm(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    h = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = herm(np.eye(n) + h @ h.conj().T / (4 * n))
    return a, b


def banded_csr(n, bw, seed, spd=False):
    rng = np.random.default_rng(seed)
    m = np.zeros((n, n), dtype=np.complex128)
    for d in range(1, bw + 1):
        v = (rng.uniform(-1, 1, n - d) + 1j * rng.uniform(-1, 1, n - d)) * (0.05 if spd else 1.0 / (1 + d))
        m[np.arange(n - d) + d, np.arange(n - d)] = v
    m = m + m.conj().T
    m[np.diag_indices(n)] = 1.0 if spd else rng.uniform(-2, 2, n)
    import scipy.sparse as sp
    s = sp.csr_matrix(m)
    s.sort_indices()
    return P.Operator.from_csr_hermitian(n, s.indptr, s.indices, s.data), m


def interval_around(a, b, k0, k):
    import scipy.linalg as sl
    ev = sl.eigh(a, b, eigvals_only=True)
    return 0.5 * (ev[k0 - 1] + ev[k0]), 0.5 * (ev[k0 + k - 1] + ev[k0 + k]), ev[k0:k0 + k]


def sin_angle_c(x, xr, b):
    def borth(v):
        g = v.conj().T @ (b @ v)
        w, u = np.linalg.eigh(0.5 * (g + g.conj().T))
        return v @ (u / np.sqrt(w))
    x, xr = borth(x), borth(xr)
    r = x - xr @ (xr.conj().T @ (b @ x))
    g = r.conj().T @ (b @ r)
    return float(np.sqrt(max(np.max(np.linalg.eigvalsh(0.5 * (g + g.conj().T))), 0.0)))


def run_gpu(A, B, lo, hi, m0, **kw):
    from paper_0901_2665_b200 import feast as F
    c = F.GpuContext(0)
    try:
        c.set_pencil_hermitian(A, B)
        return c.solve_hermitian(F.SearchInterval(lo, hi), F.FeastConfig(m0=m0, **kw))
    finally:
        c.close()


def check(r, ref, lo, hi, bmat, exact=None):
    assert r.status == ref["status"] == "converged", (r.status, ref["status"])
    assert len(r.eigenvalues) == ref["m"]
    ev = ref["eigenvalues"]
    tol = 1e-10 * np.maximum(np.abs(ev), 1e-3 * (hi - lo))
    assert np.all(np.abs(r.eigenvalues - ev) <= tol)
    if exact is not None:
        assert np.all(np.abs(r.eigenvalues - exact) <= 1e-10 * np.maximum(np.abs(exact), 1e-3 * (hi - lo)))
    assert sin_angle_c(r.eigenvectors, ref["eigenvectors"], bmat) <= 1e-8
    g = r.eigenvectors.conj().T @ (bmat @ r.eigenvectors)  # complex B-orthonormal
    assert np.max(np.abs(g - np.eye(len(g)))) <= 1e-10
    assert r.max_residual <= max(1e-9, 10 * ref["max_residual"])


def test_dense_hermitian_matches_reference():
    a, b = dense_pencil()
    lo, hi, exact = interval_around(a, b, 20, 8)
    A, B = P.Operator.from_dense_hermitian(a), P.Operator.from_dense_hermitian(b)
    r = run_gpu(A, B, lo, hi, 12)
    ref = O.feast_solve_hermitian(A, B, lo, hi, m0=12)
    check(r, ref, lo, hi, b, exact)
    assert r.loops_used == ref["loops_used"]
    assert r.subspace.shape == (60, 12)


def test_banded_hermitian_matches_reference():
    """CSR Hermitian pencil: the doubled real pencil is banded, so it takes the block-tridiagonal
    path (block Thomas factors, bulk-copy sweeps) of the real configs."""
    A, a = banded_csr(1024, 4, seed=5)
    B, b = banded_csr(1024, 4, seed=6, spd=True)
    lo, hi, exact = interval_around(a, b, 500, 12)
    r = run_gpu(A, B, lo, hi, 20)
    ref = O.feast_solve_hermitian(A, B, lo, hi, m0=20)
    check(r, ref, lo, hi, b, exact)


def test_hermitian_multiplicity():
    """a doubly degenerate eigenvalue inside the interval: the complex eigenvectors of the
    degenerate pair are B-orthonormal (the per-cluster complex Gram-Schmidt over the real pairs)"""
    n = 40
    rng = np.random.default_rng(13)  # (seeds 11, 12 end the reference in max-loops: SURVEY finding 3)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    lam = np.linspace(-3, 3, n)
    lam[21] = lam[20]
    a = herm(q @ np.diag(lam) @ q.conj().T)
    b = np.eye(n, dtype=np.complex128)
    lo, hi = 0.5 * (lam[18] + lam[19]), 0.5 * (lam[23] + lam[24])
    A, B = P.Operator.from_dense_hermitian(a), P.Operator.from_dense_hermitian(b)
    r = run_gpu(A, B, lo, hi, 8)
    ref = O.feast_solve_hermitian(A, B, lo, hi, m0=8)
    check(r, ref, lo, hi, b, np.sort(lam)[19:24])


def test_real_valued_hermitian_equals_real_path():
    """A Hermitian pencil with zero imaginary parts is the real pencil: same eigenpairs."""
    from tests.golden_problems import generate
    prob = generate("small_dense_n60")
    a, b = prob.a.dense.astype(np.complex128), prob.b.dense.astype(np.complex128)
    r = run_gpu(P.Operator.from_dense_hermitian(a), P.Operator.from_dense_hermitian(b), prob.emin, prob.emax, prob.m0)
    ref = O.feast_solve(prob)
    assert r.status == ref["status"] and len(r.eigenvalues) == ref["m"]
    assert np.all(np.abs(r.eigenvalues - ref["eigenvalues"]) <= 1e-10 * np.maximum(np.abs(ref["eigenvalues"]), 1e-3))


def test_hermitian_input_errors():
    from paper_0901_2665_b200 import feast as F
    a, b = dense_pencil(8)
    c = F.GpuContext(0)
    try:
        bad = a.copy()
        bad[0, 1] += 1e-3
        with pytest.raises(F.InputError, match="matrix is not symmetric"):
            c.set_pencil_hermitian(P.Operator.from_dense_hermitian(bad), P.Operator.from_dense_hermitian(b))
        bad = a.copy()
        bad[2, 2] += 1e-3j  # dense: the conjugate-symmetry test catches it first (operator.hpp:47-50)
        with pytest.raises(F.InputError, match="matrix is not symmetric"):
            c.set_pencil_hermitian(P.Operator.from_dense_hermitian(bad), P.Operator.from_dense_hermitian(b))
        A, _ = banded_csr(64, 2, seed=1)
        v = A.values.copy()
        k = [k for k in range(A.row_ptr[3], A.row_ptr[4]) if A.col_idx[k] == 3][0]
        v[k] += 0.5j  # CSR: the diagonal test comes first (operator.hpp:241-245)
        with pytest.raises(F.InputError, match="diagonal must be real"):
            c.set_pencil_hermitian(P.Operator.from_csr_hermitian(64, A.row_ptr, A.col_idx, v),
                                   banded_csr(64, 2, seed=2, spd=True)[0])
        A, _ = banded_csr(64, 2, seed=1)
        A.values = A.values.copy()
        A.values[1] += 0.5j  # (0, 1) no longer the conjugate of (1, 0)
        with pytest.raises(F.InputError, match="mirror entries disagree"):
            c.set_pencil_hermitian(A, banded_csr(64, 2, seed=2, spd=True)[0])
    finally:
        c.close()
