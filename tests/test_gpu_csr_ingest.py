"""CSR operators taken in on the device (csr_ingest.cu): set_pencil's device route must make the
host path's decisions and raise its errors (operator.hpp:237-268 validation, the banded-route
choice of inner_solver.hpp:84-92, the 1-norm of operator.hpp:195-212), and the blocks it
assembles must equal the ones a block-tridiagonal descriptor of the same pencil uploads, so the
solves agree bit for bit."""
import numpy as np
import pytest

from paper_0901_2665_b200.problems import Operator, banded_csr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_0901_2665_b200 import feast
    feast.load_library()
    return feast


@pytest.fixture(scope="module")
def ctx(F):
    c = F.GpuContext(0)
    yield c
    c.close()


def pencil(n=1024, bw=5, seed=11):
    rng = np.random.default_rng(seed)
    a = banded_csr(n, rng.uniform(-2, 2, n), {d: -rng.uniform(0.5, 1.5, n - d) / (1 + d) for d in range(1, bw + 1)})
    b = banded_csr(n, np.ones(n), {d: 0.02 * rng.uniform(-1, 1, n - d) for d in range(1, bw + 1)})
    return a, b


def dense_of(o):
    m = np.zeros((o.n, o.n))
    for i in range(o.n):
        for k in range(o.row_ptr[i], o.row_ptr[i + 1]):
            m[i, o.col_idx[k]] += o.values[k]
    return m


def blocktri_of(m, b):
    L = m.shape[0] // b
    diag = np.stack([m[l * b:(l + 1) * b, l * b:(l + 1) * b] for l in range(L)])
    low = np.stack([m[(l + 1) * b:(l + 2) * b, l * b:(l + 1) * b] for l in range(L - 1)])
    return Operator.from_blocktri(diag, low)


def solve(ctx, F, a, b, lo=-0.05, hi=0.05, m0=64):
    ctx.set_pencil(a, b)
    r = ctx.solve(F.SearchInterval(lo, hi), F.FeastConfig(m0=m0))
    return ctx.storage(), r


def test_device_csr_route_equals_blocktri_descriptor(ctx, F):
    a, b = pencil()
    st_csr, r_csr = solve(ctx, F, a, b)
    assert st_csr[0] == 16 and st_csr[1] == 64  # half-bandwidth 5 -> 16-row blocks
    st_bt, r_bt = solve(ctx, F, blocktri_of(dense_of(a), 16), blocktri_of(dense_of(b), 16))
    assert st_bt[:2] == st_csr[:2]
    assert r_csr.status == r_bt.status and r_csr.loops_used == r_bt.loops_used
    assert np.array_equal(r_csr.eigenvalues, r_bt.eigenvalues)
    assert np.array_equal(r_csr.eigenvectors, r_bt.eigenvectors)
    assert len(r_csr.eigenvalues) > 0


def test_unsorted_rows_and_padding(ctx, F):
    # rows permuted within themselves (the mirror check falls back to a linear scan), n not a
    # multiple of the block size (B gets a unit diagonal on the padding rows)
    a, b = pencil(n=1000, bw=7, seed=3)
    rng = np.random.default_rng(0)
    def shuffle(o):
        ci, v = o.col_idx.copy(), o.values.copy()
        for i in range(o.n):
            s, e = o.row_ptr[i], o.row_ptr[i + 1]
            p = s + rng.permutation(e - s)
            ci[s:e], v[s:e] = ci[p], v[p]
        return Operator.from_csr(o.n, o.row_ptr, ci, v)
    st1, r1 = solve(ctx, F, a, b)
    st2, r2 = solve(ctx, F, shuffle(a), shuffle(b))
    assert st1[:2] == st2[:2] == (16, 63)
    assert np.array_equal(r1.eigenvalues, r2.eigenvalues)
    assert np.array_equal(r1.eigenvectors, r2.eigenvectors)
    # against the dense route on the same pencil (different factorisation: tolerance)
    st3, r3 = solve(ctx, F, Operator.from_dense(dense_of(a)), Operator.from_dense(dense_of(b)))
    assert st3[0] == 0
    assert r3.status == r1.status and len(r3.eigenvalues) == len(r1.eigenvalues)
    assert np.max(np.abs(r3.eigenvalues - r1.eigenvalues)) <= 1e-10


def test_wide_pattern_takes_dense_route(ctx, F):
    # bandwidth above the banded policy's (3 bw + 1) 2 <= n: the dense route, from CSR
    n = 96
    rng = np.random.default_rng(5)
    m = np.diag(rng.uniform(-2, 2, n))
    m[0, n - 1] = m[n - 1, 0] = 0.3
    import scipy.sparse as sp
    s = sp.csr_matrix(m)
    a = Operator.from_csr(n, s.indptr, s.indices, s.data)
    st, r = solve(ctx, F, a, Operator.identity_csr(n), lo=-0.5, hi=0.5, m0=40)
    assert st[0] == 0
    ev = np.linalg.eigvalsh(m)
    want = ev[(ev >= -0.5) & (ev <= 0.5)]
    assert r.status == "converged" and np.allclose(r.eigenvalues, want, atol=1e-12)


@pytest.mark.parametrize("kind,msg", [("range", "triplet index out of range"),
                                      ("missing", "missing mirror entry"),
                                      ("differ", "mirror entries disagree")])
@pytest.mark.parametrize("which", ["A", "B"])
def test_device_validation_errors(ctx, F, kind, msg, which):
    a, b = pencil(n=512, bw=3, seed=7)
    o = a if which == "A" else b
    ci, v = o.col_idx.copy(), o.values.copy()
    rp = o.row_ptr.copy()
    i = 300
    k = rp[i] + (rp[i + 1] - rp[i]) - 1  # the row's last entry: (300, 303)
    assert ci[k] == i + 3
    if kind == "range":
        ci[k] = o.n + 5
    elif kind == "differ":
        v[k] += 1.0
    else:  # drop the mirror (303, 300): row 303's first entry
        kk = rp[i + 3]
        assert ci[kk] == i
        ci = np.delete(ci, kk)
        v = np.delete(v, kk)
        rp = rp.copy()
        rp[i + 4:] -= 1
    bad = Operator.from_csr(o.n, rp, ci, v)
    args = (bad, b) if which == "A" else (a, bad)
    with pytest.raises(F.InputError, match=msg):
        ctx.set_pencil(*args)
    # a well-formed pencil still loads on the same context afterwards
    ctx.set_pencil(a, b)
    assert ctx.storage()[0] == 16


def test_errors_of_a_before_b(ctx, F):
    a, b = pencil(n=256, bw=2, seed=9)
    ci = a.col_idx.copy(); ci[-1] = -1
    bad_a = Operator.from_csr(a.n, a.row_ptr, ci, a.values)
    v = b.values.copy(); v[b.row_ptr[10]] += 0.5  # row 10's first entry (10, 8): mirror differs
    bad_b = Operator.from_csr(b.n, b.row_ptr, b.col_idx, v)
    with pytest.raises(F.InputError, match="out of range"):
        ctx.set_pencil(bad_a, bad_b)
    # first failing entry in row order within one operator: row 10 before row 100
    v2 = v.copy(); v2[b.row_ptr[100]] += 0.5
    ci2 = b.col_idx.copy()
    with pytest.raises(F.InputError, match="disagree"):
        ctx.set_pencil(a, Operator.from_csr(b.n, b.row_ptr, ci2, v2))
