"""Pins the CPU checkers (oracle/) before they are trusted: every known-answer test the
reference's own suites hold for the hot path, run against BOTH the compiled
reference (oracle/_ref) and the plain-C restatement (oracle/libfeastoracle.so), plus the
committed golden fixtures generated from the reference (tests/golden/make_golden.py)."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.mt64 import MT19937_64, uniform_pm1

KINDS = [k for k in ("reference", "port") if O.available(k)]
pytestmark = pytest.mark.skipif(not KINDS, reason="no oracle built")

# test_quadrature.cpp:17-20 (positive half, 8 points)
NODES8 = [0.18343464249564980494, 0.52553240991632898582, 0.79666647741362673959, 0.96028985649753623168]
WEIGHTS8 = [0.36268378337836198297, 0.31370664587788728734, 0.22238103445337447054, 0.10122853629037625915]


@pytest.mark.parametrize("kind", KINDS)
def test_gauss_legendre_8_matches_tabulated(kind):
    x, w = O.gauss_legendre(8, kind=kind)
    for i in range(4):
        assert abs(x[4 + i] - NODES8[i]) <= 1e-15
        assert abs(x[3 - i] + NODES8[i]) <= 1e-15
        assert abs(w[4 + i] - WEIGHTS8[i]) <= 1e-15
        assert abs(w[3 - i] - WEIGHTS8[i]) <= 1e-15


@pytest.mark.parametrize("kind", KINDS)
def test_gauss_legendre_2_textbook(kind):
    x, w = O.gauss_legendre(2, kind=kind)
    assert abs(x[1] - 0.57735026918962576451) <= 1e-15 and abs(x[0] + 0.57735026918962576451) <= 1e-15
    assert w[0] == 1.0 and w[1] == 1.0


@pytest.mark.parametrize("kind", KINDS)
def test_gauss_legendre_symmetric_normalized_exact(kind):
    for n in range(1, 65):
        x, w = O.gauss_legendre(n, kind=kind)
        assert np.all(w > 0) and np.all(np.diff(x) > 0)
        assert np.array_equal(x, -x[::-1]) and np.array_equal(w, w[::-1])
        assert abs(w.sum() - 2.0) <= 1e-14
        if n <= 32:
            for k in range(2 * n):
                exact = 0.0 if k % 2 else 2.0 / (k + 1)
                assert abs(np.sum(w * x ** k) - exact) <= 1e-13
    for bad in (0, 65):
        with pytest.raises(O.OracleError) as e:
            O.gauss_legendre(bad, kind=kind)
        assert e.value.code == 4


@pytest.mark.parametrize("kind", KINDS)
def test_contour_point_on_unit_circle(kind):
    c = O.build_contour(0.0, 2.0, 8, kind=kind)  # test_quadrature.cpp:81-100
    assert c["radius"] == 1.0
    assert np.all(c["theta"] > 0) and np.all(c["theta"] < math.pi) and np.all(np.diff(c["theta"]) < 0)
    assert np.all(np.abs(np.abs(c["z"] - 1.0) - 1.0) <= 1e-14)
    assert abs(c["theta"][4] - 1.2826578641557948575) <= 1e-14
    assert abs(c["z"][4].real - 1.2841679239019287751) <= 1e-14
    assert abs(c["z"][4].imag - 0.95877452564472509392) <= 1e-14


@pytest.mark.parametrize("kind", KINDS)
def test_degenerate_interval_rejected(kind):
    with pytest.raises(O.OracleError) as e:
        O.build_contour(1e9, 1e9 + 1e-5, 8, kind=kind)
    assert e.value.code == 4
    O.build_contour(0.0, 1e-10, 8, kind=kind)


@pytest.mark.parametrize("kind", KINDS)
def test_scalar_filter_golden(kind):
    f = lambda lam, ne: O.scalar_filter(lam, -1.0, 1.0, ne, kind=kind)  # test_oracle.cpp:96-119
    for ne in range(1, 17):
        assert abs(f(0.0, ne) + 1.0) <= 1e-14
    assert abs(f(0.5, 8) - (-1.0000164802583470518)) <= 1e-15
    assert abs(f(-0.5, 8) - (-1.0000164802583470518)) <= 1e-15
    assert abs(f(1.0, 8) - (-0.5)) <= 1e-14
    assert abs(f(2.0, 8) - 1.6480258347051789577e-05) <= 5e-17
    assert abs(f(3.0, 8) - (-4.3219719641408335346e-07)) <= 5e-17
    assert abs(f(4.0, 8) - (-8.0759760015604461606e-08)) <= 5e-17
    assert abs(f(0.5, 16) - (-0.99999999976369286183)) <= 1e-15
    assert abs(f(0.25, 16) - (-1.0000000000000015399)) <= 1e-15
    assert abs(f(2.0, 16) - (-2.3630713816700372e-10)) <= 2e-16
    assert abs(f(3.0, 16) - (-3.3459037783382717e-13)) <= 2e-16


@pytest.mark.parametrize("kind", KINDS)
def test_random_block_bitstream(kind):
    # test_core.cpp:49-71, with an independent Python mt19937_64
    y = O.random_block(3, 2, 42, kind=kind)
    g = MT19937_64(42)
    for j in range(2):
        for i in range(3):
            assert y[i, j] == uniform_pm1(g)
    y2 = O.random_block(37, 5, 7, kind=kind)
    g = MT19937_64(7)
    exp = np.array([[0.0] * 5 for _ in range(37)])
    for j in range(5):
        for i in range(37):
            exp[i, j] = uniform_pm1(g)
    assert np.array_equal(y2, exp)


@pytest.mark.parametrize("kind", KINDS)
def test_centered_singleton_accumulation(kind):
    # test_core.cpp:80-92: A = 2.5, B = 1, interval [1.5, 3.5], Y = 3 -> Q = -3
    from paper_0901_2665_b200.problems import Operator
    a = Operator.from_dense(np.array([[2.5]]))
    b = Operator.identity_csr(1)
    q = O.accumulate_real(a, b, 1.5, 3.5, 8, np.array([[3.0]]), kind=kind)
    assert abs(q[0, 0] + 3.0) <= 1e-13


@pytest.mark.parametrize("kind", KINDS)
def test_hermitian_accumulation_matches_real(kind):
    # test_core.cpp:111-142: on a real symmetric pencil the Hermitian accumulation of a real
    # block equals the real accumulation (imaginary part ~0) to 1e-13
    from tests.golden_problems import fixtures, load_fixture
    prob, _ = load_fixture([p for p in fixtures() if "small_dense_n60" in p][0])
    y = O.random_block(prob.n, 7, 3)
    qr = O.accumulate_real(prob.a, prob.b, prob.emin, prob.emax, prob.n_e, y, kind=kind)
    qh = O.accumulate_hermitian(prob.a, prob.b, prob.emin, prob.emax, prob.n_e, y + 0j, kind=kind)
    scale = max(1.0, float(np.max(np.abs(qr))))
    assert np.max(np.abs(qh.real - qr)) <= 1e-13 * scale
    assert np.max(np.abs(qh.imag)) <= 1e-13 * scale


def test_hermitian_accumulation_restatement_matches_reference():
    # the C restatement's accumulate_subspace_hermitian against the compiled reference, on a
    # complex block and both storage policies (dense LU, banded LU)
    if not (O.available("reference") and O.available("port")):
        pytest.skip("needs both checkers")
    from tests.golden_problems import fixtures, load_fixture
    rng = np.random.default_rng(9)
    for name in ("small_dense_n60", "bt_L8_b48"):
        prob, _ = load_fixture([p for p in fixtures() if name in p][0])
        y = rng.standard_normal((prob.n, 5)) + 1j * rng.standard_normal((prob.n, 5))
        q0 = O.accumulate_hermitian(prob.a, prob.b, prob.emin, prob.emax, prob.n_e, y, kind="reference")
        q1 = O.accumulate_hermitian(prob.a, prob.b, prob.emin, prob.emax, prob.n_e, y, kind="port")
        assert np.max(np.abs(q0 - q1)) <= 1e-12 * max(1.0, float(np.max(np.abs(q0)))), name


@pytest.mark.parametrize("kind", KINDS)
def test_reduced_gevp_properties(kind):
    # test_linalg.cpp:272-298
    rng = np.random.default_rng(3)
    m = 20
    a = rng.uniform(-1, 1, (m, m)); a = a + a.T
    r = rng.uniform(-1, 1, (m, m)); b = r.T @ r / m + np.eye(m); b = 0.5 * (b + b.T)
    ev, phi, tr = O.reduced_gevp(a, b, kind=kind)
    assert not tr and np.all(np.diff(ev) >= 0)
    assert np.max(np.abs(a @ phi - b @ phi * ev)) <= 1e-11
    assert np.max(np.abs(phi.T @ b @ phi - np.eye(m))) <= 1e-11


from tests.golden_problems import fixtures, load_fixture  # noqa: E402


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("path", fixtures(), ids=lambda p: os.path.basename(p))
def test_golden_feast_results(kind, path):
    """The checkers reproduce the committed reference outputs: bit-exact for the reference
    build (same code, same inputs), within 1e-12 for the C restatement."""
    prob, g = load_fixture(path)
    r = O.feast_solve(prob, kind=kind)
    assert r["status"] == str(g["status"])
    assert r["m"] == int(g["m"]) and r["loops_used"] == int(g["loops_used"])
    if kind == "reference":
        assert np.array_equal(r["eigenvalues"], g["eigenvalues"])
        assert np.array_equal(r["trace_history"], g["trace_history"])
        assert np.array_equal(r["eigenvectors"], g["eigenvectors"])
    else:
        assert np.allclose(r["eigenvalues"], g["eigenvalues"], rtol=1e-12, atol=1e-13)
        assert np.allclose(r["trace_history"], g["trace_history"], rtol=1e-10, atol=1e-12)
    assert r["max_residual"] <= 1e-9
