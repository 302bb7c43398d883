"""Warm-started parameter sweep on the device (feast_gpu_sweep) against run_sweep
(run.cpp:63-125) restated over the reference's own feast_solve: A_k = add_scaled(A0, S, t_k)
(operator.hpp:282-304), a converged step's Ritz block topped up with
random_block(n, m0 - cols, seed + 1000003 (k + 1)) times B starts the next step."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_0901_2665_b200 import problems as P
from tests.golden_problems import generate

pytestmark = pytest.mark.gpu


def reference_sweep(prob, s, steps):
    """run_sweep's loop over the compiled reference (oracle/_ref): per step (result or None)."""
    import copy
    out, warm = [], None
    a0 = prob.a.to_scipy()
    for k, t in enumerate(steps):
        m = (a0 + t * s.to_scipy()).tocsr()
        m.sort_indices()
        p = copy.copy(prob)
        p.a = P.Operator.from_csr(prob.n, m.indptr, m.indices, m.data)
        try:
            r = O.feast_solve(p, initial_y=warm)
        except O.OracleError as e:
            if e.code != 5:
                raise
            out.append(None)
            warm = None
            continue
        out.append(r)
        sub = r["subspace"]
        if r["status"] == "converged" and sub.shape[1] > 0:
            if sub.shape[1] < prob.m0:
                pad = O.random_block(prob.n, prob.m0 - sub.shape[1], prob.seed + 1000003 * (k + 1))
                sub = np.hstack([sub, pad])
            warm = np.asfortranarray(prob.b.matmul(sub))
        else:
            warm = None
    return out


@pytest.mark.parametrize("which", ["bt_L16_b32", "cfg2_n2048", "small_dense_n60"])
def test_sweep_matches_reference_run_sweep(which):
    from paper_0901_2665_b200 import feast as F
    prob = generate(which)
    n = prob.n
    rng = np.random.default_rng(17)
    # a diagonal perturbation (fits every storage the pencil may take)
    s = P.Operator.from_csr(n, np.arange(n + 1), np.arange(n), rng.uniform(-1.0, 1.0, n))
    steps = [0.0, 2e-3, 4e-3, 6e-3]
    ref = reference_sweep(prob, s, steps)
    c = F.GpuContext(0)
    try:
        got = c.sweep(prob.a, prob.b, s, steps, F.SearchInterval(prob.emin, prob.emax),
                      F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol,
                                    max_loops=prob.max_loops, seed=prob.seed))
    finally:
        c.close()
    assert len(got) == len(ref)
    for k, (g, r) in enumerate(zip(got, ref)):
        assert (r is None) == isinstance(g, Exception), k
        if r is None:
            continue
        assert g.status == r["status"], (k, g.status, r["status"])
        assert g.loops_used == r["loops_used"], (k, g.loops_used, r["loops_used"])
        assert len(g.eigenvalues) == r["m"], k
        ev = r["eigenvalues"]
        assert np.all(np.abs(g.eigenvalues - ev) <= 1e-10 * np.maximum(np.abs(ev), 1e-3 * (prob.emax - prob.emin))), k
        assert g.max_residual <= max(1e-9, 10 * r["max_residual"]), k
    # the warm start pays: every converged step after the first needs at most the cold loop count
    loops = [g.loops_used for g in got if not isinstance(g, Exception)]
    assert all(x <= loops[0] for x in loops[1:]), loops


def test_sweep_input_errors():
    from paper_0901_2665_b200 import feast as F
    prob = generate("small_dense_n60")
    c = F.GpuContext(0)
    try:
        s = P.Operator.from_dense(np.eye(prob.n + 1))
        with pytest.raises(F.InputError, match="perturbation dimension mismatch"):
            c.sweep(prob.a, prob.b, s, [0.0], F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0))
        with pytest.raises(F.InputError, match="no steps given"):
            c.sweep(prob.a, prob.b, prob.a, [], F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0))
    finally:
        c.close()
