"""Full-size parity on BASELINE configs 1 and 2 (GPU vs the reference CPU oracle run on the
GPU box's host cores in the same test). Slow (tens of seconds each)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(prob):
    from paper_0901_2665_b200 import feast as F
    ctx = F.GpuContext(0)
    ctx.set_pencil(prob.a, prob.b)
    r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
                  F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol,
                                max_loops=prob.max_loops, seed=prob.seed))
    ctx.close()
    ref = O.feast_solve(prob, threads=min(prob.n_e, os.cpu_count() or 1))
    return r, ref


def _check(prob, r, ref):
    # parity policy: same status; when the oracle converges, exact count equal
    # to the oracle and to the construction/inertia count, eigenvalues 1e-10 relative
    assert r.status == ref["status"], (r.status, ref["status"], r.loops_used, ref["loops_used"])
    if ref["status"] == "converged":
        assert len(r.eigenvalues) == ref["m"] == prob.expected_count
        ev = ref["eigenvalues"]
        assert np.all(np.abs(r.eigenvalues - ev) <= 1e-10 * np.maximum(np.abs(ev), 1e-3 * (prob.emax - prob.emin)))
        assert r.max_residual <= 1e-10 and ref["max_residual"] <= 1e-10


@pytest.mark.skipif(not O.available("reference") and not O.available("port"), reason="no oracle")
def test_config1_full():
    from paper_0901_2665_b200 import problems as P
    prob = P.config1()
    r, ref = _run(prob)
    _check(prob, r, ref)


@pytest.mark.skipif(not O.available("reference") and not O.available("port"), reason="no oracle")
def test_config2_full():
    from paper_0901_2665_b200 import problems as P
    prob = P.config2()
    r, ref = _run(prob)
    _check(prob, r, ref)
