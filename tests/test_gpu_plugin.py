"""The reference-side binding (integration/feast_gpu_solver.hpp): the REFERENCE's own
feast_solve (core.hpp:264) with the GPU InnerSolver plugged in, and the loop-level forwarder,
both against the reference's CPU results on the golden fixtures."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_problems import fixtures, load_fixture

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(O.SHIM), reason="oracle/_ref/libfeastref_gpu.so not built")]


@pytest.mark.parametrize("mode", [0, 1], ids=["plugin", "forwarder"])
@pytest.mark.parametrize("path", fixtures(), ids=lambda p: p.split("/")[-1][:-4])
def test_reference_loop_with_gpu_plugin(path, mode):
    prob, g = load_fixture(path)
    r = O.shim_feast_solve(prob, mode=mode)
    assert r["status"] == str(g["status"])
    assert r["m"] == int(g["m"])
    ev = g["eigenvalues"]
    assert np.all(np.abs(r["eigenvalues"] - ev) <= 1e-10 * np.maximum(1.0, np.abs(ev)))
    assert r["max_residual"] <= 1e-9
    if mode == 0:  # the reference's loop drove every step: same loop count as its CPU run
        assert r["loops_used"] == int(g["loops_used"])
