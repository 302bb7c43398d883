"""Contour-pass error vs the reference oracle on a fixture, for the block size the GPU picks
(FEAST_MIN_BLOCK forces a larger re-blocking)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402
from tests.golden_problems import fixtures, load_fixture  # noqa: E402

for path in fixtures():
    if "bt_L16" not in path and "cfg2" not in path:
        continue
    prob, _ = load_fixture(path)
    ctx = F.GpuContext(0)
    ctx.set_pencil(prob.a, prob.b)
    ctx.prepare(prob.emin, prob.emax, prob.n_e)
    y = O.random_block(prob.n, prob.m0, 42)
    q = ctx.contour_pass(y)
    qr = O.accumulate_real(prob.a, prob.b, prob.emin, prob.emax, prob.n_e, y)
    z, _ = ctx.contour()
    rhs = np.random.default_rng(1).standard_normal((prob.n, 3)) + 1j * np.random.default_rng(2).standard_normal((prob.n, 3))
    errs = []
    for e in range(prob.n_e):
        x = ctx.solve_shift(e, rhs.copy(), False)
        xr = O.shift_solve(prob.a, prob.b, z[e], rhs, 0)
        errs.append(np.max(np.abs(x - xr)) / np.max(np.abs(xr)))
    print(os.path.basename(path), "MIN_BLOCK", os.environ.get("FEAST_MIN_BLOCK"), "Q err",
          np.max(np.abs(q - qr)) / np.max(np.abs(qr)), "solve errs", np.array2string(np.array(errs), precision=1))
    ctx.close()
