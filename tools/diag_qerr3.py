"""Contour-pass and shifted-solve error vs the reference oracle on a config-3-shaped pencil."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

for L, b in [(16, 128), (8, 256), (16, 64), (32, 32)]:
    prob = P.config3(L=L, b=b, seed=3, m0=32, want=16, yseed=7) if (L, b) in [(16, 128), (8, 256)] else None
    if prob is None:
        a, bb = P.blocktri_operators(L, b, seed=3)
        lo, hi = 0.0, 0.1
    else:
        a, bb, lo, hi = prob.a, prob.b, prob.emin, prob.emax
    ctx = F.GpuContext(0)
    ctx.set_pencil(a, bb)
    ctx.prepare(lo, hi, 8)
    y = O.random_block(a.n, 32, 42)
    q = ctx.contour_pass(y)
    qr = O.accumulate_real(a, bb, lo, hi, 8, y)
    z, _ = ctx.contour()
    rhs = np.random.default_rng(1).standard_normal((a.n, 3)) + 0j
    errs = [np.max(np.abs(ctx.solve_shift(e, rhs.copy(), False) - O.shift_solve(a, bb, z[e], rhs, 0)))
            / np.max(np.abs(O.shift_solve(a, bb, z[e], rhs, 0))) for e in range(8)]
    print(f"L={L} b={b}: Q err {np.max(np.abs(q - qr)) / np.max(np.abs(qr)):.1e}  solve errs "
          + np.array2string(np.array(errs), precision=1), flush=True)
    ctx.close()
