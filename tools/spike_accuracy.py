"""Shifted-solve accuracy of SPIKE chunkings against the reference's BandedLU (oracle/_ref):
max relative error per chunk count on config-2-shaped pencils."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

for n in (2048, 16384):
    prob = P.config2(n=n, m0=48 if n == 2048 else 192, want=24 if n == 2048 else 128)
    rng = np.random.default_rng(1)
    rhs = rng.standard_normal((prob.n, 4)) + 1j * rng.standard_normal((prob.n, 4))
    ref = {}
    for chunks in (1, 2, 4, 8, 16):
        c = F.GpuContext(0)
        c.set_spike(chunks)
        c.set_pencil(prob.a, prob.b)
        c.prepare(prob.emin, prob.emax, 8)
        z, _ = c.contour()
        errs = []
        for e in (0, 3, 7):
            if e not in ref:
                ref[e] = O.shift_solve(prob.a, prob.b, z[e], rhs, 0)
            x = c.solve_shift(e, rhs, False)
            errs.append(float(np.max(np.abs(x - ref[e])) / np.max(np.abs(ref[e]))))
        c.close()
        print(f"n={n} chunks={chunks} max rel err per node {['%.1e' % v for v in errs]}", flush=True)
