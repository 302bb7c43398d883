"""Times the on-device reduced generalized eigensolve (C-ABI reduced_gevp) on random and
on nearly diagonal pencils (the FEAST steady state)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402

ctx = F.GpuContext(0)
rng = np.random.default_rng(0)
for m in [int(a) for a in (sys.argv[1:] or ["64", "192", "300", "600"])]:
    a = rng.uniform(-1, 1, (m, m)); a = a + a.T
    r = rng.uniform(-1, 1, (m, m)); b = r.T @ r / m + np.eye(m); b = 0.5 * (b + b.T)
    d = np.sort(rng.uniform(-1, 1, m)); q = np.eye(m) + 1e-7 * rng.standard_normal((m, m))
    a2 = q.T @ np.diag(d) @ q; a2 = 0.5 * (a2 + a2.T); b2 = q.T @ q; b2 = 0.5 * (b2 + b2.T)
    for name, (A, B) in (("random", (a, b)), ("near-diag", (a2, b2))):
        ctx.reduced_gevp(A, B)
        t = time.perf_counter()
        for _ in range(3):
            ev, phi, tr = ctx.reduced_gevp(A, B)
        dt = (time.perf_counter() - t) / 3
        err = np.max(np.abs(A @ phi - B @ phi * ev))
        print(f"m={m:4d} {name:9s} {dt*1e3:8.2f} ms  resid {err:.1e}", flush=True)
