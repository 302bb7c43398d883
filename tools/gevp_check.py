"""Reduced generalized eigensolve (C-ABI reduced_gevp) against scipy at the given sizes:
random, graded-mass and nearly diagonal pencils; prints the worst eigenvalue / residual /
B-orthonormality errors per case."""
import os
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402

ctx = F.GpuContext(0)
rng = np.random.default_rng(0)
for m in [int(a) for a in (sys.argv[1:] or ["192", "300", "600", "768"])]:
    a = rng.uniform(-1, 1, (m, m)); a = a + a.T
    r = rng.uniform(-1, 1, (m, m)); b = r.T @ r / m + np.eye(m); b = 0.5 * (b + b.T)
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    bg = (q * np.logspace(-8, 0, m)) @ q.T; bg = 0.5 * (bg + bg.T)
    for name, (A, B) in (("random", (a, b)), ("graded", (a, bg)), ("identity", (a, np.eye(m)))):
        ev, phi, tr = ctx.reduced_gevp(A, B)
        ref = sl.eigh(A, B, eigvals_only=True)
        e1 = np.max(np.abs(ev - ref[-len(ev):] if tr else ev - ref) / np.maximum(1, np.abs(ref).max()))
        e2 = np.max(np.abs(A @ phi - B @ phi * ev))
        e3 = np.max(np.abs(phi.T @ B @ phi - np.eye(phi.shape[1])))
        print(f"m={m:4d} {name:9s} trunc={tr} ev_err={e1:.1e} resid={e2:.1e} borth={e3:.1e}", flush=True)
