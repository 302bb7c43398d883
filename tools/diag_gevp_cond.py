"""reduced_gevp on ill-conditioned B (FEAST's filtered subspaces): GPU vs reference oracle,
eigenpair residuals |A phi - lam B phi| / (|A| |phi|) and B-orthonormality."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402

ctx = F.GpuContext(0)
rng = np.random.default_rng(5)
for m, cond in [(32, 1e6), (32, 1e10), (64, 1e10), (192, 1e8), (192, 1e11)]:
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    b = u @ np.diag(np.logspace(0, -np.log10(cond), m)) @ u.T
    b = 0.5 * (b + b.T)
    a = rng.standard_normal((m, m)); a = 0.5 * (a + a.T)
    a = b @ a @ b  # A_Q = Q^T A Q shares the scaling of B_Q = Q^T B Q
    a = 0.5 * (a + a.T)
    out = []
    for name, fn in (("gpu", ctx.reduced_gevp), ("ref", O.reduced_gevp)):
        ev, phi, tr = fn(a, b)
        res = np.abs(a @ phi - b @ phi * ev).max() / (np.abs(a).max() * np.abs(phi).max())
        orth = np.abs(phi.T @ b @ phi - np.eye(phi.shape[1])).max()
        out.append(f"{name}: k={len(ev)} trunc={tr} res={res:.1e} orth={orth:.1e}")
    print(f"m={m} cond={cond:.0e}  " + "  |  ".join(out), flush=True)
