"""Scaled config 5 (L = 32, b = 512, M0 = 768) consistency checks on the device: contour pass
of the full block vs. column chunks, and Rayleigh-Ritz projections vs. numpy on the same Q."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
m = int(sys.argv[2]) if len(sys.argv) > 2 else 768
prob = P.config5(L=L)
ctx = F.GpuContext(0)
ctx.set_pencil(prob.a, prob.b)
ctx.prepare(prob.emin, prob.emax, prob.n_e)
y = ctx.random_block(prob.n, m, 42)
q = ctx.contour_pass(y)
for w in (20, 64, 128, 256):
    qc = np.concatenate([ctx.contour_pass(np.ascontiguousarray(y[:, i:i + w])) for i in range(0, m, w)], axis=1)
    print(f"chunks of {w:3d}: max |Q - Q_chunks| / max|Q| = {np.max(np.abs(q - qc)) / np.max(np.abs(q)):.2e}",
          flush=True)
A = prob.a.to_scipy() if hasattr(prob.a, "to_scipy") else None
res = ctx.rayleigh_ritz(q)
print("rayleigh_ritz returned", [getattr(x, "shape", x) for x in res] if isinstance(res, tuple) else type(res))
ev, x, tr = res
Ad, Bd = prob.a.to_dense(), prob.b.to_dense()
aq = q.T @ (Ad @ q); aq = 0.5 * (aq + aq.T)
bq = q.T @ (Bd @ q); bq = 0.5 * (bq + bq.T)
w = np.linalg.eigvalsh(bq)
print(f"B_Q eigenvalues: min {w[0]:.3e} max {w[-1]:.3e}  (GPU truncated={tr}, mo={len(ev)})")
evg, phig, trg = ctx.reduced_gevp(aq, bq)
print(f"reduced_gevp on numpy projections: mo={len(evg)} trunc={trg}; max |ev_rr - ev_numpy_proj| = "
      f"{np.max(np.abs(np.sort(ev) - np.sort(evg))) if len(ev) == len(evg) else 'size differs'}")
inside = (ev >= prob.emin) & (ev <= prob.emax)
print("in-interval Ritz values (GPU RR):", int(inside.sum()))
r = Ad @ x - (Bd @ x) * ev
print("Ritz residuals (in interval): max", float(np.max(np.linalg.norm(r[:, inside], axis=0))) if inside.any() else None)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (checker only)
import time  # noqa: E402
t = time.perf_counter()
evr, phir, trr = O.reduced_gevp(aq, bq, kind="reference")
print(f"reference reduced_gevp: mo={len(evr)} trunc={trr} ({time.perf_counter() - t:.1f} s)")
for name, (e_, p_) in (("gpu", (evg, phig)), ("ref", (evr, phir))):
    xx = q @ p_
    ins = (e_ >= prob.emin) & (e_ <= prob.emax)
    rr = Ad @ xx[:, ins] - (Bd @ xx[:, ins]) * e_[ins]
    nr = np.linalg.norm(rr, axis=0) / np.maximum(np.linalg.norm(Ad @ xx[:, ins], axis=0), 1e-300)
    print(f"{name}: in-interval {int(ins.sum())}, residual < 1e-6: {int((nr < 1e-6).sum())}, "
          f"< 1e-2: {int((nr < 1e-2).sum())}, median {np.median(nr):.1e}")
