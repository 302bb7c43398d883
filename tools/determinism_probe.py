"""Which stage of a config is not bit-reproducible: repeated factorisations, contour passes and
Rayleigh-Ritz steps on the same inputs, compared bit for bit."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from tests.golden import make_fullsize as MF  # noqa: E402

prob = MF.problem(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
c = F.GpuContext(0)
c.set_pencil(prob.a, prob.b)
c.prepare(prob.emin, prob.emax, prob.n_e)
y = c.random_block(prob.n, prob.m0, prob.seed)
q0 = c.contour_pass(y)
print("contour_pass", [bool(np.array_equal(c.contour_pass(y), q0)) for _ in range(reps)], flush=True)
qs = []
for _ in range(3):
    c.prepare(prob.emin, prob.emax, prob.n_e)
    qs.append(c.contour_pass(y))
print("refactor + contour_pass", [bool(np.array_equal(q, q0)) for q in qs], flush=True)
ev0, x0, _ = c.rayleigh_ritz(q0)
out = []
for _ in range(reps):
    ev, x, _ = c.rayleigh_ritz(q0)
    out.append((bool(np.array_equal(ev, ev0)), bool(np.array_equal(x, x0)), float(np.max(np.abs(ev - ev0)))))
print("rayleigh_ritz (ev, x, max dev)", out, flush=True)
aq = np.asfortranarray(q0.T @ prob.a.matmul(q0)); aq = 0.5 * (aq + aq.T)
bq = np.asfortranarray(q0.T @ prob.b.matmul(q0)); bq = 0.5 * (bq + bq.T)
e0, p0, _ = c.reduced_gevp(aq, bq)
out = []
for _ in range(reps):
    e, p, _ = c.reduced_gevp(aq, bq)
    out.append((bool(np.array_equal(e, e0)), bool(np.array_equal(p, p0))))
print("reduced_gevp (ev, phi)", out, flush=True)
c.close()
