"""Repeated full-size config-3 solves (fresh contexts): at which pass, if any, does a run's trace history first
differ from the first run's? (Non-intrusive: the per-pass traces are part of the result.)
usage: trace_repeat.py [runs]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.golden import make_fullsize as MF
from paper_0901_2665_b200 import feast as F
prob = MF.problem("cfg3")
hist = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    c = F.GpuContext(0); c.set_pencil(prob.a, prob.b)
    r = c.solve(F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed))
    c.close()
    hist.append(np.asarray(r.trace_history).copy())
ref = hist[0]
for i, h in enumerate(hist[1:], 1):
    d = np.nonzero(h != ref)[0]
    if len(d):
        print("   rel dev per pass:", " ".join("%.0e" % (abs(a - b) / abs(b)) for a, b in zip(h, ref)))
    print(i, "identical" if len(d) == 0 else ("first differs at pass %d (rel %.1e), %d passes differ" % (d[0], abs(h[d[0]] - ref[d[0]]) / abs(ref[d[0]]), len(d))))
