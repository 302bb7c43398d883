"""Repeated full solves of a full-size config in one process: are the results bit-reproducible?
usage: cfg3_repeat.py [name] [reps] [lookahead 0/1]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from tests.golden import make_fullsize as MF  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
if name in ("cfg1", "cfg2"):
    import bench
    prob = bench.make_problem(name)
else:
    prob = MF.problem(name)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
la = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
sums = []
for i in range(reps):
    c = F.GpuContext(0)
    c.set_lookahead(la)
    c.set_pencil(prob.a, prob.b)
    r = c.solve(F.SearchInterval(prob.emin, prob.emax),
                F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed))
    c.close()
    sums.append(repr(float(np.sum(r.eigenvalues))))
print("lookahead", la, "distinct results:", len(set(sums)), sums, flush=True)
