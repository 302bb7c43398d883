"""Config-3-shaped problem (L=16, b=128): GPU vs reference oracle, loops and residuals."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config3(L=16, b=128, seed=3, m0=32, want=16, yseed=7)
ctx = F.GpuContext(0)
ctx.set_pencil(prob.a, prob.b)
r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
              F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed))
ref = O.feast_solve(prob, threads=8)
print("gpu loops", r.loops_used, "ref loops", ref["loops_used"])
print("gpu res", np.array2string(np.asarray(r.residuals), precision=2))
print("ref res", np.array2string(np.asarray(ref["residuals"]), precision=2))
print("gpu trace", np.array2string(np.asarray(r.trace_history), precision=16))
print("ref trace", np.array2string(np.asarray(ref["trace_history"]), precision=16))
