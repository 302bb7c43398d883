"""Complete FEAST solve of a BASELINE config through the C-ABI; prints status, count vs the
construction/inertia count, loops, residuals and timings as one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

name = sys.argv[1]
kw = dict(a.split("=") for a in sys.argv[2:])
gen = {"cfg1": P.config1, "cfg2": P.config2, "cfg3": P.config3, "cfg4": P.config4, "cfg5": P.config5}[name]
t = time.perf_counter()
prob = gen(**{k: int(v) for k, v in kw.items()})
tgen = time.perf_counter() - t
ctx = F.GpuContext(0)
t = time.perf_counter()
ctx.set_pencil(prob.a, prob.b)
r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
              F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops,
                            seed=prob.seed))
tsolve = time.perf_counter() - t
out = dict(config=prob.name, n=prob.n, m0=prob.m0, n_e=prob.n_e, status=r.status, count=len(r.eigenvalues),
           expected=prob.expected_count, loops=r.loops_used, max_residual=r.max_residual,
           trace_history=[float(x) for x in r.trace_history], counts=[int(x) for x in r.in_interval_counts],
           timings=r.timings.__dict__, wall_s=tsolve, gen_s=tgen, passes_per_s=(r.loops_used + 1) / tsolve)
print(json.dumps(out), flush=True)
