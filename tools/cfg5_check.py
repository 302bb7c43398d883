"""Scaled config 5 (L layers of b = 512, seed 5, M0 = 768, Ne = 16) solved with every node
resident and with streamed node batches of 1 (the full-size memory plan); prints status,
count and trace of both (they must agree bit for bit)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
prob = P.config5(L=L)
out = {}
for batch in (0, 1):
    ctx = F.GpuContext(0)
    if batch:
        ctx.set_node_batch(batch)
    ctx.set_pencil(prob.a, prob.b)
    r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
                  F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops,
                                seed=prob.seed))
    out[batch] = dict(status=r.status, count=len(r.eigenvalues), loops=r.loops_used, max_residual=r.max_residual,
                      counts=[int(x) for x in r.in_interval_counts], trace=[float(x) for x in r.trace_history][:6])
    print(batch, json.dumps(out[batch]), flush=True)
    ctx.close()
print("identical" if out[0] == out[1] else "DIFFERENT")
