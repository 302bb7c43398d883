"""Full-size config 5 on one GPU (L = 2048, b = 512, N = 1,048,576, M0 = 768, Ne = 16): the
streamed memory plan (node batches of one, every pass refactors each node) for two passes
(max_loops = 1), with FEAST_TRACE=2 phase marks on stderr; prints one JSON line with the
per-pass device times (FeastTimings) and wall clock."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

t = time.perf_counter()
prob = P.config5()
t_gen = time.perf_counter() - t
ctx = F.GpuContext(0)
ctx.set_node_batch(int(os.environ.get("FEAST_CFG5_BATCH", "1")))
t = time.perf_counter()
ctx.set_pencil(prob.a, prob.b)
t_pencil = time.perf_counter() - t
t = time.perf_counter()
r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
              F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=1, seed=prob.seed))
t_solve = time.perf_counter() - t
print(json.dumps(dict(config=prob.name, passes=r.loops_used + 1, status=r.status, counts=[int(x) for x in r.in_interval_counts],
                      timings=r.timings.__dict__, solve_wall_s=t_solve, set_pencil_s=t_pencil, generate_s=t_gen,
                      wall_per_pass_s=t_solve / (r.loops_used + 1))), flush=True)
