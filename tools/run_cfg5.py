"""Full-size BASELINE config 5 on one GPU: L = 2048 layers of b = 512 (N = 1,048,576),
seed 5, M0 = 768, Ne = 16, interval from tools/cfg5_interval.py (512 eigenvalues by inertia
count). The factors (25.8 GB per node) of 16 nodes do not fit one B200, so the streamed memory
plan runs with node batches of FEAST_CFG5_BATCH (default 1: two slots with their W/T workspaces exceed 180 GB beside the pencil and the five N x M0 blocks): each pass refactors every batch
(the reference's low_memory trade-off). Prints one JSON line with status, count vs the inertia
count, residuals, timings."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

mem = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout.split("\n")[1].split()
avail = int(mem[6]) if len(mem) > 6 else 0
print(f"host memory available: {avail} GB", flush=True)
if avail < 80:
    print(json.dumps({"config": "cfg5", "skipped": f"host has {avail} GB available, needs ~80"}))
    sys.exit(0)
t = time.perf_counter()
prob = P.config5()
print(f"generated {prob.name} in {time.perf_counter() - t:.0f} s, interval [{prob.emin}, {prob.emax}]", flush=True)
ctx = F.GpuContext(0)
ctx.set_node_batch(int(os.environ.get("FEAST_CFG5_BATCH", "1")))
t = time.perf_counter()
ctx.set_pencil(prob.a, prob.b)
t_pencil = time.perf_counter() - t
print(f"set_pencil {t_pencil:.1f} s, storage {ctx.storage()}", flush=True)
t = time.perf_counter()
r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
              F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops,
                            seed=prob.seed))
t_solve = time.perf_counter() - t
out = dict(config=prob.name, n=prob.n, m0=prob.m0, n_e=prob.n_e, status=r.status, count=len(r.eigenvalues),
           expected=prob.expected_count, loops=r.loops_used, max_residual=r.max_residual,
           counts=[int(x) for x in r.in_interval_counts], trace_history=[float(x) for x in r.trace_history],
           timings=r.timings.__dict__, set_pencil_s=t_pencil, solve_wall_s=t_solve,
           node_batch=int(os.environ.get("FEAST_CFG5_BATCH", "1")))
print(json.dumps(out), flush=True)
