"""Host-side phase breakdown of one complete feast_solve through the C-ABI (bench.py's e2e
leg): runs the config twice in one process (cold: first context of the process; warm: a fresh
context after that) with FEAST_TRACE (default 2 = stream-synced marks) and prints the wall
clock of set_pencil + solve for each."""
import os
import sys
import time

os.environ.setdefault("FEAST_TRACE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = {"cfg1": P.config1, "cfg2": P.config2, "cfg3": P.config3, "cfg4": P.config4}[name]()
for rep in ("cold", "warm"):
    print(f"--- {rep} ---", file=sys.stderr, flush=True)
    ctx = F.GpuContext(0)
    t0 = time.perf_counter()
    ctx.set_pencil(prob.a, prob.b)
    r = ctx.solve(F.SearchInterval(prob.emin, prob.emax),
                  F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol,
                                max_loops=prob.max_loops, seed=prob.seed))
    t = time.perf_counter() - t0
    ctx.close()
    print(f"{rep}: {name} status={r.status} passes={r.loops_used + 1} wall={t * 1e3:.1f} ms "
          f"({(r.loops_used + 1) / t:.1f} passes/s) timings={r.timings}", file=sys.stderr, flush=True)
