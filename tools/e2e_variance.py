"""End-to-end solve times on config 2 (fresh context each), look-ahead on and off, and a cold
process breakdown; prints one line per solve."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.perf_counter()
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402
t_import = time.perf_counter() - t0
prob = P.config2()
cfg = F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed)
iv = F.SearchInterval(prob.emin, prob.emax)
for la in (True, False, True):
    for k in range(6):
        t0 = time.perf_counter()
        c = F.GpuContext(0)
        t1 = time.perf_counter()
        c.set_lookahead(la)
        c.set_pencil(prob.a, prob.b)
        t2 = time.perf_counter()
        r = c.solve(iv, cfg)
        t3 = time.perf_counter()
        c.close()
        t4 = time.perf_counter()
        print(f"la={int(la)} k={k} create {1e3*(t1-t0):7.2f} pencil {1e3*(t2-t1):6.2f} solve {1e3*(t3-t2):6.2f} "
              f"close {1e3*(t4-t3):6.2f} passes {r.loops_used + 1} timings {r.timings}", flush=True)
print("import", t_import)
