"""A cold process's config-2 solve, phase by phase: library load, CUDA context, set_pencil, solve
(FEAST_TRACE=2 marks on stderr), close."""
import os
import sys
import time

t0 = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config2()
t1 = time.perf_counter()
from paper_0901_2665_b200 import feast as F  # noqa: E402
F.load_library()
t2 = time.perf_counter()
c = F.GpuContext(0)
t3 = time.perf_counter()
c.set_pencil(prob.a, prob.b)
t4 = time.perf_counter()
r = c.solve(F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0, n_e=prob.n_e, seed=prob.seed))
t5 = time.perf_counter()
c.close()
t6 = time.perf_counter()
print(f"generate {t1 - t0:.3f}  load {t2 - t1:.3f}  context {t3 - t2:.3f}  set_pencil {t4 - t3:.3f}  "
      f"solve {t5 - t4:.3f}  close {t6 - t5:.3f}  passes {r.loops_used + 1}", flush=True)
