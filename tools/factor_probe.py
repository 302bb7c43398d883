"""config 4 (or cfg1): set_pencil + prepare only (for ncu timing of the factorisation kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = {"cfg1": P.config1, "cfg4": P.config4}[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]()
c = F.GpuContext(0)
c.set_pencil(prob.a, prob.b)
for _ in range(2):
    t0 = time.perf_counter()
    c.prepare(prob.emin, prob.emax, prob.n_e)
    print("prepare %.3f s" % (time.perf_counter() - t0), flush=True)
