"""Runs W+1 FEAST passes of a config through the C-ABI (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = {"cfg1": P.config1, "cfg2": P.config2, "cfg3": P.config3, "cfg4": P.config4}[cfg]()
import time  # noqa: E402

ctx = F.GpuContext(0)
t0 = time.perf_counter()
ctx.set_pencil(prob.a, prob.b)
t1 = time.perf_counter()
ctx.prepare(prob.emin, prob.emax, prob.n_e)
t2 = time.perf_counter()
print(f"{cfg}: set_pencil {t1 - t0:.3f}s  prepare(factor) {t2 - t1:.3f}s", flush=True)
ctx.bench_init(prob.m0, prob.seed)
ms, ph = ctx.bench_passes(passes, 0)
print(f"{cfg}: {passes} passes {ms:.3f} ms  phases {ph}")
