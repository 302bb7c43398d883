"""config 2 passes/s, contour-solve time and factorisation time for SPIKE chunk counts 1..16."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config2()
for chunks in (1, 2, 4, 8, 16):
    for la in (True, False):
        c = F.GpuContext(0)
        c.set_spike(chunks)
        c.set_lookahead(la)
        c.set_pencil(prob.a, prob.b)
        t0 = time.perf_counter()
        c.prepare(prob.emin, prob.emax, prob.n_e)
        tf = time.perf_counter() - t0
        c.bench_init(prob.m0, prob.seed)
        c.bench_passes(3, 256 << 20)
        ms, ph = c.bench_passes(20, 256 << 20)
        c.close()
        c2 = F.GpuContext(0)
        c2.set_spike(chunks)
        c2.set_lookahead(la)
        t0 = time.perf_counter()
        c2.set_pencil(prob.a, prob.b)
        r = c2.solve(F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0, n_e=prob.n_e, seed=prob.seed))
        te = time.perf_counter() - t0
        c2.close()
        print(json.dumps(dict(chunks=chunks, lookahead=la, passes_per_s=20 / (ms / 1e3), contour_ms=ph[0] / 20,
                              rr_ms=ph[2] / 20, factor_ms=1e3 * tf, e2e_ms=1e3 * te, e2e_passes=r.loops_used + 1,
                              status=r.status, count=len(r.eigenvalues))), flush=True)
