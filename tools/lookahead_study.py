"""Look-ahead admission study: per-pass cancellation factors K (FEAST_TRACE output) and the
difference between look-ahead and reference-order solves for several admission bounds."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402
from tests.golden_problems import generate  # noqa: E402

probs = {n: generate(n) for n in ["small_dense_n60", "small_dense_std_n80", "cfg1_n256", "cfg2_n2048", "bt_L16_b32", "bt_L8_b48"]}
probs["cfg2"] = P.config2()
probs["cfg1_y7"] = P.config1(yseed=7)
probs["cfg3_L16_b128"] = P.config3(L=16, b=128, seed=3, m0=32, want=16, yseed=7)


def run(prob, la, kmax):
    c = F.GpuContext(0)
    c.set_lookahead(la, kmax)
    c.set_pencil(prob.a, prob.b)
    n0 = c.lookahead_count()
    r = c.solve(F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed))
    used = c.lookahead_count() - n0
    c.close()
    return r, used


for name, prob in probs.items():
    ref, _ = run(prob, False, 0)
    for kmax in (8, 64, 1e3, 1e6):
        r, used = run(prob, True, kmax)
        same = r.status == ref.status and r.loops_used == ref.loops_used and len(r.eigenvalues) == len(ref.eigenvalues)
        ev = float(np.max(np.abs(r.eigenvalues - ref.eigenvalues) / np.maximum(np.abs(ref.eigenvalues), 1e-3 * (prob.emax - prob.emin)))) if same and len(r.eigenvalues) else -1
        print(f"{name:16s} kmax={kmax:8.0e} used={used:2d}/{ref.loops_used + 1:2d} status {r.status}/{ref.status} loops {r.loops_used}/{ref.loops_used} ev_rel={ev:.1e} maxres {r.max_residual:.1e}/{ref.max_residual:.1e}", flush=True)
