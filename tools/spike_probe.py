"""config 2 contour passes with a given SPIKE chunk count (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config2()
c = F.GpuContext(0)
c.set_spike(int(sys.argv[1]))
c.set_lookahead(False)
c.set_pencil(prob.a, prob.b)
c.prepare(prob.emin, prob.emax, prob.n_e)
c.bench_init(prob.m0, prob.seed)
ms, ph = c.bench_passes(4, 0)
print(ms / 4, ph / 4)
