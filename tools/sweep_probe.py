"""config 2: three contour passes (for ncu timing of the sweep kernel alone)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config2()
c = F.GpuContext(0)
c.set_spike(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
c.set_pencil(prob.a, prob.b)
c.prepare(prob.emin, prob.emax, prob.n_e)
y = np.asfortranarray(np.random.default_rng(1).standard_normal((prob.n, prob.m0)))
for _ in range(3):
    q = c.contour_pass(y)
print("norm", float(np.linalg.norm(q)))
