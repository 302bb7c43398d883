"""Reduced eigensolve at several sizes (for an ncu launch list of the tridiagonal kernels)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402

ctx = F.GpuContext(0)
rng = np.random.default_rng(0)
for m in [int(a) for a in sys.argv[1:]]:
    a = rng.uniform(-1, 1, (m, m)); a = a + a.T
    b = np.eye(m)
    ctx.reduced_gevp(a, b)
