"""config 2 contour-solve time with the sweep running alone (no look-ahead overlap), per SPIKE chunk count."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402

prob = P.config2()
for chunks in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1").split(",")]:
    c = F.GpuContext(0)
    c.set_spike(chunks)
    c.set_lookahead(False)
    c.set_pencil(prob.a, prob.b)
    c.prepare(prob.emin, prob.emax, prob.n_e)
    c.bench_init(prob.m0, prob.seed)
    c.bench_passes(3, 256 << 20)
    ms, ph = c.bench_passes(20, 256 << 20)
    c.close()
    print(json.dumps(dict(chunks=chunks, contour_ms=ph[0] / 20, sweep_kernel_ms=ph[3] / 20, rr_ms=ph[2] / 20,
                          pass_ms=ms / 20)), flush=True)
