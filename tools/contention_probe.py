"""Two contexts on one device, one host thread each: A repeats a contour pass, B repeats the reduced
eigensolve; each compares its results with its first, bit for bit. Finds kernels whose results change
when another kernel shares the GPU (a race that lockstep execution hides)."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import feast as F  # noqa: E402
from tests.golden import make_fullsize as MF  # noqa: E402

prob = MF.problem(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
a = F.GpuContext(0)
a.set_pencil(prob.a, prob.b)
a.prepare(prob.emin, prob.emax, prob.n_e)
y = a.random_block(prob.n, prob.m0, prob.seed)
q0 = a.contour_pass(y)
aq = np.asfortranarray(q0.T @ prob.a.matmul(q0)); aq = 0.5 * (aq + aq.T)
bq = np.asfortranarray(q0.T @ prob.b.matmul(q0)); bq = 0.5 * (bq + bq.T)
b = F.GpuContext(0)
e0, p0, _ = b.reduced_gevp(aq, bq)
out = {"sweep": [], "eig": []}
stop = threading.Event()


def loop_a():
    for _ in range(reps):
        out["sweep"].append(bool(np.array_equal(a.contour_pass(y), q0)))
    stop.set()


def loop_b():
    while not stop.is_set():
        e, p, _ = b.reduced_gevp(aq, bq)
        out["eig"].append(bool(np.array_equal(e, e0) and np.array_equal(p, p0)))


ta, tb = threading.Thread(target=loop_a), threading.Thread(target=loop_b)
ta.start(); tb.start(); ta.join(); tb.join()
print("sweep identical:", out["sweep"])
print("eigensolve identical: %d of %d" % (sum(out["eig"]), len(out["eig"])))
a.close(); b.close()
