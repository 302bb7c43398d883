"""Generates tests/golden/*.npz: inputs + the REFERENCE's own feast_solve outputs
(oracle/_ref, compiled from /root/reference). Run in the build container:
    python tests/golden/make_golden.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.golden_problems import GOLDEN, NAMES, generate, save_fixture  # noqa: E402

if __name__ == "__main__":
    assert O.available("reference"), "build oracle/_ref first (make -C oracle reference)"
    for name in NAMES:
        prob = generate(name)
        r = O.feast_solve(prob, kind="reference")
        out = {k: r[k] for k in ("eigenvalues", "eigenvectors", "residuals", "trace_history",
                                 "in_interval_counts", "subspace")}
        out.update(status=r["status"], m=r["m"], loops_used=r["loops_used"], max_residual=r["max_residual"])
        save_fixture(prob, out, os.path.join(GOLDEN, name + ".npz"))
        print(name, r["status"], r["m"], r["loops_used"], f"{r['max_residual']:.1e}")
