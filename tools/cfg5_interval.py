"""Search interval for the full-size config 5 (L = 2048, b = 512, N = 1,048,576, seed 5) holding
512 eigenvalues, from inertia (Sturm) counts of A - sigma B (block-LDL^T Schur complements,
problems.inertia_count). The full gap-midpoint search of problems.interval_with_count needs
~200 counts (~80 s each here), so this uses lo = 0 and bisects the first eigenvalue above the
512th one to a third of the mean spacing (hi = the bracket's left end, count exactly
c0 + 512); ~16 counts. Writes intervals.json["blocktri_L2048_b512_s5_k512"]."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2665_b200 import problems as P  # noqa: E402

# usage: cfg5_interval.py [L [tol]]   (the scaled config 5 of SURVEY 8(c): L = 64, tol ~ a third of the spacing)
L, b, seed, want = (int(sys.argv[1]) if len(sys.argv) > 1 else 2048), 512, 5, 512
TOL = float(sys.argv[2]) if len(sys.argv) > 2 else 3e-6
t0 = time.time()
a, bb = P.blocktri_operators(L, b, seed)
print(f"generated in {time.time() - t0:.0f} s", flush=True)


def count(s):
    t = time.time()
    c = P.inertia_count(a, bb, s)
    print(f"count({s:.9g}) = {c}  ({time.time() - t:.0f} s)", flush=True)
    return c


lo = 0.0
c0 = count(lo)
target = c0 + want
x, y = lo, 0.004
cy = count(y)
while cy <= target:
    x, y = y, 2 * y
    cy = count(y)
cx = c0 if x == lo else count(x)
# bisection: keep count(x) <= target < count(y)
while y - x > TOL:
    mid = 0.5 * (x + y)
    cm = count(mid)
    if cm <= target:
        x, cx = mid, cm
    else:
        y, cy = mid, cm
while cx < target:  # x must hold exactly target eigenvalues below it
    mid = 0.5 * (x + y)
    cm = count(mid)
    if cm <= target:
        x, cx = mid, cm
    else:
        y, cy = mid, cm
hi = x
assert count(hi) - c0 == want
path = os.path.join(os.path.dirname(P.__file__), "intervals.json")
data = json.load(open(path))
data[f"blocktri_L{L}_b{b}_s{seed}_k{want}"] = {"lo": lo, "hi": hi, "count_lo": c0, "count_hi": c0 + want,
                                               "first_above_bracket": [x, y],
                                               "method": "tools/cfg5_interval.py (lo = 0, bisection)"}
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
if os.path.isdir(out):  # (run on the GPU box: only gpurun_out/ travels back)
    json.dump({f"blocktri_L{L}_b{b}_s{seed}_k{want}": data[f"blocktri_L{L}_b{b}_s{seed}_k{want}"]},
              open(os.path.join(out, f"interval_L{L}.json"), "w"), indent=1, sort_keys=True)
print(f"interval [{lo}, {hi}] holds {want}; total {time.time() - t0:.0f} s", flush=True)
