"""Small named problems shared by the golden fixtures, the oracle pins and the GPU parity
tests. Inputs are stored inside each fixture (tests/golden/*.npz), so every machine sees
the same bits regardless of BLAS threading."""
import os

import numpy as np

from paper_0901_2665_b200 import abi
from paper_0901_2665_b200 import problems as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def generate(name):
    if name == "small_dense_n60":
        return P.small_dense(60, seed=7, want=6, m0=10)
    if name == "small_dense_std_n80":
        return P.small_dense(80, seed=8, want=8, m0=14, gen=False)
    if name == "cfg1_n256":
        return P.config1(n=256, m0=40)
    if name == "cfg2_n2048":
        return P.config2(n=2048, bw=16, m0=48, want=24)
    if name == "bt_L16_b32":
        a, b = P.blocktri_operators(16, 32, seed=11)
        lo, hi = P._cached_interval("bt_L16_b32_s11_k20", lambda: P.interval_with_count(a, b, 20, 0.0, 0.25))
        return P.Problem("bt_L16_b32", a, b, lo, hi, 32, expected_count=20)
    if name == "bt_L8_b48":
        a, b = P.blocktri_operators(8, 48, seed=12)
        lo, hi = P._cached_interval("bt_L8_b48_s12_k12", lambda: P.interval_with_count(a, b, 12, 0.0, 0.25))
        return P.Problem("bt_L8_b48", a, b, lo, hi, 20, expected_count=12)
    raise KeyError(name)


NAMES = ["small_dense_n60", "small_dense_std_n80", "cfg1_n256", "cfg2_n2048", "bt_L16_b32", "bt_L8_b48"]


def _pack(prefix, op, d):
    d[prefix + "kind"] = op.kind
    d[prefix + "n"] = op.n
    for f in ("dense", "row_ptr", "col_idx", "values", "diag", "lower"):
        v = getattr(op, f)
        if v is not None:
            d[prefix + f] = v
    d[prefix + "nblocks"] = op.nblocks
    d[prefix + "bsize"] = op.bsize


def _unpack(prefix, g):
    kind = int(g[prefix + "kind"])
    n = int(g[prefix + "n"])
    get = lambda f: np.array(g[prefix + f]) if (prefix + f) in g.files else None
    op = P.Operator(kind, n, dense=None if get("dense") is None else np.asfortranarray(get("dense")),
                    row_ptr=get("row_ptr"), col_idx=get("col_idx"), values=get("values"),
                    nblocks=int(g[prefix + "nblocks"]), bsize=int(g[prefix + "bsize"]),
                    diag=get("diag"), lower=get("lower"))
    return op


def save_fixture(prob, outputs, path):
    d = {}
    _pack("a_", prob.a, d)
    _pack("b_", prob.b, d)
    d.update(name=prob.name, emin=prob.emin, emax=prob.emax, m0=prob.m0, n_e=prob.n_e,
             trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed,
             expected_count=-1 if prob.expected_count is None else prob.expected_count)
    for k, v in outputs.items():
        d["out_" + k] = v
    np.savez_compressed(path, **d)


def load_fixture(path):
    g = np.load(path, allow_pickle=False)
    prob = P.Problem(str(g["name"]), _unpack("a_", g), _unpack("b_", g), float(g["emin"]), float(g["emax"]),
                     int(g["m0"]), n_e=int(g["n_e"]), trace_tol=float(g["trace_tol"]),
                     max_loops=int(g["max_loops"]), seed=int(g["seed"]),
                     expected_count=int(g["expected_count"]))
    out = {k[4:]: g[k] for k in g.files if k.startswith("out_")}
    return prob, out


def fixtures():
    if not os.path.isdir(GOLDEN):
        return []
    # (full_*.npz are the full-size reference runs of tests/golden/make_fullsize.py: outputs only)
    return sorted(os.path.join(GOLDEN, f) for f in os.listdir(GOLDEN)
                  if f.endswith(".npz") and not f.startswith("full_"))
