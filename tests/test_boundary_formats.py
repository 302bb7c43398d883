"""Boundary formats: FEASTOP1 binary operator files (pencil_io.py) and the
RunReport JSON / CSV (report.py) against the reference's schema contract
(docs/run_report.schema.json, read from the reference tree when present)."""
import io
import json
import os
import re

import numpy as np
import pytest

from paper_0901_2665_b200 import abi
from paper_0901_2665_b200 import pencil_io as IO
from paper_0901_2665_b200 import report as R
from paper_0901_2665_b200.feast import FeastConfig, FeastResult, FeastTimings, InputError
from tests.golden_problems import generate

SCHEMA = "/root/reference/proj/docs/run_report.schema.json"


@pytest.mark.parametrize("name", ["small_dense_n60", "cfg2_n2048", "bt_L16_b32"])
@pytest.mark.parametrize("mmap", [True, False])
def test_operator_file_round_trip(tmp_path, name, mmap):
    prob = generate(name)
    for op in (prob.a, prob.b):
        path = tmp_path / "op.bin"
        IO.save_operator(path, op)
        back = IO.load_operator(path, mmap=mmap)
        assert back.kind == op.kind and back.n == op.n and back.nblocks == op.nblocks and back.bsize == op.bsize
        for f in ("dense", "row_ptr", "col_idx", "values", "diag", "lower"):
            x, y = getattr(op, f), getattr(back, f)
            assert (x is None) == (y is None), f
            if x is not None:
                assert np.array_equal(np.asarray(x), np.asarray(y)), f


def test_operator_file_rejects_bad_input(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTFEAST" + b"\0" * 56)
    with pytest.raises(InputError, match="not a FEASTOP1"):
        IO.load_operator(p)
    prob = generate("bt_L16_b32")
    IO.save_operator(p, prob.a)
    data = p.read_bytes()
    p.write_bytes(data[: len(data) // 2])
    with pytest.raises(InputError, match="truncated payload"):
        IO.load_operator(p)


def _fake_result():
    return FeastResult(eigenvalues=np.array([0.25, 0.5]), eigenvectors=np.zeros((3, 2)), residuals=np.array([1e-14, 2e-14]),
                       residual_absolute_only=np.array([False, False]), max_residual=2e-14, loops_used=2,
                       trace_history=np.array([0.7, 0.75, 0.75]), in_interval_counts=np.array([2, 2, 2], dtype=np.int32),
                       status="converged", subspace=np.zeros((3, 2)), timings=FeastTimings(0.1, 0.2, 0.3, 0.6))


def _validate(obj, schema, root=None):
    """The draft-07 subset docs/run_report.schema.json uses: type, required,
    additionalProperties false, minimum, pattern, items."""
    root = root or schema
    t = schema.get("type")
    types = {"object": dict, "array": list, "string": str, "integer": int, "number": (int, float)}
    if t:
        assert isinstance(obj, types[t]) and not (t in ("integer", "number") and isinstance(obj, bool)), (obj, t)
    if t == "object":
        for k in schema.get("required", []):
            assert k in obj, k
        props = schema.get("properties", {})
        if schema.get("additionalProperties") is False:
            assert set(obj) <= set(props), set(obj) - set(props)
        for k, v in obj.items():
            if k in props:
                _validate(v, props[k], root)
    if t == "array" and "items" in schema:
        for v in obj:
            _validate(v, schema["items"], root)
    if "minimum" in schema:
        assert obj >= schema["minimum"]
    if "pattern" in schema:
        assert re.search(schema["pattern"], obj), obj


def test_run_report_fields_and_order():
    prob = generate("small_dense_n60")
    rep = R.run_report(_fake_result(), prob.a, prob.emin, prob.emax, FeastConfig(m0=10, n_e=8, seed=42), "gen:small")
    j = R.report_to_json(rep)
    assert list(j) == ["n", "nnz", "lambda_min", "lambda_max", "m0", "ne", "loops", "status", "eigenvalues",
                       "residuals", "max_residual", "trace_history", "in_interval_counts", "timings", "seed",
                       "source"]  # report.cpp:11-35
    assert j["nnz"] == 60 * 60 and j["loops"] == 2 and j["status"] == "converged"
    assert "timings" not in R.report_to_json(rep, include_timings=False)
    assert json.loads(R.dumps(rep)) == j
    buf = io.StringIO()
    R.write_report_csv(buf, rep)
    assert buf.getvalue() == "index,eigenvalue,residual\n0,0.25,1e-14\n1,0.5,2e-14\n"  # C printf %.17g


@pytest.mark.skipif(not os.path.exists(SCHEMA), reason="reference tree not present")
def test_run_report_matches_reference_schema():
    schema = json.load(open(SCHEMA))
    prob = generate("cfg2_n2048")
    cfg = FeastConfig(m0=prob.m0, n_e=8, seed=42)
    rep = R.run_report(_fake_result(), prob.a, prob.emin, prob.emax, cfg, "cfg2")
    _validate(R.report_to_json(rep), schema)
    _validate(R.report_to_json(rep, include_timings=False), schema)
    reps = R.sweep_reports([_fake_result(), InputError("BicgstabShiftSystem: inner solve did not reach tolerance")],
                           prob.a, prob.a, [0.0, 0.5], prob.emin, prob.emax, cfg, "cfg2")
    assert reps[1].status.startswith("error: ") and reps[1].source == "cfg2 + 0.500000*S"
    for r in reps:
        _validate(R.report_to_json(r), schema)
    assert re.search(schema["properties"]["status"]["pattern"], "subspace-breakdown")
    assert schema["properties"]["status"]["pattern"] == R.STATUS_PATTERN
    assert sorted(abi.STATUS_NAMES) == sorted(R.STATUS_PATTERN[2:-4].split("|")[:5])


@pytest.mark.gpu
def test_solve_from_operator_files_is_bit_identical(tmp_path):
    """A memory-mapped FEASTOP1 pencil streams through the pinned stage (no re-blocking copy) and
    solves to the same bits as the in-memory pencil."""
    from paper_0901_2665_b200 import feast as F
    prob = generate("bt_L16_b32")
    IO.save_operator(tmp_path / "a.bin", prob.a)
    IO.save_operator(tmp_path / "b.bin", prob.b)
    a, b = IO.load_operator(tmp_path / "a.bin"), IO.load_operator(tmp_path / "b.bin")
    cfg = F.FeastConfig(m0=prob.m0, n_e=prob.n_e, seed=prob.seed)
    out = []
    for pa, pb in ((prob.a, prob.b), (a, b)):
        c = F.GpuContext(0)
        try:
            c.set_pencil(pa, pb)
            out.append(c.solve(F.SearchInterval(prob.emin, prob.emax), cfg))
        finally:
            c.close()
    assert np.array_equal(out[0].eigenvalues, out[1].eigenvalues)
    assert np.array_equal(out[0].eigenvectors, out[1].eigenvectors)
    rep = R.run_report(out[1], a, prob.emin, prob.emax, cfg, f"{tmp_path}/a.bin {tmp_path}/b.bin")
    if os.path.exists(SCHEMA):
        _validate(R.report_to_json(rep), json.load(open(SCHEMA)))
