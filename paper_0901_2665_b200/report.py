"""RunReport at the boundary: the reference harness's per-solve record
(`RunReport`, include/feast/report.hpp:19-36), its JSON form (`report_to_json`,
src/report.cpp:11-35: same keys in the same order, timings optional for byte-stable comparison)
and CSV form (`write_report_csv`, src/report.cpp:37-45), filled from a GPU `FeastResult` the
way `solve_pencil` fills it (src/run.cpp:14-44) and from `GpuContext.sweep` steps the way
`run_sweep` does (src/run.cpp:63-125: a failed step carries "error: <message>").
The schema contract is docs/run_report.schema.json of the reference (checked by
tests/test_report.py when the reference tree is present)."""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi

STATUS_PATTERN = r"^(converged|max-loops|no-eigenvalues-in-interval|subspace-saturated|subspace-breakdown|error: .*)$"


@dataclass
class RunReport:
    n: int = 0
    nnz: int = 0
    lambda_min: float = 0.0
    lambda_max: float = 0.0
    m0: int = 0
    ne: int = 0
    loops: int = 0
    status: str = ""
    eigenvalues: List[float] = field(default_factory=list)
    residuals: List[float] = field(default_factory=list)
    max_residual: float = 0.0
    trace_history: List[float] = field(default_factory=list)
    in_interval_counts: List[int] = field(default_factory=list)
    timings: Optional[dict] = None
    seed: int = 0
    source: str = ""


def operator_nnz(op) -> int:
    """SymmetricOperator::nnz (operator.hpp): stored entries, symmetric-complete for sparse
    storage, n * n for dense; block-tridiagonal storage counts its nonzero entries both ways."""
    if op.kind == abi.STORAGE_DENSE:
        return op.n * op.n
    if op.kind == abi.STORAGE_CSR:
        return int(op.row_ptr[op.n])
    return int(np.count_nonzero(op.diag) + 2 * np.count_nonzero(op.lower))


def union_nnz(a0, s) -> int:
    """nnz of add_scaled(a0, s, t) (operator.hpp:282-304): the union pattern when both are sparse."""
    if a0.kind == abi.STORAGE_DENSE or s.kind == abi.STORAGE_DENSE:
        return a0.n * a0.n
    return int((abs(a0.to_scipy()) + abs(s.to_scipy())).nnz)


def run_report(result, a, lambda_min, lambda_max, config, source="") -> RunReport:
    """solve_pencil's report (run.cpp:26-42) of one FeastResult."""
    t = result.timings
    return RunReport(n=a.n, nnz=operator_nnz(a), lambda_min=float(lambda_min), lambda_max=float(lambda_max),
                     m0=int(config.m0), ne=int(config.n_e), loops=int(result.loops_used), status=result.status,
                     eigenvalues=[float(x) for x in result.eigenvalues],
                     residuals=[float(x) for x in result.residuals], max_residual=float(result.max_residual),
                     trace_history=[float(x) for x in result.trace_history],
                     in_interval_counts=[int(x) for x in result.in_interval_counts],
                     timings=dict(factorize_s=t.factorize_s, solve_s=t.solve_s, reduce_s=t.reduce_s,
                                  total_s=t.total_s),
                     seed=int(config.seed), source=source)


def sweep_reports(results, a0, s, steps, lambda_min, lambda_max, config, source="") -> List[RunReport]:
    """run_sweep's reports (run.cpp:77-104): one per step, source "<base> + <t>*S" with
    std::to_string's six decimals, failed steps as "error: <message>"."""
    out = []
    for t, r in zip(steps, results):
        src = f"{source} + {t:.6f}*S"
        if isinstance(r, Exception):
            out.append(RunReport(n=a0.n, nnz=union_nnz(a0, s), lambda_min=float(lambda_min), lambda_max=float(lambda_max),
                                 m0=int(config.m0), ne=int(config.n_e), status=f"error: {r}",
                                 seed=int(config.seed), source=src))
        else:
            out.append(run_report(r, a0, lambda_min, lambda_max, config, src))
    return out


def report_to_json(r: RunReport, include_timings: bool = True) -> dict:
    """report_to_json (report.cpp:11-35): the same keys in the same order."""
    j = dict(n=r.n, nnz=r.nnz, lambda_min=r.lambda_min, lambda_max=r.lambda_max, m0=r.m0, ne=r.ne, loops=r.loops,
             status=r.status, eigenvalues=list(r.eigenvalues), residuals=list(r.residuals),
             max_residual=r.max_residual, trace_history=list(r.trace_history),
             in_interval_counts=list(r.in_interval_counts))
    if include_timings and r.timings is not None:
        j["timings"] = {k: r.timings[k] for k in ("factorize_s", "solve_s", "reduce_s", "total_s")}
    j["seed"] = r.seed
    j["source"] = r.source
    return j


def dumps(r: RunReport, include_timings: bool = True) -> str:
    return json.dumps(report_to_json(r, include_timings), indent=2)


def write_report_csv(out, r: RunReport):
    """write_report_csv (report.cpp:37-45): index,eigenvalue,residual with %.17g."""
    out.write("index,eigenvalue,residual\n")
    for i, (ev, res) in enumerate(zip(r.eigenvalues, r.residuals)):
        out.write("%d,%.17g,%.17g\n" % (i, ev, res))
