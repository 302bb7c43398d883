#!/usr/bin/env python
"""bench.py — FEAST iterations/s on BASELINE config 2 (the headline workload).

Workload (BASELINE.json configs[1]): generalized banded pencil N=16384, half-bandwidth 16,
interval holding 128 eigenvalues (inertia count), M0=192, Ne=8. One STEP = one FEAST pass
(the loop body of core.hpp:334-388): Ne complex-shifted multi-RHS block-Thomas solves with
the fused quadrature epilogue, the ordered Q reduction (+ NCCL allreduce when N>1),
Rayleigh-Ritz with the reduced eigensolve on device, trace/count, Y = B X.

  value : passes/s, whole job, device-timed (CUDA events, max over ranks), inputs resident,
          L2 flushed (256 MiB write) between passes outside the timed events.
  e2e   : passes/s of one complete feast_solve through the C-ABI with HOST buffers
          (pencil H2D, factorisation, all passes, result D2H), wall clock around the call.
  --impl reference : the reference's own CPU loop body (oracle/_ref, the feastlite C++
          library compiled from /root/reference) on the host cores, same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FP64_TFLOPS = 37.1  # DMMA m8n8k4 f64, measured on this pool's B200 (profiles/fp64_peak.txt)
# the contour-solve kernel bench.py's roofline reports (config 2: b = 16, twisted, bulk-copy
# pipeline, 8-column CTAs; sweep_small.cu) and its DRAM traffic key in profiles/r01_traffic.json
SWEEP_KERNEL = "bt_sweep_bulk_kernel<16,8,1,0,1>"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_ready(self, timeout=5.0):
        """nvidia-smi needs a moment before its first sample; start timing after it."""
        t0 = time.monotonic()
        while self.proc and not self.lines and time.monotonic() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, region=None):
        """Samples taken during `region` (monotonic t0, t1), widened by one sampling period
        on each side so short regions still get the samples that straddle them."""
        sm, smax, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            if region and not (region[0] - 0.12 <= t <= region[1] + 0.12):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_problem(name):
    from paper_0901_2665_b200 import problems as P
    if name == "cfg2":
        return P.config2()
    if name == "cfg1":
        return P.config1()
    if name == "cfg3":
        return P.config3()
    if name == "cfg4":
        return P.config4()
    raise SystemExit(f"unknown config {name}")


def sweep_flops(prob, ctx_b=None):
    """Algorithmic flops of one contour-solve launch (all Ne nodes, M0 columns).
    block-Thomas: per node (3L-2) complex b x b by b x M0 products = 8*(3L-2)*b^2*M0 flops.
    dense LU solve: 8*N^2*M0 flops per node (two triangular solves)."""
    from paper_0901_2665_b200 import abi
    m0, ne = prob.m0, prob.n_e
    if prob.a.kind == abi.STORAGE_DENSE:
        return 8.0 * prob.n ** 2 * m0 * ne, 16.0 * prob.n ** 2 * ne + 48.0 * prob.n * m0 * ne
    b = ctx_b or 16
    L = (prob.n + b - 1) // b
    flops = 8.0 * (3 * L - 2) * b * b * m0 * ne
    bytes_ = 16.0 * (2 * L - 1) * b * b * ne + 16.0 * (L - 1) * b * b + 48.0 * L * b * m0 * ne
    return flops, bytes_


def run_reference(args, prob, world, rank):
    if rank != 0:
        return
    from oracle import oracle as O
    nproc = os.cpu_count() or 1
    threads = max(1, min(prob.n_e, nproc))
    kind = "reference" if O.available("reference") else "port"
    # one step = one reference loop body; factorisation once (outside the steps)
    O.bench_passes(prob, 0, threads=threads, kind=kind)  # warms the library
    t_s = []
    for i in range(args.warmup + args.steps):
        r = O.bench_passes(prob, 1, threads=threads, kind=kind)
        if i >= args.warmup:
            t_s.append(r["solve_s"] + r["reduce_s"])
    tot = sum(t_s)
    v = args.steps / tot
    line = {
        "impl": "reference", "metric": "feast_iterations_per_sec", "value": v, "unit": "iter/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, problems.py)",
        "config": {"workload": prob.name, "n": prob.n, "m0": prob.m0, "n_e": prob.n_e,
                   "interval": [prob.emin, prob.emax]},
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": threads, "kind": kind,
                         "sample": f"{args.steps} passes of the reference loop body "
                                   f"(accumulate_subspace_real + rayleigh_ritz + B*X), factors "
                                   f"prepared once, threads={threads} of nproc={nproc}"},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush-mib", type=int, default=256)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)

    prob = make_problem(args.config)
    if args.impl == "reference":
        run_reference(args, prob, world, rank)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_0901_2665_b200 import feast as F
    ctx = F.GpuContext(local)
    if world > 1:
        import torch
        uid = F.GpuContext.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
        dist.broadcast(t, 0)
        ctx.set_comm(bytes(t.numpy().tobytes()), rank, world)
    ctx.set_pencil(prob.a, prob.b)
    ctx.prepare(prob.emin, prob.emax, prob.n_e)
    ctx.bench_init(prob.m0, prob.seed)
    flush = args.flush_mib << 20
    ctx.bench_passes(args.warmup, flush)
    if dist:
        dist.barrier()
    l0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        clk.wait_ready()
        t_region = time.monotonic()
        ms, ph = ctx.bench_passes(args.steps, flush)
        t_region = (t_region, time.monotonic())
        time.sleep(0.15)  # the sample straddling the end of the region
    launches = ctx.launch_count() - l0
    if dist:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        dist.barrier()
    value = args.steps / (ms / 1e3)

    # e2e: complete solves through the C-ABI with host buffers, each on a fresh context (pencil
    # upload, factorisation, all passes, result download); one untimed warm-up solve, then
    # E2E_REPS timed ones (wall clock, median, max over ranks)
    from paper_0901_2665_b200 import abi
    E2E_REPS = 5

    def e2e_solve():
        ctx2 = F.GpuContext(local)
        if world > 1:
            import torch
            uid = F.GpuContext.nccl_unique_id() if rank == 0 else bytes(128)
            t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
            dist.broadcast(t, 0)
            ctx2.set_comm(bytes(t.numpy().tobytes()), rank, world)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        ctx2.set_pencil(prob.a, prob.b)
        r = ctx2.solve(F.SearchInterval(prob.emin, prob.emax),
                       F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol,
                                     max_loops=prob.max_loops, seed=prob.seed))
        dt = time.perf_counter() - t0
        ctx2.close()
        return r, dt

    e2e_solve()
    times, passes_total = [], 0
    for _ in range(E2E_REPS):
        res, dt = e2e_solve()
        times.append(dt)
        passes_total += res.loops_used + 1
    # median of the repetitions: single solves on this pool's boxes occasionally run 2x slow
    # (host-side stalls between the ~1 ms kernels), which a mean of few samples would report
    e2e_s = float(sorted(times)[len(times) // 2])
    if dist:
        import torch
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    passes_e2e = passes_total / E2E_REPS

    def op_bytes(o):
        tot = 0
        for arr in (o.dense, o.row_ptr, o.col_idx, o.values, o.diag, o.lower):
            if arr is not None:
                tot += arr.nbytes
        return tot
    # inputs: the pencil (the initial block is drawn on the device, random_block_device)
    h2d = (op_bytes(prob.a) + op_bytes(prob.b)) / passes_e2e
    d2h = (8 * prob.n * (len(res.eigenvalues) + res.subspace.shape[1]) + 8 * prob.m0 * 3) / passes_e2e

    b_used = 16 if prob.a.kind != abi.STORAGE_DENSE else None
    # DRAM traffic of the same kernel from the committed ncu --set full capture (profiles/)
    traffic = None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")) as f:
            tr = json.load(f).get(SWEEP_KERNEL)
        if b_used and tr and tr["config"].startswith(prob.name):
            traffic = tr["dram_bytes_read_per_launch"] + tr["dram_bytes_write_per_launch"]
    except (OSError, ValueError, KeyError):
        traffic = None
    flops, bytes_ = sweep_flops(prob, b_used)
    k_ms = ph[3] / args.steps
    achieved = flops / (k_ms * 1e-3) / 1e12
    out = {
        "metric": "feast_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, problems.py)",
        "config": {"workload": prob.name, "n": prob.n, "m0": prob.m0, "n_e": prob.n_e,
                   "interval": [prob.emin, prob.emax], "nodes_per_gpu": prob.n_e / world,
                   "l2": f"flushed ({args.flush_mib} MiB write) between passes, outside timing",
                   "parallelism": f"contour nodes sharded over {world} GPU(s)"},
        "phase_ms_per_step": {"contour_solves": ph[0] / args.steps, "q_reduce_allreduce": ph[1] / args.steps,
                              "rayleigh_ritz": ph[2] / args.steps},
        "eigenpairs_per_sec": len(res.eigenvalues) / e2e_s,
        "e2e": {"value": passes_e2e / e2e_s, "unit": "iter/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "passes": passes_e2e, "status": res.status,
                "eigenpairs": len(res.eigenvalues), "seconds": e2e_s,
                "method": f"wall clock of set_pencil + solve on a fresh context, median of {E2E_REPS} "
                          "solves after one untimed warm-up solve",
                "samples_s": [round(t_, 6) for t_ in times]},
        "roofline": {"kernel": SWEEP_KERNEL if b_used else "dense_solve (zgemm chain)",
                     "bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu, profiles/r01_traffic.json)",
                     "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": bytes_,
                     "hbm_frac": bytes_ / (k_ms * 1e-3) / 1e9 / peaks().get("hbm_gbs", 6650.0),
                     "avg_launch_ms": k_ms, "peak_source": "measured DMMA f64 (tools/microbench/fp64_peak.cu)"},
        "gpu_launches": launches,
        "clocks": clk.summary(t_region),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            nproc = os.cpu_count() or 1
            threads = max(1, min(prob.n_e, nproc))
            kind = "reference" if O.available("reference") else "port"
            r = O.bench_passes(prob, 2, threads=threads, kind=kind)
            v = 2 / (r["solve_s"] + r["reduce_s"])
            out["cpu_baseline"] = {"value": v, "unit": "iter/s", "cores": threads, "kind": kind,
                                   "sample": "2 passes of the reference loop body, factors once "
                                             f"({r['factorize_s']:.2f}s), threads={threads}/{nproc}"}
        except Exception as e:  # reported, never fatal
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    ctx.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
