"""The multi-rank path of the C++ library on ONE GPU.

* NCCL itself: a one-rank NCCL communicator (feast_gpu_set_comm with nranks = 1) routes every
  collective through ncclAllReduce / ncclAllGather; results must equal the no-communicator run
  bit for bit.
* R ranks: R contexts on device 0 joined as a loopback group (feast_gpu_set_group), one host thread
  each (ctypes releases the GIL), run the sharded contour (contiguous node blocks, per-rank
  ascending sums, allreduce) and the row-distributed Rayleigh-Ritz (slab applies and projections,
  allreduce of 2 M0^2 values, slab allgathers). Against the one-rank run: the contour pass's Q to
  1e-13 (the partial sums add in a different order), the full solve to the parity tolerances
  (same status, counts and loops; eigenvalues 1e-10; principal angles 1e-8), and every rank must
  return the same bits (the replicated decisions agree).
"""
import threading

import numpy as np
import pytest

from tests.golden_problems import generate
from tests.test_gpu_parity import sin_max_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_0901_2665_b200 import feast
    feast.load_library()
    return feast


def cfg_of(F, prob):
    return F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops,
                         seed=prob.seed)


def solve_one(F, prob, lookahead=True):
    c = F.GpuContext(0)
    try:
        c.set_lookahead(lookahead)
        c.set_pencil(prob.a, prob.b)
        return c.solve(F.SearchInterval(prob.emin, prob.emax), cfg_of(F, prob))
    finally:
        c.close()


def run_ranks(F, nranks, body, row_dist=True, lookahead=True):
    """body(ctx, rank) on nranks contexts of a loopback group, one thread each."""
    g = F.LocalGroup(nranks)
    ctxs = [F.GpuContext(0) for _ in range(nranks)]
    out, errs = [None] * nranks, [None] * nranks

    def work(r):
        try:
            ctxs[r].set_group(g, r)
            ctxs[r].set_row_distribution(row_dist)
            ctxs[r].set_lookahead(lookahead)
            out[r] = body(ctxs[r], r)
        except Exception as e:  # re-raised below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in ctxs:
        c.close()
    g.close()
    for e in errs:
        if e is not None:
            raise e
    return out


def test_one_rank_nccl_communicator(F):
    prob = generate("cfg2_n2048")
    ref = solve_one(F, prob)
    c = F.GpuContext(0)
    try:
        c.set_comm(F.GpuContext.nccl_unique_id(), 0, 1)
        c.set_pencil(prob.a, prob.b)
        r = c.solve(F.SearchInterval(prob.emin, prob.emax), cfg_of(F, prob))
    finally:
        c.close()
    assert r.status == ref.status and r.loops_used == ref.loops_used
    assert np.array_equal(r.eigenvalues, ref.eigenvalues)
    assert np.array_equal(r.eigenvectors, ref.eigenvectors)


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("which", ["cfg2_n2048", "small_dense_n60"])
def test_sharded_contour_pass_sums_to_one_rank(F, which, nranks):
    prob = generate(which)
    y = np.random.default_rng(9).uniform(-1, 1, (prob.n, prob.m0))
    c = F.GpuContext(0)
    try:
        c.set_pencil(prob.a, prob.b)
        c.prepare(prob.emin, prob.emax, prob.n_e)
        q1 = c.contour_pass(y)
    finally:
        c.close()

    def body(ctx, r):
        ctx.set_pencil(prob.a, prob.b)
        ctx.prepare(prob.emin, prob.emax, prob.n_e)
        return ctx.contour_pass(y)
    qs = run_ranks(F, nranks, body)
    for q in qs:
        assert np.array_equal(q, qs[0])
        assert np.max(np.abs(q - q1)) <= 1e-13 * max(1.0, np.max(np.abs(q1)))


@pytest.mark.parametrize("row_dist,lookahead", [(True, True), (True, False), (False, True)])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("which", ["cfg2_n2048", "bt_L16_b32", "bt_L8_b48", "small_dense_n60", "cfg1_n256"])
def test_sharded_solve_matches_one_rank(F, which, nranks, row_dist, lookahead):
    prob = generate(which)
    ref = solve_one(F, prob, lookahead)

    def body(ctx, r):
        ctx.set_pencil(prob.a, prob.b)
        return ctx.solve(F.SearchInterval(prob.emin, prob.emax), cfg_of(F, prob))
    rs = run_ranks(F, nranks, body, row_dist=row_dist, lookahead=lookahead)
    for r in rs[1:]:  # every rank took the same decisions on the same bits
        assert r.status == rs[0].status and r.loops_used == rs[0].loops_used
        assert np.array_equal(r.eigenvalues, rs[0].eigenvalues)
        assert np.array_equal(r.eigenvectors, rs[0].eigenvectors)
    r = rs[0]
    # the sharded sums (and the SPIKE chunking each rank picks for its share of the nodes) round
    # differently, and FEAST's 1e-13 trace-stagnation test may then stop a pass or two apart; the
    # status and the eigenpairs must agree
    assert r.status == ref.status and abs(r.loops_used - ref.loops_used) <= 2, (r.loops_used, ref.loops_used)
    if r.loops_used == ref.loops_used:
        assert np.array_equal(r.in_interval_counts, ref.in_interval_counts)
    tol = 1e-10 * np.maximum(np.abs(ref.eigenvalues), 1e-3 * (prob.emax - prob.emin))
    assert len(r.eigenvalues) == len(ref.eigenvalues)
    assert np.all(np.abs(r.eigenvalues - ref.eigenvalues) <= tol)
    if len(r.eigenvalues):
        assert sin_max_angle(r.eigenvectors, ref.eigenvectors, prob.b.to_dense()) <= 1e-8
    assert r.max_residual <= max(1e-9, 10 * ref.max_residual)


def test_sharded_rayleigh_ritz_matches_one_rank(F):
    """feast_gpu_rayleigh_ritz with a full Q on every rank: slab projections + allreduce."""
    prob = generate("bt_L16_b32")
    q = np.random.default_rng(4).standard_normal((prob.n, 24))
    c = F.GpuContext(0)
    try:
        c.set_pencil(prob.a, prob.b)
        ev1, x1, _ = c.rayleigh_ritz(q)
    finally:
        c.close()

    def body(ctx, r):
        ctx.set_pencil(prob.a, prob.b)
        return ctx.rayleigh_ritz(q)
    outs = run_ranks(F, 3, body)
    for ev, x, _ in outs:
        assert np.array_equal(ev, outs[0][0]) and np.array_equal(x, outs[0][1])
        assert np.max(np.abs(ev - ev1)) <= 1e-10 * max(1.0, np.max(np.abs(ev1)))
        assert sin_max_angle(x, x1, prob.b.to_dense()) <= 1e-8
