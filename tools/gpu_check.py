"""Developer smoke check on a GPU box: every stage of the boundary against the reference
oracle (oracle/_ref). Prints one line per check; never raises on mismatch."""
import os
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_0901_2665_b200 import feast as F  # noqa: E402
from paper_0901_2665_b200 import problems as P  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))


def check(name, fn):
    t = time.time()
    try:
        msg = fn()
        print(f"[ok ] {name}: {msg} ({time.time()-t:.2f}s)", flush=True)
    except Exception as e:
        print(f"[ERR] {name}: {e!r} ({time.time()-t:.2f}s)", flush=True)
        traceback.print_exc()


def rgevp(m, seed, trunc=False):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (m, m)); a = a + a.T
    r = rng.uniform(-1, 1, (m, m))
    if trunc:
        r[:, : m // 3] = 0.0
        b = r.T @ r / m
    else:
        b = r.T @ r / m + np.eye(m)
    b = 0.5 * (b + b.T)
    return a, b


def main():
    ctx = F.GpuContext(0)
    for m in [8, 50, 160, 192, 300]:
        def f(m=m):
            a, b = rgevp(m, m)
            ev, phi, tr = ctx.reduced_gevp(a, b)
            rev, rphi, rtr = O.reduced_gevp(a, b)
            orth = np.max(np.abs(phi.T @ b @ phi - np.eye(phi.shape[1])))
            res = np.max(np.abs(a @ phi - b @ phi * ev))
            return f"m={m} trunc={tr}/{rtr} ev_rel={rel(ev, rev):.2e} orth={orth:.2e} res={res:.2e}"
        check(f"reduced_gevp m={m}", f)

    def ftr():
        a, b = rgevp(40, 3, trunc=True)
        ev, phi, tr = ctx.reduced_gevp(a, b)
        rev, rphi, rtr = O.reduced_gevp(a, b)
        return f"trunc={tr}/{rtr} k={len(ev)}/{len(rev)} ev_rel={rel(ev, rev) if len(ev)==len(rev) else -1:.2e}"
    check("reduced_gevp truncation", ftr)

    probs = [P.small_dense(60), P.config1(n=256, m0=40), P.config2(n=2048, bw=16, m0=48, want=24)]
    try:
        a, bb = P.blocktri_operators(16, 32, seed=11)
        lo, hi, _ = P.interval_with_count(a, bb, 20, 0.0, 0.25)
        probs.append(P.Problem("bt_L16_b32", a, bb, lo, hi, 32, expected_count=20))
    except Exception as e:
        print("blocktri gen failed", e)
    for p in probs:
        def fs(p=p):
            ctx.set_pencil(p.a, p.b)
            ctx.prepare(p.emin, p.emax, p.n_e)
            n = p.n
            rng = np.random.default_rng(5)
            rhs = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
            z, c = ctx.contour()
            out = []
            for mode in (0, 1):
                x = ctx.solve_shift(0, rhs, bool(mode))
                xr = O.shift_solve(p.a, p.b, z[0], rhs, mode)
                out.append(f"mode{mode} rel={rel(x, xr):.2e}")
            return " ".join(out)
        check(f"solve_shift {p.name}", fs)

        def fq(p=p):
            y = O.random_block(p.n, min(p.m0, 24), 42)
            q = ctx.contour_pass(y)
            qr = O.accumulate_real(p.a, p.b, p.emin, p.emax, p.n_e, y)
            return f"rel={rel(q, qr):.2e}"
        check(f"contour_pass {p.name}", fq)

        def frr(p=p):
            y = O.random_block(p.n, p.m0, 42)
            q = O.accumulate_real(p.a, p.b, p.emin, p.emax, p.n_e, y)
            ev, x, tr = ctx.rayleigh_ritz(q)
            rev, rx, rtr = O.rayleigh_ritz(p.a, p.b, q)
            k = min(len(ev), len(rev))
            return f"trunc={tr}/{rtr} m={len(ev)}/{len(rev)} ev_rel={rel(ev[:k], rev[:k]):.2e}"
        check(f"rayleigh_ritz {p.name}", frr)

        def fsolve(p=p):
            t = time.time()
            r = ctx.solve(F.SearchInterval(p.emin, p.emax),
                          F.FeastConfig(m0=p.m0, n_e=p.n_e, trace_tol=p.trace_tol, max_loops=p.max_loops,
                                        seed=p.seed))
            tg = time.time() - t
            t = time.time()
            ref = O.feast_solve(p, threads=8)
            tc = time.time() - t
            k = min(len(r.eigenvalues), len(ref["eigenvalues"]))
            return (f"gpu {r.status} m={len(r.eigenvalues)} loops={r.loops_used} maxres={r.max_residual:.1e} "
                    f"| ref {ref['status']} m={ref['m']} loops={ref['loops_used']} maxres={ref['max_residual']:.1e} "
                    f"| expected={p.expected_count} ev_rel={rel(r.eigenvalues[:k], ref['eigenvalues'][:k]):.2e} "
                    f"| t_gpu={tg:.2f}s t_ref={tc:.2f}s")
        check(f"feast_solve {p.name}", fsolve)
    print("launches", ctx.launch_count())


if __name__ == "__main__":
    main()
