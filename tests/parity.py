"""Shared parity checks for the full-size tests: the SURVEY §8(c) policy against a reference run
(live or from a committed fixture), the north-star residual and principal angles.

  (ii)  the reference converged: same status, in-interval count equal to the reference's and to
        the construction / inertia count, eigenvalues within 1e-10 relative (denominator
        max(|lambda|, 1e-3 * interval width): the reference's own acceptance test avoids
        |lambda| ~ 0, acceptance.cpp:352-357), max principal angle <= 1e-8, north-star residual
        ||Ax - lambda Bx|| / (||A|| ||x||) <= 1e-10;
  (iii) the reference ended in max-loops (spurious Ritz pairs, SURVEY finding 3): same status;
        the pairs each side validates (its own reference-metric residual <= VALIDATED) must be
        the same pairs (eigenvalues within the (ii) tolerance), as many as the construction /
        inertia count, with the north-star residual <= 1e-10 on the GPU's validated pairs.
"""
import numpy as np

# Validation threshold on the reference-metric residual (residual.hpp: relative to |lambda|).
# Spurious Ritz pairs sit at ~1e-1 .. 1, converged ones at <= ~1e-8: on full-size config 3 the pair
# at lambda = 6.2e-5 (|lambda| tiny, so the metric amplifies an absolute residual of ~1e-12 by
# 1.6e4) has 9e-10 in the reference and 1.5e-8 on the GPU (b = 256 explicit block inverses; its
# north-star residual, asserted below, is <= 1e-10). The threshold only has to separate the two
# populations.
VALIDATED = 1e-6


def norm1(op):
    from paper_0901_2665_b200 import abi
    if op.kind == abi.STORAGE_DENSE:
        return float(np.max(np.abs(op.dense).sum(axis=0)))
    return float(np.max(np.asarray(abs(op.to_scipy()).sum(axis=0)).ravel()))


def north_star_residual(prob, lam, x):
    """||Ax - lambda Bx||_2 / (||A|| ||x||_2) per column (||A||_1 = ||A||_inf >= ||A||_2)."""
    if x.shape[1] == 0:
        return np.zeros(0)
    res = prob.a.matmul(x) - prob.b.matmul(x) * lam
    return np.linalg.norm(res, axis=0) / (norm1(prob.a) * np.linalg.norm(x, axis=0))


def ev_tol(prob, ev):
    return 1e-10 * np.maximum(np.abs(ev), 1e-3 * (prob.emax - prob.emin))


def sin_max_angle(x, xr, bmat_apply):
    """max principal angle between span(x) and span(xr) in the B inner product, via sines:
    sigma_max((I - Xr Xr^T B) X) with B-orthonormal X, Xr."""
    def borth(v):
        g = v.T @ bmat_apply(v)
        w, u = np.linalg.eigh(0.5 * (g + g.T))
        return v @ (u / np.sqrt(w))
    x, xr = borth(x), borth(xr)
    r = x - xr @ (xr.T @ bmat_apply(x))
    g = r.T @ bmat_apply(r)
    return float(np.sqrt(max(np.max(np.linalg.eigvalsh(0.5 * (g + g.T))), 0.0)))


def clusters(ev, rel_gap=1e-6):
    """Index groups of consecutive eigenvalues closer than rel_gap * max|ev| (their individual
    eigenvectors are not determined, only the cluster's subspace)."""
    if len(ev) == 0:
        return []
    scale = max(1e-300, float(np.max(np.abs(ev))))
    groups, cur = [], [0]
    for i in range(1, len(ev)):
        if ev[i] - ev[i - 1] <= rel_gap * scale:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def sketched_sines(sx, sxr, ev):
    """Per-cluster sine of the largest principal angle between the Euclidean spans of the
    sketched blocks S X and S X_ref (a K-row Gaussian sketch preserves these angles to
    ~3/sqrt(K) relative for the few-dimensional cluster subspaces)."""
    out = []
    for g in clusters(ev):
        q, _ = np.linalg.qr(sx[:, g])
        qr, _ = np.linalg.qr(sxr[:, g])
        r = q - qr @ (qr.T @ q)
        out.append(float(np.linalg.norm(r, 2)))
    return np.array(out)


def match(ev, ev_ref, prob):
    """For each reference eigenvalue the nearest GPU one; max |diff| / tolerance."""
    if len(ev_ref) == 0:
        return 0.0
    idx = np.searchsorted(ev, ev_ref)
    best = np.full(len(ev_ref), np.inf)
    for d in (-1, 0):
        j = np.clip(idx + d, 0, len(ev) - 1)
        best = np.minimum(best, np.abs(ev[j] - ev_ref))
    return float(np.max(best / ev_tol(prob, ev_ref)))


def check_policy(prob, r, ref, x_ref=None, sketch=None, sketch_ref=None, expected=None):
    """r: the GPU FeastResult; ref: dict with status, m, eigenvalues, residuals (the reference's
    FeastResult, live or from a fixture). Returns a dict of the measured figures."""
    expected = prob.expected_count if expected is None else expected
    out = {"status": r.status, "ref_status": ref["status"], "count": len(r.eigenvalues),
           "ref_count": int(ref["m"])}
    assert r.status == ref["status"], out
    lam, x = r.eigenvalues, r.eigenvectors
    ns = north_star_residual(prob, lam, x)
    if ref["status"] == "converged":
        assert len(lam) == int(ref["m"]), out
        if expected is not None:
            assert len(lam) == expected, out
        ev = np.asarray(ref["eigenvalues"])
        assert np.all(np.abs(lam - ev) <= ev_tol(prob, ev)), np.max(np.abs(lam - ev) / ev_tol(prob, ev))
        out["ev_err_over_tol"] = float(np.max(np.abs(lam - ev) / ev_tol(prob, ev))) if len(ev) else 0.0
        assert np.max(ns, initial=0.0) <= 1e-10, np.max(ns)
        out["north_star_residual"] = float(np.max(ns, initial=0.0))
        if x_ref is not None and len(lam):
            s = sin_max_angle(x, x_ref, prob.b.matmul)
            assert s <= 1e-8, s
            out["sin_max_angle"] = s
        if sketch is not None and sketch_ref is not None and len(lam):
            sines = sketched_sines(sketch @ x, sketch_ref, ev)
            assert np.max(sines) <= 1e-8, np.max(sines)
            out["sketched_sin_max"] = float(np.max(sines))
    else:
        gv = np.asarray(r.residuals) <= VALIDATED
        rv = np.asarray(ref["residuals"]) <= VALIDATED
        lam_v, ev_v = lam[gv], np.asarray(ref["eigenvalues"])[rv]
        out.update(validated=int(gv.sum()), ref_validated=int(rv.sum()),
                   top_residuals=[float(v) for v in np.sort(np.asarray(r.residuals))[-4:]],
                   ref_top_residuals=[float(v) for v in np.sort(np.asarray(ref["residuals"]))[-4:]])
        assert gv.sum() == rv.sum(), out
        if expected is not None:
            assert gv.sum() == expected, out
        out["ev_err_over_tol"] = match(lam_v, ev_v, prob)
        assert out["ev_err_over_tol"] <= 1.0, out
        assert np.max(ns[gv], initial=0.0) <= 1e-10, np.max(ns[gv])
        out["north_star_residual"] = float(np.max(ns[gv], initial=0.0))
    return out
