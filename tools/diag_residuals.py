import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from paper_0901_2665_b200 import feast as F, problems as P
prob = P.config2()
ctx = F.GpuContext(0)
ctx.set_pencil(prob.a, prob.b)
r = ctx.solve(F.SearchInterval(prob.emin, prob.emax), F.FeastConfig(m0=prob.m0, n_e=prob.n_e, trace_tol=prob.trace_tol, max_loops=prob.max_loops, seed=prob.seed))
x = r.eigenvectors
ax = prob.a.matmul(x); bx = prob.b.matmul(x)
res = ax - bx * r.eigenvalues
an = float(np.max(np.abs(prob.a.to_scipy()).sum(axis=0)))
rel = np.linalg.norm(res, axis=0) / (an * np.linalg.norm(x, axis=0))
r1 = np.abs(res).sum(axis=0) / np.abs(ax).sum(axis=0)
j = int(np.argmax(rel))
print("status", r.status, "loops", r.loops_used, "m", len(r.eigenvalues))
print("worst j", j, "lam", r.eigenvalues[j], "rel", rel[j], "r1", r1[j], "gpu residual", r.residuals[j])
print("neighbours", r.eigenvalues[max(0,j-2):j+3])
print("emin/emax", prob.emin, prob.emax)
print("sorted rel top5", np.sort(rel)[-5:])
