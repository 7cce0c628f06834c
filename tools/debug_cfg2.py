import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
vals = CF.spectrum(idx, O.uniform_fill)
c = CF.resolved(idx, vals)
t0 = time.time()
Q = O.seeded_orthogonal(len(vals), 1000 + idx)
A = O.assemble_matrix(vals, Q)
print("fixture", time.time() - t0, c)
n, p = c["n"], c["m0"]
X = P.make_initial_guess(n, p, 42)
Xo = O.make_initial_guess(n, p, 42)
print("guess equal", np.array_equal(X, Xo))
rule = P.build_contour_rule(P.SearchInterval(c["lo"], c["hi"]), c["n_c"])
one = P.ContourRule(rule.interval, rule.nodes[:2], rule.weights[:2])
Y = P.apply_filter(A, one, X)
oone = O.ContourRule(O.SearchInterval(c["lo"], c["hi"]), rule.nodes[:2], rule.weights[:2])
Yo = O.apply_filter(A, oone, X)
print("2-node filter rel", np.linalg.norm(Y - Yo) / np.linalg.norm(Yo))
cfg = P.SolverConfig(m0=p, n_c=c["n_c"], tol=c["tol"], max_iter=6)
t0 = time.time()
sol = P.feast_solve(A, P.SearchInterval(c["lo"], c["hi"]), cfg, keep_first=True)
print("gpu solve", time.time() - t0)
for t in sol.trace: print(t)
Yf = sol.first_filtered
Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(c["lo"], c["hi"]), c["n_c"]), X)
print("Y1 rel", np.linalg.norm(Yf - Yo) / np.linalg.norm(Yo))
U, r = P.orthonormalize(Yf, 1e-10)
Uo, ro = O.orthonormalize(Yo, 1e-10)
print("rank", r, ro, "span", np.linalg.norm(U @ (U.T @ Uo) - Uo))
rr = P.rayleigh_ritz(A, Uo, P.SearchInterval(c["lo"], c["hi"]))
rro = O.rayleigh_ritz(A, Uo, O.SearchInterval(c["lo"], c["hi"]))
print("rr dvals", np.abs(rr.values - rro.values).max(), "inside", rr.inside_flags.sum(), rro.inside_flags.sum())
ins = rro.inside_flags
print("max res inside gpu/oracle", rr.residual_norms[rr.inside_flags].max(), rro.residual_norms[ins].max())
