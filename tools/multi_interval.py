# Throughput of independent interval solves on one GPU: sequential vs
# solve_many with 1/2/4/8 worker contexts.
#   python tools/multi_interval.py [n] [intervals] -> JSON line
import json, sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
vals = O.uniform_fill(n, -1.0, 1.0, 2000)
A = O.assemble_matrix(vals, O.seeded_orthogonal(n, 1000))
S = P.SymmetricMatrix(A)
edges = np.linspace(-0.8, 0.8, k + 1)
jobs = []
for lo, hi in zip(edges[:-1], edges[1:]):
    inside = int(((vals > lo) & (vals < hi)).sum())
    jobs.append(("feast", P.SearchInterval(float(lo), float(hi)),
                 P.SolverConfig(m0=int(1.5 * inside), n_c=8, tol=1e-10, max_iter=20)))
P.solve_many(S, jobs[:1], per_device=1)  # warm
t0 = time.perf_counter()
seq = [P.feast_solve(S, iv, cfg) for _, iv, cfg in jobs]
t_seq = time.perf_counter() - t0
out = {"n": n, "intervals": k, "eigenpairs": int(sum(len(s.eigenvalues) for s in seq)),
       "sequential_s": round(t_seq, 3)}
for per in (1, 2, 4, 8):
    t0 = time.perf_counter()
    got = P.solve_many(S, jobs, per_device=per)
    out[f"concurrent_{per}_s"] = round(time.perf_counter() - t0, 3)
    assert all(g["error"] is None for g in got)
    assert all(np.array_equal(g["eigenvalues"], s.eigenvalues) for g, s in zip(got, seq))
print(json.dumps(out), flush=True)
