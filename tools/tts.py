import sys, time
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
idx = int(sys.argv[1])
vals = CF.spectrum(idx, O.uniform_fill); c = CF.resolved(idx, vals)
A = CF.laplacian_2d() if idx == 3 else O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
S = P.SymmetricMatrix(A)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    t0 = time.time()
    sol = P.feast_solve(S, P.SearchInterval(c["lo"], c["hi"]), P.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"]))
    print(f"cfg{idx} tts {time.time()-t0:.3f}s iters {sol.iterations} conv {sol.converged}", flush=True)
