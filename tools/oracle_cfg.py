# oracle (CPU) reference runs of a config's drivers; prints traces as JSON lines
import json, sys, time
sys.path.insert(0, '.')
import numpy as np
import oracle as O
from paper_1605_08771_b200 import configs as CF
idx = int(sys.argv[1])
drivers = sys.argv[2].split(",")
s = int(sys.argv[3]) if len(sys.argv) > 3 else None
vals = CF.spectrum(idx, O.uniform_fill); c = CF.resolved(idx, vals)
A = CF.laplacian_2d() if idx == 3 else O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
for d in drivers:
    t = time.time()
    sol = getattr(O, d)(A, O.SearchInterval(c["lo"], c["hi"]),
                        O.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=s or c["s"]))
    print(json.dumps({"cfg": idx, "driver": d, "s": s or c["s"], "seconds": round(time.time() - t, 2),
                      "iterations": sol.iterations, "converged": sol.converged, "m": len(sol.eigenvalues),
                      "inside": c["inside"], "m0": c["m0"],
                      "trace": [[t.iter, t.subspace_dim, t.rhs_cumulative, t.max_residual, t.m_found] for t in sol.trace],
                      "recovery": sol.recovery_events}), flush=True)
