# Appendix-B evidence: the oracle itself changes XFEAST/RFEAST decisions on cfg1
# when only the OpenBLAS thread count (reduction order) changes.
import json, sys, time
sys.path.insert(0, '.')
import oracle as O
from paper_1605_08771_b200 import configs as CF
idx = 1
vals = CF.spectrum(idx, O.uniform_fill); c = CF.resolved(idx, vals)
A = O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
for d in sys.argv[1].split(","):
    for th in (1, 8):
        O.set_threads(th)
        t = time.time()
        s = getattr(O, d)(A, O.SearchInterval(c["lo"], c["hi"]),
                          O.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=c["s"]))
        print(json.dumps({"driver": d, "threads": th, "iterations": s.iterations, "converged": s.converged,
                          "m": len(s.eigenvalues), "dims": [t.subspace_dim for t in s.trace],
                          "seconds": round(time.time() - t, 1)}), flush=True)
