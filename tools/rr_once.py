"""One feast_solve on a bench workload (device-built fixture, no oracle), for
ncu captures of the Rayleigh-Ritz tail:  python tools/rr_once.py [cfg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
A, _, c = bench.build_workload(cfg, 0)
S = P.SymmetricMatrix(A.cpu().numpy().T.copy(order="F"))
del A
sol = P.feast_solve(S, P.SearchInterval(c["lo"], c["hi"]),
                    P.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"]))
print("rr_once", cfg, sol.iterations, sol.converged, len(sol.eigenvalues))
