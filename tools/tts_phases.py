"""Time-to-solution of feast_solve on a bench workload with the per-phase
wall times (FEASTLAB_TIME=1, stderr).  python tools/tts_phases.py [cfg] [lu|ldlt] [cache]"""
import os
import sys
import time

os.environ.setdefault("FEASTLAB_TIME", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
fac = sys.argv[2] if len(sys.argv) > 2 else "lu"
cache = len(sys.argv) > 3 and sys.argv[3] == "cache"
ctx = P.default_context()
ctx.set_factorization(fac)
A, vals, c = bench.build_workload(cfg, 0)
Ah = A.cpu().numpy().T.copy(order="F")
del A
t0 = time.perf_counter()
S = P.SymmetricMatrix(Ah)
print(f"python SymmetricMatrix {time.perf_counter() - t0:.3f} s", flush=True)
for rep in range(2):
    t0 = time.perf_counter()
    sol = P.feast_solve(S, P.SearchInterval(c["lo"], c["hi"]),
                        P.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"],
                                       max_iter=c["max_iter"], cache_factorizations=cache))
    print(f"cfg{cfg} {fac} cache={cache} rep {rep}: tts {time.perf_counter() - t0:.3f} s, "
          f"{sol.iterations} iterations, converged {sol.converged}", flush=True)
