# time-to-solution breakdown on a config (GPU), with the oracle TTS beside it optional
import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
drivers = sys.argv[2].split(",") if len(sys.argv) > 2 else ["feast_solve"]
vals = CF.spectrum(idx, O.uniform_fill)
c = CF.resolved(idx, vals)
A = CF.laplacian_2d() if idx == 3 else O.assemble_matrix(vals, O.seeded_orthogonal(len(vals), 1000 + idx))
ctx = P.default_context()
S = P.SymmetricMatrix(A)
for d in drivers:
    cfg = P.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=c["s"])
    ctx.set_profiling(True)
    t0 = time.time()
    sol = getattr(P, d)(S, P.SearchInterval(c["lo"], c["hi"]), cfg)
    t = time.time() - t0
    prof = {k: ctx.profile(k)[0] for k in P.Context.KERNEL_CLASSES + P.Context.PHASE_CLASSES}
    ctx.set_profiling(False)
    print(f"cfg{idx} {d}: tts {t:.3f}s iters {sol.iterations} conv {sol.converged} m {len(sol.eigenvalues)} "
          f"(inside {c['inside']}) last r {sol.trace[-1].max_residual:.2e}", flush=True)
    print("   ms:", {k: round(v, 1) for k, v in prof.items() if v > 0}, flush=True)
    print("   dims:", [t.subspace_dim for t in sol.trace], flush=True)
