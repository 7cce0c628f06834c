# eigen-accuracy of the drivers on cfg0/cfg1 under the current FEASTLAB_ZGEMM mode
import os, sys
sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
mode = os.environ.get("FEASTLAB_ZGEMM", "3m")
for idx in [int(a) for a in sys.argv[1:]] or [0, 1]:
    vals = CF.spectrum(idx, O.uniform_fill); c = CF.resolved(idx, vals)
    Q = O.seeded_orthogonal(len(vals), 1000 + idx); A = O.assemble_matrix(vals, Q)
    inside = (vals > c["lo"]) & (vals < c["hi"])
    Qi = Q[:, inside]
    for drv in ["feast_solve", "xfeast_solve", "rfeast_solve"]:
        cfg = P.SolverConfig(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=c["s"])
        sol = getattr(P, drv)(A, P.SearchInterval(c["lo"], c["hi"]), cfg)
        V = sol.eigenvectors
        sine = np.linalg.norm(V - Qi @ (Qi.T @ V), 2) if sol.converged and V.shape[1] == Qi.shape[1] else float('nan')
        ev = np.abs(np.sort(sol.eigenvalues) - vals[inside]).max() if len(sol.eigenvalues) == inside.sum() else float('nan')
        print(f"{mode} cfg{idx} {drv}: it {sol.iterations} conv {sol.converged} m {len(sol.eigenvalues)} "
              f"maxres {max(sol.residual_norms) if len(sol.residual_norms) else 0:.2e} eig_err {ev:.2e} sine {sine:.2e}", flush=True)
