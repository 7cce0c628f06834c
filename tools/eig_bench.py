# device symmetric eigensolver (fl_sym_eig) on random / clustered matrices
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
for p in [int(a) for a in sys.argv[1:]] or [150, 512, 768, 1386]:
    rng = np.random.default_rng(p)
    M = rng.standard_normal((p, p)); M = np.asfortranarray(0.5 * (M + M.T))
    P.sym_eig(M)
    t0 = time.perf_counter(); w, V = P.sym_eig(M); dt = time.perf_counter() - t0
    wr = np.linalg.eigvalsh(M)
    err = np.abs(w - wr).max() / np.abs(wr).max()
    orth = np.abs(V.T @ V - np.eye(p)).max()
    res = np.abs(M @ V - V * w).max() / np.abs(wr).max()
    print(f"p={p}: {1e3*dt:.1f} ms  eig err {err:.1e} orth {orth:.1e} res {res:.1e}", flush=True)
