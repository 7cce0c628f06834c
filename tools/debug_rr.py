import sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1605_08771_b200 as P

for p in (64, 130, 300, 700, 768):
    M = O.random_symmetric(p, 5)
    w, V = P.sym_eig(M)
    wr, Vr = np.linalg.eigh(M)
    res = np.linalg.norm(M @ V - V * w) / np.linalg.norm(M)
    print(f"sym_eig p={p}: max|dw|={np.abs(w-wr).max():.2e} resid={res:.2e} orth={np.abs(V.T@V-np.eye(p)).max():.2e}")
n = 1100
for p in (150, 700, 768):
    A = O.random_symmetric(n, 3) / np.sqrt(n)
    X = O.random_block(n, p, 4)
    U, r = P.orthonormalize(X, 1e-10)
    Ur, rr_ = O.orthonormalize(X, 1e-10)
    print(f"orth p={p}: rank {r} vs {rr_}; orth err {np.abs(U.T@U-np.eye(r)).max():.2e}; span {np.linalg.norm(U@U.T-Ur@Ur.T):.2e}")
    rr = P.rayleigh_ritz(A, Ur, P.SearchInterval(-0.5, 0.5))
    ro = O.rayleigh_ritz(A, Ur, O.SearchInterval(-0.5, 0.5))
    print(f"  rr: dvals {np.abs(rr.values-ro.values).max():.2e} dnorms {np.abs(rr.residual_norms-ro.residual_norms).max():.2e} inside {rr.inside_flags.sum()} vs {ro.inside_flags.sum()}")
