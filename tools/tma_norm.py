"""||Y|| of one seeded filter application (compare FEASTLAB_ZGEMM_TMA=0 / 1 runs):
python tools/tma_norm.py n n_c p [streams]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
n, nc, p = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(1)
A = rng.standard_normal((n, n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
X = np.asfortranarray(rng.standard_normal((n, p)))
if len(sys.argv) > 4:
    P.default_context().set_streams(int(sys.argv[4]))
Y = P.apply_filter(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), X)
print(n, nc, p, "norm %.15e" % np.linalg.norm(Y), flush=True)
