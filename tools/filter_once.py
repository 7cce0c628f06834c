# one filter application on a cfg-shaped workload (for ncu launch lists):
#   python tools/filter_once.py [cfg_index in 0,2,3,4] [streams]
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = CF.CONFIGS[idx]
lo, hi = (c.lo, c.hi) if idx != 3 else CF.cfg3_interval()[:2]
rng = np.random.default_rng(idx)
A = rng.standard_normal((c.n, c.n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(c.n))
X = np.asfortranarray(rng.standard_normal((c.n, c.m0)))
ctx = P.default_context()
ctx.set_streams(streams)
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(lo, hi), c.n_c), ctx=ctx)
Y = f.apply(X)
print("filter_once", idx, c.n, c.m0, c.n_c, float(np.linalg.norm(Y)))
