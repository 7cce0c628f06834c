"""One filter application (random symmetric n x n, nc nodes, p columns) for
profiling single kernels under ncu.  python tools/one_filter.py [n] [nc] [p]"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = int(sys.argv[3]) if len(sys.argv) > 3 else 64
rng = np.random.default_rng(0)
A = rng.standard_normal((n, n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
X = np.asfortranarray(rng.standard_normal((n, p)))
rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc)
f = P.FilterApplier(A, rule)
Y = f.apply(X)
print("ok", float(np.linalg.norm(Y)))
