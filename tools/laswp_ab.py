# A/B of the two laswp forms (FEASTLAB_LASWP=smem: shared-memory gather,
# default: warp per column). Row interchanges are pure data movement, so the
# filtered block Y must be bitwise identical; prints Y's digest and the
# application time.  python tools/laswp_ab.py [cfg] [--save path]
import hashlib
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CF.CONFIGS[idx]
lo, hi = (c.lo, c.hi) if idx != 3 else CF.cfg3_interval()[:2]
rng = np.random.default_rng(idx)
n = c.n
A = rng.standard_normal((n, n))
A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
X = np.asfortranarray(rng.standard_normal((n, c.m0)))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(lo, hi), c.n_c))
Y = f.apply(X)  # first call (captures the graph)
torch.cuda.synchronize()
ts = []
for _ in range(2):
    t = time.perf_counter()
    Y = f.apply(X)
    ts.append(time.perf_counter() - t)
d = hashlib.sha256(np.ascontiguousarray(Y).tobytes()).hexdigest()[:16]
import os
print(f"laswp={os.environ.get('FEASTLAB_LASWP', 'warp')} cfg{idx} n={n} digest={d} "
      f"ms={1e3 * min(ts):.1f}")
