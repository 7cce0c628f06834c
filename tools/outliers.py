# which kernel class grows in the slow filter applications (profiled, eager)
import ctypes, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
n, p, nc, streams, reps = (int(a) for a in sys.argv[1:6])
ctx = P.default_context()
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n))); A = 0.5 * (A + A.T) / np.sqrt(n)
X = np.asfortranarray(np.random.default_rng(1).standard_normal((n, p)))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), ctx=ctx)
ctx.set_streams(streams)
f.apply(X)
names = ["shift", "panel", "laswp", "trsm", "zgemm", "permute", "accumulate", "allreduce"]
buf = (ctypes.c_double * (4 * 200000))()
for r in range(reps):
    ctx.set_profiling(True)
    f.apply(X)
    cnt = _lib.lib().fl_ctx_profile_dump(ctx.handle, buf, 200000)
    ctx.set_profiling(False)
    rec = np.frombuffer(buf, dtype=np.float64, count=4 * cnt).reshape(-1, 4)
    span = rec[:, 2].max() - rec[:, 1].min()
    parts = []
    for ci, nm in enumerate(names[:5]):
        rr = rec[rec[:, 0] == ci]
        d = rr[:, 2] - rr[:, 1]
        parts.append(f"{nm} {d.sum():6.1f} (max {d.max() if len(d) else 0:5.2f})")
    print(f"span {span:6.1f} | " + " | ".join(parts), flush=True)
