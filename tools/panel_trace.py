"""Per-warp timeline of the on-chip panel's column steps (first panel, node 0,
ranks 0 and CL-1), from a build with -DFL_PANEL_TRACE:
  PANEL_FLAGS=-DFL_PANEL_TRACE ./tools/prof_panel_build.sh ... (or run after it)"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
A = rng.standard_normal((n, n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
X = np.asfortranarray(rng.standard_normal((n, 64)))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), 1))
f.apply(X)
buf = (ctypes.c_longlong * (64 * 2 * 8 * 8))()
_lib.lib().fl_debug_panel_trace(buf, len(buf))
t = np.array(buf, dtype=np.int64).reshape(64, 2, 8, 8)
names = ["start", "bar_in", "bar_out", "wait_in", "wait_out", "reduced", "pushed"]
for jl in (3, 4, 5, 20, 21, 40):
    for r in (0, 1):
        tt = t[jl, r, :, :7]
        t0 = tt[:, 0].min()
        nxt = t[jl + 1, r, :, 0].min() if jl + 1 < 64 else 0
        print(f"col {jl} rank {'0' if r == 0 else 'last'} (next column starts +{nxt - t0})")
        for w in range(8):
            print("   warp", w, " ".join(f"{names[i]}:{tt[w, i] - t0}" for i in (0, 1, 2, 5, 6, 3, 4)))
# column-averaged phase durations over warps of rank 0, columns 1..63 within leaves
d = t[:, 0, :, :5].astype(float)
st = d[:, :, 0]
d = t[:, 0, :, :7].astype(float)
inleaf = [c for c in range(63) if c % 16 != 15]
nx = np.array([d[c + 1, :, 0] - d[c, :, 4] for c in inleaf])
print("mean per column (rank 0, in-leaf): start->bar_in %.0f  bar %.0f  CTA reduce %.0f  push %.0f  deferred %.0f  wait %.0f  wait_out->next start %.0f" % (
    np.mean(d[inleaf, :, 1] - d[inleaf, :, 0]), np.mean(d[inleaf, :, 2] - d[inleaf, :, 1]),
    np.mean(d[inleaf, :, 5] - d[inleaf, :, 2]), np.mean(d[inleaf, :, 6] - d[inleaf, :, 5]),
    np.mean(d[inleaf, :, 3] - d[inleaf, :, 6]), np.mean(d[inleaf, :, 4] - d[inleaf, :, 3]), np.mean(nx)))
