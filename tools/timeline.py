# per-class busy time and overlap timeline of one filter application
import ctypes, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
n, p, nc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
streams = int(sys.argv[4]) if len(sys.argv) > 4 else 4
ctx = P.default_context()
if len(sys.argv) > 5:
    ctx.set_factorization(sys.argv[5])
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n))); A = 0.5 * (A + A.T) / np.sqrt(n)
X = np.asfortranarray(np.random.default_rng(1).standard_normal((n, p)))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), ctx=ctx)
ctx.set_streams(streams)
f.apply(X)
ctx.set_profiling(True)
f.apply(X)
buf = (ctypes.c_double * (4 * 200000))()
cnt = _lib.lib().fl_ctx_profile_dump(ctx.handle, buf, 200000)
ctx.set_profiling(False)
rec = np.frombuffer(buf, dtype=np.float64, count=4 * cnt).reshape(-1, 4)
names = ["shift", "panel", "laswp", "trsm", "zgemm", "permute", "accumulate", "allreduce"]
T = rec[:, 2].max()
print(f"n={n} p={p} nc={nc} streams={streams}: span {T:.1f} ms, {cnt} records")
# busy union per class and overall
grid = np.linspace(0, T, 20001)
busy = {}
for ci, nm in enumerate(names):
    r = rec[rec[:, 0] == ci]
    if len(r) == 0: continue
    act = np.zeros(len(grid), bool)
    for a, b in r[:, 1:3]:
        act[(grid >= a) & (grid < b)] = True
    busy[nm] = act
    print(f"  {nm:10s} busy {100*act.mean():5.1f}% of span ({act.mean()*T:.1f} ms)")
if "panel" in busy and "zgemm" in busy:
    pn, gm = busy["panel"], busy["zgemm"]
    print(f"  panel-only (no zgemm running) {100*(pn & ~gm).mean():.1f}%  ({(pn & ~gm).mean()*T:.1f} ms)")
    anyb = np.zeros(len(grid), bool)
    for v in busy.values(): anyb |= v
    print(f"  idle {100*(~anyb).mean():.1f}%")
# phase split of the span: factor vs solve (first permute start)
perm = rec[rec[:, 0] == 5]
if len(perm):
    print(f"  first solve starts at {perm[:,1].min():.1f} ms, last at {perm[:,1].max():.1f} ms")
# zgemm launches by work size: efficiency per bucket (launch-duration based)
z = rec[rec[:, 0] == 4]
if len(z):
    dur = z[:, 2] - z[:, 1]
    w = z[:, 3]
    print(f"  zgemm: {len(z)} launches, {w.sum()/dur.sum()/1e9:.2f} TF/s avg over launch durations")
    edges = [0, 1e9, 1e10, 5e10, 1e11, 2e11, 1e13]
    for lo, hi in zip(edges[:-1], edges[1:]):
        m = (w >= lo) & (w < hi)
        if m.any():
            print(f"    work [{lo:.0e},{hi:.0e}): {m.sum():4d} launches, {dur[m].sum():7.2f} ms, "
                  f"{w[m].sum()/dur[m].sum()/1e9:6.2f} TF/s")

perm = rec[rec[:, 0] == 5]
pan = rec[rec[:, 0] == 1]
if len(perm) and len(pan):
    print(f"  factor phase ends {perm[:, 1].min():.2f} ms (first solve starts), last panel ends "
          f"{pan[:, 2].max():.2f} ms, span {T:.2f} ms; panel launches {len(pan)}, "
          f"mean panel {np.mean(pan[:, 2] - pan[:, 1]) * 1e3:.1f} us")
