import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
ctx = P.default_context()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
A = 0.5 * (A + A.T) / np.sqrt(n)
X = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 64)))
for nc in (1, 4, 16):
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc)
    f = P.FilterApplier(A, rule, ctx=ctx)
    try:
        f.apply(X)
    except Exception as e:  # timing experiments may produce singular nodes
        pass
    for streams in (1, 4):
        ctx.set_streams(streams)
        ctx.set_profiling(True)
        t0 = time.time()
        try:
            f.apply(X)
        except Exception:
            pass
        t1 = time.time()
        out = {k: ctx.profile(k) for k in ("panel", "laswp", "trsm", "zgemm")}
        ctx.set_profiling(False)
        print(f"n={n} nc={nc} streams={streams} wall={1e3*(t1-t0):.1f}ms " +
              " ".join(f"{k}:{v[0]:.1f}ms/{v[2]}" for k, v in out.items()), flush=True)
import ctypes
from paper_1605_08771_b200 import _lib
out = (ctypes.c_double * 8)()
_lib.lib().fl_debug_panel_profile(out, 1)
rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.2), 1)
f = P.FilterApplier(A, rule, ctx=ctx)
f.apply(X)
_lib.lib().fl_debug_panel_profile(out, 1)
import os
names = (["cand+publish", "cluster.sync", "pivot fetch", "update", "leaf store+sync", "perm+sync", "trsm", "inner update"]
         if os.environ.get("FEASTLAB_PANEL") == "reg" else
         ["load/store/Linv", "cand", "BAR+CTAred", "push", "deferred", "mbar wait", "red+update", "transitions"])
tot = sum(out)
print("panel phases per column (cycles, mean over the 8 warps of rank 0, node 0):", {k: int(v / 8 / n) for k, v in zip(names, out)}, "total", int(tot / 8 / n))
