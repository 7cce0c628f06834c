"""Per-shape-class breakdown of the GEMM launches of one filter application
(CUDA events per launch, fl_ctx_profile_dump's shape tags):
  python tools/zgemm_classes.py [cfg=4] [streams=1] [lu|ldlt]
Prints one JSON object: per (role, K) class the launches, summed ms,
algorithmic TFLOP/s and the issued fraction of the DMMA peak (3M: 6 of 8
flops), plus the wall time of the profiled application."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402
from paper_1605_08771_b200 import _lib  # noqa: E402

ROLES = {1: "trailing update", 2: "in-block panel-column update", 3: "in-block U12 update (K=64)",
         4: "in-block U rows of a panel column", 5: "solve update", 6: "in-block solve update (K=64)",
         7: "L_kk^-1 product (SET)", 8: "solve diagonal-block product (SET)"}
PEAK = 37.08
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = P.default_context()
ctx.set_factorization(sys.argv[3] if len(sys.argv) > 3 else "lu")
ctx.set_streams(streams)
A, vals, c = bench.build_workload(cfg, 0)
n, p, nc = c["n"], c["m0"], c["n_c"]
X = torch.from_numpy(np.ascontiguousarray(P.make_initial_guess(n, p, 42).T)).cuda()
Y = torch.empty((p, n), dtype=torch.float64, device="cuda")
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
f = P.FilterApplier(None, P.build_contour_rule(P.SearchInterval(c["lo"], c["hi"]), nc), False,
                    ctx=ctx, device_matrix=dA)
torch.cuda.synchronize()
f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)  # warm (graph capture; not profiled)
ctx.sync()
ctx.set_profiling(True)
f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
ctx.sync()
cap = 400000
buf = (C.c_double * (5 * cap))()
cnt = _lib.lib().fl_ctx_profile_dump(ctx.handle, buf, cap)
rec = np.frombuffer(buf, dtype=np.float64)[:5 * cnt].reshape(cnt, 5)
ctx.set_profiling(False)
wall = rec[:, 2].max() - rec[:, 1].min()
out = {"cfg": cfg, "streams": streams, "records": int(cnt), "application_ms": round(float(wall), 2), "classes": []}
tags = rec[:, 4].astype(np.int64)
role = tags >> 30
K = (tags & 1023) * 16
Nt = (tags >> 10) & 1023
tot_ms = 0.0
for r in sorted(set(role[role > 0])):
    for wide in (False, True):
        for k in sorted(set(K[role == r])):
            m = (role == r) & (K == k) & ((Nt > 1) == wide)
            if not m.any():
                continue
            ms = float((rec[m, 2] - rec[m, 1]).sum())
            w = float(rec[m, 3].sum())
            tot_ms += ms
            out["classes"].append({"role": ROLES[int(r)], "K": int(k), "N_tiles": "many" if wide else "1",
                                   "launches": int(m.sum()), "ms": round(ms, 2),
                                   "algorithmic_tflops": round(w / ms / 1e9, 2),
                                   "issued_frac_of_dmma_peak": round(0.75 * w / ms / 1e9 / PEAK, 3),
                                   "share_of_flops": round(w / (nc * (8 / 3 * n ** 3 + 8.0 * n * n * p)), 4)})
out["gemm_class_ms"] = round(tot_ms, 2)
for cl in out["classes"]:
    cl["share_of_gemm_ms"] = round(cl["ms"] / tot_ms, 4)
print(json.dumps(out))
