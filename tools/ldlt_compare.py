"""LU vs complex-symmetric LDL^T filter on a bench workload: ms per
application (CUDA events on the library stream) and the relative difference
of the two Y's.  python tools/ldlt_compare.py [cfg] [steps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = P.default_context()
A, vals, c = bench.build_workload(cfg, 0)
n, p, nc = c["n"], c["m0"], c["n_c"]
dev = torch.device("cuda", 0)
X = torch.from_numpy(np.ascontiguousarray(P.make_initial_guess(n, p, 42).T)).to(dev)
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
rule = P.build_contour_rule(P.SearchInterval(c["lo"], c["hi"]), nc)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
out = {"config": cfg, "n": n, "m0": p, "n_c": nc}
Ys = {}
for mode in ("lu", "ldlt"):
    ctx.set_factorization(mode)
    filt = P.FilterApplier(None, rule, False, ctx=ctx, device_matrix=dA)
    Y = torch.empty((p, n), dtype=torch.float64, device=dev)
    filt.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        filt.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
    e1.record(stream)
    e1.synchronize()
    ctx.sync()
    out[mode + "_ms"] = e0.elapsed_time(e1) / steps
    Ys[mode] = Y.double()
    del filt
out["rel_diff"] = float(torch.linalg.norm(Ys["ldlt"] - Ys["lu"]) / torch.linalg.norm(Ys["lu"]))
out["speedup"] = out["lu_ms"] / out["ldlt_ms"]
print(json.dumps(out))
