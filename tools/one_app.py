"""One filter application on a bench workload (for ncu launch lists):
python tools/one_app.py [cfg] [lu|ldlt] [streams]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = P.default_context()
ctx.set_factorization(sys.argv[2] if len(sys.argv) > 2 else "lu")
if len(sys.argv) > 3:
    ctx.set_streams(int(sys.argv[3]))
A, vals, c = bench.build_workload(cfg, 0)
n, p, nc = c["n"], c["m0"], c["n_c"]
X = torch.from_numpy(np.ascontiguousarray(P.make_initial_guess(n, p, 42).T)).cuda()
Y = torch.empty((p, n), dtype=torch.float64, device="cuda")
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
f = P.FilterApplier(None, P.build_contour_rule(P.SearchInterval(c["lo"], c["hi"]), nc), False,
                    ctx=ctx, device_matrix=dA)
torch.cuda.synchronize()
f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
ctx.sync()
print("ok", float(torch.linalg.norm(Y)))
