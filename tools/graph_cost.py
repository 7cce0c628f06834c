"""Wall time of the 1st (eager, host-paced launches), 2nd (stream capture +
instantiate + launch) and 3rd (graph replay) filter application on a bench
workload.  python tools/graph_cost.py [cfg] [lu|ldlt]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1605_08771_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
fac = sys.argv[2] if len(sys.argv) > 2 else "lu"
ctx = P.default_context()
ctx.set_factorization(fac)
A, vals, c = bench.build_workload(cfg, 0)
n, p, nc = c["n"], c["m0"], c["n_c"]
dev = torch.device("cuda", 0)
X = torch.from_numpy(np.ascontiguousarray(P.make_initial_guess(n, p, 42).T)).to(dev)
Y = torch.empty((p, n), dtype=torch.float64, device=dev)
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
rule = P.build_contour_rule(P.SearchInterval(c["lo"], c["hi"]), nc)
filt = P.FilterApplier(None, rule, False, ctx=ctx, device_matrix=dA)
torch.cuda.synchronize()
for k in range(4):
    l0 = ctx.launches()
    t0 = time.perf_counter()
    filt.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    print(f"cfg{cfg} {fac} application {k}: enqueue {t1 - t0:.3f} s, total {t2 - t0:.3f} s, "
          f"launches {ctx.launches() - l0}", flush=True)
