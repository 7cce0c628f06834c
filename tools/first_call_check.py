"""Filter output of calls 1..3 (first-call graph capture, replay) against the
known answer Q diag(rho(lambda)) Q^T X for a seeded A = Q diag(lambda) Q^T.
python tools/first_call_check.py [n] [nc] [p] [lu|ldlt] [cache]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_08771_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = int(sys.argv[3]) if len(sys.argv) > 3 else 256
fac = sys.argv[4] if len(sys.argv) > 4 else "ldlt"
cache = len(sys.argv) > 5 and sys.argv[5] == "cache"
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
Q, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g))
vals = torch.rand(n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
A = ((Q * vals) @ Q.T)
A = (0.5 * (A + A.T)).contiguous()
ctx = P.default_context()
ctx.set_factorization(fac)
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
X = torch.randn(p, n, dtype=torch.float64, device=dev, generator=g)
rule = P.build_contour_rule(P.SearchInterval(-0.2, 0.2), nc)
rho = torch.tensor([P.filter_value(rule, float(v)) for v in vals.cpu()], dtype=torch.float64,
                   device=dev)
Yx = Q @ (rho[:, None] * (Q.T @ X.T))
keep = None
if os.environ.get("KEEP_LU"):  # an LU filter applied first and kept alive
    ctx.set_factorization("lu")
    keep = P.FilterApplier(None, rule, False, ctx=ctx, device_matrix=dA)
    Yk = torch.empty_like(X)
    keep.apply_device(X.data_ptr(), n, p, Yk.data_ptr(), n)
    ctx.sync()
    print("LU first:", (torch.linalg.norm(Yk.T - Yx) / torch.linalg.norm(Yx)).item(),
          "free GB", torch.cuda.mem_get_info()[0] / 1e9, flush=True)
    ctx.set_factorization(fac)
f = P.FilterApplier(None, rule, cache, ctx=ctx, device_matrix=dA)
torch.cuda.synchronize()
for k in range(3):
    Y = torch.full_like(X, float("nan"))
    torch.cuda.synchronize()
    f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
    ctx.sync()
    rel = (torch.linalg.norm(Y.T - Yx) / torch.linalg.norm(Yx)).item()
    print(f"n={n} nc={nc} p={p} {fac} cache={cache} call {k}: rel {rel:.2e}", flush=True)
