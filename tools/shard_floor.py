"""Timing-only: rank 0's node shard at G GPUs (tools/shard_time.py) with
FEASTLAB_DEBUG_SKIP set by the caller (1: no panels, 4: no laswp) — the
floor that panel work can reach. Results are wrong by design; singular-node
errors are ignored."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import configs as CF
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = CF.CONFIGS[cfg]
n, nc, p = c.n, c.n_c, c.m0 or 660
dev = torch.device("cuda", 0)
A = torch.randn(n, n, dtype=torch.float64, device=dev)
A = (A + A.T) * (0.5 / n ** 0.5)
ctx = P.default_context()
dA = P.DeviceMatrix.from_device(A.data_ptr(), n, n, ctx)
X = torch.randn(p, n, dtype=torch.float64, device=dev)
Y = torch.empty_like(X)
rule = P.build_contour_rule(P.SearchInterval(c.lo, c.hi), nc)
k = nc // G
sub = P.ContourRule(rule.interval, rule.nodes[:k], rule.weights[:k])
f = P.FilterApplier(None, sub, False, ctx=ctx, device_matrix=dA)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
for _ in range(2):
    try:
        f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n); ctx.sync()
    except Exception:
        pass
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(3):
    try:
        f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
    except Exception:
        pass
e1.record(stream)
e1.synchronize()
try:
    ctx.sync()
except Exception:
    pass
print(f"cfg{cfg} G={G} nodes/GPU={k} skip={os.environ.get('FEASTLAB_DEBUG_SKIP','0')} ms/step {e0.elapsed_time(e1)/3:.2f}")
