# per-application GPU time (CUDA events on the context stream), device buffers
import gc, os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
n, p, nc, streams, reps = (int(a) for a in sys.argv[1:6])
ctx = P.default_context()
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n))); A = 0.5 * (A + A.T) / np.sqrt(n)
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), ctx=ctx)
ctx.set_streams(streams)
X = torch.randn(p, n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
st = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3): f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n)
if os.environ.get("NOGC"): gc.collect(); gc.freeze(); gc.disable()
ts = []
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); f.apply_device(X.data_ptr(), n, p, Y.data_ptr(), n); e1.record(st); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
tag = os.environ.get("TAG", "")
print(f"{tag} streams={streams}: n>155 {(ts > 155).sum()} min {ts.min():.1f} med {np.median(ts):.1f} max {ts.max():.1f} | " + " ".join(f"{t:.0f}" for t in ts), flush=True)
