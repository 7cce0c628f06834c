# filter wall time vs node-chunk concurrency, no profiling
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
n = int(sys.argv[1]); p = int(sys.argv[2]); nc = int(sys.argv[3])
ctx = P.default_context()
A = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n))); A = 0.5 * (A + A.T) / np.sqrt(n)
X = np.asfortranarray(np.random.default_rng(1).standard_normal((n, p)))
rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc)
f = P.FilterApplier(A, rule, ctx=ctx)
F = nc * (8 / 3 * n ** 3 + 8 * n * n * p)
for s in [int(a) for a in sys.argv[4:]] or (1, 2, 3, 4):
    ctx.set_streams(s)
    f.apply(X)
    t0 = time.time()
    for _ in range(3): f.apply(X)
    dt = (time.time() - t0) / 3
    print(f"n={n} p={p} nc={nc} streams={s}: {1e3*dt:.1f} ms  {F/dt/1e12:.2f} TF/s (host buffers)", flush=True)
