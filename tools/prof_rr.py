# Rayleigh-Ritz / orthonormalisation cost split on device blocks:
#   python tools/prof_rr.py n p
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib as L
n, p = int(sys.argv[1]), int(sys.argv[2])
ctx = P.default_context()
rng = np.random.default_rng(0)
A = rng.standard_normal((n, n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
dA = P.DeviceMatrix(A, ctx)
X = np.linalg.qr(rng.standard_normal((n, p)))[0]
dX = P.DeviceBlock(n, p, ctx).set(np.asfortranarray(X))
dV = P.DeviceBlock(n, p, ctx); dU = P.DeviceBlock(n, p, ctx)
vals = np.zeros(p); norms = np.zeros(p); inside = np.zeros(p, dtype=np.uint8)
lib = L.lib()
def rr():
    err = L.Err()
    st = lib.fl_rayleigh_ritz(ctx.handle, dA.handle, dX.handle, -0.1, 0.1, vals.ctypes.data, dV.handle,
                              norms.ctypes.data, inside.ctypes.data, C.byref(err))
    assert st == 0, err.msg
def orth():
    err = L.Err(); r = C.c_int()
    st = lib.fl_orthonormalize(ctx.handle, dX.handle, 1e-12, 0, dU.handle, C.byref(r), C.byref(err))
    assert st == 0, err.msg
for fn, name in ((rr, "rayleigh_ritz"), (orth, "orthonormalize")):
    fn()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(3): fn()
    ctx.sync()
    dt = (time.perf_counter() - t0) / 3
    ctx.set_profiling(True); fn(); ctx.sync()
    e = ctx.profile("eig")
    ctx.set_profiling(False)
    print(f"n={n} p={p} {name}: {1e3*dt:.1f} ms per call; eig {e[0]:.1f} ms", flush=True)
