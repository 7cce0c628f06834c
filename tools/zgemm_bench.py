import ctypes as C, sys
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
ctx = P.default_context()
for (M, N, K, b) in [(4032, 4032, 64, 4), (4032, 4032, 128, 4), (4032, 4032, 256, 4), (4032, 4032, 1024, 2),
                     (2048, 768, 64, 16), (1024, 1024, 64, 16), (4096, 4096, 64, 16)]:
    ms = C.c_double(); err = _lib.Err()
    st = _lib.lib().fl_debug_zgemm(ctx.handle, M, N, K, b, 5, C.byref(ms), C.byref(err))
    fl = 8.0 * M * N * K * b
    print(f"M={M} N={N} K={K} batch={b}: {ms.value:.3f} ms  {fl/ms.value/1e9:.2f} TF/s  ({100*fl/ms.value/1e9/37.08:.1f}% of DMMA peak) st={st}", flush=True)
