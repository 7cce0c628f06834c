# one zgemm shape (for ncu captures): python tools/zgemm_one.py M N K batch [iters]
import ctypes as C, sys
sys.path.insert(0, '.')
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
M, N, K, b = (int(a) for a in sys.argv[1:5])
it = int(sys.argv[5]) if len(sys.argv) > 5 else 3
ctx = P.default_context()
ms = C.c_double(); err = _lib.Err()
st = _lib.lib().fl_debug_zgemm(ctx.handle, M, N, K, b, it, C.byref(ms), C.byref(err))
print(f"M={M} N={N} K={K} batch={b}: {ms.value:.3f} ms {8.0*M*N*K*b/ms.value/1e9:.2f} TF/s (8MNK) st={st}")
