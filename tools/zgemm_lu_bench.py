"""Times the planar-complex DMMA GEMM on operands laid out as in an LU trailing
update (fl_debug_zgemm_lu): N x N factor planes, strided tiles. One JSON line
per shape; `checksum` compares kernel variants (FEASTLAB_ZGEMM_* switches).
Usage: python tools/zgemm_lu_bench.py [small]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib

PEAK = 37.08
ctx = P.default_context()
SHAPES = [  # N, M, Nc, K, batch, set
    (16384, 14336, 14336, 1024, 2, 0),  # an early trailing update of a cfg4 chunk
    (16384, 8192, 8192, 1024, 2, 0),
    (16384, 4096, 4096, 1024, 2, 0),
    (16384, 15360, 1024, 1024, 2, 0),   # the next block's columns
    (16384, 14336, 64, 512, 2, 0),      # in-block panel update (look-ahead stream)
    (16384, 8192, 512, 256, 2, 0),      # blocked solve update (W: here inside F)
    (4096, 3072, 3072, 256, 4, 0),      # cfg2-like
]
if len(sys.argv) > 1 and sys.argv[1] == "one":  # a single launch shape (ncu captures)
    SHAPES = [(16384, 8192, 8192, 1024, 2, 0)]
if len(sys.argv) > 1 and sys.argv[1] == "small":
    SHAPES = [(4096, 2048, 2048, 1024, 2, 0), (4096, 3072, 64, 512, 2, 0), (1024, 512, 512, 128, 1, 0)]
VARIANT = int(os.environ.get("ZGEMM_VARIANT", "0"))  # 1: the TMA-fed kernel
for (N, M, Nc, K, b, st) in SHAPES:
    ms, cs, err = C.c_double(), C.c_double(), _lib.Err()
    md = (C.c_double * 2)()
    rc = _lib.lib().fl_debug_zgemm_lu(ctx.handle, N, M, Nc, K, b, 3, VARIANT, C.byref(ms), C.byref(cs), md,
                                      C.byref(err))
    if rc:
        print(json.dumps({"rc": rc, "msg": err.msg.decode(errors="replace")}))
        continue
    fl = 8.0 * M * Nc * K * b
    tf = fl / ms.value / 1e9 if ms.value > 0 else 0.0
    print(json.dumps({"N": N, "M": M, "Nc": Nc, "K": K, "batch": b, "variant": VARIANT, "maxdiff": md[0], "max_abs": md[1], "rc": rc, "ms": round(ms.value, 4),
                      "algorithmic_tflops": round(tf, 2), "issued_frac_of_dmma_peak": round(0.75 * tf / PEAK, 4),
                      "checksum": repr(cs.value)}), flush=True)
