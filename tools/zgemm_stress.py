"""Repeats the TMA-fed trailing-update product against the cp.async kernel on
the same operands and reports the largest difference seen (a rare in-kernel
race shows up as an occasional large maxdiff):
python tools/zgemm_stress.py [calls=30] [N,M,Nc,K,batch]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 30
N, M, Nc, K, b = 16384, 8192, 8192, 1024, 2
if len(sys.argv) > 2:
    N, M, Nc, K, b = (int(x) for x in sys.argv[2].split(","))
ctx = P.default_context()
worst, bad = 0.0, 0
for i in range(calls):
    ms, cs, err = C.c_double(), C.c_double(), _lib.Err()
    md = (C.c_double * 2)()
    rc = _lib.lib().fl_debug_zgemm_lu(ctx.handle, N, M, Nc, K, b, 1, int(os.environ.get('ZGEMM_VARIANT', '1')), C.byref(ms), C.byref(cs), md, C.byref(err))
    assert rc == 0, err.msg
    worst = max(worst, md[0])
    bad += md[0] > 1e-12
print(json.dumps({"shape": [N, M, Nc, K, b], "calls": calls, "worst_maxdiff": worst, "calls_with_error": bad}))
