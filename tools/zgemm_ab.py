"""A/B of the trailing-update GEMM kernels inside one process (the boxes of
the pool differ by a few percent, so variants are interleaved and repeated):
python tools/zgemm_ab.py [reps=3]  -> one JSON line per variant (median ms)."""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib

PEAK = 37.08
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = P.default_context()
N, M, Nc, K, b = 16384, 8192, 8192, 1024, 2
if len(sys.argv) > 2:
    N, M, Nc, K, b = (int(x) for x in sys.argv[2].split(","))
VARIANTS = [("cp.async 3M", 0, None, "0"), ("tma", 1, None, "0")]
times = {v[0]: [] for v in VARIANTS}
diff = {}
for r in range(reps):
    for name, var, sched, l2 in VARIANTS:
        os.environ["FEASTLAB_TMA_L2AHEAD"] = l2
        if sched is not None:
            os.environ["FEASTLAB_TMA_SCHED"] = sched  # read once per process: A/B needs one process per schedule
        ms, cs, err = C.c_double(), C.c_double(), _lib.Err()
        md = (C.c_double * 2)()
        rc = _lib.lib().fl_debug_zgemm_lu(ctx.handle, N, M, Nc, K, b, 3, var, C.byref(ms), C.byref(cs), md, C.byref(err))
        if rc:
            print(json.dumps({"variant": name, "rc": rc, "msg": err.msg.decode(errors="replace")}), flush=True)
            continue
        times[name].append(ms.value)
        diff[name] = md[0]
for name, _, _, _ in VARIANTS:
    if not times[name]:
        continue
    ms = statistics.median(times[name])
    tf = 8.0 * M * Nc * K * b / ms / 1e9
    print(json.dumps({"variant": name, "shape": [N, M, Nc, K, b], "ms_median": round(ms, 3), "ms_all": [round(x, 3) for x in times[name]],
                      "algorithmic_tflops": round(tf, 2), "issued_frac_of_dmma_peak": round(0.75 * tf / PEAK, 4),
                      "maxdiff_vs_cp_async": diff.get(name)}), flush=True)
