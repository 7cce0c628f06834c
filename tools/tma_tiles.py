"""Tile sums of the cached factors of one seeded filter application, saved to
gpurun_out/<tag>.npy (compare a FEASTLAB_ZGEMM_TMA=0 run with TMA runs):
python tools/tma_tiles.py n n_c tag [streams]; python tools/tma_tiles.py cmp a.npy b.npy"""
import os, sys
import numpy as np
if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    d = np.abs(a - b) / np.maximum(np.abs(a), 1e-300)
    bad = np.argwhere(d > 1e-9)
    print("differing tiles", len(bad), "of", a.size)
    if len(bad):
        # (node, tile col, tile row): report per node the smallest tile column, and in it the smallest row
        for node in sorted(set(bad[:, 0])):
            bb = bad[bad[:, 0] == node]
            c = bb[:, 1].min()
            rows = sorted(bb[bb[:, 1] == c][:, 2])
            print(f" node {node}: {len(bb)} tiles; first tile column {c}: rows {rows[:12]}{'...' if len(rows) > 12 else ''}; "
                  f"min row over all {bb[:, 2].min()}")
    sys.exit(0)
import ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_08771_b200 as P
from paper_1605_08771_b200 import _lib
n, nc, tag = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
rng = np.random.default_rng(1)
A = rng.standard_normal((n, n)); A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
X = np.asfortranarray(rng.standard_normal((n, 64)))
if len(sys.argv) > 4:
    P.default_context().set_streams(int(sys.argv[4]))
f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), nc), True)
Y = f.apply(X)
NB = (n + 63) // 64
out = np.zeros(nc * NB * NB)
rc = _lib.lib().fl_debug_factor_tilesums(f.handle, nc, out.ctypes.data_as(C.c_void_p))
assert rc == 0, rc
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/{tag}.npy", out.reshape(nc, NB, NB))
print(n, nc, tag, "norm %.15e" % np.linalg.norm(Y), flush=True)
