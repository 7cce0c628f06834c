"""LU outer-block and triangular-solve block widths (FEASTLAB_LU_PANELS,
FEASTLAB_SOLVE_PANELS: 1..16 LU panels, 1..8 solve tiles of 64): every width, including
ragged last blocks (N / 64 not a multiple of the width), gives the oracle's
filter (proj/src/filterop.cpp:62-84) to rounding level. The defaults pick 16
panels (K = 1024 trailing updates) for >= 8 local nodes of N >= 12288 (8 for
fewer nodes), 4 for >= 8 local nodes of smaller N, and 2 below."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,n_c", [(700, 8), (1000, 16)])
@pytest.mark.parametrize("lu,solve", [(1, 1), (2, 2), (3, 3), (4, 4), (4, 1), (1, 4), (3, 2),
                                      (8, 8), (6, 3), (7, 5), (12, 4), (16, 8)])
def test_block_widths_match_oracle(n, n_c, lu, solve, monkeypatch):
    import paper_1605_08771_b200 as P
    monkeypatch.setenv("FEASTLAB_LU_PANELS", str(lu))
    monkeypatch.setenv("FEASTLAB_SOLVE_PANELS", str(solve))
    A = O.random_symmetric(n, 17) / np.sqrt(n)
    X = O.random_block(n, 96, 18)
    I = (-0.35, 0.25)
    Y = P.apply_filter(A, P.build_contour_rule(P.SearchInterval(*I), n_c), X)
    ref = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(*I), n_c), X)
    rel = np.linalg.norm(Y - ref) / np.linalg.norm(ref)
    assert rel <= 1e-12, rel


def test_cached_factors_with_wide_blocks(monkeypatch):
    """Cached factorisations (SolverConfig.cache_factorizations) reuse the
    wide-block LU: the second application solves only and matches the oracle."""
    import paper_1605_08771_b200 as P
    monkeypatch.setenv("FEASTLAB_LU_PANELS", "4")
    n = 900
    A = O.random_symmetric(n, 21) / np.sqrt(n)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.3), 8)
    orule = O.build_contour_rule(O.SearchInterval(-0.3, 0.3), 8)
    f = P.FilterApplier(A, rule, True)
    acc = P.SolveAccounting()
    for seed in (1, 2):
        X = O.random_block(n, 40, seed)
        Y = f.apply(X, acc)
        ref = O.apply_filter(A, orule, X)
        assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-12
    assert acc.factorizations == 8


_LASWP_CHILD = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
import oracle as O
import paper_1605_08771_b200 as P
n = 1000
A = O.random_symmetric(n, 31) / np.sqrt(n)
X = O.random_block(n, 72, 32)
Y = P.apply_filter(A, P.build_contour_rule(P.SearchInterval(-0.3, 0.2), 8), X)
print(hashlib.sha256(np.ascontiguousarray(Y).tobytes()).hexdigest())
"""


def test_laswp_forms_bitwise_equal():
    """The warp-per-column laswp (default) and the shared-memory form
    (FEASTLAB_LASWP=smem, read once per process) move the same rows: the
    filtered block is bitwise identical."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _LASWP_CHILD.format(root=root)
    out = {}
    for form in ("warp", "smem"):
        env = dict(os.environ)
        env.pop("FEASTLAB_LASWP", None)
        if form == "smem":
            env["FEASTLAB_LASWP"] = "smem"
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[form] = r.stdout.strip().splitlines()[-1]
    assert out["warp"] == out["smem"]


@pytest.mark.parametrize("n,lu", [(1000, 2), (1000, 4), (1500, 7), (2200, 16), (2048, 16)])
def test_composed_block_interchanges_bitwise_equal(n, lu, monkeypatch):
    """The outer block's np net permutations composed and applied in one pass
    (launch_laswp_block, default) move the same rows as one pass per panel
    (FEASTLAB_LASWP_BLOCK=0): the filtered block is bitwise identical, on
    ragged last blocks and on blocks that end the matrix too."""
    import paper_1605_08771_b200 as P
    monkeypatch.setenv("FEASTLAB_LU_PANELS", str(lu))
    A = O.random_symmetric(n, 41) / np.sqrt(n)
    X = O.random_block(n, 72, 42)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.2), 8)
    out = {}
    for form in ("0", "1"):
        monkeypatch.setenv("FEASTLAB_LASWP_BLOCK", form)
        out[form] = [P.apply_filter(A, rule, X) for _ in range(2)]  # eager, then graph
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][0])
    ref = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.3, 0.2), 8), X)
    assert np.linalg.norm(out["1"][0] - ref) / np.linalg.norm(ref) <= 1e-12
