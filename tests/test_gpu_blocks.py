"""LU outer-block and triangular-solve block widths (FEASTLAB_LU_PANELS,
FEASTLAB_SOLVE_PANELS: 1..8 panels / tiles of 64): every width, including
ragged last blocks (N / 64 not a multiple of the width), gives the oracle's
filter (proj/src/filterop.cpp:62-84) to rounding level. The defaults pick 8
panels (K = 512 trailing updates) for >= 8 local nodes of N >= 12288, 4 for
>= 8 local nodes of smaller N, and 2 below."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,n_c", [(700, 8), (1000, 16)])
@pytest.mark.parametrize("lu,solve", [(1, 1), (2, 2), (3, 3), (4, 4), (4, 1), (1, 4), (3, 2),
                                      (8, 8), (6, 3), (7, 5)])
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
