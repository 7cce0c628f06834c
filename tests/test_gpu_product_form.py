"""3M vs 4M complex product forms of the DMMA GEMMs (gemm.cu).

The filter's trailing updates and blocked solves run in the 3M form by
default (3 real DMMA products per complex product). Both forms must give the
oracle's filtered block to the north-star tolerance (1e-9 relative Frobenius)
and agree with each other to rounding level; node solves must reach the same
backward error.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def restore_mode():
    import paper_1605_08771_b200 as P
    old = P.zgemm_mode()
    yield P
    P.zgemm_mode(old)


def _problem(n, p, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
    X = np.asfortranarray(rng.standard_normal((n, p)))
    return A, X


@pytest.mark.parametrize("n,p,nc", [(300, 40, 8), (1000, 150, 8), (777, 65, 4)])
def test_filter_both_forms_match_oracle(restore_mode, n, p, nc):
    P = restore_mode
    A, X = _problem(n, p, n)
    I = (-0.1, 0.1)
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(*I), nc), X)
    rule = P.build_contour_rule(P.SearchInterval(*I), nc)
    Y = {}
    for mode in ("4m", "3m"):
        assert P.zgemm_mode(mode) == mode
        Y[mode] = P.apply_filter(A, rule, X)
        rel = np.linalg.norm(Y[mode] - Yo) / np.linalg.norm(Yo)
        assert rel <= 1e-9, (mode, rel)
    assert np.linalg.norm(Y["3m"] - Y["4m"]) / np.linalg.norm(Y["4m"]) <= 1e-11


@pytest.mark.parametrize("mode", ["3m", "4m"])
def test_node_solve_backward_error(restore_mode, mode):
    P = restore_mode
    P.zgemm_mode(mode)
    A, X = _problem(640, 96, 7)
    z = complex(0.05, 0.02)
    Z = P.node_solve(A, z, X)
    M = z * np.eye(640) - A
    berr = np.linalg.norm(M @ Z - X) / (np.linalg.norm(M) * np.linalg.norm(Z) + np.linalg.norm(X))
    assert berr <= 1e-14, berr


def test_mode_validation(restore_mode):
    P = restore_mode
    with pytest.raises(ValueError):
        P.zgemm_mode("5m")
