"""Re-expresses proj/tests/test_ritz.cpp and acceptance C3
(proj/tests/acceptance.cpp:118-132) against both the CPU oracle (pin) and the B200 path (F = b200, -m gpu)."""
import numpy as np
import pytest

import oracle as O


def _qr_basis(X, k):
    Q, _ = np.linalg.qr(X)
    return Q[:, :k]


@pytest.mark.parametrize("method", ["svd", "qr"])
def test_orthonormalize_basis_and_span(F, method):
    X = O.random_block(20, 8, 51)
    U, rank = F.orthonormalize(X, 1e-10, method)
    assert rank == 8
    assert np.abs(U.T @ U - np.eye(8)).max() <= 1e-12
    Q = _qr_basis(X, 8)
    assert np.linalg.norm(U @ U.T - Q @ Q.T) <= 1e-10


def test_orthonormalize_rank_deficiency(F):
    v = O.random_block(10, 1, 3)[:, 0]
    X = np.stack([v, 2.0 * v], axis=1)
    U, rank = F.orthonormalize(X, 1e-10)
    assert rank == 1
    assert abs(abs(U[:, 0] @ (v / np.linalg.norm(v))) - 1.0) <= 1e-12
    with pytest.raises(F.FeastRuntimeError):
        F.orthonormalize(np.zeros((5, 3)), 1e-10)


def test_orthonormalize_passthrough(F):
    Q = _qr_basis(O.random_block(15, 4, 77), 4)
    U, rank = F.orthonormalize(Q, 1e-10)
    assert rank == 4
    assert np.abs(U.T @ U - np.eye(4)).max() <= 1e-12
    assert np.linalg.norm(U @ U.T - Q @ Q.T) <= 1e-12


def test_rr_coordinate_case(F):
    A = np.diag([1.0, 2.0, 3.0])
    X = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])
    rr = F.rayleigh_ritz(A, X, O.SearchInterval(0, 10))
    assert rr.size() == 2
    assert rr.values[0] == pytest.approx(1.0, rel=1e-14)
    assert rr.values[1] == pytest.approx(2.0, rel=1e-14)
    assert rr.residual_norms.max() <= 1e-14
    assert abs(abs(rr.vectors[0, 0]) - 1.0) <= 1e-14


def test_rr_invariant_subspace(F):
    A = O.random_symmetric(12, 9)
    w, V = O.dense_eig(A)
    rr = F.rayleigh_ritz(A, V[:, 3:5], O.SearchInterval(-100, 100))
    scale = np.linalg.norm(A)
    assert abs(rr.values[0] - w[3]) <= 1e-12 * scale
    assert abs(rr.values[1] - w[4]) <= 1e-12 * scale
    assert rr.residual_norms.max() <= 1e-11 * scale


def test_rr_brute_force_reduced_oracle(F):
    A = O.random_symmetric(16, 33)
    Q = _qr_basis(O.random_block(16, 5, 34), 5)
    rr = F.rayleigh_ritz(A, Q, O.SearchInterval(-1, 1))
    red = Q.T @ A @ Q
    ref, _ = O.dense_eig(0.5 * (red + red.T))
    bounds, _ = O.dense_eig(A)
    s = np.linalg.norm(A)
    for k in range(5):
        assert abs(rr.values[k] - ref[k]) <= 1e-12 * s
        assert rr.values[k] >= bounds[0] - 1e-10 * s
        assert rr.values[k] <= bounds[15] + 1e-10 * s
        assert abs(np.linalg.norm(rr.vectors[:, k]) - 1.0) <= 1e-12


def test_rr_cholesky_failure_reports_pivot(F):
    A = O.random_symmetric(8, 12)
    v = O.random_block(8, 1, 13)[:, 0]
    X = np.stack([v, np.zeros(8)], axis=1)
    with pytest.raises(F.CholeskyError) as ei:
        F.rayleigh_ritz(A, X, O.SearchInterval(-1, 1))
    assert ei.value.pivot <= 1e-12
    assert ei.value.index == 1


def test_residual_orthogonality_20_seeds(F):
    for seed in range(20):
        n = 10 + seed % 7
        A = O.random_symmetric(n, 100 + seed)
        U, _ = F.orthonormalize(O.random_block(n, 4, 200 + seed), 1e-10)
        rr = F.rayleigh_ritz(A, U, O.SearchInterval(-1, 1))
        R = F.compute_residual_block(A, rr)
        assert np.abs(rr.vectors.T @ R).max() <= 1e-10 * np.linalg.norm(A)


def test_acceptance_c3(F):
    for k in range(20):
        n = 10 + k
        A = O.random_symmetric(n, 3000 + k)
        U, _ = F.orthonormalize(O.random_block(n, 5, 4000 + k), 1e-10)
        rr = F.rayleigh_ritz(A, U, O.SearchInterval(-1, 1))
        R = F.compute_residual_block(A, rr)
        assert np.abs(rr.vectors.T @ R).max() <= 1e-10 * np.linalg.norm(A)


def test_residual_block_2x2(F):
    A = np.diag([1.0, 2.0])
    s = 1 / np.sqrt(2.0)
    trial = F.RitzSet(np.array([1.5]), np.array([[s], [s]]), np.zeros(1), np.array([True]))
    R = F.compute_residual_block(A, trial)
    assert R[0, 0] == pytest.approx(-0.5 * s, rel=1e-14)
    assert R[1, 0] == pytest.approx(0.5 * s, rel=1e-14)
    assert abs(trial.vectors[:, 0] @ R[:, 0]) <= 1e-15


def test_exact_pairs_zero_residual(F):
    A = O.random_symmetric(7, 55)
    w, V = O.dense_eig(A)
    ex = F.RitzSet(w[:3], V[:, :3], np.zeros(3), np.ones(3, bool))
    assert np.abs(F.compute_residual_block(A, ex)).max() <= 1e-13 * np.linalg.norm(A)


def _make_ritz(values, residuals, I):
    n = len(values)
    return O.RitzSet(np.array(values, float), np.eye(n), np.array(residuals, float),
                     np.array([I.contains(v) for v in values]))


def test_select_inside_then_outside(F):
    I = O.SearchInterval(-1, 1)
    rs = _make_ritz([-0.9, -0.5, 0.0, 0.4, 0.8, 1.5, 1.6, 1.7, 1.8, 1.9, 2.0],
                    [1e-3, 2e-3, 3e-3, 4e-3, 5e-3, 9e-2, 1e-4, 5e-2, 2e-4, 8e-2, 3e-4], I)
    sel = F.select_pairs(rs, 8, I)
    assert sel.size() == 8 and F.count_inside(sel) == 5
    outside = [v for v, f in zip(sel.values, sel.inside_flags) if not f]
    assert outside == [1.6, 1.8, 2.0]


def test_select_lowest_residual_inside_past_m0(F):
    I = O.SearchInterval(-1, 1)
    rs = _make_ritz([-0.8, -0.6, -0.4, -0.2, 0.0, 0.2, 0.4, 0.6, 0.8, 0.9],
                    [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-11], I)
    sel = F.select_pairs(rs, 4, I)
    assert sel.size() == 4 and np.all(sel.residual_norms <= 1e-8)


def test_select_nothing_inside(F):
    I = O.SearchInterval(-1, 1)
    sel = F.select_pairs(_make_ritz([2.0, 3.0, 4.0], [3e-3, 1e-5, 7e-4], I), 2, I)
    assert list(sel.residual_norms) == [1e-5, 7e-4]


def test_select_ties_break_toward_center_then_index(F):
    I = O.SearchInterval(-1, 1)
    rs = _make_ritz([0.5, -0.2, 0.2, 0.9], [1e-3, 1e-3, 1e-3, 1e-3], I)
    assert list(F.select_indices(rs, 4, I)) == [1, 2, 0, 3]


def test_count_inside(F):
    I = O.SearchInterval(-1, 1)
    assert F.count_inside(_make_ritz([2.0, 3.0], [1e-3, 1e-3], I)) == 0
    assert F.count_inside(_make_ritz([0.5, 2.0, -0.5], [1e-3] * 3, I)) == 2
