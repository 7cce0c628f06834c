"""RFEAST's Cholesky recovery on the B200 path (proj/src/drivers.cpp:210-219,
proj/src/ritz.cpp:64-79): when the expanded block [Xp, R] spans more columns
than the matrix has rows, its Gram matrix is singular, the column-by-column
Cholesky of the Rayleigh-Ritz reduction meets a non-positive pivot, the
driver counts a recovery event, orthonormalises the block and redoes the
Rayleigh-Ritz step. The instances make the failure structural (rank deficit
of s*m0 - n columns, so a deficient pivot is rounding noise of either sign on
both sides and the first non-positive one is met with near certainty), and
the test asserts the oracle and the device agree on the recovery count, the
trace and the eigenpairs."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _instance(n, inside, seed):
    rng = np.random.default_rng(seed)
    vals = np.sort(np.concatenate([rng.uniform(-0.28, 0.28, inside),
                                   rng.uniform(0.31, 0.9, (n - inside) // 2),
                                   -rng.uniform(0.31, 0.9, n - inside - (n - inside) // 2)]))
    return O.assemble_matrix(vals, O.seeded_orthogonal(n, 500 + seed)), vals


@pytest.mark.parametrize("n,m0,s,inside", [(48, 28, 2, 8), (48, 28, 3, 8), (300, 160, 2, 20),
                                           (300, 110, 3, 20)])
def test_rfeast_cholesky_recovery_matches_oracle(n, m0, s, inside):
    import paper_1605_08771_b200 as P
    A, vals = _instance(n, inside, n + s)
    kw = dict(m0=m0, n_c=4, tol=1e-10, max_iter=10, s=s)
    ref = O.rfeast_solve(A, O.SearchInterval(-0.3, 0.3), O.SolverConfig(**kw))
    sol = P.rfeast_solve(A, P.SearchInterval(-0.3, 0.3), P.SolverConfig(**kw))
    print(f"n={n} m0={m0} s={s}: oracle it={ref.iterations} rec={ref.recovery_events} "
          f"m={len(ref.eigenvalues)} | b200 it={sol.iterations} rec={sol.recovery_events} "
          f"m={len(sol.eigenvalues)}")
    assert ref.recovery_events >= 1  # the instance does reach the recovery path
    assert sol.recovery_events == ref.recovery_events
    assert sol.iterations == ref.iterations and sol.converged == ref.converged
    assert [(t.iter, t.subspace_dim, t.rhs_cumulative, t.m_found) for t in sol.trace] == \
        [(t.iter, t.subspace_dim, t.rhs_cumulative, t.m_found) for t in ref.trace]
    assert len(sol.eigenvalues) == len(ref.eigenvalues) == inside
    assert np.abs(np.asarray(sol.eigenvalues) - np.asarray(ref.eigenvalues)).max() <= 1e-10
    exact = vals[(vals > -0.3) & (vals < 0.3)]
    assert np.abs(np.sort(sol.eigenvalues) - exact).max() <= 1e-10
    assert sol.accounting.rhs_solved == ref.accounting.rhs_solved
    assert sol.accounting.factorizations == ref.accounting.factorizations
