"""B200 vs oracle parity on the BASELINE configurations (north-star gates):
first filtered subspace <= 1e-9 relative Frobenius; eigenvalues <= 1e-10
(relative to max(|lambda|, ||A||_2)); eigenvector subspace sine <= 1e-8;
identical converged count, iteration count and trace accounting."""
import numpy as np
import pytest

import oracle as O
from paper_1605_08771_b200 import configs as CF

pytestmark = pytest.mark.gpu


def _matrix(index):
    vals = CF.spectrum(index, O.uniform_fill)
    if index == 3:
        A = CF.laplacian_2d()
    else:
        Q = O.seeded_orthogonal(len(vals), 1000 + index)
        A = O.assemble_matrix(vals, Q)
    return A, vals, CF.resolved(index, vals)


def _sine(Vref, V):
    Q, _ = np.linalg.qr(Vref)
    return np.linalg.norm(V - Q @ (Q.T @ V), 2)


def _compare(sol, ref, A, tol_ev=1e-10, tol_sine=1e-8):
    assert sol.converged == ref.converged
    assert sol.iterations == ref.iterations
    assert len(sol.eigenvalues) == len(ref.eigenvalues)
    assert [t.rhs_cumulative for t in sol.trace] == [t.rhs_cumulative for t in ref.trace]
    assert [t.subspace_dim for t in sol.trace] == [t.subspace_dim for t in ref.trace]
    assert [t.m_found for t in sol.trace] == [t.m_found for t in ref.trace]
    assert sol.recovery_events == ref.recovery_events
    if len(ref.eigenvalues):
        normA = np.abs(ref.eigenvalues).max()
        scale = np.maximum(np.abs(ref.eigenvalues), max(normA, 1.0))
        assert np.all(np.abs(sol.eigenvalues - ref.eigenvalues) <= tol_ev * scale)
        assert _sine(ref.eigenvectors, sol.eigenvectors) <= tol_sine


@pytest.mark.parametrize("index", [0])
def test_first_filtered_subspace_and_feast(index):
    import paper_1605_08771_b200 as P
    A, vals, c = _matrix(index)
    cfg = dict(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"])
    I = (c["lo"], c["hi"])
    ref = O.feast_solve(A, O.SearchInterval(*I), O.SolverConfig(**cfg))
    sol = P.feast_solve(A, P.SearchInterval(*I), P.SolverConfig(**cfg), keep_first=True)
    Y1 = sol.first_filtered
    rel = np.linalg.norm(Y1 - ref.first_filtered) / np.linalg.norm(ref.first_filtered)
    assert rel <= 1e-9, rel
    _compare(sol, ref, A)
    assert len(sol.eigenvalues) == c["inside"]


@pytest.mark.slow
@pytest.mark.parametrize("driver", ["feast_solve", "xfeast_solve", "rfeast_solve"])
def test_cfg1_hard_edge_drivers(driver):
    import paper_1605_08771_b200 as P
    A, vals, c = _matrix(1)
    kw = dict(m0=c["m0"], n_c=c["n_c"], tol=c["tol"], max_iter=c["max_iter"], s=c["s"])
    I = (c["lo"], c["hi"])
    ref = getattr(O, driver)(A, O.SearchInterval(*I), O.SolverConfig(**kw))
    sol = getattr(P, driver)(A, P.SearchInterval(*I), P.SolverConfig(**kw))
    _compare(sol, ref, A)
