"""Concurrent independent solves (solve_concurrently / fl_solve_many,
SURVEY §8(f)(2)): intervals of one spectrum and compare-style cells run on
several worker contexts at once must return exactly what each solve returns
alone (deterministic kernels, private streams and workspaces), in job order;
a failing job reports its error while the others complete (the CLI's compare
semantics, feastlab_cli.cpp:245-294)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _matrix():
    vals = np.linspace(-1.0, 1.0, 400) + 1e-3 * np.sin(np.arange(400))
    Q = O.seeded_orthogonal(400, 7)
    return O.assemble_matrix(vals, Q), vals


def test_concurrent_intervals_match_sequential():
    import paper_1605_08771_b200 as P
    A, vals = _matrix()
    edges = [-0.6, -0.3, 0.0, 0.3, 0.6]
    jobs = []
    for lo, hi in zip(edges[:-1], edges[1:]):
        inside = int(((vals > lo) & (vals < hi)).sum())
        cfg = P.SolverConfig(m0=int(1.5 * inside) + 4, n_c=8, tol=1e-11, max_iter=20)
        jobs.append(("feast", P.SearchInterval(lo, hi), cfg))
    jobs.append(("xfeast", P.SearchInterval(-0.3, 0.0),
                 P.SolverConfig(m0=60, n_c=8, tol=1e-11, max_iter=20, s=2)))
    jobs.append(("feast", P.SearchInterval(-0.1, 0.1), P.SolverConfig(m0=401, n_c=8)))  # m0 > n
    got = P.solve_many(A, jobs, devices=[0], per_device=3)
    assert len(got) == len(jobs)
    for (variant, interval, cfg), g in zip(jobs[:-1], got[:-1]):
        ref = getattr(P, f"{variant}_solve")(A, interval, cfg)
        assert g["error"] is None
        assert g["iterations"] == ref.iterations and g["converged"] == ref.converged
        assert np.array_equal(g["eigenvalues"], ref.eigenvalues)
    assert got[-1]["error"] and "m0" in got[-1]["error"]
    # the four intervals tile (-0.6, 0.6): together they find every eigenvalue once
    found = np.sort(np.concatenate([g["eigenvalues"] for g in got[:4]]))
    exact = np.sort(vals[(vals > -0.6) & (vals < 0.6)])
    assert len(found) == len(exact)
    assert np.abs(found - exact).max() <= 1e-12
