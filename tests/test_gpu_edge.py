"""Edge cases the reference exercises on the B200 path: options
(generalized_reduced, qr orthogonalizer, factor cache), a singular shift
(non-finite entries) reported with the node index, full subspace m0 = n,
single-column blocks and single-node rules."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
I11 = O.SearchInterval(-1, 1)


def _instance(seed, n=40, inside=6):
    lay = O.SpectrumLayout(n, O.SearchInterval(-0.9, 0.9), inside, O.SearchInterval(1.6, 12.0),
                           n - inside, seed=seed)
    return O.assemble_matrix(*O.generate_spectrum(lay))


@pytest.mark.parametrize("opt", [dict(generalized_reduced=True), dict(orthogonalizer="qr"),
                                 dict(cache_factorizations=True)])
def test_driver_options_match_oracle(opt):
    import paper_1605_08771_b200 as P
    A = _instance(71)
    kw = dict(m0=9, n_c=8, tol=1e-10, max_iter=20, **opt)
    sol = P.feast_solve(A, P.SearchInterval(-1, 1), P.SolverConfig(**kw))
    ref = O.feast_solve(A, I11, O.SolverConfig(**kw))
    assert sol.converged == ref.converged and sol.iterations == ref.iterations
    assert len(sol.eigenvalues) == len(ref.eigenvalues)
    assert np.abs(sol.eigenvalues - ref.eigenvalues).max() <= 1e-10 * np.abs(A).max()
    assert [t.subspace_dim for t in sol.trace] == [t.subspace_dim for t in ref.trace]
    if opt.get("cache_factorizations"):
        assert sol.accounting.factorizations == 8


def test_singular_node_is_reported():
    import paper_1605_08771_b200 as P
    A = np.eye(70)
    A[3, 3] = np.inf
    rule = P.build_contour_rule(P.SearchInterval(-1, 1), 4)
    with pytest.raises(P.FeastRuntimeError) as ei:
        P.apply_filter(A, rule, np.ones((70, 2)))
    assert "singular factorization at node 0" in str(ei.value)


def test_full_subspace_and_single_columns():
    import paper_1605_08771_b200 as P
    A = _instance(73, n=24, inside=5)
    sol = P.feast_solve(A, P.SearchInterval(-1, 1), P.SolverConfig(m0=24, n_c=8, tol=1e-10))
    ref = O.feast_solve(A, I11, O.SolverConfig(m0=24, n_c=8, tol=1e-10))
    assert len(sol.eigenvalues) == len(ref.eigenvalues) == 5
    assert np.abs(sol.eigenvalues - ref.eigenvalues).max() <= 1e-10 * np.abs(A).max()
    rule = P.build_contour_rule(P.SearchInterval(-0.5, 0.5), 1)
    x = O.random_block(24, 1, 3)
    y = P.apply_filter(A, rule, x)
    yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.5, 0.5), 1), x)
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)


def test_run_to_run_bitwise_determinism():
    # C10-style gate (proj/tests/acceptance.cpp:429-450) at a size that uses
    # every kernel path (several 128-column blocks, node chunks on 4 streams)
    import paper_1605_08771_b200 as P
    lay = O.SpectrumLayout(700, O.SearchInterval(-0.3, 0.3), 40, O.SearchInterval(0.5, 4.0), 660,
                           seed=5)
    A = O.assemble_matrix(*O.generate_spectrum(lay))
    cfg = P.SolverConfig(m0=60, n_c=8, s=2, tol=1e-10, max_iter=6)
    for d in (P.feast_solve, P.xfeast_solve, P.rfeast_solve):
        a = d(A, P.SearchInterval(-0.35, 0.35), cfg)
        b = d(A, P.SearchInterval(-0.35, 0.35), cfg)
        assert P.write_trace_csv(a.trace) == P.write_trace_csv(b.trace)
        assert np.array_equal(a.eigenvalues, b.eigenvalues)
        assert np.array_equal(a.eigenvectors, b.eigenvectors)


def test_singular_node_device_path_is_raised_at_next_sync():
    """Device-resident applications do not wait for the singular-node verdict;
    the next host wait on the context raises it (capi.cu resolve_pending)."""
    import torch
    import paper_1605_08771_b200 as P
    ctx = P.Context(0)
    A = np.eye(70)
    A[3, 3] = np.inf
    f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-1, 1), 4), ctx=ctx)
    X = torch.ones((2, 70), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    torch.cuda.synchronize()
    f.apply_device(X.data_ptr(), 70, 2, Y.data_ptr(), 70)  # returns without waiting
    with pytest.raises(P.FeastRuntimeError) as ei:
        ctx.sync()
    assert "singular factorization at node 0" in str(ei.value)
    ctx.sync()  # the verdict is consumed once


def test_context_outlives_its_objects_in_any_destruction_order():
    """fl_ctx is reference counted by its matrices, blocks and filters: the
    owner may destroy it first (as a garbage collector breaking a cycle may)
    and the objects stay usable until they are destroyed themselves."""
    import ctypes as C
    import paper_1605_08771_b200 as P
    from paper_1605_08771_b200 import _lib as L
    lib = L.lib()
    n, p = 96, 8
    A = np.asfortranarray(np.diag(np.linspace(-1, 1, n)))
    X = np.asfortranarray(np.random.default_rng(0).standard_normal((n, p)))
    ctx, mat, flt, blk = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    err = L.Err()
    assert lib.fl_ctx_create(0, C.byref(ctx), C.byref(err)) == 0
    assert lib.fl_matrix_create(ctx, A.ctypes.data, n, n, L.FL_HOST, C.byref(mat), C.byref(err)) == 0
    rule = P.build_contour_rule(P.SearchInterval(-0.5, 0.5), 4)
    zr, zi, wr, wi = (np.ascontiguousarray(v) for v in rule.parts())
    assert lib.fl_filter_create(ctx, mat, 4, zr.ctypes.data, zi.ctypes.data, wr.ctypes.data,
                                wi.ctypes.data, 0, C.byref(flt), C.byref(err)) == 0
    assert lib.fl_block_create(ctx, n, p, C.byref(blk), C.byref(err)) == 0
    assert lib.fl_ctx_destroy(ctx) == 0          # owner gone first
    Y = np.zeros((n, p), order="F")
    rhs, facts = C.c_longlong(), C.c_longlong()
    assert lib.fl_filter_apply_raw(flt, X.ctypes.data, n, p, Y.ctypes.data, n, L.FL_HOST,
                                   C.byref(rhs), C.byref(facts), C.byref(err)) == 0, err.msg
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.5, 0.5), 4), X)
    assert np.linalg.norm(Y - Yo) <= 1e-12 * np.linalg.norm(Yo)
    assert lib.fl_block_destroy(blk) == 0
    assert lib.fl_filter_destroy(flt) == 0
    assert lib.fl_matrix_destroy(mat) == 0       # last reference: context torn down here
