"""CUDA-graph replay of filter applications (capi.cu filter_apply_dev).

Small problems (N < 2048): call 1 runs eagerly, call 2 with the same launch
key is captured and launched, later calls replay. Large ones capture on the
first call; with cached factorizations the factoring application is captured
and launched once, the solve-only applications are captured and replayed. Every path must give bitwise the same Y as
the eager run, a changed key (new X buffer, new block width) must re-capture,
and the launch counter must keep counting the replayed kernels.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _setup(n=500, p=70, nc=6, seed=3):
    import paper_1605_08771_b200 as P
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    A = np.asfortranarray(0.5 * (A + A.T) / np.sqrt(n))
    X = np.asfortranarray(rng.standard_normal((n, p)))
    rule = P.build_contour_rule(P.SearchInterval(-0.2, 0.3), nc)
    return P, A, X, rule


def test_replay_is_bitwise_identical_to_eager():
    P, A, X, rule = _setup()
    ctx = P.Context(0)
    f = P.FilterApplier(A, rule, ctx=ctx)
    Ys = [f.apply(X) for _ in range(4)]  # eager, capture, replay, replay
    for Y in Ys[1:]:
        assert np.array_equal(Y, Ys[0])
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.2, 0.3), 6), X)
    assert np.linalg.norm(Ys[0] - Yo) / np.linalg.norm(Yo) <= 1e-9


def test_key_change_recaptures_and_launches_are_counted():
    P, A, X, rule = _setup()
    ctx = P.Context(0)
    f = P.FilterApplier(A, rule, ctx=ctx)
    l0 = ctx.launches(); f.apply(X); l1 = ctx.launches()
    f.apply(X); l2 = ctx.launches()
    f.apply(X); l3 = ctx.launches()
    assert l1 - l0 == l2 - l1 == l3 - l2 > 0
    X2 = np.asfortranarray(X[:, :33])  # narrower block: new key
    Y2 = [f.apply(X2) for _ in range(3)]
    assert np.array_equal(Y2[0], Y2[2])
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.2, 0.3), 6), X2)
    assert np.linalg.norm(Y2[2] - Yo) / np.linalg.norm(Yo) <= 1e-9
    assert np.array_equal(f.apply(X), f.apply(X))  # back to the first key


def test_device_buffers_replay():
    import torch
    P, A, X, rule = _setup(n=384, p=64)
    ctx = P.Context(0)
    f = P.FilterApplier(A, rule, ctx=ctx)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Yd = torch.empty_like(Xd)
    torch.cuda.synchronize()  # Xd is written on torch's stream, read on the context's
    outs = []
    for _ in range(3):
        f.apply_device(Xd.data_ptr(), 384, 64, Yd.data_ptr(), 384)
        ctx.sync()
        outs.append(Yd.cpu().numpy().T.copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    assert np.array_equal(outs[0], f.apply(X))


def test_large_first_call_capture_and_cached_phases():
    """N >= 2048: every call runs as a graph. Cached factors: call 1 (factor +
    solve graph), call 2 (solve-only capture), call 3 (replay) agree bitwise
    with each other and with the uncached filter, and factor once."""
    P, A, X, rule = _setup(n=2100, p=64, nc=2, seed=5)
    ctx = P.Context(0)
    acc = P.SolveAccounting()
    fc = P.FilterApplier(A, rule, True, ctx=ctx)
    Yc = [fc.apply(X, acc) for _ in range(3)]
    assert acc.factorizations == 2 and acc.rhs_solved == 3 * 2 * 64
    f = P.FilterApplier(A, rule, ctx=ctx)
    Y = [f.apply(X) for _ in range(2)]
    for y in Yc[1:] + Y:
        assert np.array_equal(y, Yc[0])
    Yo = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.2, 0.3), 2), X)
    assert np.linalg.norm(Yc[0] - Yo) / np.linalg.norm(Yo) <= 1e-12
