"""Ownership and error-path semantics of the drop-in filter objects on the B200:
NodeFactorization owns one device factor (proj/src/filterop.cpp:9-33: factor in
the constructor, solve() against it), a singular node found by a cached
factoring application survives a second application issued before the host
syncs, rules with more nodes than one kernel launch batches (kMaxNodes = 64)
filter exactly as the oracle, and A is uploaded once per context."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _rule80(P, lo, hi, k=40):
    """An 80-node rule through contour_rule_from_nodes (gauss_legendre stops at
    64 nodes, proj/src/contour.cpp:17-20; external node sets have no limit):
    the k-node Gauss rules of two overlapping circles, concatenated."""
    a = P.build_contour_rule(P.SearchInterval(lo, hi), k)
    b = P.build_contour_rule(P.SearchInterval(lo * 0.9, hi * 1.1), k)
    nodes = np.concatenate([a.nodes, b.nodes])
    weights = np.concatenate([a.weights, b.weights]) * 0.5
    return nodes, weights


def _A(n, seed):
    lay = O.SpectrumLayout(n, O.SearchInterval(-0.5, 0.5), 12, O.SearchInterval(1.0, 6.0), n - 12,
                           seed=seed)
    return O.assemble_matrix(*O.generate_spectrum(lay))


def test_node_factorization_owns_its_factor():
    import paper_1605_08771_b200 as P
    ctx = P.Context(0)
    n = 150
    A = _A(n, 3)
    z = complex(0.1, 0.35)
    rng = np.random.default_rng(4)
    B = rng.standard_normal((n, 7)) + 1j * rng.standard_normal((n, 7))
    l0 = ctx.launches()
    nf = P.NodeFactorization(A, z, ctx=ctx)
    l_factor = ctx.launches() - l0
    W1 = nf.solve(B)
    l1 = ctx.launches()
    W2 = nf.solve(B)
    l_solve = ctx.launches() - l1
    # the second solve reuses the factor: no shift, panel, swap or trailing-update launches
    assert l_solve < l_factor / 2, (l_solve, l_factor)
    assert np.array_equal(W1, W2)
    ref = O.node_solve(A, z, B)
    assert np.linalg.norm(W1 - ref) / np.linalg.norm(ref) <= 1e-12
    # real right-hand side: the reference casts to complex (filterop.cpp:26-28)
    Wr = nf.solve(B.real)
    assert np.linalg.norm(Wr - O.node_solve(A, z, B.real)) <= 1e-12 * np.linalg.norm(Wr)


def test_node_factorization_singular_at_construction():
    import paper_1605_08771_b200 as P
    A = np.eye(70)
    A[5, 5] = np.inf
    with pytest.raises(P.FeastRuntimeError) as ei:
        P.NodeFactorization(A, complex(0.0, 0.5), node_index=5)
    assert "singular factorization at node 5" in str(ei.value)


def test_cached_singular_verdict_survives_a_second_application():
    """a solve-only application (cached factors) must not
    reset the singular-node verdict of the factoring application before it."""
    import torch
    import paper_1605_08771_b200 as P
    ctx = P.Context(0)
    A = np.eye(70)
    A[3, 3] = np.inf
    f = P.FilterApplier(A, P.build_contour_rule(P.SearchInterval(-1, 1), 4), True, ctx=ctx)
    X = torch.ones((2, 70), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    torch.cuda.synchronize()
    f.apply_device(X.data_ptr(), 70, 2, Y.data_ptr(), 70)  # factors: finds node 0 singular
    f.apply_device(X.data_ptr(), 70, 2, Y.data_ptr(), 70)  # solve-only, before any host wait
    with pytest.raises(P.FeastRuntimeError) as ei:
        ctx.sync()
    assert "singular factorization at node 0" in str(ei.value)
    ctx.sync()
    # the bad factors were dropped: the next application factors again and raises again
    with pytest.raises(P.FeastRuntimeError):
        f.apply(np.ones((70, 2)))


@pytest.mark.parametrize("cache", [False, True])
def test_rule_with_more_nodes_than_one_launch_batch(cache):
    """n_c = 80 > kMaxNodes: the accumulation continues the ascending sum over
    launches, so Y matches the oracle as closely as an 8-node rule does."""
    import paper_1605_08771_b200 as P
    n, p = 200, 12
    A = _A(n, 9)
    X = O.random_block(n, p, 10)
    nodes, weights = _rule80(P, -0.4, 0.45)
    rule = P.contour_rule_from_nodes(P.SearchInterval(-0.4, 0.45), nodes, weights)
    acc = P.SolveAccounting()
    Y = P.FilterApplier(A, rule, cache).apply(X, acc)
    ref = O.apply_filter(A, O.contour_rule_from_nodes(O.SearchInterval(-0.4, 0.45), nodes,
                                                      weights), X)
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-12
    assert acc.rhs_solved == 80 * p and acc.factorizations == 80


def test_ordered_reduction_more_than_64_nodes_is_bitwise_plain():
    import paper_1605_08771_b200 as P
    n, p = 130, 10
    A = _A(n, 21)
    X = O.random_block(n, p, 22)
    nodes, weights = _rule80(P, -0.3, 0.4, k=35)  # 70 nodes
    rule = P.contour_rule_from_nodes(P.SearchInterval(-0.3, 0.4), nodes, weights)
    Y0 = P.FilterApplier(A, rule, ctx=P.Context(0)).apply(X)
    nccl = P.Context(0, nccl_id=P.Context.nccl_unique_id(), rank=0, nranks=1)
    nccl.set_reduction("ordered")
    Y1 = P.FilterApplier(A, rule, ctx=nccl).apply(X)
    assert np.array_equal(Y0, Y1)
