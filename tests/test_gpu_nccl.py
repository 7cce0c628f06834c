"""The NCCL data path on the one GPU this tier has: a clique of one rank runs
ncclCommInitRank and the in-library ncclAllReduce of the filter sum (and of
the cached-factorisation count); results must equal the collective-free path
bit for bit (an all-reduce over one rank is a copy)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cache", [False, True])
def test_single_rank_nccl_clique_matches(cache):
    import paper_1605_08771_b200 as P
    n, p = 300, 20
    A = O.random_symmetric(n, 5) / np.sqrt(n)
    X = O.random_block(n, p, 6)
    rule = P.build_contour_rule(P.SearchInterval(-0.4, 0.3), 8)
    plain = P.Context(0)
    nccl = P.Context(0, nccl_id=P.Context.nccl_unique_id(), rank=0, nranks=1)
    accs = []
    outs = []
    for ctx in (plain, nccl):
        f = P.FilterApplier(A, rule, cache, ctx=ctx)
        acc = P.SolveAccounting()
        outs.append([f.apply(X, acc) for _ in range(2)])
        accs.append((acc.rhs_solved, acc.factorizations))
    assert accs[0] == accs[1] == (2 * 8 * p, 8 if cache else 16)
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    ref = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.4, 0.3), 8), X)
    assert np.linalg.norm(outs[1][0] - ref) / np.linalg.norm(ref) <= 1e-12


def test_ordered_reduction_single_rank_is_bitwise_plain():
    """FL_REDUCE_ORDERED (node terms -> ncclAllGather -> ascending-k sum) on a
    one-rank clique reproduces the collective-free accumulate bit for bit:
    the same per-node rounding and the same association."""
    import paper_1605_08771_b200 as P
    n, p = 260, 24
    A = O.random_symmetric(n, 15) / np.sqrt(n)
    X = O.random_block(n, p, 16)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.4), 8)
    plain = P.Context(0)
    nccl = P.Context(0, nccl_id=P.Context.nccl_unique_id(), rank=0, nranks=1)
    nccl.set_reduction("ordered")
    Y0 = P.FilterApplier(A, rule, ctx=plain).apply(X)
    f = P.FilterApplier(A, rule, ctx=nccl)
    Ys = [f.apply(X) for _ in range(3)]  # eager, captured, replayed
    for Y in Ys:
        assert np.array_equal(Y, Y0)
    with pytest.raises(P.InvalidArgument):
        nccl.set_reduction("median")
