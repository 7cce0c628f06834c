"""Every shard of a G-GPU filter job on the one GPU this tier has
(fl_ctx_create_virtual: rank r of G for the node sharding, no communicator).
Rank r's context factors and solves exactly the contour nodes
fl_node_shard(n_c, r, G) gives it and returns their ascending partial sum,
which is what a rank of a real NCCL clique holds just before its all-reduce
(capi.cu filter_apply_dev). The shard sums must add up to the oracle's filter
(SURVEY.md §8(e)), each shard must be bitwise the one-rank filter of the
sub-rule it owns, and the accounting must count only local work."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _A(n, seed):
    lay = O.SpectrumLayout(n, O.SearchInterval(-0.4, 0.4), 20, O.SearchInterval(0.8, 5.0), n - 20,
                           seed=seed)
    return O.assemble_matrix(*O.generate_spectrum(lay))


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("cache", [False, True])
def test_virtual_shards_sum_to_the_filter(G, cache):
    import paper_1605_08771_b200 as P
    from paper_1605_08771_b200 import dist as D
    n, p, nc = 520, 40, 16
    A = _A(n, 31)
    X = O.random_block(n, p, 32)
    I = P.SearchInterval(-0.45, 0.45)
    rule = P.build_contour_rule(I, nc)
    zr, zi, wr, wi = rule.parts()
    parts, facts = [], 0
    for r in range(G):
        ctx = P.Context(0, rank=r, nranks=G, virtual=True)
        acc = P.SolveAccounting()
        f = P.FilterApplier(A, rule, cache, ctx=ctx)
        Yr = f.apply(X, acc)
        f.apply(X, acc)  # a second application: replayed graph / cached factors
        kb, ke = D.node_shard(nc, r, G)
        assert acc.rhs_solved == 2 * nc * p  # the reference's per-application count
        facts += acc.factorizations
        # the shard is exactly the one-rank filter of the sub-rule it owns
        sub = P.contour_rule_from_nodes(I, list(zr[kb:ke] + 1j * zi[kb:ke]),
                                        list(wr[kb:ke] + 1j * wi[kb:ke]))
        Ysub = P.FilterApplier(A, sub, ctx=P.Context(0)).apply(X)
        assert np.array_equal(Yr, Ysub), (G, r)
        parts.append(Yr)
        del f
    # non-cached: every rank counts the whole rule per application, as every
    # rank of a clique does; cached: each node's factorization once, summed
    # over the shards (the clique all-reduces this count)
    assert facts == (nc if cache else 2 * nc * G)
    Y = np.zeros_like(parts[0])
    for Yr in parts:  # the all-reduce's sum (rank order)
        Y = Y + Yr
    ref = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.45, 0.45), nc), X)
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-12


def test_virtual_rank_owns_no_nodes_when_G_exceeds_nc():
    import paper_1605_08771_b200 as P
    from paper_1605_08771_b200 import dist as D
    n, p, nc, G = 130, 6, 4, 8
    A = _A(n, 41)
    X = O.random_block(n, p, 42)
    rule = P.build_contour_rule(P.SearchInterval(-0.3, 0.3), nc)
    Y = np.zeros((n, p))
    empty = 0
    for r in range(G):
        kb, ke = D.node_shard(nc, r, G)
        Yr = P.FilterApplier(A, rule, ctx=P.Context(0, rank=r, nranks=G, virtual=True)).apply(X)
        if ke == kb:
            empty += 1
            assert not Yr.any()  # a rank without nodes contributes zeros
        Y = Y + Yr
    assert empty == G - nc
    ref = O.apply_filter(A, O.build_contour_rule(O.SearchInterval(-0.3, 0.3), nc), X)
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-12
