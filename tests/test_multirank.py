"""N > 1 host path on CPU with gloo (world_size 2): node sharding, the
rendezvous helpers of bench.py, and the sharded filter sum (each rank's
ascending partial sum over its contiguous node shard, then a sum all-reduce)
reproducing the single-process filter. The CUDA/NCCL data path itself needs
GPUs (the round's GPU tier has one); its host logic is what runs here."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    """The product's host-side multi-rank logic on `world` CPU ranks: the NCCL
    id rendezvous of dist.make_context (fl_nccl_unique_id on rank 0, broadcast
    over gloo), the contour rule built by the product's host code (bitwise the
    same on every rank), the node shard of fl_node_shard, the max-over-ranks
    timing helper, and the loud failure of the data-path context without a GPU.
    Each rank's shard of the filter is computed by the oracle (the checker: the
    product's kernels need the B200) and the sum all-reduced, reproducing the
    single-process filter."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle as O
        import paper_1605_08771_b200 as P
        from paper_1605_08771_b200 import dist as D
        # NCCL id rendezvous (dist.make_context): identical 128 bytes on every rank
        uid = D.rendezvous_nccl_id(rank)
        ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(ids, torch.tensor(list(uid), dtype=torch.uint8))
        assert all(torch.equal(ids[0], t) for t in ids) and any(uid)
        assert D.max_over_ranks(float(rank + 1)) == float(world)
        # no GPU here: the multi-rank context must fail loudly, never fall back
        try:
            D.make_context(rank, world, 0)
            raise AssertionError("make_context succeeded without a GPU")
        except P.FeastCudaError:
            pass
        # the product's rule (host C++) is bitwise rank-invariant
        n, p, nc = 40, 3, 8
        rule = P.build_contour_rule(P.SearchInterval(-0.5, 0.5), nc)
        zr, zi, wr, wi = (np.ascontiguousarray(v) for v in rule.parts())
        mine = torch.from_numpy(np.concatenate([zr, zi, wr, wi]))
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        assert all(torch.equal(allr[0], t) for t in allr)
        # sharded filter: rank r sums its contiguous nodes in ascending order
        A = O.random_symmetric(n, 77) / np.sqrt(n)
        X = O.random_block(n, p, 78)
        orule = O.contour_rule_from_nodes(O.SearchInterval(-0.5, 0.5), list(zr + 1j * zi),
                                          list(wr + 1j * wi))
        kb, ke = D.node_shard(nc, rank, world)
        part = O.ContourRule(orule.interval, orule.nodes[kb:ke], orule.weights[kb:ke])
        Y = O.apply_filter(A, part, X) if ke > kb else np.zeros((n, p))
        t = torch.from_numpy(np.ascontiguousarray(Y))
        dist.all_reduce(t)
        if rank == 0:
            full = O.apply_filter(A, orule, X)
            out.put(("ok", float(np.linalg.norm(t.numpy() - full) / np.linalg.norm(full))))
    except BaseException as e:  # report to the parent
        out.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_node_shards_partition_the_rule():
    from paper_1605_08771_b200 import dist as D
    for nc in (1, 8, 16, 32, 5, 64):
        for world in (1, 2, 4, 8):
            covered = []
            for r in range(world):
                kb, ke = D.node_shard(nc, r, world)
                assert 0 <= kb <= ke <= nc
                covered.extend(range(kb, ke))
            assert covered == list(range(nc))
    with pytest.raises(ValueError):
        D.node_shard(8, 2, 2)


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_host_path_and_sharded_filter_sum_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
    status, val = q.get(timeout=10)
    assert status == "ok", val
    assert val <= 1e-13


def _ordered_worker(rank, world, port, out):
    """FL_REDUCE_ORDERED host logic (capi.cu filter_apply_dev): rank r writes
    its nodes' terms Re(w_k W_k) at slots r*Lmax + (k - kb), the slots are
    all-gathered, every rank sums the n_c terms in ascending global k."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle as O
        from paper_1605_08771_b200 import dist as D
        n, p, nc = 36, 4, 8
        A = O.random_symmetric(n, 91) / np.sqrt(n)
        X = O.random_block(n, p, 92)
        rule = O.build_contour_rule(O.SearchInterval(-0.4, 0.6), nc)
        z = np.asarray(rule.nodes)
        w = np.asarray(rule.weights)

        def term(k):  # Re(w W) as two rounded products and a rounded difference
            W = O.node_solve(A, z[k], X)
            return w[k].real * W.real - w[k].imag * W.imag

        Lmax = -(-nc // world)
        kb, ke = D.node_shard(nc, rank, world)
        local = np.zeros((Lmax, n, p))
        for k in range(kb, ke):
            local[k - kb] = term(k)
        gathered = [torch.zeros(Lmax, n, p, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(local))
        slots = {}
        for r in range(world):
            b0, b1 = D.node_shard(nc, r, world)
            for k in range(b0, b1):
                slots[k] = (r, k - b0)
        Y = np.zeros((n, p))
        for k in range(nc):  # ascending global order
            r, i = slots[k]
            Y = Y + gathered[r][i].numpy()
        single = np.zeros((n, p))
        for k in range(nc):
            single = single + term(k)
        if rank == 0:
            out.put(("ok", bool(np.array_equal(Y, single))))
    except Exception as e:
        out.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ordered_reduction_is_bitwise_rank_invariant_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ordered_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(180)
    status, val = q.get(timeout=10)
    assert status == "ok", val
    assert val is True
