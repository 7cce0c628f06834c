"""Multi-GPU plumbing: one process per GPU (torchrun), torch.distributed for the
rendezvous only; the data-path collective (all-reduce of the filter sum) is
NCCL inside libfeastlab_b200.so (fl_ctx_create_nccl)."""
from __future__ import annotations

import ctypes as C
import os

from . import _lib as L


def env_ranks():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def node_shard(n_c: int, rank: int, nranks: int):
    """Contour nodes [k_begin, k_end) of `rank` (fl_node_shard)."""
    kb, ke = C.c_int(), C.c_int()
    st = L.lib().fl_node_shard(n_c, rank, nranks, C.byref(kb), C.byref(ke))
    if st != L.FL_OK:
        raise ValueError(f"bad shard request n_c={n_c} rank={rank} nranks={nranks}")
    return kb.value, ke.value


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast a small byte string (the 128-byte ncclUniqueId) from `src`."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8)
    if dist.get_rank() == src:
        t[:] = torch.tensor(list(payload), dtype=torch.uint8)
    dist.broadcast(t, src)
    return bytes(t.tolist())


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rendezvous_nccl_id(rank: int) -> bytes:
    """Rank 0 makes the ncclUniqueId (fl_nccl_unique_id); every rank receives it
    over the torch.distributed rendezvous group."""
    from .feastlab import Context
    uid = Context.nccl_unique_id() if rank == 0 else None
    return broadcast_bytes(uid, 128, 0)


def make_context(rank: int, world: int, local_rank: int):
    """fl_ctx for this rank: NCCL clique over all ranks when world > 1."""
    from .feastlab import Context
    if world == 1:
        return Context(local_rank)
    uid = rendezvous_nccl_id(rank)
    return Context(local_rank, nccl_id=uid, rank=rank, nranks=world)
