"""Process-group plumbing around the C ABI's NCCL communicator.

One process per GPU.  torch.distributed (any backend) only carries the
128-byte NCCL unique id from rank 0 to the others; all data-path collectives
run inside libpsb.so on its own communicator.
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def broadcast_unique_id(make_uid, group=None) -> bytes:
    """Rank 0 calls make_uid() (psb_comm_unique_id) and every rank returns it."""
    import torch.distributed as dist
    obj: List[Optional[bytes]] = [make_uid() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(ctx, group=None) -> None:
    """psb_comm_init for this process' rank of the default process group."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    uid = broadcast_unique_id(type(ctx).unique_id, group) if world > 1 else None
    ctx.comm_init(rank, world, uid)


def worker_ids(rank: int, local_workers: int) -> range:
    """Global worker ids owned by `rank`: the reference's canonical worker
    order is preserved across ranks (worker id = rank * W + w)."""
    return range(rank * local_workers, (rank + 1) * local_workers)


def q8_shards(n: int, block: int, world: int) -> List[Tuple[int, int]]:
    """Block-shards of the dense 8-bit all-reduce (psb_ctx.cu:q8_step): rank q
    reduces blocks [q*nbs, min((q+1)*nbs, nb)) with nbs = ceil(nb / world)."""
    nb = (n + block - 1) // block
    nbs = (nb + world - 1) // world
    return [(q * nbs, min((q + 1) * nbs, nb)) for q in range(world)]
