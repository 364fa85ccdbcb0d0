"""Multi-GPU plumbing: one process per GPU, batch sharding, and the
bootstrap of the library's NCCL communicator through torch.distributed.

The batch members are independent problems ("each batch is independently and
randomly initialized"), so the only exchange is the MIN all-reduce of the best key
(u << 32 | global member) per check interval and the broadcast of the winner's bits,
both done inside libgalois over NCCL. This module only computes slices and moves the
128-byte ncclUniqueId from rank 0 to the other ranks (host logic, testable with gloo).
"""
from __future__ import annotations

from typing import Tuple

NO_MEMBER_KEY = (1 << 64) - 1


def batch_slice(batch: int, world: int, rank: int) -> Tuple[int, int, int]:
    """Members owned by `rank`: (first global member b0, local count, b_per) with
    b_per = roundup(ceil(B / world), 32) — the rule of galois.h / engine.cu."""
    per = -(-batch // world)
    per = -(-per // 32) * 32
    b0 = per * rank
    return b0, max(0, min(per, batch - b0)), per


def owner_rank(global_b: int, batch: int, world: int) -> int:
    return global_b // batch_slice(batch, world, 0)[2]


def best_key(unsat: int, global_b: int) -> int:
    """The all-reduced key: lexicographic (unsat, member) in one uint64."""
    return (int(unsat) << 32) | int(global_b)


def decode_key(key: int) -> Tuple[int, int]:
    return key >> 32, key & 0xFFFFFFFF


def share_nccl_id(make_id, rank: int, src: int = 0) -> bytes:
    """Rank `src` calls make_id() (galois_comm_unique_id) and every rank receives the
    128-byte id through torch.distributed (any backend)."""
    import torch.distributed as dist
    obj = [make_id() if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    nid = obj[0]
    assert isinstance(nid, (bytes, bytearray)) and len(nid) == 128
    return bytes(nid)


def engine_for_rank(cnf, batch: int, steps: int, lr: float = 0.5, seed: int = 0, **kw):
    """Create this rank's Engine (torch.distributed must be initialised; one GPU per
    process, torch.cuda.current_device() = LOCAL_RANK)."""
    import torch.distributed as dist
    from . import galois as G
    rank, world = dist.get_rank(), dist.get_world_size()
    nid = share_nccl_id(G.galois_comm_unique_id, rank) if world > 1 else None
    return G.Engine(cnf, batch, steps, lr, seed, rank=rank, world=world, nccl_id=nid, **kw)
