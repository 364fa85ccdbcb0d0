"""N > 1 host logic on CPU with gloo, world size 2 (-m "not gpu"): the batch slices of
galois.h, the 128-byte id bootstrap, and that sharding the batch over ranks and MIN-
reducing the best key reproduces the single-process best exactly (members are
independent and their RNG counters are global; the per-rank engine is stood in for by
the fp64 oracle run on that rank's slice)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2603_28796_b200 import dist as D
from paper_2603_28796_b200 import instances as I


def test_batch_slices_cover_the_batch():
    for B in (1, 31, 32, 33, 100, 1000, 3000, 4096, 65536):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b0, nb, per = D.batch_slice(B, world, r)
                assert per % 32 == 0 and b0 % 32 == 0
                seen.extend(range(b0, b0 + nb))
            assert seen == list(range(B))
            for b in (0, B - 1):
                r = D.owner_rank(b, B, world)
                b0, nb, _ = D.batch_slice(B, world, r)
                assert b0 <= b < b0 + nb


def test_key_order_is_lexicographic():
    keys = [D.best_key(u, b) for u, b in [(3, 7), (2, 9), (2, 4), (5, 0)]]
    assert D.decode_key(min(keys)) == (2, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) the 128-byte id reaches every rank unchanged
        blob = bytes(np.random.default_rng(123).integers(0, 256, 128, dtype=np.uint8))
        nid = D.share_nccl_id(lambda: blob, rank)
        # 2) sharded run + MIN all-reduce of the key
        inst = I.random_ksat(30, 128, 3, 4)
        f = O.Cnf(inst.n, inst.offsets, inst.lits)
        B, T = 80, 12
        b0, nb, _ = D.batch_slice(B, world, rank)
        res = O.run(f, O.Config(seed=5), b0, nb, T, 1) if nb else None
        key = D.best_key(res["best_unsat"], res["best_b"]) if nb else D.NO_MEMBER_KEY
        # (u, t, b) lexicographic: reduce (u, t) first via a packed key, then b
        ut = torch.tensor([(res["best_unsat"] << 20 | res["best_t"]) if nb else (1 << 62)], dtype=torch.int64)
        dist.all_reduce(ut, op=dist.ReduceOp.MIN)
        cand = torch.tensor([res["best_b"] if nb and (res["best_unsat"] << 20 | res["best_t"]) == ut.item()
                             else (1 << 62)], dtype=torch.int64)
        dist.all_reduce(cand, op=dist.ReduceOp.MIN)
        out[rank] = (nid == blob, int(ut.item()) >> 20, int(ut.item()) & ((1 << 20) - 1), int(cand.item()), key)
    finally:
        dist.destroy_process_group()


def test_sharded_best_equals_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    inst = I.random_ksat(30, 128, 3, 4)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    full = O.run(f, O.Config(seed=5), 0, 80, 12, 1)
    for r in range(world):
        ok, u, t, b, _ = out[r]
        assert ok
        assert (u, t, b) == (full["best_unsat"], full["best_t"], full["best_b"])
