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
    """One rank of the exchange protocol of galois.h set_comm / engine.cu, on CPU: the rank's
    slice is stepped by the fp64 oracle; at every check the rank keeps its own record (strictly
    smaller count, bits extracted then), the 8-byte key (u << 32 | b) of the check is MIN
    all-reduced, the global record follows k_gfinalize's rule, and a global count of 0 stops
    every rank; the winner's bits are broadcast from the owner's own record."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) the 128-byte id reaches every rank unchanged
        blob = bytes(np.random.default_rng(123).integers(0, 256, 128, dtype=np.uint8))
        nid = D.share_nccl_id(lambda: blob, rank)
        results = []
        for (n, m, seed, B, T, K) in CASES:
            inst = I.random_ksat(n, m, 3, seed)
            f = O.Cnf(inst.n, inst.offsets, inst.lits)
            cfg = O.Config(seed=seed)
            b0, nb, per = D.batch_slice(B, world, rank)
            st = O.State.init(inst.n, b0, max(nb, 1), seed)
            local = (1 << 62, -1, -1)                 # this rank's record (u, t, b)
            local_bits = np.zeros(inst.n, np.uint8)
            g = (1 << 62, -1, -1)                     # the global record (k_gfinalize)
            r, u = O.round_and_check(f, cfg, st)
            t = 0
            while True:
                if t == 0 or t % K == 0 or t == T:
                    key = D.NO_MEMBER_KEY
                    if nb:
                        i = int(np.argmin(u[:nb]))
                        key = D.best_key(int(u[i]), b0 + i)
                        if u[i] < local[0]:
                            local = (int(u[i]), t, b0 + i)
                            local_bits = r[i].copy()
                    kt = torch.tensor([key - (1 << 63)], dtype=torch.int64)   # uint64 order in int64
                    dist.all_reduce(kt, op=dist.ReduceOp.MIN)
                    gu, gb = D.decode_key(int(kt.item()) + (1 << 63))
                    if gu < g[0]:
                        g = (gu, t, gb)
                    if g[0] == 0:
                        break
                if t == T:
                    break
                t += 1
                out_ = O.step(f, cfg, st)
                r, u = out_["r"], out_["unsat"]
            owner = g[2] // per
            bits = torch.from_numpy(local_bits.astype(np.int64))
            dist.broadcast(bits, src=owner)
            if rank == owner:
                assert local == g, (local, g)          # the owner's own record is the global one
            results.append((g, bits.numpy().astype(np.uint8).tobytes()))
        out[rank] = (nid == blob, results)
    finally:
        dist.destroy_process_group()


# (n, m, seed, B, T, K): a SAT stop, a budget run, a check interval, a short last rank
CASES = [(30, 128, 4, 80, 12, 1), (40, 176, 6, 96, 10, 1), (40, 176, 7, 70, 9, 4)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_best_equals_single_process(world):
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for ci, (n, m, seed, B, T, K) in enumerate(CASES):
        inst = I.random_ksat(n, m, 3, seed)
        f = O.Cnf(inst.n, inst.offsets, inst.lits)
        full = O.run(f, O.Config(seed=seed), 0, B, T, K)
        for r in range(world):
            ok, results = out[r]
            assert ok
            g, bits = results[ci]
            assert g == (full["best_unsat"], full["best_t"], full["best_b"])
            assert bits == full["best_r"].tobytes()
