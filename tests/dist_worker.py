"""torchrun worker of tests/test_gpu_multi.py (one process per GPU, NCCL): the batch
sharded over the ranks with libgalois's exchange (galois.h set_comm) against a 1-GPU engine
of the same global batch on rank 0 and the fp64 oracle. Writes a JSON verdict per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2603_28796_b200 import dist as D  # noqa: E402
from paper_2603_28796_b200 import galois as G  # noqa: E402
from paper_2603_28796_b200 import instances as I  # noqa: E402

# (n, m, seed, B, T, K, sub_batch): a SAT stop (configs[0] shape), a budget run with
# unequal slices, a check interval, sub-batch windows in lock step
CASES = [(50, 213, 0, 1024, 100, 1, 0), (300, 1290, 5, 3000, 40, 1, 0), (300, 1290, 5, 4096, 30, 3, 0),
         (200, 852, 9, 2048, 20, 1, 512)]


def run_case(case, rank, world, local):
    n, m, seed, B, T, K, sub = case
    inst = I.random_ksat(n, m, 3, seed)
    cnf = G.Cnf.from_instance(inst)
    nid = D.share_nccl_id(G.galois_comm_unique_id, rank)
    eng = G.Engine(cnf, B, T, 0.5, seed, rank=rank, world=world, nccl_id=nid, check_interval=K, sub_batch=sub)
    rc = eng.run()
    best = eng.best_assignment()
    counts, b0 = eng.unsat_counts()
    info = eng.info()
    eng.free()
    # gather every rank's counts on rank 0 (member order)
    per = D.batch_slice(B, world, 0)[2]
    buf = torch.full((per,), -1, dtype=torch.int64, device=f"cuda:{local}")
    buf[:len(counts)] = torch.from_numpy(counts.astype(np.int64))
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, parts, dst=0)
    out = None
    if rank == 0:
        allc = torch.cat(parts).cpu().numpy()
        allc = allc[allc >= 0]
        ref = G.Engine(cnf, B, T, 0.5, seed, check_interval=K, sub_batch=sub)
        rrc = ref.run()
        rb = ref.best_assignment()
        rcounts, _ = ref.unsat_counts()
        rinfo = ref.info()
        ref.free()
        from oracle import oracle as O
        f = O.Cnf(inst.n, inst.offsets, inst.lits)
        orc = O.run(f, O.Config(seed=seed), 0, B, T, K)
        out = dict(
            case=list(case),
            rc=[rc, rrc],
            best=[[best["unsat"], best["step"], best["global_b"]], [rb["unsat"], rb["step"], rb["global_b"]]],
            oracle_best=[orc["best_unsat"], orc["best_t"], orc["best_b"]],
            bits_equal=bool((best["values"] == rb["values"]).all()),
            bits_reproduce=int(O.unsat_count(f, best["values"])) == best["unsat"],
            counts_equal=bool(len(allc) == len(rcounts) and (allc == rcounts).all()) if rc != G.SAT else None,
            steps=[info["steps_done"], rinfo["steps_done"]],
        )
    cnf.free()
    return out


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    results = [run_case(c, rank, world, local) for c in CASES]
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        with open(sys.argv[1], "w") as fh:
            json.dump(results, fh)


if __name__ == "__main__":
    main()
