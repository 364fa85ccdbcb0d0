"""Drive every kernel of libgalois once on small shapes, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py [part ...]

parts: small (k_small_run, cooperative grid barrier: C1 through run()), tma (the
TMA-pipelined updates k_update_pair / k_update_tma, sweep, hub partials, k_extract), lanes (2 lanes on
their own streams, CUDA graph chunks), loop (k_sweep<kLoop>), v4 (b_pad < 1024 sweep and
k_update_st), soft (SOFT mode), select (theta_sel / pool / top-|S| / cube variables),
tseitin (device normalisation), window (f4 sub-batching), smallw (sub-1024 windows: k_update_smallw,
the fused scalar sweep, k_init's row packing, the units-only pool with a global-memory sort). Default: all.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2603_28796_b200 import galois as G  # noqa: E402
from paper_2603_28796_b200 import instances as I  # noqa: E402


def hub_instance(n=3000, m=9000, seed=5):
    """3-SAT with two hub variables (degree > 256) so the hub partial kernel runs."""
    inst = I.random_ksat(n, m, 3, seed)
    lits = inst.lits.copy()
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(lits), 1200, replace=False)
    lits[idx[:600]] = np.where(lits[idx[:600]] > 0, 1, -1) * 7
    lits[idx[600:]] = np.where(lits[idx[600:]] > 0, 1, -1) * 11
    # keep variables distinct within a clause: duplicates are legal (kept verbatim) anyway
    return I.Instance("hub", n, inst.offsets, lits)


def part_small():
    inst = I.random_ksat(50, 213, 3, 0)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 1024, 60, 0.5, 0)
    e.run()
    e.best_assignment()
    e.unsat_counts()
    e.free()
    cnf.free()


def part_tma():
    inst = hub_instance()
    cnf = G.Cnf.from_instance(inst)
    for K in (1, 3):
        e = G.Engine(cnf, 2048, 6, 0.5, 1, check_interval=K)
        e.enqueue(6)
        e.best_assignment()
        e.unsat_counts()
        e.free()
    e = G.Engine(cnf, 2048, 3, 0.5, 1, debug=True)
    e.step()
    e.get_grad()
    e.free()
    cnf.free()
    # k_update_pair with adjacent rows (B = 1024), an odd n (a lone last variable), hubs and
    # pairs that go variable by variable
    inst = I.industrial(2501, 30_000, 21, occ_exp=0.9)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 1024, 3, 0.5, 2)
    e.enqueue(3)
    e.best_assignment()
    e.free()
    cnf.free()


def part_lanes():
    inst = I.random_ksat(400, 1700, 3, 2)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 4096, 40, 0.5, 3, lanes=2, graphs=1)
    e.run()
    e.best_assignment()
    e.unsat_counts()
    e.free()
    cnf.free()


def part_loop():
    # kLoop: the X/R slices of all chunks exceed the sweep's L2 budget -> chunk loop
    inst = I.random_ksat(100_000, 420_000, 3, 4)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 8192, 2, 0.5, 0)
    e.enqueue(2)
    e.best_assignment()
    e.free()
    cnf.free()


def part_v4():
    inst = hub_instance(1000, 4200, 6)
    cnf = G.Cnf.from_instance(inst)
    for B in (96, 512):
        e = G.Engine(cnf, B, 4, 0.5, 2)
        e.enqueue(4)
        e.best_assignment()
        e.free()
    cnf.free()


def part_soft():
    inst = I.random_ksat(200, 850, 3, 1)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 256, 3, 0.5, 0, mode=1, debug=True)
    e.step()
    e.get_grad()
    e.get_loss()
    e.free()
    cnf.free()


def part_select():
    inst = I.random_ksat(3000, 12000, 3, 3)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 2048, 4, 0.5, 0)
    e.run()
    s = e.select_member(0)
    e.candidate_pool(s["global_b"], 16, 0.01, 5)
    e.cube_variables(s["global_b"], 12)
    e.free()
    cnf.free()


def part_tseitin():
    inst = I.industrial(5000, 20000, 0)
    cnf = G.Cnf.from_instance(inst)
    c3 = cnf.normalize(3)
    c3.csr()
    e = G.Engine(c3, 1024, 2, 0.5, 0)
    e.run()
    e.free()
    c3.free()
    cnf.free()


def part_window():
    inst = I.random_ksat(500, 2100, 3, 7)
    cnf = G.Cnf.from_instance(inst)
    e = G.Engine(cnf, 3000, 5, 0.5, 0, sub_batch=1024)
    e.run()
    e.best_assignment()
    e.unsat_counts()
    e.free()
    cnf.free()


def part_smallw():
    # k_update_smallw for every power-of-two window (W = 1..16) on an odd n with hubs, the
    # fused scalar sweep (W = 1, 3), the small-window k_init mapping, and the units-only pool
    # with |S| > 4096 (global-memory sort) on a normalised CNF
    inst = I.industrial(2501, 30_000, 21, occ_exp=0.9)
    cnf = G.Cnf.from_instance(inst)
    for B in (32, 64, 96, 128, 256, 512):
        e = G.Engine(cnf, B, 3, 0.5, 1, cubes=(1, 2) if B == 64 else ())
        e.enqueue(3)
        e.best_assignment()
        e.free()
    e = G.Engine(cnf, 600, 4, 0.5, 0, sub_batch=64)
    e.run()
    e.best_assignment()
    e.free()
    cnf.free()
    inst = I.industrial(12_000, 48_000, 13)
    cnf0 = G.Cnf.from_instance(inst)
    cnf = cnf0.normalize(3)
    e = G.Engine(cnf, 64, 3, 0.5, 3)
    e.run()
    s = e.select_member(0)
    e.candidate_pool(s["global_b"], 3, 0.4, 9, arrays=False)
    e.free()
    cnf.free()
    cnf0.free()


PARTS = dict(small=part_small, tma=part_tma, lanes=part_lanes, loop=part_loop, v4=part_v4, soft=part_soft,
             select=part_select, tseitin=part_tseitin, window=part_window, smallw=part_smallw)

if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    for name in (sys.argv[1:] or list(PARTS)):
        PARTS[name]()
        print(f"part {name} ok", flush=True)
