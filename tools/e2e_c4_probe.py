"""Breakdown of bench.py's e2e leg on C4: CNF upload/build, engine prepare, run, read-back."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_2603_28796_b200 import galois as G
W = sys.argv[1] if len(sys.argv) > 1 else "C4"
inst = bench.make_instance(W)
B = bench.WORKLOADS[W]["batch"]
off = np.ascontiguousarray(inst.offsets, dtype=np.int64)
lits = np.ascontiguousarray(inst.lits, dtype=np.int32)
torch.cuda.set_device(0)
hold = G.Engine(G.Cnf(inst.n, off, lits), B, 10, 0.5, 1, cubes=inst.pins)   # like bench: its engine is alive
hold.enqueue(2)
for rep in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cnf = G.Cnf(inst.n, off, lits); torch.cuda.synchronize(); t1 = time.perf_counter()
    eng = G.Engine(cnf, B, 100, 0.5, 0, cubes=inst.pins, lanes=bench.default_lanes(B))
    eng.info(); torch.cuda.synchronize(); t2 = time.perf_counter()
    eng.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
    eng.unsat_counts(); eng.best_assignment(); torch.cuda.synchronize(); t4 = time.perf_counter()
    eng.free(); cnf.free()
    print(f"{W} rep {rep}: load {1e3*(t1-t0):.1f} prepare {1e3*(t2-t1):.1f} run {1e3*(t3-t2):.1f} "
          f"read {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f} ms", flush=True)
