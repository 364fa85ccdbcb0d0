"""Phase breakdown of bench.py's e2e path (CNF upload/build, create+init+run, read-back)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_28796_b200 import galois as G  # noqa: E402

W = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = bench.make_instance(W)
B = bench.WORKLOADS[W]["batch"]
off = np.ascontiguousarray(inst.offsets, dtype=np.int64)
lits = np.ascontiguousarray(inst.lits, dtype=np.int32)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cnf = G.Cnf(inst.n, off, lits)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng = G.Engine(cnf, B, 100, 0.5, 0, cubes=inst.pins)
    eng.info()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng.run()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    counts, _ = eng.unsat_counts()
    best = eng.best_assignment()
    t4 = time.perf_counter()
    eng.free()
    cnf.free()
    print(f"{W} rep {rep}: load {1e3*(t1-t0):.2f} ms, create+init {1e3*(t2-t1):.2f} ms, run {1e3*(t3-t2):.2f} ms, "
          f"read {1e3*(t4-t3):.2f} ms")
