"""Per-step clause-unsat density of the sample (Lambda / m) and of the rounding (unsat / m)
for a bench workload — what the sweep's per-member counters see.

    python tools/density.py C4 [steps]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_28796_b200 import galois as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
inst = bench.make_instance(name)
batch = bench.WORKLOADS[name]["batch"]
cnf = G.Cnf.from_instance(inst)
eng = G.Engine(cnf, batch, steps, 0.5, 0)
for t in range(1, steps + 1):
    rc = eng.step()
    if t in (1, 2, 5, 10, 20, 50, 100) or rc != G.OK:
        lam = eng.get_loss()
        u, _ = eng.unsat_counts()
        print(f"t={t} lambda/m mean {lam.mean() / inst.m:.4%} max {lam.max() / inst.m:.4%}  "
              f"unsat/m mean {u.mean() / inst.m:.4%} min {u.min()}", flush=True)
    if rc != G.OK:
        break
