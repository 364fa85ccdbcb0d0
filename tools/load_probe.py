"""Where the sporadic e2e stalls come from: CNF load alone, then load + engine create/free
cycles (C4), host wall per call bracketed by device syncs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2603_28796_b200 import galois as G
inst = bench.make_instance("C4")
torch.cuda.set_device(0)
off = torch.from_numpy(np.ascontiguousarray(inst.offsets, dtype=np.int64)).pin_memory().numpy()
lits = torch.from_numpy(np.ascontiguousarray(inst.lits, dtype=np.int32)).pin_memory().numpy()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - a)
out = []
for rep in range(10):
    cnf, tl = t(lambda: G.Cnf(inst.n, off, lits))
    _, tf = t(lambda: cnf.free())
    out.append(f"{tl:.1f}/{tf:.1f}")
print("load/free alone:", " ".join(out), flush=True)
out = []
for rep in range(10):
    cnf, tl = t(lambda: G.Cnf(inst.n, off, lits))
    eng, tc = t(lambda: (lambda e: (e.info(), e)[1])(G.Engine(cnf, 1024, 100, 0.5, 0)))
    _, tr = t(lambda: eng.enqueue(3))
    _, tf = t(lambda: (eng.free(), cnf.free()))
    out.append(f"{tl:.1f}/{tc:.1f}/{tr:.1f}/{tf:.1f}")
print("load/create/3 steps/free:", " ".join(out), flush=True)
