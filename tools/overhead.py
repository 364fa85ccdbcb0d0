"""Host-side overheads of the public API on a tiny instance (C1 shape): create, prepare
(first call), steps, best_assignment, free."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2603_28796_b200 import galois as G, instances as I  # noqa: E402

inst = I.random_ksat(50, 213, 3, 0)
cnf = G.Cnf.from_instance(inst)
torch.cuda.synchronize()
for rep in range(4):
    t0 = time.perf_counter(); eng = G.Engine(cnf, 1024, 100, 0.5, 0); t1 = time.perf_counter()
    G.lib().galois_engine_info(eng.handle, None, None, None, None); torch.cuda.synchronize(); t2 = time.perf_counter()
    for _ in range(10):
        eng.step()
    t3 = time.perf_counter()
    eng.enqueue(20); torch.cuda.synchronize(); t4 = time.perf_counter()
    eng.best_assignment(); t5 = time.perf_counter()
    eng.free(); torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.3f} prepare {1e3*(t2-t1):.3f} step x10 {1e3*(t3-t2):.3f} "
          f"enqueue20 {1e3*(t4-t3):.3f} best {1e3*(t5-t4):.3f} free {1e3*(t6-t5):.3f} ms")
