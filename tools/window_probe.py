import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, json, sys, torch
from paper_2603_28796_b200 import galois as G, instances as I
inst = I.CONFIGS["C4"][0]()
dev = torch.device("cuda:0")
cnf = G.Cnf.from_instance(inst)
if os.environ.get("WINDOW_NORM"):
    cnf = cnf.normalize(3)
print("bytes/member", cnf.bytes_per_member(), flush=True)
for sub in [int(x) for x in os.environ.get('WINDOW_SUBS', '1024,512,256,128,64,32').split(',')]:
    for rep in range(3):
        eng = G.Engine(cnf, 3072 if sub >= 256 else 1024, 10, 0.5, 0, sub_batch=sub)
        if rep == 2: eng.set_profiling(True)
        torch.cuda.synchronize(dev); t0 = time.perf_counter()
        eng.run(); torch.cuda.synchronize(dev); dt = time.perf_counter() - t0
        B = 3072 if sub >= 256 else 1024
        if rep == 2: print(json.dumps({k: v for k, v in eng.kernel_times().items() if v[1]}), flush=True)
        if rep == 1: print(json.dumps({"sub": sub, "B": B, "s": dt, "ms_per_member_step": dt * 1e3 / (B * 10),
                                  "levals": inst.L * B * 10 / dt, "best": eng.best_assignment()["unsat"]}), flush=True)
        eng.free()
