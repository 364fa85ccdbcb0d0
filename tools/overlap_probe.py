"""Probe: does splitting the batch into independent lanes on separate streams overlap
the sweep of one lane with the update of another?  python tools/overlap_probe.py W"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_28796_b200 import galois as G

W = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = bench.make_instance(W)
B = bench.WORKLOADS[W]["batch"]
torch.cuda.set_device(0)
cnf = G.Cnf.from_instance(inst)
K = 100
for lanes in (1, 2, 4):
    if B // lanes < 1024:
        continue
    sts = [torch.cuda.Stream() for _ in range(lanes)]
    engs = [G.Engine(cnf, B // lanes, K + 10, 0.5, i, cubes=inst.pins, stream=s.cuda_stream) for i, s in enumerate(sts)]
    for e in engs:
        e.enqueue(5)
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in sts]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in sts]
    for e, s in zip(ev0, sts):
        e.record(s)
    for k in range(K):
        for e in engs:
            e.enqueue(1)
    for e, s in zip(ev1, sts):
        e.record(s)
    torch.cuda.synchronize()
    t = max(ev0[0].elapsed_time(e) for e in ev1)
    print(f"{os.environ.get('GALOIS_LIB', 'default')} {W} lanes={lanes} ms/step {t / K:.4f}", flush=True)
    for e in engs:
        e.free()
