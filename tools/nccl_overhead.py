"""Per-step cost of the NCCL exchange on one GPU: the bench workload with a 1-rank NCCL
communicator (MIN all-reduce of the best key per check, per lane) against no communicator.
    python tools/nccl_overhead.py [W] [lanes]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_28796_b200 import galois as G  # noqa: E402

W = sys.argv[1] if len(sys.argv) > 1 else "C2"
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else bench.default_lanes(bench.WORKLOADS[W]["batch"])
inst = bench.make_instance(W)
B = bench.WORKLOADS[W]["batch"]
torch.cuda.set_device(0)
st = torch.cuda.Stream()
cnf = G.Cnf.from_instance(inst)
for K in (1, 10):
    for nccl in (False, True):
        eng = G.Engine(cnf, B, 215, 0.5, 0, cubes=inst.pins, stream=st.cuda_stream, lanes=lanes, check_interval=K,
                       nccl_id=G.galois_comm_unique_id() if nccl else None)
        eng.enqueue(5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        eng.enqueue(200)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{W} lanes={lanes} K={K} nccl={nccl}: {e0.elapsed_time(e1) / 200:.4f} ms/step", flush=True)
        eng.free()
