# step time without per-kernel events (no profiling): bash tools/noprof_ab.sh lib... -- workloads
libs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done; shift
for W in "$@"; do for L in "${libs[@]}"; do GALOIS_LIB=$L W=$W python - <<'PY'
import os, torch
import bench
from paper_2603_28796_b200 import galois as G
W = os.environ["W"]; inst = bench.make_instance(W); B = bench.WORKLOADS[W]["batch"]
torch.cuda.set_device(0); st = torch.cuda.Stream(); torch.cuda.set_stream(st)
cnf = G.Cnf.from_instance(inst)
eng = G.Engine(cnf, B, 205, 0.5, 0, cubes=inst.pins, stream=st.cuda_stream)
eng.enqueue(5); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); eng.enqueue(200); e1.record(st); torch.cuda.synchronize()
print(os.environ["GALOIS_LIB"], W, "ms/step (no per-kernel events)", round(e0.elapsed_time(e1) / 200, 4))
PY
done; done
