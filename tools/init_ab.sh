# time k_init alone through the engine (profiling on): bash tools/init_ab.sh lib...
for L in "$@"; do GALOIS_LIB=$L python - <<'PY'
import os, numpy as np
from paper_2603_28796_b200 import galois as G, instances as I
import bench
for wl in ("C2", "C4"):
    inst = bench.make_instance(wl)
    cnf = G.Cnf.from_instance(inst)
    for rep in range(2):
        eng = G.Engine(cnf, bench.WORKLOADS[wl]["batch"], 1, 0.5, 0)
        eng.set_profiling(True)
        eng.info()
        kt = eng.kernel_times()
        eng.free()
    print(os.environ["GALOIS_LIB"], wl, "init ms", kt["init"])
PY
done
