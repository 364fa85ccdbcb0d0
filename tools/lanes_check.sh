#!/usr/bin/env bash
# lanes: GPU tests + bench A/B of the lane count
set -u
OUT=gpurun_out/${1:-lanes}
mkdir -p $OUT
python -m paper_2603_28796_b200.build > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_lanes.py -x -q > $OUT/pytest_lanes.log 2>&1; tail -15 $OUT/pytest_lanes.log
for W in C2 C3a C5; do for L in 1 2 4; do
  timeout 600 python bench.py --workload $W --lanes $L --no-cpu-baseline --no-e2e --no-tts > $OUT/b_${W}_$L.json 2> $OUT/b_${W}_$L.err
  python -c "import json,sys; d=json.loads(open('$OUT/b_${W}_$L.json').read().strip().splitlines()[-1]); print('$W lanes=$L', round(d['ms_per_step'],4), '%.3e'%d['value'], d['config']['lanes_per_gpu'], d['gpu_launches'], d['completed_all_steps'], round(d['roofline']['frac'],3))" || tail -3 $OUT/b_${W}_$L.err
done; done
