#!/usr/bin/env bash
# Focused ncu --set full captures (one launch each, after `skip` matching launches):
#   gpurun -- 'bash tools/prof.sh <tag> <workload>:<kernel regex>:<skip> ...'
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -m paper_2603_28796_b200.build > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
for spec in "$@"; do
    IFS=: read -r W K S <<< "$spec"
    timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
        -o "$OUT/${W}_$K" python bench.py --workload $W --steps $((S + 4)) --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e \
        > "$OUT/${W}_$K.log" 2>&1
    echo "$spec rc=$?"
done
