#!/usr/bin/env bash
# round-2 session C: full gpu tests, racecheck of the TMA rings, A/B vs HEAD, ncu of the C4 update
set -u
TAG=${1:-r02e}
PARTS=${2:-"tests race ab ncu4"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
has() { [[ " $PARTS " == *" $1 "* ]]; }
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
if has tests; then
    timeout 2400 python -m pytest tests -m gpu -q -x -rf --durations=10 > "$OUT/pytest_gpu.log" 2>&1
    tail -15 "$OUT/pytest_gpu.log"
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; tail -2 "$OUT/smoke.log"
fi
if has race; then
    for part in tma loop lanes window; do
        timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize.py $part > "$OUT/san_racecheck_$part.log" 2>&1
        echo "racecheck $part rc=$? $(grep 'RACECHECK SUMMARY' $OUT/san_racecheck_$part.log | tail -1)"
    done
fi
if has ab; then
    bash tools/ab.sh paper_2603_28796_b200/libgalois.so tools/ab/lib_head.so -- C4 C2 C5 C3a 2>&1 | tee "$OUT/ab.txt"
fi
if has ncu4; then
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_update_tma|k_sweep" -s 6 -c 2 \
        -o "$OUT/full_C4" python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-tts > "$OUT/full_C4.log" 2>&1
    echo "ncu full C4 rc=$?"
fi
