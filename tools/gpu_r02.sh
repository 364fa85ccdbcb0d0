#!/usr/bin/env bash
# Round-2 GPU session: gpurun --timeout T -- 'bash tools/gpu_r02.sh <tag> "<parts>"'
# parts: tests newtests smoke bench benchall sanitize launches full
set -u
TAG=${1:-r02}
PARTS=${2:-"tests smoke bench"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
python -m paper_2603_28796_b200.build > "$OUT/build.log" 2>&1 || { tail -30 "$OUT/build.log"; exit 1; }
has() { [[ " $PARTS " == *" $1 "* ]]; }
CS=/usr/local/cuda/bin/compute-sanitizer
NCU=/usr/local/cuda/bin/ncu
if has newtests; then
    timeout 1500 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_variants.py tests/test_gpu_edges.py tests/test_gpu_lanes.py -m gpu -q -x -rA --durations=15 > "$OUT/pytest_new.log" 2>&1
    tail -25 "$OUT/pytest_new.log"
fi
if has tests; then
    timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 > "$OUT/pytest_gpu.log" 2>&1
    tail -30 "$OUT/pytest_gpu.log"
fi
if has smoke; then
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
    tail -2 "$OUT/smoke.log"
fi
if has bench; then
    timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
    tail -c 1500 "$OUT/bench.json"; echo
fi
if has benchall; then
    for W in C2 C1 C3a C3b C5; do
        timeout 600 python bench.py --workload $W --no-cpu-baseline > "$OUT/bench_$W.json" 2> "$OUT/bench_$W.err"
        tail -c 300 "$OUT/bench_$W.json"; echo
    done
fi
if has sanitize; then
    for tool in memcheck racecheck synccheck; do
        for part in small tma lanes loop v4 soft select tseitin window; do
            timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py $part > "$OUT/san_${tool}_$part.log" 2>&1
            echo "sanitize $tool $part rc=$? $(grep -c 'ERROR SUMMARY' $OUT/san_${tool}_$part.log) $(grep 'ERROR SUMMARY' $OUT/san_${tool}_$part.log | tail -1)"
        done
    done
fi
if has launches; then
    timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches_C4.csv" python bench.py --steps 4 --warmup 3 \
        --no-cpu-baseline --no-e2e --no-tts > "$OUT/launches_C4.log" 2>&1
    echo "launches rc=$?"
fi
if has full; then
    for K in k_sweep k_update_tma k_hub_partial_tma; do
        timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 \
            -o "$OUT/full_C4_$K" python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-tts \
            > "$OUT/full_C4_$K.log" 2>&1
        echo "full $K rc=$?"
    done
fi
