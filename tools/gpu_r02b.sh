#!/usr/bin/env bash
# round-2 session B: sweep A/B, sanitizer, ncu captures of C3a/C3b/C5 (usage: bash tools/gpu_r02b.sh <tag> "<parts>")
set -u
TAG=${1:-r02d}
PARTS=${2:-"ab sanitize ncu3"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
has() { [[ " $PARTS " == *" $1 "* ]]; }
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
if has ab; then
    bash tools/ab.sh paper_2603_28796_b200/libgalois.so tools/ab/lib_nohint.so tools/ab/lib_tmaloop.so tools/ab/lib_tmaall.so -- C4 C5 C2 2>&1 | tee "$OUT/ab.txt"
fi
if has sanitize; then
    for tool in memcheck racecheck synccheck; do
        for part in small tma lanes loop v4 soft select tseitin window; do
            timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py $part > "$OUT/san_${tool}_$part.log" 2>&1
            echo "sanitize $tool $part rc=$? $(grep 'ERROR SUMMARY' $OUT/san_${tool}_$part.log | tail -1)"
        done
    done 2>&1 | tee "$OUT/sanitize_summary.txt"
fi
if has ncu3; then
    for W in C3a C3b C5; do
        timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_sweep|k_update_tma|k_hub_partial_tma" -s 6 -c 3 \
            -o "$OUT/full_$W" python bench.py --workload $W --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --no-tts \
            > "$OUT/full_$W.log" 2>&1
        echo "ncu full $W rc=$?"
    done
fi
