#!/usr/bin/env bash
# One GPU session's evidence: tests, smoke, bench lines, launch list and ncu captures.
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh <tag> [parts]'
# parts (default all): tests bench launches full paper
set -u
TAG=${1:-r01}
PARTS=${2:-"tests bench launches full paper"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -m paper_2603_28796_b200.build > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
    timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1
    tail -3 "$OUT/pytest_gpu.log"
    timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$OUT/smoke.log" 2>&1
    tail -1 "$OUT/smoke.log"
fi
if has bench; then
    for W in C2 C1 C3a C3b C4 C5; do
        extra="--no-cpu-baseline"
        [ "$W" = C4 ] && extra=""
        timeout 600 python bench.py --workload $W $extra > "$OUT/bench_$W.json" 2> "$OUT/bench_$W.err"
        tail -c 400 "$OUT/bench_$W.json"; echo
    done
    timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
    tail -c 300 "$OUT/bench_reference.json"; echo
fi
NCU=/usr/local/cuda/bin/ncu
if has launches; then
    for W in C2 C4; do
        timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
            --log-file "$OUT/launches_$W.csv" python bench.py --workload $W --steps 4 --warmup 3 \
            --no-cpu-baseline --no-e2e --no-tts > "$OUT/launches_$W.log" 2>&1
        echo "launches $W rc=$?"
    done
fi
if has full; then
    for W in C2 C4; do
        for K in k_update_pair k_sweep k_hub_partial_tma; do
            timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
                -o "$OUT/full_${W}_$K" python bench.py --workload $W --steps 24 --warmup 3 --lanes 1 --no-cpu-baseline \
                --no-e2e > "$OUT/full_${W}_$K.log" 2>&1
            echo "full $W $K rc=$?"
        done
    done
fi
if has sanitize; then
    CS=/usr/local/cuda/bin/compute-sanitizer
    for tool in memcheck racecheck synccheck; do
        for part in small tma lanes loop v4 soft select tseitin window; do
            timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py $part > "$OUT/san_${tool}_$part.log" 2>&1
            echo "sanitize $tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/san_${tool}_$part.log | tail -1)"
        done
    done 2>&1 | tee "$OUT/sanitize_summary.txt"
fi
if has paper; then
    timeout 900 python bench.py --workload P4 > "$OUT/paper_P4.json" 2> "$OUT/paper_P4.err"
    tail -c 400 "$OUT/paper_P4.json"; echo
    timeout 1500 python bench.py --workload PL > "$OUT/paper_PL.json" 2> "$OUT/paper_PL.err"
    tail -c 600 "$OUT/paper_PL.json"; echo
    timeout 1800 python tools/pl_parity.py > "$OUT/pl_parity.json" 2> "$OUT/pl_parity.err"
    echo "pl_parity rc=$?"; tail -c 600 "$OUT/pl_parity.json"; echo
fi
