#!/usr/bin/env bash
# A/B the per-kernel times of library variants: bash tools/ab.sh "<lib>[@ENV=V,...]" ... -- <workloads>
# e.g. bash tools/ab.sh tools/ab/lib_2_3.so tools/ab/lib_0_4.so@GALOIS_SWEEP_CTAS=4 -- C4 C2
set -u
libs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
shift
for W in "$@"; do
    for spec in "${libs[@]}"; do
        lib=${spec%%@*}
        envs=""
        [[ "$spec" == *@* ]] && envs=${spec#*@}
        out=$(env ${envs//,/ } GALOIS_LIB=$lib timeout 600 python bench.py --workload $W --no-cpu-baseline --no-e2e --no-tts 2>/dev/null | tail -1)
        echo "$W $spec: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v, 4) for k, v in d['kernels_ms_per_step'].items()})" 2>/dev/null | tail -1)"
    done
done
