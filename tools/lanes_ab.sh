#!/usr/bin/env bash
# bash tools/lanes_ab.sh "<libs>" "<lanes>" <workloads...>: ms/step of each (lib, lanes)
libs=$1; lanes=$2; shift 2
for W in "$@"; do for L in $libs; do for n in $lanes; do
  out=$(GALOIS_LIB=$L timeout 600 python bench.py --workload $W --lanes $n --no-cpu-baseline --no-e2e --no-tts 2>/dev/null | tail -1)
  echo "$W $L lanes=$n: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v, 4) for k, v in d['kernels_ms_per_step'].items()})" 2>/dev/null)"
done; done; done
