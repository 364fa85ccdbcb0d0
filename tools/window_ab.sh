#!/usr/bin/env bash
# bash tools/window_ab.sh <out> lib1 lib2 ...: tools/window_probe.py per library variant (raw lines)
out=$1; shift; mkdir -p gpurun_out/$out
for L in "$@"; do GALOIS_LIB=$L timeout 300 python tools/window_probe.py > gpurun_out/$out/$(basename $L .so).txt 2>&1; done
