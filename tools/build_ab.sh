#!/usr/bin/env bash
# Build variant libraries for A/B timing: bash tools/build_ab.sh name "<nvcc -D flags>" [name "<flags>"]...
set -eu
mkdir -p tools/ab
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  GALOIS_NVCC_EXTRA="$flags" GALOIS_OBJ_DIR=build/ab_$name GALOIS_LIB_OUT=tools/ab/lib_$name.so \
    python -m paper_2603_28796_b200.build > /dev/null &
done
wait
ls tools/ab
