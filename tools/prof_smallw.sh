#!/usr/bin/env bash
# ncu --set full of the small-window kernels (f4 at P:559's scale), via tools/window_probe.py
set -u
OUT=gpurun_out/psw; mkdir -p $OUT
python -m paper_2603_28796_b200.build > $OUT/build.log 2>&1 || exit 1
NCU=/usr/local/cuda/bin/ncu
run() {   # name, kernel regex, env
  env $3 timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$2 -s 12 -c 1 \
      -o $OUT/$1 python tools/window_probe.py > $OUT/$1.log 2>&1
  echo "$1 rc=$?"
  $NCU -i $OUT/$1.ncu-rep --page raw --csv > $OUT/raw_$1.csv 2>&1
}
run upd_w1_norm k_update_smallw "WINDOW_NORM=1 WINDOW_SUBS=32"
run fwd_w1_norm k_clauses_st "WINDOW_NORM=1 WINDOW_SUBS=32"
run upd_w8 k_update_smallw "WINDOW_SUBS=256"
run fwd_w8 k_clauses_v4 "WINDOW_SUBS=256"
