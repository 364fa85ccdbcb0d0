set -u
OUT=gpurun_out/p1; mkdir -p $OUT
python -m paper_2603_28796_b200.build > $OUT/build.log 2>&1 || exit 1
NCU=/usr/local/cuda/bin/ncu
for K in k_update_pair k_sweep; do
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
  -o $OUT/full_C4_$K python bench.py --workload C4 --steps 24 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --no-tts > $OUT/full_$K.log 2>&1
echo "$K rc=$?"
$NCU -i $OUT/full_C4_$K.ncu-rep --page source --csv --print-source sass > $OUT/src_$K.csv 2>&1
echo "src rc=$?"
done
