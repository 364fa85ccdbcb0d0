python -m paper_2603_28796_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/san3
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in smallw select window v4 tma; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py $part > gpurun_out/san3/san_${tool}_$part.log 2>&1
    echo "sanitize $tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san3/san_${tool}_$part.log | tail -1)"
  done
done 2>&1 | tee gpurun_out/san3/summary.txt
