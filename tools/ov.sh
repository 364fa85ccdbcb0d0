python -m paper_2603_28796_b200.build > /dev/null
for L in paper_2603_28796_b200/libgalois.so tools/ab/lib_c3.so tools/ab/lib_c2.so; do
  for W in C2 C3a C5; do GALOIS_LIB=$L timeout 300 python tools/overlap_probe.py $W 2>&1 | grep -v Warn; done
done
