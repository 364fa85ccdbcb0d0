python -m paper_2603_28796_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
bash tools/ab.sh ${LIB_A:-tools/ab/lib_noucf.so} paper_2603_28796_b200/libgalois.so -- ${WLS:-C3a C2}
