python -m paper_2603_28796_b200.build > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/t2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t2/pytest.log 2>&1; tail -5 gpurun_out/t2/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/t2/c2.json 2> gpurun_out/t2/c2.err; tail -c 600 gpurun_out/t2/c2.json
