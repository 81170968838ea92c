mkdir -p gpurun_out
python paper_1105_4204_b200/build.py > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python scripts/e2e_breakdown.py 2 > gpurun_out/e2e45.log 2>&1; echo e2e_rc=$?
timeout 300 python bench.py --cpu-budget 5 > gpurun_out/bench45.json 2> gpurun_out/bench45.err; echo bench_rc=$?
