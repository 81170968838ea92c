mkdir -p gpurun_out
python paper_1105_4204_b200/build.py > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in 2 3 4; do timeout 300 python scripts/sweep_options.py $c > gpurun_out/sweep44_$c.log 2>&1; echo sweep$c rc=$?; done
