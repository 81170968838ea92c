mkdir -p gpurun_out
python paper_1105_4204_b200/build.py > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for c in 2 3 4; do timeout 300 python scripts/sweep_options.py $c > gpurun_out/sweep43_$c.log 2>&1; echo sweep$c rc=$?; done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain43.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass1|pass2" -s 6 -c 2 -o gpurun_out/prof43_cfg2 -f $CMD > gpurun_out/ncu43.log 2>&1; echo full_rc=$?
