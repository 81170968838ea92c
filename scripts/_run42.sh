set -x
mkdir -p gpurun_out
SFU=$PWD/paper_1105_4204_b200/_lib/libtrigbf_b200_sfu.so
TRIGBF_B200_LIB=$SFU timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sfu.log 2>&1; echo pytest_sfu_rc=$?
TRIGBF_B200_LIB=$SFU timeout 300 python scripts/probe_parity.py > gpurun_out/probe_sfu.log 2>&1; echo probe_rc=$?
for c in 2 3 5 1; do
  for v in base sfu; do
    if [ $v = sfu ]; then export TRIGBF_B200_LIB=$SFU; else unset TRIGBF_B200_LIB; fi
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b42_${c}_$v.json 2> gpurun_out/b42_${c}_$v.err; echo cfg$c $v rc=$?
  done
done
