#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02h
mkdir -p $O
./probes/staging > $O/probe_staging.txt 2>&1
cat $O/probe_staging.txt
timeout 2400 python -m pytest tests -x -q -m gpu --durations=8 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -14 $O/pytest_gpu.log
bash scripts/gpu_ncu_r02.sh > $O/ncu_script.log 2>&1
tail -20 $O/ncu_script.log
