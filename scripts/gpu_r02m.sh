#!/bin/bash
# round 2 production evidence (final kernels): GPU suite (incl. the checked build), set_surfaces phases, bench, ncu
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02m
mkdir -p $O
timeout 3000 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
NM_CELL_VERBOSE=1 python scripts/cells_quick.py 5 > $O/set_surfaces_cfg5.txt 2>&1
python scripts/quick_time.py 2 5:2000000 > $O/quick_time.txt 2>&1
timeout 1800 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
rm -rf gpurun_out/ncu_r02
bash scripts/gpu_ncu_r02.sh > $O/ncu_script.log 2>&1
tail -3 $O/ncu_script.log
