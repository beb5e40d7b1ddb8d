#!/bin/bash
# round 2: batched fp64 fix-up + refinement oracle on the GPU + timing
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02e
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=20 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
python scripts/quick_time.py 2 5:2000000 3:2000000 > $O/quick_time.txt 2>&1
python scripts/cells_quick.py 5 > $O/cells_cfg5.txt 2>&1
python scripts/cells_quick.py 3 > $O/cells_cfg3.txt 2>&1
tail -25 $O/pytest_gpu.log; cat $O/quick_time.txt $O/cells_cfg5.txt $O/cells_cfg3.txt
