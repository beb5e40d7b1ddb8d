#!/bin/bash
# round 2: chunked fp64 fix-up, position-indexed k_label outputs, sidecar
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
python scripts/quick_time.py 2 5:2000000 3:2000000 > $O/quick_time.txt 2>&1
python scripts/cells_quick.py 5 > $O/cells_cfg5.txt 2>&1
tail -16 $O/pytest_gpu.log; cat $O/quick_time.txt $O/cells_cfg5.txt
