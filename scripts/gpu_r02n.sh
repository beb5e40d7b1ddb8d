#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02n
mkdir -p $O
timeout 3000 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
for c in 5 3; do NM_CELL_VERBOSE=1 python scripts/cells_quick.py $c > $O/set_surfaces_cfg$c.txt 2>&1; done
cat $O/set_surfaces_cfg5.txt
python scripts/quick_time.py 2 5:2000000 > $O/quick_time.txt 2>&1; cat $O/quick_time.txt
