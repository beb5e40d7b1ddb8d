#!/bin/bash
# two-stage fix-up (hybrid far terms, oracle-order stage 2): GPU suite, fix-up timings
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ba
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
for c in 5 3 2; do python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1; done
timeout 600 python scripts/quick_time.py 5:2000000 3:2000000 2 > $O/quick.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cells.csv \
    python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
