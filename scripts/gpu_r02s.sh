#!/bin/bash
# device geometry (extents/13-DOP, Morton clusters) + transpose certify: full GPU suite, set_surfaces phases, launches
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 4 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 2 > $O/surf_cfg3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_surf.csv \
    python scripts/surf_quick.py 5 1 > $O/ncu_launches.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
ls -la $O
