#!/bin/bash
# superclusters: cell tests, set_surfaces phases, launches
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cell or cull" > $O/pytest_cells.log 2>&1
echo "pytest exit $?" >> $O/pytest_cells.log
NM_CELL_VERBOSE=2 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
python scripts/surf_quick.py 2 3 > $O/surf_cfg2.txt 2>&1
python scripts/cells_quick.py 5 > $O/cells_cfg5.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_surf.csv \
    python scripts/surf_quick.py 5 1 > $O/ncu_launches.log 2>&1
