#!/bin/bash
# k_pair_resolve: cell/cull parity tests, node pass with and without, masks vs 13-DOP culling
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ae
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -x -q -m gpu -k "cell or cull or cfg5 or cfg3" > $O/pytest_cells.log 2>&1
echo "pytest exit $?" >> $O/pytest_cells.log
python scripts/cells_quick.py 5 > $O/cells_cfg5.txt 2>&1
NM_NO_RESOLVE=1 python scripts/cells_quick.py 5 > $O/cells_cfg5_noresolve.txt 2>&1
python scripts/cells_quick.py 3 > $O/cells_cfg3.txt 2>&1
python scripts/cells_quick.py 2 > $O/cells_cfg2.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cells.csv \
    python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
