#!/bin/bash
# device memory pool: set_surfaces phases, then the full GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v
mkdir -p $O
NM_CELL_VERBOSE=2 python scripts/surf_quick.py 5 6 > $O/surf_cfg5.txt 2>&1
NM_CELL_VERBOSE=2 python scripts/surf_quick.py 3 4 > $O/surf_cfg3.txt 2>&1
python scripts/surf_quick.py 2 4 > $O/surf_cfg2.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
