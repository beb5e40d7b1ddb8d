#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aw
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
python scripts/surf_quick.py 2 3 > $O/surf_cfg2.txt 2>&1
