#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02u
mkdir -p $O
NM_CELL_VERBOSE=3 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
NM_CELL_VERBOSE=3 python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
