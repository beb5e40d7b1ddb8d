#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ab
mkdir -p $O
NM_CELL_VERBOSE=3 python scripts/surf_quick.py 5 2 > $O/surf_cfg5_cold.txt 2>&1
