#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02au
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 5 1 > $O/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"certify_all" -c 2 -o $O/prof_certify_all \
    python scripts/surf_quick.py 5 1 > $O/ncu_certify.log 2>&1
