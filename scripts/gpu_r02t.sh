#!/bin/bash
# deferred frees (Retired): set_surfaces phases + ncu of the child certification
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
python scripts/surf_quick.py 2 3 > $O/surf_cfg2.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"child_certify_all" -c 1 -o $O/prof_child \
    python scripts/surf_quick.py 5 1 > $O/ncu_child.log 2>&1
ls -la $O
