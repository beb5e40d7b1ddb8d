#!/bin/bash
# set_surfaces phases (absolute timestamps per thread) + ncu of the certification kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02p
mkdir -p $O
nproc > $O/nproc.txt
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 4 > $O/surf_cfg5.txt 2>&1
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
python scripts/surf_quick.py 5 1 > $O/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_child_certify|k_cell_certify" -s 2 -c 2 -o $O/prof_certify \
    python scripts/surf_quick.py 5 1 > $O/ncu_certify.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_surf.csv \
    python scripts/surf_quick.py 5 1 > $O/ncu_launches.log 2>&1
ls -la $O
