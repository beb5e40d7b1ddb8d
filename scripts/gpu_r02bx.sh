#!/bin/bash
# set_surfaces (cfg5, cells) kernel launch list + --set full of the two certification kernels, final build
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bx
mkdir -p $O
python scripts/surf_quick.py 5 2 > $O/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_set_surfaces_cfg5.csv \
    python scripts/surf_quick.py 5 2 > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_child_certify_all|k_cell_certify_all" -s 2 -c 2 -o $O/prof_certify \
    python scripts/surf_quick.py 5 2 > $O/ncu_full.log 2>&1
ls -la $O
