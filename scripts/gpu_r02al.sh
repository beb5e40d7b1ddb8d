#!/bin/bash
# profile of one certified-cell node pass after the resolve step
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02al
mkdir -p $O
python scripts/cells_quick.py 5 > $O/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cells.csv \
    python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pair_resolve" -s 1 -c 1 -o $O/prof_resolve \
    python scripts/cells_quick.py 5 > $O/ncu_resolve.log 2>&1
