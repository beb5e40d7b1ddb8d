#!/bin/bash
# ncu --set full of the one-launch certification kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02r
mkdir -p $O
python scripts/surf_quick.py 5 1 > $O/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"certify_all" -c 2 -o $O/prof_certify_all \
    python scripts/surf_quick.py 5 1 > $O/ncu_certify.log 2>&1
ls -la $O
