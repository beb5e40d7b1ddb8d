#!/bin/bash
# round 2: watertight subtile frames — accuracy diagnosis + GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02d
mkdir -p $O
python scripts/diag_err_full.py 2 0 > $O/diag_cfg2_strips.txt 2>&1
python scripts/diag_err_full.py 2 1 > $O/diag_cfg2_tris.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
head -3 $O/diag_cfg2_strips.txt $O/diag_cfg2_tris.txt
tail -25 $O/pytest_gpu.log
