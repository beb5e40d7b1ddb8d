#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bb
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for c in 5 3 2; do python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1; done
timeout 600 python scripts/quick_time.py 5:2000000 3:2000000 2 > $O/quick.txt 2>&1
