#!/bin/bash
# ball chains in their own kernel (one warp per pending pair): parity tests, node pass timings
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ap
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_dropin.py -x -q -m gpu > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for c in 5 3 2; do python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cells.csv python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
