#!/bin/bash
# point -> cell lookups by multiplication: cell tests, node pass timings
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02br
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -x -q -m gpu > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for c in 5 3 2; do python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"classify" -c 6 --csv --log-file $O/classify.csv python scripts/cells_quick.py 5 > $O/ncu.log 2>&1
