#!/bin/bash
# sphere-traced ball chains in k_pair_resolve: parity tests, node pass with / without tracing
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ag
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -x -q -m gpu -k "cell or cull or cfg5 or cfg3 or resolve" > $O/pytest_cells.log 2>&1
echo "pytest exit $?" >> $O/pytest_cells.log
for c in 5 3 2; do
  python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/trace0.so python scripts/cells_quick.py $c > $O/cells_cfg${c}_trace0.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cells.csv \
    python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
