#!/bin/bash
# child runs joined to certified parents across y / z faces: cell tests, set_surfaces, node passes
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bs
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cell or cull or resolve" > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 4 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
for c in 5 3 2; do python scripts/cells_quick.py $c > $O/cells_cfg${c}.txt 2>&1; done
