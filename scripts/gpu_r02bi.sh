#!/bin/bash
# packing with pre-snapped vertices: bitwise s vs the previous build (stored), set_surfaces phases
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bi
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 5 > $O/surf_cfg5.txt 2>&1
python scripts/surf_quick.py 3 3 > $O/surf_cfg3.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -x -q -m gpu > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for c in 2 5; do
  python scripts/pack_bitwise.py $c /tmp/s_new_$c.npy
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/oldpack.so python scripts/pack_bitwise.py $c /tmp/s_old_$c.npy
  python -c "import numpy as np; a=np.load('/tmp/s_new_$c.npy'); b=np.load('/tmp/s_old_$c.npy'); print('cfg$c bitwise equal:', bool(np.array_equal(a.view(np.uint64), b.view(np.uint64))), a.shape)" >> $O/bitwise.txt
  rm -f /tmp/s_new_$c.npy /tmp/s_old_$c.npy
done
