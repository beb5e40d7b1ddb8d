#!/bin/bash
# A/B: exact certification tests batched across the warp (NM_CERT_BATCH) vs the per-cube loop
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02by
mkdir -p $O
L=paper_2203_10000_b200/lib
for rep in 1 2; do
  for v in base certbatch certbatch3; do
    if [ $v = base ]; then lib=$L/libnestmesh_label.so; else lib=$L/variants/$v.so; fi
    echo "== rep $rep $v" >> $O/ab.txt
    NM_LABEL_LIB=$lib timeout 300 python scripts/surf_quick.py 5 4 2>&1 | cut -c1-200 >> $O/ab.txt
    NM_LABEL_LIB=$lib timeout 300 python scripts/surf_quick.py 3 3 2>&1 | cut -c1-200 >> $O/ab.txt
  done
done
NM_LABEL_LIB=$L/variants/certbatch.so timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cell" > $O/pytest_cells_certbatch.log 2>&1
echo "exit $?" >> $O/pytest_cells_certbatch.log
tail -2 $O/pytest_cells_certbatch.log
