#!/bin/bash
# ball-chain tracing variants (steps, early stop when the balls shrink, step fraction)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ah
mkdir -p $O
for c in 5 3 2; do
  python scripts/cells_quick.py $c > $O/cells_cfg${c}_base.txt 2>&1
  for v in trace0 s4 s8 s8shr s12shr s24shr99; do
    NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so python scripts/cells_quick.py $c > $O/cells_cfg${c}_$v.txt 2>&1
  done
done
