#!/bin/bash
# ball-chain tracing: steps and compartment-size threshold
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bo
mkdir -p $O
for c in 5 3 2; do
  python scripts/cells_quick.py $c > $O/cells_cfg${c}_base.txt 2>&1
  for v in lb3 lb4; do
    NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so python scripts/cells_quick.py $c > $O/cells_cfg${c}_$v.txt 2>&1
  done
done
