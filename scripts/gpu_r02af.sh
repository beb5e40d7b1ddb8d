#!/bin/bash
# k_pair_resolve neighbourhood reach A/B (1 = 26 neighbours, 2 = 124 (default), 3 = 342)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02af
mkdir -p $O
for c in 5 3 2; do
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/reach1.so python scripts/cells_quick.py $c > $O/cells_cfg${c}_reach1.txt 2>&1
  python scripts/cells_quick.py $c > $O/cells_cfg${c}_reach2.txt 2>&1
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/reach3.so python scripts/cells_quick.py $c > $O/cells_cfg${c}_reach3.txt 2>&1
done
