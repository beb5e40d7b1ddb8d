#!/bin/bash
# launch-bounds A/B: certification (set_surfaces) and fix-up (cells node pass)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bp
mkdir -p $O
for rep in 1 2; do
for v in base c3 c4; do
  echo "== rep $rep $v" >> $O/surf.txt
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so python scripts/surf_quick.py 5 4 2>&1 | tail -3 >> $O/surf.txt
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so python scripts/surf_quick.py 3 3 2>&1 | tail -2 >> $O/surf.txt
done
for v in base f8 f12; do
  echo "== rep $rep $v" >> $O/fix.txt
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so timeout 300 python scripts/quick_time.py 5:2000000 3:2000000 2 >> $O/fix.txt 2>&1
  NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so python scripts/cells_quick.py 5 2>&1 | grep "mode': 2" | tail -1 >> $O/fix.txt
done
done
