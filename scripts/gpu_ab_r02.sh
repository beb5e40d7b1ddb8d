#!/bin/bash
# round 2 A/B of k_label pipeline variants (lib/variants/*.so), alternating
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_r02
mkdir -p $O
out=$O/variants_ab.log
: > $out
for rep in 1 2; do
  for v in paper_2203_10000_b200/lib/variants/*.so; do
    echo "== rep $rep $(basename $v)" >> $out
    NM_LABEL_LIB=$v timeout 300 python scripts/quick_time.py 5:2000000 3:2000000 2 >> $out 2>&1
  done
done
cat $out
