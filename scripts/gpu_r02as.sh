#!/bin/bash
# k_label occupancy A/B: 4 CTAs/SM (base, 119 regs) vs 5 (96 regs, small spills)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02as
mkdir -p $O
out=$O/mb5_ab.log
: > $out
for rep in 1 2 3; do
  for v in base mb5; do
    echo "== rep $rep $v" >> $out
    NM_LABEL_LIB=paper_2203_10000_b200/lib/variants/$v.so timeout 300 python scripts/quick_time.py 5:2000000 3:2000000 2 >> $out 2>&1
  done
done
cat $out
