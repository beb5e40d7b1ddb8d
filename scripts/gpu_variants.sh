#!/bin/bash
# Time every built variant under paper_2203_10000_b200/lib/variants on the same slabs.
mkdir -p gpurun_out
out=gpurun_out/variants.log
: > $out
for v in paper_2203_10000_b200/lib/variants/*.so; do
  echo "== $(basename $v)" >> $out
  NM_LABEL_LIB=$v timeout 300 python scripts/quick_time.py ${NM_VARIANT_ARGS:-5:2000000 3:2000000 2} >> $out 2>&1
done
cat $out
