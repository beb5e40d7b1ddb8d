#!/bin/bash
# Alternating A/B of the built variants (lib/variants/*.so): node-pass timing
# on cfg5/cfg3 slabs twice each, plus the fp32 error profile of each variant.
mkdir -p gpurun_out
out=gpurun_out/variants_ab.log
: > $out
for rep in 1 2; do
  for v in paper_2203_10000_b200/lib/variants/*.so; do
    echo "== rep $rep $(basename $v)" >> $out
    NM_LABEL_LIB=$v timeout 300 python scripts/quick_time.py ${NM_VARIANT_ARGS:-5:2000000 3:2000000} >> $out 2>&1
  done
done
for v in paper_2203_10000_b200/lib/variants/*.so; do
  echo "== err $(basename $v)" >> $out
  NM_LABEL_LIB=$v timeout 300 python scripts/diag_err.py >> $out 2>&1
done
cat $out
