#!/bin/bash
# FP32 lane-ops per eval and full-mesh DRAM bytes of k_label on cfg2 / cfg3
# (the cfg5 pair is from gpu_ncu_r02.sh), so those bench lines carry a frac.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bu
mkdir -p $O
python scripts/kernel_hash.py > $O/sass_hash.txt
for c in "2 stride:1" "3 stride:5"; do
  set -- $c
  python scripts/ncu_label.py $1 $2 > $O/plain_ops_cfg$1.log 2>&1 &&
  ncu --metrics sass__thread_inst_executed_true_per_opcode,sass__inst_executed_per_opcode,gpu__time_duration.sum \
      --print-metric-instances details -k regex:k_label -s 1 -c 1 --csv --log-file $O/opcounts_cfg$1.csv \
      python scripts/ncu_label.py $1 $2 > $O/ncu_ops_cfg$1.log 2>&1
  python scripts/ncu_label.py $1 full 1 > $O/plain_full_cfg$1.log 2>&1 &&
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
      -k regex:k_label -c 1 --csv --log-file $O/traffic_cfg$1.csv python scripts/ncu_label.py $1 full 1 > $O/ncu_traffic_cfg$1.log 2>&1
done
ls -la $O
