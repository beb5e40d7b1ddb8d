#!/bin/bash
# round 2 ncu evidence for the CURRENT build (run after a plain bench passed):
#   1. per-opcode thread-instruction counts of one k_label launch on a strided
#      1/5 cfg5 node sample (FP32 lane-ops per eval for bench.py's roofline)
#   2. DRAM bytes of one FULL-mesh cfg5 k_label launch (roofline.traffic)
#   3. --set full of k_label on a 600k-node slab (pipe utilisation, stalls)
#   4. --set full of the fix-up kernels + k_cell_classify on the cfg5 cell pass
# plus the SASS hash of k_label<1,true,0> the captures belong to.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ncu_r02
mkdir -p $O
python scripts/kernel_hash.py > $O/sass_hash.txt
python scripts/ncu_label.py 5 stride:5 > $O/plain_stride5.log 2>&1 &&
ncu --metrics sass__thread_inst_executed_true_per_opcode,sass__inst_executed_per_opcode,gpu__time_duration.sum \
    --print-metric-instances details -k regex:k_label -s 1 -c 1 --csv --log-file $O/opcounts_stride5.csv \
    python scripts/ncu_label.py 5 stride:5 > $O/ncu_opcounts.log 2>&1
python scripts/ncu_label.py 5 full 1 > $O/plain_full.log 2>&1 &&
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    -k regex:k_label -c 1 --csv --log-file $O/traffic_full.csv python scripts/ncu_label.py 5 full 1 > $O/ncu_traffic.log 2>&1
python scripts/ncu_label.py 5 600000 > $O/plain_600k.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_label -s 1 -c 1 -o $O/prof_k_label \
    python scripts/ncu_label.py 5 600000 > $O/ncu_full.log 2>&1
python scripts/cells_quick.py 5 > $O/plain_cells.log 2>&1 &&
ncu --set full --clock-control none -k regex:"k_fixup|k_fix_finalize|k_cell_classify|k_unpermute" -s 4 -c 4 -o $O/prof_aux \
    python scripts/cells_quick.py 5 > $O/ncu_aux.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cells.csv \
    python scripts/cells_quick.py 5 > $O/ncu_launches.log 2>&1
ls -la $O
