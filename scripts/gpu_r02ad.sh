#!/bin/bash
# (1) fix-up with two accumulator chains: cells node pass timing + ncu of k_fixup
# (2) where k_label's DRAM writes come from: L2 write sectors from the SMs vs DRAM writes,
#     with ncu's cache flush and without
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ad
mkdir -p $O
python scripts/kernel_hash.py > $O/sass_hash.txt
python scripts/cells_quick.py 5 > $O/cells_cfg5.txt 2>&1 &&
ncu --set full --clock-control none -k regex:"k_fixup" -s 2 -c 1 -o $O/prof_fixup \
    python scripts/cells_quick.py 5 > $O/ncu_fixup.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_srcunit_ltcfabric.sum,gpu__time_duration.sum
python scripts/ncu_label.py 5 stride:5 1 > $O/plain_stride5.log 2>&1 &&
ncu --metrics $M -k regex:k_label -c 1 --csv --log-file $O/writes_flush.csv python scripts/ncu_label.py 5 stride:5 1 > $O/ncu_w1.log 2>&1
ncu --metrics $M --cache-control none -k regex:k_label -c 1 --csv --log-file $O/writes_noflush.csv python scripts/ncu_label.py 5 stride:5 1 > $O/ncu_w2.log 2>&1
ls -la $O
