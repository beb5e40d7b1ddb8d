#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02j
mkdir -p $O
bash scripts/gpu_ab_r02.sh > $O/ab.log 2>&1
grep -E "^==|cfg5|cfg3|cfg2" gpurun_out/ab_r02/variants_ab.log | sed 's/near\/far.*//' 
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
tail -7 $O/cpp_e2e_timing.txt
# DRAM traffic of the full-mesh k_label launch: cache control all vs none, plus SM->L2 writes
python scripts/ncu_label.py 5 full 1 > $O/plain_full.log 2>&1 &&
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum \
    --cache-control none -k regex:k_label -c 1 --csv --log-file $O/traffic_none.csv python scripts/ncu_label.py 5 full 1 > $O/ncu1.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    --cache-control all -k regex:k_unpermute -c 1 --csv --log-file $O/traffic_unpermute.csv python scripts/ncu_label.py 5 full 1 > $O/ncu2.log 2>&1
grep -E "dram|lts" $O/traffic_none.csv $O/traffic_unpermute.csv | cut -d, -f5,13- | head -20
