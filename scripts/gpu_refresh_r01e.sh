# Round-1 refresh after the complex-product operand order (vos.cuh seg_far):
# smoke, pytest -m gpu, the bench configs, the reference arm, the dense-kernel
# ncu capture and the bench launch list (with DRAM bytes per launch).
set -x
mkdir -p gpurun_out/r01e
o=gpurun_out/r01e
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $o/pytest_gpu.log 2>&1
python bench.py > $o/bench_cfg5.json 2> $o/bench_cfg5.err
python bench.py --config 3 --cpu-seconds 8 --quality > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python bench.py --config 2 --cpu-seconds 8 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
python scripts/ncu_label.py 5 600000 > $o/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_label -c 1 -o $o/prof_k_label python scripts/ncu_label.py 5 600000 > $o/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 400 --csv --log-file $o/launches_bench_cfg5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-cull > $o/ncu_launch.log 2>&1
tail -2 $o/pytest_gpu.log; cat $o/smoke.log
