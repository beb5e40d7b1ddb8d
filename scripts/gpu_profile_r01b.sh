# Round-1 refresh after strip chains: ncu full capture of k_label on a cfg5
# slab, the bench launch list (with DRAM bytes), and the secondary configs.
set -x
mkdir -p gpurun_out
python scripts/ncu_label.py 5 600000 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_label -c 1 -o gpurun_out/prof_k_label_chain python scripts/ncu_label.py 5 600000 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_cfg5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-cull > gpurun_out/ncu_launch.log 2>&1
python bench.py --config 3 --cpu-seconds 8 --quality > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 2 --cpu-seconds 8 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 4 --steps 1 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
