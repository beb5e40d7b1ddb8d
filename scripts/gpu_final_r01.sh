# Round-1 final refresh: tests, smoke, every bench config, the reference arm,
# the dense-kernel ncu capture + bench launch list, the culled-pass captures.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config 3 --cpu-seconds 8 --quality > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 2 --cpu-seconds 8 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 4 --steps 1 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python scripts/ncu_label.py 5 600000 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_label -c 1 -o gpurun_out/prof_k_label_final python scripts/ncu_label.py 5 600000 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_cfg5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-cull > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_label -s 1 -c 1 -o gpurun_out/prof_sparse5 python scripts/ncu_cells.py 5 > gpurun_out/ncu_sparse_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cells5.csv python scripts/ncu_cells.py 5 > /dev/null 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
