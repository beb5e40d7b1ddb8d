set -e
python -c "import __graft_entry__ as g; g.smoke()"
python -m pytest tests -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench_cfg5.json
cat gpurun_out/bench_cfg5.json
python bench.py --config 3 --cpu-seconds 8 > gpurun_out/bench_cfg3.json
cat gpurun_out/bench_cfg3.json
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_ncu.log 2>&1
