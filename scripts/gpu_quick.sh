python -m pytest tests -q -m gpu -x 2>&1 | tail -15
python bench.py --config 4 --steps 1 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; cat gpurun_out/bench_cfg4.json; tail -3 gpurun_out/bench_cfg4.err
