set -e
python -c "import __graft_entry__ as g; g.smoke()"
python -m pytest tests -q -m gpu 2>&1 | tail -2
python bench.py > gpurun_out/bench_cfg5.json
python bench.py --config 3 --cpu-seconds 8 --quality > gpurun_out/bench_cfg3.json
python bench.py --config 2 --cpu-seconds 8 > gpurun_out/bench_cfg2.json
python bench.py --config 4 --steps 1 --warmup 3 > gpurun_out/bench_cfg4.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json
