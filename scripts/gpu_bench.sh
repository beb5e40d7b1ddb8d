set -e
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --config 2 --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_cfg2.json
cat gpurun_out/bench_cfg2.json
python bench.py > gpurun_out/bench_cfg5.json
cat gpurun_out/bench_cfg5.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json
cat gpurun_out/bench_ref.json
