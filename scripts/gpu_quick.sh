python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -3
python scripts/quick_time.py 5:2000000 3:2000000
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_cull.json && python -c "import json;d=json.load(open('gpurun_out/b_cull.json'));print(d['value'], d['full_mesh_labeling_time_s'], d['cull_outside'])"
