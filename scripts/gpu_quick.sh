python -m pytest tests/test_gpu_dropin.py -q -m gpu -k "stream or nccl" 2>&1 | tail -3
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_cull.json && python -c "import json;d=json.load(open('gpurun_out/b_cull.json'));print(d['value'], d['full_mesh_labeling_time_s'], d['roofline']['kernel_share_of_step'], d['cull_outside'])"
