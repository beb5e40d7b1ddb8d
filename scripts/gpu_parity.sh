nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -30
python scripts/quick_time.py 1 2 5:2000000 3:2000000
