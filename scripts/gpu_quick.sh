python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
python scripts/quick_time.py 5:2000000 3:2000000 2
