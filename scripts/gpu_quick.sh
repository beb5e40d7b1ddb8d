python -m pytest tests/test_gpu_dropin.py -q -m gpu -k recursive 2>&1 | tail -5
