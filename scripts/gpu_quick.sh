python -m pytest tests/test_gpu_dropin.py -q -m gpu -k cpp 2>&1 | tail -3
