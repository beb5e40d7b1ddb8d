python -m pytest tests/test_gpu_dropin.py -q -m gpu -x 2>&1 | tail -15
