python -m pytest tests/test_gpu_dropin.py -q -m gpu -k validation 2>&1 | tail -8
