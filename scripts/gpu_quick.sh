python -m pytest tests/test_gpu_parity.py -q -m gpu -k "distance" 2>&1 | tail -8
