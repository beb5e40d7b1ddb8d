python -m pytest tests/test_gpu_parity.py -q -m gpu -k "lattice or boundary" 2>&1 | tail -4
