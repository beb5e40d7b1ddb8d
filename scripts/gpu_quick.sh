python -m pytest tests/test_gpu_dropin.py -q -m gpu -k "multi_rank or nccl" 2>&1 | tail -15
