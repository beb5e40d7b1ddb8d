python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -5
python scripts/quick_time.py 2 5:2000000 3:2000000
NM_LAYOUT=1 python scripts/quick_time.py 5:2000000
