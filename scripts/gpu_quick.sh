python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
python scripts/quick_time.py 5:2000000 3:2000000 2
NM_LABEL_LIB=probes/libnl_cta.so python scripts/quick_time.py 5:2000000 3:2000000 2
