python scripts/quick_time.py 5:2000000 3:2000000
NM_LABEL_LIB=probes/libnl_nopair.so python scripts/quick_time.py 5:2000000 3:2000000
python scripts/quick_time.py 5:2000000 3:2000000
