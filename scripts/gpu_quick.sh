NM_PAIRS=2 python scripts/quick_time.py 5:2000000 3:2000000
