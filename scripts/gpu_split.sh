# quick timing of small shards (compartment split) — development aid
python scripts/quick_time.py 2 5:1259712 3:964141 5:2000000
