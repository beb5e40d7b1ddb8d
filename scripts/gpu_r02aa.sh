#!/bin/bash
# cell_axis sweep with the faster build; bench cfg5 refresh
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aa
mkdir -p $O
python scripts/cell_axis_sweep.py 5 120 144 168 200 240 > $O/axis_cfg5.txt 2>&1
python scripts/cell_axis_sweep.py 3 120 168 240 > $O/axis_cfg3.txt 2>&1
python scripts/cell_axis_sweep.py 2 120 168 240 > $O/axis_cfg2.txt 2>&1
timeout 1800 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
