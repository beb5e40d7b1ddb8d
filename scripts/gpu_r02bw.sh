#!/bin/bash
# stripify with bitset degree buckets (same strips): set_surfaces phases, GPU suite, bench cfg5, smoke
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bw
mkdir -p $O
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 4 > $O/set_surfaces_cfg5.txt 2>&1
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 3 3 > $O/set_surfaces_cfg3.txt 2>&1
timeout 3000 python -m pytest tests -x -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
timeout 1800 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
