#!/bin/bash
# round 2 final refresh (classify multiply, face-neighbour child runs): GPU suite, bench lines (cfg5 default + cfg2/3/4 + reference arm), set_surfaces phases
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bt
mkdir -p $O
timeout 3000 python -m pytest tests -x -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
NM_CELL_VERBOSE=1 python scripts/surf_quick.py 5 4 > $O/set_surfaces_cfg5.txt 2>&1
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
timeout 1800 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in 2 3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python smoke_check.py > /dev/null 2>&1 || true
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
