#!/bin/bash
# bench lines with the per-config stamped opcount/traffic files (cfg2, cfg3) + cfg5 check
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bv
mkdir -p $O
for c in 2 3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 1800 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
