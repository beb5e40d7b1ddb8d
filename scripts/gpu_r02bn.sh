#!/bin/bash
# final ncu evidence: the certified-cell pass kernels (--set full) and the bench launch list
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bn
mkdir -p $O
python scripts/cells_quick.py 5 > $O/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_pair_chain|k_fixup|k_label" -s 6 -c 6 -o $O/prof_cells \
    python scripts/cells_quick.py 5 > $O/ncu_cells.log 2>&1
timeout 1500 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_plain.json 2> $O/bench_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
ls -la $O
