#!/bin/bash
# chunked tet labels under the tet upload: GPU suite, C++ e2e phases, bench cfg5/cfg3 e2e lines
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02at
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
python scripts/cpp_e2e_timing.py 3 > $O/cpp_e2e_timing_cfg3.txt 2>&1
timeout 1800 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
