#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02k
mkdir -p $O
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
tail -7 $O/cpp_e2e_timing.txt
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_sidecar.py -x -q -m gpu > $O/pytest.log 2>&1; tail -3 $O/pytest.log
