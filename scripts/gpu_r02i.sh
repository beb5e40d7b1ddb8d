#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02i
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python scripts/cpp_e2e_timing.py 5 > $O/cpp_e2e_timing.txt 2>&1
tail -30 $O/cpp_e2e_timing.txt
timeout 1500 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02i/bench.json").read().strip().splitlines()[-1])
print(json.dumps({k: d[k] for k in ("value", "ms_per_step", "e2e", "cpp_dropin_e2e", "clocks")}, indent=1)[:3000])
PY
rm -rf gpurun_out/ncu_r02
bash scripts/gpu_ncu_r02.sh > $O/ncu_script.log 2>&1
tail -5 $O/ncu_script.log
