#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=8 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
tail -12 $O/pytest_gpu.log
timeout 1500 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02g/bench.json").read().strip().splitlines()[-1])
print(json.dumps({k: d[k] for k in ("value", "ms_per_step", "e2e", "roofline", "cpp_dropin_e2e", "clocks")}, indent=1)[:4000])
print(json.dumps(d["cull_outside"], indent=1)[:2500])
PY
