#!/bin/bash
# round 2: compute-sanitizer memcheck (ONE tool per call) on the smoke path
# (dense + certified-cell labeling, cfg1) after a plain run has exited 0.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_plain.log 2>&1 || { echo "plain smoke failed"; exit 1; }
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1
echo "memcheck exit $?" >> $O/memcheck_smoke.log
tail -5 $O/memcheck_smoke.log
