"""GPU: the C++ drop-in (labeling.hpp over the reference types) and the NCCL
path of the partitioner (torchrun, one rank, real all_gather)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_dropin_binary(tmp_path):
    exe = ROOT / "build" / "dropin_test"
    if not exe.exists():
        pytest.skip("build/dropin_test not built (needs the reference headers at build time)")
    out = tmp_path / "labels.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    labels = np.fromfile(out, dtype=np.int32)
    S = synth.concat_surfaces([synth.icosphere(6.0, 3), synth.icosphere(10.0, 3)], labels=[3, 9])
    nodes, tets = synth.lattice_mesh((-12.0, -12.0, -12.0), 0.75, (32, 32, 32))
    ref = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
    np.testing.assert_array_equal(labels, ref)


def test_bench_nccl_path_one_rank(tmp_path):
    """bench.py under torchrun with --force-dist: the NCCL process group, the
    mask all-gather and max-over-ranks timing run for real (world size 1)."""
    env = dict(os.environ, NM_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29533", str(ROOT / "bench.py"), "--config", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["config"]["distributed"] is True
