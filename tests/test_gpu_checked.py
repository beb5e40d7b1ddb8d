"""Memory-safety evidence for the kernels (compute-sanitizer is closed on this
GPU pool: profiles/r02/compute_sanitizer_refusal.log). The checked build
(lib/checked/libnestmesh_label.so, -DNM_CHECKED, csrc/check.cuh) bounds-checks
every global index the main kernels form (points, tiles, positions, fix-up
pairs and partials, tet node ids) and traps on a violation. This test runs
the GPU parity suites against that build in a subprocess: a failed check
fails the launch and the test."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_gpu_suites_under_checked_build():
    lib = ROOT / "paper_2203_10000_b200" / "lib" / "checked" / "libnestmesh_label.so"
    if not lib.exists():
        pytest.skip("checked build missing (paper_2203_10000_b200.build.build_checked_lib)")
    env = dict(os.environ, NM_LABEL_LIB=str(lib))
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
           str(ROOT / "tests" / "test_gpu_parity.py"), str(ROOT / "tests" / "test_gpu_refine_oracle.py"),
           str(ROOT / "tests" / "test_sidecar.py"), "-k", "not cfg5_full_size and not boundary_distance_median"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "NM_DCHECK failed" not in r.stdout + r.stderr
