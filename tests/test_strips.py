"""The strip decomposition of nm_set_surfaces (csrc/strips.h), on the CPU.

The packed tiles — hence every fp32 partial sum of k_label — depend on the
exact strips, so a faster stripify must return the SAME strips. The
checksums below were recorded from the round-1 implementation (before the
bucket queue and the vertex-range incidence lists); tests/cpp/strips_check.cpp
also checks that every triangle is in exactly one strip and that each strip
triangle's vertices are the strip's three consecutive vertices."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2203_10000_b200 import synth

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = {  # config -> (checksum, strips, triangles)
    2: ("538b755764538a1e", 400, 35840),
    3: ("49def4fe3a392fb7", 2480, 363520),
    5: ("aa7f97d5449d92a3", 3840, 983040),
}


@pytest.fixture(scope="module")
def strips_exe(tmp_path_factory):
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    exe = tmp_path_factory.mktemp("strips") / "strips_check"
    subprocess.run([cxx, "-O2", "-std=c++17", f"-I{ROOT / 'paper_2203_10000_b200' / 'csrc'}",
                    str(ROOT / "tests" / "cpp" / "strips_check.cpp"), "-o", str(exe)], check=True)
    return exe


@pytest.mark.parametrize("cfg_id", [2, 3, 5])
def test_stripify_matches_round1_strips(strips_exe, tmp_path, cfg_id):
    S = synth.config(cfg_id).surfaces
    tri = np.ascontiguousarray(S.tri, np.uint32)
    off = np.ascontiguousarray(S.comp_off, np.uint32)
    f = tmp_path / "surf.bin"
    with open(f, "wb") as fh:
        np.array([S.xyz.shape[0], tri.shape[0], off.shape[0] - 1], np.uint64).tofile(fh)
        tri.tofile(fh)
        off.tofile(fh)
    r = subprocess.run([str(strips_exe), str(f)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr)
    checksum, nstrips, ntris, _ms = r.stdout.split()
    assert (checksum, int(nstrips), int(ntris)) == GOLDEN[cfg_id]


def test_stripify_ragged_and_nonmanifold(strips_exe, tmp_path):
    """Open patches, a non-manifold fan (three triangles on one edge),
    degenerate triangles and an empty compartment still give a partition."""
    tri = np.array([[0, 1, 2], [1, 3, 2], [0, 1, 4], [0, 1, 5],   # edge (0,1) shared by three
                    [6, 6, 7], [7, 8, 9], [8, 9, 10]], np.uint32)  # a degenerate triangle
    off = np.array([0, 4, 4, 7], np.uint32)                        # middle compartment empty
    f = tmp_path / "surf.bin"
    with open(f, "wb") as fh:
        np.array([11, tri.shape[0], off.shape[0] - 1], np.uint64).tofile(fh)
        tri.tofile(fh)
        off.tofile(fh)
    r = subprocess.run([str(strips_exe), str(f)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stderr)
    assert int(r.stdout.split()[2]) == 7


def test_bitset_buckets_equal_heap_order(tmp_path):
    """csrc/strips.h's exact bitset degree buckets pick the same next strip
    start as the lazy heaps they replaced (tests/cpp/strips_heap_ref.h), on
    random soups with non-manifold edges and degenerate triangles."""
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    exe = tmp_path / "strips_equiv"
    subprocess.run([cxx, "-O2", "-std=c++17", f"-I{ROOT / 'paper_2203_10000_b200' / 'csrc'}",
                    f"-I{ROOT / 'tests' / 'cpp'}", str(ROOT / "tests" / "cpp" / "strips_equiv.cpp"), "-o", str(exe)],
                   check=True)
    for seed in (7, 11):
        r = subprocess.run([str(exe), str(seed), "3000"], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
