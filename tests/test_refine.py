"""Host refinement of the recursive driver (csrc/refine.cpp).
CPU only: nm_refine is host code inside libnestmesh_label.so."""
import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import NativeError, refine

from test_synth import _faces_conforming, _volumes


def _check(nodes, tets, new_nodes, new_tets, new_labels, parent, labels, n_old):
    assert np.array_equal(new_nodes[:n_old], nodes)            # old nodes keep their ids/positions
    v = _volumes(new_nodes, new_tets)
    assert np.all(v > 0)                                         # oriented (mesh.hpp:44-48)
    v0 = _volumes(nodes, tets)
    assert abs(v.sum() - v0.sum()) <= 1e-12 * v0.sum()          # SPEC.md:304 volume conservation
    ok, _ = _faces_conforming(new_tets)
    assert ok                                                    # SPEC.md:305 conformity
    np.testing.assert_array_equal(new_labels, labels[parent])   # SPEC.md:288 inherit labels
    # per-parent volume is preserved too
    vp = np.zeros(tets.shape[0])
    np.add.at(vp, parent, v)
    np.testing.assert_allclose(vp, v0, rtol=1e-12, atol=0)


def test_single_tet_eight_children():
    """one isolated tet -> 8 children, volume preserved."""
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float64)
    tets = np.array([[0, 1, 2, 3]], np.uint32)
    nn, nt, nl, par, n_old = refine(nodes, tets, np.array([5], np.int32), [0])
    assert nt.shape[0] == 8 and nn.shape[0] == 10 and n_old == 4
    _check(nodes, tets, nn, nt, nl, par, np.array([5], np.int32), n_old)
    # midpoints at (p_a + p_b) * 0.5 in ascending edge-key order
    keys = sorted((a, b) for a in range(4) for b in range(a + 1, 4))
    for i, (a, b) in enumerate(keys):
        np.testing.assert_array_equal(nn[4 + i], (nodes[a] + nodes[b]) * 0.5)


def test_one_tet_of_cube_conforming():
    """one tet of a 5-tet cube -> neighbours get transition
    templates; the result is conforming."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (1, 1, 1))
    labels = np.arange(1, 6, dtype=np.int32)
    for sel in range(5):
        nn, nt, nl, par, n_old = refine(nodes, tets, labels, [sel])
        _check(nodes, tets, nn, nt, nl, par, labels, n_old)


def test_empty_selection_identity():
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (2, 2, 2))
    labels = np.ones(tets.shape[0], np.int32)
    nn, nt, nl, par, n_old = refine(nodes, tets, labels, [])
    assert np.array_equal(nn, nodes) and np.array_equal(nt, tets) and np.array_equal(par, np.arange(tets.shape[0]))


def test_invalid_selection():
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (1, 1, 1))
    with pytest.raises(NativeError, match="InvalidSelection"):
        refine(nodes, tets, None, [99])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_selections_conforming(seed):
    nodes, tets = synth.lattice_mesh((-1.0, 0.5, 2.0), 0.8, (4, 3, 5))
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 4, tets.shape[0]).astype(np.int32)
    sel = np.flatnonzero(rng.random(tets.shape[0]) < 0.15)
    nn, nt, nl, par, n_old = refine(nodes, tets, labels, sel)
    _check(nodes, tets, nn, nt, nl, par, labels, n_old)
    if oracle.ref_available():
        import ctypes
        R = oracle.ref()
        D = ctypes.POINTER(ctypes.c_double)
        U = ctypes.POINTER(ctypes.c_uint32)
        assert R.ref_validate_mesh_ok(nn.ctypes.data_as(D), nn.shape[0], nt.ctypes.data_as(U), nt.shape[0]) == 1


def test_two_levels_straddle_refinement_relabels_to_initial():
    """The recursive driver on a small cfg4 analogue: straddle tets are refined
    twice; masks of old nodes are reused, only new nodes are evaluated; the
    result equals initial labeling of the refined mesh (oracle)."""
    R = 10.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 2), synth.icosphere(R, 2)], labels=[1, 2])
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, R / 4, (11, 11, 11))
    masks = oracle.label_nodes(nodes, S)
    labels = oracle.label_tets(tets, masks, S.label_ids)
    for level in range(2):
        sel = oracle.flag_boundary(tets, masks)
        nodes2, tets2, inherited, parent, n_old = refine(nodes, tets, labels, sel)
        new_masks = oracle.label_nodes(nodes2[n_old:], S)
        masks = np.concatenate([masks, new_masks])
        labels = oracle.label_tets(tets2, masks, S.label_ids)
        full = oracle.label_tets(tets2, oracle.label_nodes(nodes2, S), S.label_ids)
        np.testing.assert_array_equal(labels, full)
        nodes, tets = nodes2, tets2
    ok, _ = _faces_conforming(tets)
    assert ok


def test_sample_surface_area_uniform_and_deterministic():
    """area-weighted samples with a fixed seed."""
    from paper_2203_10000_b200._native import sample_surface
    xyz = np.array([[0, 0, 0], [4, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]], np.float64)
    tri = np.array([[0, 1, 2], [3, 4, 5]], np.uint32)   # areas 2.0 (z=0) and 0.5 (z=1)
    a = sample_surface(xyz, tri, 20000, seed=7)
    b = sample_surface(xyz, tri, 20000, seed=7)
    np.testing.assert_array_equal(a, b)
    assert np.all(a[:, 0] >= 0) and np.all(a[:, 1] >= 0)
    on_big = a[:, 2] == 0
    assert abs(on_big.mean() - 0.8) < 0.015                    # area-weighted triangle choice
    assert np.all(a[on_big, 0] + 4 * a[on_big, 1] <= 4 + 1e-12)  # inside the big triangle
    x = a[on_big, 0]
    assert abs(np.mean(x) - 4 / 3) < 0.03                      # uniform within it (centroid x = 4/3)


def test_oracle_point_triangle_distance_kats():
    tri = np.array([[0, 1, 2]], np.uint32)
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float64)
    pts = np.array([[0.2, 0.2, 0.5], [2.0, 0.0, 0.0], [-1.0, -1.0, 0.0], [0.5, -2.0, 0.0], [0.6, 0.6, 0.0]])
    d = oracle.point_surface_distance(pts, xyz, tri)
    np.testing.assert_allclose(d, [0.5, 1.0, np.sqrt(2.0), 2.0, np.sqrt(2) * 0.1], rtol=1e-12)


def test_refine_under_sanitizers(tmp_path):
    """csrc/refine.cpp (host code of the C ABI) built with AddressSanitizer +
    UBSan and driven through nm_refine / nm_mesh_* on random selections
    (tests/cpp/refine_asan.cpp): no memory or UB finding, invariants hold."""
    import shutil
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    cuda = Path("/usr/local/cuda")
    if shutil.which("g++") is None or not (cuda / "include" / "cuda_runtime.h").exists():
        pytest.skip("g++ or CUDA headers missing")
    exe = tmp_path / "refine_asan"
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-fno-omit-frame-pointer", f"-I{root / 'include'}", f"-I{cuda / 'include'}",
           str(root / "tests" / "cpp" / "refine_asan.cpp"), str(root / "paper_2203_10000_b200" / "csrc" / "refine.cpp"),
           f"-L{cuda / 'lib64'}", "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "refine_asan ok" in r.stdout
