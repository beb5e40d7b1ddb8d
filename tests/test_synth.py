"""The caller-side generators (csrc/synth.cpp) pinned against the UNMODIFIED
reference generators (oracle/_ref: primitives.hpp, lattice.hpp), directly when
the reference is present and through committed sha256 fixtures otherwise;
plus the reference's own lattice tests (proj/tests/test_lattice.cpp)
re-expressed without Catch2. CPU only."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_icosphere_matches_reference_fixture():
    g = json.loads((GOLDEN / "ref_generators.json").read_text())
    for lvl in range(0, 7):
        assert sha(*synth.icosphere(1.0, lvl)) == g[f"icosphere_1_L{lvl}"], lvl
    assert sha(*synth.icosphere(10.0, 3)) == g["icosphere_10_L3"]
    assert sha(*synth.icosphere(100.0, 4, (3.0, -7.0, 11.0))) == g["icosphere_100_L4_off"]


def test_lattice_matches_reference_fixture():
    g = json.loads((GOLDEN / "ref_generators.json").read_text())
    for (o, h, n) in [((-12.0, -12.0, -12.0), 0.75, (32, 32, 32)), ((-2.0, 1.0, 0.5), 1.25, (3, 4, 2)),
                      ((0.0, 0.0, 0.0), 1.0, (1, 1, 1))]:
        assert sha(*synth.lattice_mesh(o, h, n)) == g[f"lattice_{o}_{h}_{n}"]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_generators_bitwise_vs_reference_live():
    import ctypes
    R = oracle.ref()
    D = ctypes.POINTER(ctypes.c_double)
    U = ctypes.POINTER(ctypes.c_uint32)
    for r, lvl, c in [(1.0, 5, (0, 0, 0)), (37.5, 2, (1.5, -2.0, 3.25))]:
        x, t = synth.icosphere(r, lvl, c)
        rx, rt = np.empty_like(x), np.empty_like(t)
        cc = np.asarray(c, np.float64)
        R.ref_icosphere(r, lvl, cc.ctypes.data_as(D), rx.ctypes.data_as(D), rt.ctypes.data_as(U))
        np.testing.assert_array_equal(x, rx)
        np.testing.assert_array_equal(t, rt)
    for n in [(1, 1, 1), (2, 3, 4), (5, 1, 2)]:
        nodes, tets = synth.lattice_mesh((0.5, -1.0, 2.0), 0.7, n)
        rn, rt = np.empty_like(nodes), np.empty_like(tets)
        o = np.array([0.5, -1.0, 2.0])
        R.ref_lattice_mesh(o.ctypes.data_as(D), 0.7, *n, rn.ctypes.data_as(D), rt.ctypes.data_as(U))
        np.testing.assert_array_equal(nodes, rn)
        np.testing.assert_array_equal(tets, rt)
    bx, bt = synth.box_surface([0, 1, 2], [3, 5, 7])
    rx, rt = np.empty_like(bx), np.empty_like(bt)
    lo, hi = np.array([0.0, 1, 2]), np.array([3.0, 5, 7])
    R.ref_box_surface(lo.ctypes.data_as(D), hi.ctypes.data_as(D), rx.ctypes.data_as(D), rt.ctypes.data_as(U))
    np.testing.assert_array_equal(bx, rx)
    np.testing.assert_array_equal(bt, rt)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_config_surfaces_closed_and_outward():
    """Labeling precondition: every compartment closed
    (surface.hpp:80-104) and outward (signed volume > 0, surface.hpp:40-45)."""
    import ctypes
    R = oracle.ref()
    D = ctypes.POINTER(ctypes.c_double)
    U = ctypes.POINTER(ctypes.c_uint32)
    for cid in (1, 2, 3, 5):
        S = synth.config(cid).surfaces
        for k in range(S.K):
            x, t = S.compartment(k)
            x = np.ascontiguousarray(x)
            t = np.ascontiguousarray(t)
            assert R.ref_validate_closed(x.ctypes.data_as(D), x.shape[0], t.ctypes.data_as(U), t.shape[0]) == 0
            assert R.ref_signed_volume(x.ctypes.data_as(D), x.shape[0], t.ctypes.data_as(U), t.shape[0]) > 0


def _volumes(nodes, tets):
    a, b, c, d = (nodes[tets[:, i]] for i in range(4))
    return np.einsum("ij,ij->i", b - a, np.cross(c - a, d - a)) / 6.0


def _faces_conforming(tets):
    """Every interior face shared by exactly 2 tets with opposite orientation
    (the check of mesh.hpp:194-235, vectorised)."""
    F = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])
    f = tets[:, F].reshape(-1, 3).astype(np.int64)
    key = np.sort(f, axis=1)
    inv = (f[:, 0] > f[:, 1]).astype(int) + (f[:, 0] > f[:, 2]) + (f[:, 1] > f[:, 2])
    _, idx, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    par = np.zeros(cnt.size, int)
    np.add.at(par, idx.ravel(), inv & 1)
    return bool(np.all(cnt <= 2) and np.all(par[cnt == 2] == 1)), int(np.sum(cnt == 1))


def test_lattice_single_cell():
    """test_lattice.cpp:10-23: 8 nodes, 5 tets, volumes {1/6 x4, 1/3}."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (1, 1, 1))
    assert nodes.shape == (8, 3) and tets.shape == (5, 4)
    v = np.sort(_volumes(nodes, tets))
    np.testing.assert_allclose(v, [1 / 6] * 4 + [1 / 3], atol=1e-15)


def test_lattice_conformity_and_volume():
    """test_lattice.cpp:25-75: 2^3 -> 27 nodes / 40 tets; all counts in
    {1..4}^3 conforming with 5 tets/cell and exact volume; boundary faces =
    2 x boundary quads."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (2, 2, 2))
    assert nodes.shape[0] == 27 and tets.shape[0] == 40
    h = 1.25
    for nx in range(1, 5):
        for ny in range(1, 5):
            for nz in range(1, 5):
                nodes, tets = synth.lattice_mesh((-2.0, 1.0, 0.5), h, (nx, ny, nz))
                assert tets.shape[0] == 5 * nx * ny * nz
                v = _volumes(nodes, tets)
                assert np.all(v > 0)
                assert abs(v.sum() - nx * ny * nz * h ** 3) <= 1e-9 * nx * ny * nz * h ** 3
                ok, nb = _faces_conforming(tets)
                assert ok
                assert nb == 2 * 2 * (nx * ny + ny * nz + nx * nz)


def test_lattice_deterministic():
    """test_lattice.cpp:77-86: identical spec -> bit-identical mesh."""
    a = synth.lattice_mesh((0.1, 0.2, 0.3), 0.9, (4, 3, 5))
    b = synth.lattice_mesh((0.1, 0.2, 0.3), 0.9, (4, 3, 5))
    assert sha(*a) == sha(*b)


def test_config_shapes():
    c1 = synth.config(1)
    assert (c1.surfaces.K, c1.surfaces.n_triangles, c1.n, c1.n_nodes) == (1, 1280, (32, 32, 32), 35937)
    c2 = synth.config(2)
    assert c2.surfaces.K == 4 and c2.surfaces.n_triangles == 35840
    c3 = synth.config(3)
    assert c3.surfaces.K == 20 and c3.surfaces.n_triangles == 363520 and c3.n == (174, 214, 204)
    assert list(c3.surfaces.priorities) == list(range(1, 21))
    c5 = synth.config(5)
    assert c5.surfaces.K == 12 and c5.surfaces.n_triangles == 983040
    assert c5.n == (215, 215, 215) and c5.n_nodes == 10077696 and c5.n_tets == 49691875
