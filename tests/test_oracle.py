"""The CPU oracle (oracle/labeling_oracle.cpp) pinned before it is trusted:
SPEC.md known-answer examples, analytic values, an independent formula
(L'Huilier), the SPEC invariants (:253-257) and the committed golden fixture.
CPU only."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden"


def _surface(spec):
    if spec[0] == "icosphere":
        return synth.single_surface(*synth.icosphere(spec[1], spec[2]))
    return synth.single_surface(*synth.box_surface(spec[1], spec[2]))


def test_spec_kats():
    kats = json.loads((GOLDEN / "spec_kats.json").read_text())
    for case in kats["cases"]:
        S = _surface(case["surface"])
        s = oracle.enclosure(np.array([case["point"]], np.float64), S)[0, 0]
        assert abs(s - case["expect"]) <= case["tol"], case


def test_golden_cfg1():
    g = json.loads((GOLDEN / "oracle_cfg1.json").read_text())
    cfg = synth.config(1)
    nodes, tets = cfg.lattice_mesh()
    m, s = oracle.label_nodes(nodes, cfg.surfaces, want_s=True)
    lab = oracle.label_tets(tets, m, cfg.surfaces.label_ids)
    assert int(m.sum()) == g["inside_nodes"] == 9795
    assert hashlib.sha256(m.tobytes()).hexdigest() == g["mask_sha256"]
    assert hashlib.sha256(lab.tobytes()).hexdigest() == g["label_sha256"]
    np.testing.assert_array_equal(s[g["s_idx"], 0], np.array(g["s"]))


def test_lhuilier_cross_check():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        p, a, b, c = rng.normal(size=(4, 3)) * rng.uniform(0.1, 100)
        S = synth.single_surface(np.array([a, b, c]), np.array([[0, 1, 2]], np.uint32))
        vos = 4 * np.pi * oracle.enclosure(p[None], S)[0, 0]
        lh = oracle.lhuilier(p, a, b, c)
        assert abs(vos - lh) <= 1e-9 * max(1.0, abs(lh)), (vos, lh)


def test_additivity_split_box():
    """a box split into two boxes sharing an interface."""
    big = synth.single_surface(*synth.box_surface([0, 0, 0], [2, 1, 1]))
    a = synth.single_surface(*synth.box_surface([0, 0, 0], [1, 1, 1]))
    b = synth.single_surface(*synth.box_surface([1, 0, 0], [2, 1, 1]))
    pts = np.random.default_rng(4).uniform(-1, 3, (500, 3))
    pts = pts[np.abs(pts[:, 0] - 1) > 1e-3]
    sb, sa, sc = (oracle.enclosure(pts, X)[:, 0] for X in (big, a, b))
    np.testing.assert_allclose(sb, sa + sc, atol=1e-12)


def test_rigid_invariance():
    """translation/rotation invariance to 1e-9."""
    xyz, tri = synth.icosphere(5.0, 3)
    pts = np.random.default_rng(5).uniform(-8, 8, (300, 3))
    s0 = oracle.enclosure(pts, synth.single_surface(xyz, tri))
    th = 0.7
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]]) @ \
        np.array([[1, 0, 0], [0, np.cos(0.3), -np.sin(0.3)], [0, np.sin(0.3), np.cos(0.3)]])
    t = np.array([13.0, -4.0, 120.0])
    s1 = oracle.enclosure(pts @ R.T + t, synth.single_surface(xyz @ R.T + t, tri))
    np.testing.assert_allclose(s0, s1, atol=1e-9)


def test_worker_count_independence():
    """SPEC.md:265 / acceptance #8: bit-identical for any worker count."""
    cfg = synth.config(2)
    pts = cfg.lattice_nodes()[::997]
    ref = oracle.enclosure(pts, cfg.surfaces, workers=1)
    for w in (2, 3, 8):
        np.testing.assert_array_equal(oracle.enclosure(pts, cfg.surfaces, workers=w), ref)


def _lattice_over(R, h, margin=1.7):
    n = int(np.ceil(2 * margin * R / h))
    return synth.lattice_mesh((-margin * R,) * 3, h, (n, n, n))


def _tet_volumes(nodes, tets):
    a, b, c, d = (nodes[tets[:, i]] for i in range(4))
    return np.einsum("ij,ij->i", b - a, np.cross(c - a, d - a)) / 6.0, (a + b + c + d) / 4.0


def test_sphere_volume_kat():
    """SPEC.md:240 'labeled-tet volume / sphere volume in [0.9, 1.0] at
    h = R/10'. With the paper's node rule ('four nodes inside')
    the labeled set is an inner approximation whose deficit is ~3ch/R: at
    h = R/10 it is 0.81 on the 5-tet lattice, and it enters SPEC's band at
    h = R/20 (DESIGN.md §7 records this deviation). The tet-centroid reading
    lands within 1 % of the sphere already at R/10."""
    R = 10.0
    S = synth.single_surface(*synth.icosphere(R, 4))
    V = 4 / 3 * np.pi * R ** 3
    for div, lo in ((10, 0.78), (20, 0.9)):
        nodes, tets = _lattice_over(R, R / div)
        vol, cen = _tet_volumes(nodes, tets)
        assert np.all(vol > 0)
        lab = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
        ratio = vol[lab == 1].sum() / V
        assert lo <= ratio <= 1.0, (div, ratio)
        if div == 10:
            mc = oracle.label_nodes(cen, S)
            assert abs(vol[mc == 1].sum() / V - 1.0) <= 0.01


def test_monotone_nesting_and_enclosing():
    """concentric spheres nest; an enclosing surface
    labels everything."""
    R = 10.0
    S = synth.concat_surfaces([synth.icosphere(R, 4), synth.icosphere(1.5 * R, 4)], labels=[1, 2])
    nodes, tets = _lattice_over(R, R / 10)
    m = oracle.label_nodes(nodes, S)
    assert np.all(((m & 1) != 0) <= ((m & 2) != 0))  # inside inner => inside outer
    lab = oracle.label_tets(tets, m, S.label_ids)
    inner_only = oracle.label_tets(tets, m & 1, S.label_ids) == 1
    outer_any = oracle.label_tets(tets, m & 2, S.label_ids) == 2
    assert np.all(inner_only <= outer_any)
    assert set(np.unique(lab)) == {0, 1, 2}
    big = synth.single_surface(*synth.icosphere(10 * R, 3), label=7)
    mb = oracle.label_nodes(nodes, big)
    assert np.all(oracle.label_tets(tets, mb, big.label_ids) == 7)


def test_priority_after_threshold():
    """intersecting surfaces -> the innermost-listed wins."""
    a = synth.icosphere(5.0, 3, center=(-2.0, 0, 0))
    b = synth.icosphere(5.0, 3, center=(2.0, 0, 0))
    S = synth.concat_surfaces([a, b], labels=[11, 22])
    pts = np.array([[0.0, 0, 0], [-5.0, 0, 0], [5.0, 0, 0], [20.0, 0, 0]])
    m = oracle.label_nodes(pts, S)
    assert list(m) == [3, 1, 2, 0]
    tets = np.array([[0, 0, 0, 0], [1, 1, 1, 1], [2, 2, 2, 2], [3, 3, 3, 3], [0, 1, 2, 3]], np.uint32)
    assert list(oracle.label_tets(tets, m, S.label_ids)) == [11, 11, 22, 0, 0]


def test_flag_boundary_oracle():
    masks = np.array([0b01, 0b01, 0b11, 0b00], np.uint32)
    tets = np.array([[0, 1, 0, 1], [0, 1, 2, 0], [0, 1, 3, 0], [2, 2, 2, 2]], np.uint32)
    assert list(oracle.flag_boundary(tets, masks)) == [1, 2]
    assert list(oracle.flag_boundary(tets, masks, active_mask=0b10)) == [1]


@pytest.fixture(scope="module")
def two_sphere():
    """Acceptance #2 fixture: two concentric spheres (R, 0.6 R)."""
    R = 30.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 3), synth.icosphere(R, 3)], labels=[1, 2])
    return R, S


@pytest.mark.parametrize("div", [6, 10])
def test_relabel_equals_initial(two_sphere, div):
    """SPEC.md:249 / acceptance #2: recursive relabel == initial labeling at
    h in {R/6, R/10}, starting from labels inherited from a coarser surface."""
    R, S = two_sphere
    h = R / div
    n = int(np.ceil(2.6 * R / h))
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, h, (n, n, n))
    init = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
    coarse = synth.concat_surfaces([synth.icosphere(0.6 * R, 1), synth.icosphere(R, 1)], labels=[1, 2])
    prev = oracle.label_tets(tets, oracle.label_nodes(nodes, coarse), coarse.label_ids)
    assert np.any(prev != init)
    lab, passes, conv, ev = oracle.relabel_recursive(nodes, tets, S, prev)
    assert conv
    np.testing.assert_array_equal(lab, init)
    assert ev.sum() < nodes.shape[0]  # only a boundary band was evaluated


def test_relabel_fixed_point_and_single_fix(two_sphere):
    """converged input -> 1 pass, no change; one mislabeled
    boundary tet -> corrected within <= 2 passes."""
    R, S = two_sphere
    h = R / 6
    n = int(np.ceil(2.6 * R / h))
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, h, (n, n, n))
    init = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
    lab, passes, conv, _ = oracle.relabel_recursive(nodes, tets, S, init)
    assert conv and passes == 1
    np.testing.assert_array_equal(lab, init)
    # flip one tet next to the 1|2 interface
    bad = init.copy()
    i = int(np.flatnonzero(init == 1)[0])
    bad[i] = 2
    lab, passes, conv, _ = oracle.relabel_recursive(nodes, tets, S, bad)
    assert conv and passes <= 2
    np.testing.assert_array_equal(lab, init)
