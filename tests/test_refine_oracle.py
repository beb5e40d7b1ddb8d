"""Refinement parity against the independent fp64 oracle (oracle/refine_oracle.cpp,
SPEC.md:285-321) and the SPEC's refinement properties. CPU tests: the
product's host refine_volume (nm_refine, csrc/refine.cpp); the device
refinement (refine.cuh) is compared with the same oracle in
tests/test_gpu_refine_oracle.py.

Comparison: node arrays bit for bit (old nodes first, midpoints in
ascending edge order, fp64 0.5 (a + b)); children as (parent, sorted node
ids, label) tables (the SPEC fixes the templates, the shortest-diagonal rule
and the lowest-index tie-breaks, not the order of children inside a parent);
every child positively oriented."""
import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import refine

from test_synth import _faces_conforming, _volumes

F = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])


def assert_same_refinement(prod, orc):
    pn, pt, pl, pp = prod[:4]
    on, ot, ol, op = orc
    np.testing.assert_array_equal(pn, on)
    assert pt.shape == ot.shape
    np.testing.assert_array_equal(oracle.canonical_children(pt, pl, pp), oracle.canonical_children(ot, ol, op))
    assert np.all(_volumes(pn, pt) > 0) and np.all(_volumes(on, ot) > 0)


def interface_tets(tets, labels, a, b):
    """refine_boundary's selection: tets labeled a or b sharing
    a face with a tet of the other label."""
    f = np.sort(tets[:, F].reshape(-1, 3).astype(np.int64), axis=1)
    key = (f[:, 0] << 42) | (f[:, 1] << 21) | f[:, 2]
    order = np.argsort(key, kind="stable")
    k = key[order]
    same = np.flatnonzero(k[1:] == k[:-1])
    t1, t2 = order[same] // 4, order[same + 1] // 4
    sel = np.zeros(tets.shape[0], bool)
    for x, y in ((t1, t2), (t2, t1)):
        m = ((labels[x] == a) & (labels[y] == b)) | ((labels[x] == b) & (labels[y] == a))
        sel[x[m]] = True
    return np.flatnonzero(sel)


def interface_faces(tets, labels, a, b):
    f = np.sort(tets[:, F].reshape(-1, 3).astype(np.int64), axis=1)
    lab = np.repeat(labels, 4)
    key = (f[:, 0] << 42) | (f[:, 1] << 21) | f[:, 2]
    order = np.argsort(key, kind="stable")
    k = key[order]
    same = np.flatnonzero(k[1:] == k[:-1])
    i, j = order[same], order[same + 1]
    m = ((lab[i] == a) & (lab[j] == b)) | ((lab[i] == b) & (lab[j] == a))
    return f[i[m]]


def test_oracle_single_tet_and_identity():
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float64)
    tets = np.array([[0, 1, 2, 3]], np.uint32)
    on, ot, ol, op = oracle.refine_volume(nodes, tets, [7], [0])
    assert ot.shape[0] == 8 and on.shape[0] == 10 and np.all(ol == 7)
    v = _volumes(on, ot)
    assert np.all(v > 0) and abs(v.sum() - 1.0 / 6.0) < 1e-15
    on, ot, ol, op = oracle.refine_volume(nodes, tets, [7], [])
    np.testing.assert_array_equal(on, nodes)
    np.testing.assert_array_equal(ot, tets)
    with pytest.raises(ValueError, match="InvalidSelection"):
        oracle.refine_volume(nodes, tets, [7], [3])


@pytest.mark.parametrize("sel", range(5))
def test_host_refine_equals_oracle_cube(sel):
    """one tet of a 5-tet cube."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (1, 1, 1))
    labels = np.arange(1, 6, dtype=np.int32)
    assert_same_refinement(refine(nodes, tets, labels, [sel]), oracle.refine_volume(nodes, tets, labels, [sel]))


@pytest.mark.parametrize("seed,frac", [(0, 0.02), (1, 0.1), (2, 0.3), (3, 0.6)])
def test_host_refine_equals_oracle_random(seed, frac):
    """Random selections on a perturbed lattice (no diagonal ties) and on the
    exact lattice (every octahedron has tied diagonals: the lowest-index
    tie-break decides)."""
    rng = np.random.default_rng(seed)
    nodes, tets = synth.lattice_mesh((-1.0, 0.5, 2.0), 0.8, (7, 6, 8))
    labels = rng.integers(0, 4, tets.shape[0]).astype(np.int32)
    sel = np.flatnonzero(rng.random(tets.shape[0]) < frac)
    for pts in (nodes, nodes + rng.normal(scale=0.02, size=nodes.shape)):
        prod = refine(pts, tets, labels, sel)
        orc = oracle.refine_volume(pts, tets, labels, sel)
        assert_same_refinement(prod, orc)
        ok, _ = _faces_conforming(orc[1])
        assert ok


def test_escalation_patterns():
    """Transition patterns outside Fig. 2(c-e) escalate to the 1:8 split
    (SPEC.md:321): two tets whose split edges end up opposite / spread over
    4 vertices; checked against the oracle on every pair selection of a
    2x2x2 lattice."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (2, 2, 2))
    labels = np.ones(tets.shape[0], np.int32)
    rng = np.random.default_rng(5)
    for _ in range(40):
        sel = rng.choice(tets.shape[0], 2, replace=False)
        prod = refine(nodes, tets, labels, sel)
        orc = oracle.refine_volume(nodes, tets, labels, sel)
        assert_same_refinement(prod, orc)
        # more children than the 2 x 8 selected ones: neighbours got templates or escalated
        assert orc[1].shape[0] > tets.shape[0] + 14


def test_refine_straddle_selection_equals_oracle():
    """The recursive driver's selection (straddle tets of a labeled two-sphere
    mesh), two levels, product == oracle at each level."""
    R = 10.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 2), synth.icosphere(R, 2)], labels=[1, 2])
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, R / 5, (13, 13, 13))
    masks = oracle.label_nodes(nodes, S)
    labels = oracle.label_tets(tets, masks, S.label_ids)
    for _ in range(2):
        sel = oracle.flag_boundary(tets, masks)
        prod = refine(nodes, tets, labels, sel)
        orc = oracle.refine_volume(nodes, tets, labels, sel)
        assert_same_refinement(prod, orc)
        nodes, tets, labels = orc[0], orc[1], orc[2]
        masks = oracle.label_nodes(nodes, S)


def test_volume_conservation_and_conformity():
    """SPEC.md:304-305 on the oracle's own output."""
    rng = np.random.default_rng(11)
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (6, 6, 6))
    nodes = nodes + rng.normal(scale=0.05, size=nodes.shape)
    sel = np.flatnonzero(rng.random(tets.shape[0]) < 0.2)
    on, ot, ol, op = oracle.refine_volume(nodes, tets, None, sel)
    v0, v = _volumes(nodes, tets), _volumes(on, ot)
    assert abs(v.sum() - v0.sum()) <= 1e-12 * v0.sum()
    vp = np.zeros(tets.shape[0])
    np.add.at(vp, op, v)
    np.testing.assert_allclose(vp, v0, rtol=1e-12, atol=0)
    ok, _ = _faces_conforming(ot)
    assert ok
    if oracle.ref_available():
        import ctypes
        D, U = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint32)
        assert oracle.ref().ref_validate_mesh_ok(on.ctypes.data_as(D), on.shape[0], ot.ctypes.data_as(U),
                                                 ot.shape[0]) == 1


def _half_cube(n=6):
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (n, n, n))
    cen = nodes[tets].mean(axis=1)
    labels = np.where(cen[:, 0] < n / 2, 1, 2).astype(np.int32)
    return nodes, tets, labels


def test_repeated_boundary_refinement_quadruples_linear_density():
    """refine_boundary twice -> 4x linear density at the
    interface. Both sides' layers are split 1:8, so every interface face is
    split 1:4 per level: after two levels the interface edges are exactly a
    quarter of the original ones, 16 faces per original face."""
    nodes, tets, labels = _half_cube()
    f0 = interface_faces(tets, labels, 1, 2)
    n, t, l = nodes, tets, labels
    for _ in range(2):
        sel = interface_tets(t, l, 1, 2)
        prod = refine(n, t, l, sel)
        orc = oracle.refine_volume(n, t, l, sel)
        assert_same_refinement(prod, orc)
        n, t, l = orc[0], orc[1], orc[2]
    f2 = interface_faces(t, l, 1, 2)
    assert f2.shape[0] == 16 * f0.shape[0]

    def edge_lengths(P, faces):
        e = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [0, 2]]])
        e = np.unique(np.sort(e, axis=1), axis=0)
        return np.linalg.norm(P[e[:, 0]] - P[e[:, 1]], axis=1)

    l0, l2 = np.sort(edge_lengths(nodes, f0)), np.sort(edge_lengths(n, f2))
    np.testing.assert_allclose(np.unique(l2), np.unique(l0) / 4.0, rtol=1e-14)
    assert abs(np.median(l2) - np.median(l0) / 4.0) < 1e-12


def test_subdivision_consistency():
    """after two levels, the nodes on every original interface
    edge (a, b) are the direct 4x-split points a + k/4 (b - a), k = 1, 2, 3
    (bit for bit on the dyadic lattice)."""
    nodes, tets, labels = _half_cube(4)
    f0 = interface_faces(tets, labels, 1, 2)
    n, t, l = nodes, tets, labels
    for _ in range(2):
        n, t, l, _ = oracle.refine_volume(n, t, l, interface_tets(t, l, 1, 2))
    have = {tuple(p) for p in n.tolist()}
    e = np.unique(np.sort(np.concatenate([f0[:, [0, 1]], f0[:, [1, 2]], f0[:, [0, 2]]]), axis=1), axis=0)
    for a, b in e:
        A, B = nodes[a], nodes[b]
        for k in (1, 2, 3):
            assert tuple((A + (B - A) * (k / 4.0)).tolist()) in have
