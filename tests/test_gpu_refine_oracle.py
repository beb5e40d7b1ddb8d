"""Device refinement and the recursive driver against the independent fp64
refinement oracle (oracle/refine_oracle.cpp), plus the
SPEC's relabel_recursive examples on the GPU path and the
refinement quality property of SPEC.md:308."""
import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200.quality import boundary_distance

from test_refine_oracle import assert_same_refinement, interface_tets

pytestmark = pytest.mark.gpu


def test_device_refine_equals_oracle_cfg2_straddle(ctx):
    """cfg2 full lattice (1.17M nodes, 6.1M tets): the straddle selection of
    the GPU masks, refined on the device (nm_refine_device) == the oracle's
    refinement of the same selection (nodes bitwise, children as sets)."""
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    labels, masks, _ = ctx.label_mesh(nodes, tets, want_masks=True)
    sel = ctx.flag_boundary(tets, masks)
    np.testing.assert_array_equal(sel, oracle.flag_boundary(tets, masks))
    assert sel.size > 100_000
    dev = ctx.refine_device(nodes, tets, labels, sel)
    orc = oracle.refine_volume(nodes, tets, labels, sel)
    assert_same_refinement(dev, orc)


def test_refine_relabel_levels_equal_oracle_chain(ctx):
    """nm_refine_relabel, 2 levels on a cfg2-like nested-sphere mesh: each
    level's mesh equals the oracle refinement of the straddle selection of the
    previous level's (oracle-checked) masks; final masks/labels equal the
    oracle's labeling of the final mesh."""
    R = 40.0
    S = synth.concat_surfaces([synth.icosphere(0.7 * R, 4), synth.icosphere(R, 4)], labels=[3, 5])
    nodes, tets = synth.lattice_mesh((-1.2 * R,) * 3, R / 8, (20, 20, 20))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    n2, t2, lab, masks, st = ctx.refine_relabel(nodes, tets, levels=2)
    m = oracle.label_nodes(nodes, S)
    n, t, l = nodes, tets, oracle.label_tets(tets, m, S.label_ids)
    for _ in range(2):
        on, ot, ol, op = oracle.refine_volume(n, t, l, oracle.flag_boundary(t, m))
        m = np.concatenate([m, oracle.label_nodes(on[n.shape[0]:], S)])
        n, t, l = on, ot, oracle.label_tets(ot, m, S.label_ids)
    np.testing.assert_array_equal(n2, n)
    np.testing.assert_array_equal(np.sort(np.sort(t2, axis=1), axis=0), np.sort(np.sort(t, axis=1), axis=0))
    np.testing.assert_array_equal(masks, m)
    # labels per tet (as node-id sets) agree
    a = oracle.canonical_children(t2, lab, np.zeros(t2.shape[0]))
    b = oracle.canonical_children(t, l, np.zeros(t.shape[0]))
    np.testing.assert_array_equal(a, b)


def test_refine_boundary_device_equals_oracle(ctx):
    """refine_boundary on the device, twice: each level
    == oracle refine_volume of the interface layers."""
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (8, 8, 8))
    cen = nodes[tets].mean(axis=1)
    labels = np.where(np.linalg.norm(cen - 4.0, axis=1) < 2.7, 1, 2).astype(np.int32)
    n, t, l = nodes, tets, labels
    for _ in range(2):
        dn, dt, dl, dp, _ = ctx.refine_boundary(n, t, l, 1, 2)
        orc = oracle.refine_volume(n, t, l, interface_tets(t, l, 1, 2))
        assert_same_refinement((dn, dt, dl, dp), orc)
        n, t, l = dn, dt, dl


def _two_sphere(div):
    R = 30.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 3), synth.icosphere(R, 3)], labels=[1, 2])
    coarse = synth.concat_surfaces([synth.icosphere(0.6 * R, 1), synth.icosphere(R, 1)], labels=[1, 2])
    h = R / div
    n = int(np.ceil(2.6 * R / h))
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, h, (n, n, n))
    return S, coarse, nodes, tets


def test_relabel_nonconvergence_reported(ctx):
    """max_iters passes without a fixed point -> NonConvergence
    (converged = 0) with the best labels; the oracle agrees on the pass count
    and the labels after the same capped iteration."""
    S, coarse, nodes, tets = _two_sphere(6)
    prev = oracle.label_tets(tets, oracle.label_nodes(nodes, coarse), coarse.label_ids)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    lab_full, passes_full, conv_full, _, _ = ctx.relabel(nodes, tets, prev)
    assert conv_full and passes_full >= 2
    lab1, passes1, conv1, _, _ = ctx.relabel(nodes, tets, prev, max_iters=1)
    assert passes1 == 1 and not conv1
    lo, po, co, _ = oracle.relabel_recursive(nodes, tets, S, prev, max_iters=1)
    assert po == 1 and not co
    np.testing.assert_array_equal(lab1, lo)


def test_single_misassigned_tet_fixed_within_two_passes(ctx):
    """SPEC.md:251 (Fig. 3 analogue) on the GPU path: one boundary tet with a
    wrong label is corrected in <= 2 passes, result == initial_label."""
    S, _, nodes, tets = _two_sphere(8)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    init, masks, _ = ctx.label_mesh(nodes, tets, want_masks=True)
    boundary = ctx.flag_boundary(tets, masks)
    rng = np.random.default_rng(3)
    for t in rng.choice(boundary, 5, replace=False):
        prev = init.copy()
        prev[t] = 2 if init[t] != 2 else 1
        lab, passes, conv, ev, st = ctx.relabel(nodes, tets, prev, want_evaluated=True)
        assert conv and passes <= 2
        np.testing.assert_array_equal(lab, init)
        assert ev.sum() < nodes.shape[0] // 2       # only the frontier of the label-change faces was evaluated


def test_boundary_distance_median_does_not_increase(ctx):
    """after refine_boundary + relabel_recursive the boundary-
    distance median (quality.boundary_distance of the extracted compartment
    boundary to the segmentation surface) does not increase; two rounds."""
    sx, st_ = synth.icosphere(20.0, 4, center=(0.3, -0.2, 0.1))
    S = synth.single_surface(sx, st_, label=1)
    nodes, tets = synth.lattice_mesh((-26.0,) * 3, 4.0, (13, 13, 13))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    labels, _, _ = ctx.label_mesh(nodes, tets)
    medians = []
    for level in range(3):
        btri, _ = ctx.extract_boundary(tets, labels, [1])
        medians.append(boundary_distance(ctx, nodes, btri, sx, st_, samples=20000, seed=level)["median"])
        if level == 2:
            break
        nodes, tets, inherited, _, _ = ctx.refine_boundary(nodes, tets, labels, 1, 0)
        labels, passes, conv, _, _ = ctx.relabel(nodes, tets, inherited)
        assert conv
        full, _, _ = ctx.label_mesh(nodes, tets)
        np.testing.assert_array_equal(labels, full)     # relabel == initial
    assert medians[1] <= medians[0] and medians[2] <= medians[1], medians
