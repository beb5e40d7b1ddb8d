"""GPU parity: the sm_100a labeling path (through the C ABI) against the fp64
CPU oracle on the same seeded inputs.

Bars:
  * node masks and tet labels bit-exact with the oracle, except pairs whose
    oracle ratio lies within TIE_EPS of T (counted, must be none here);
  * per-(point, compartment) |s_gpu - s_oracle| <= S_TOL (SPEC.md:262's 1e-4;
    the kernel is expected to land ~1e-6).
"""
import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth

pytestmark = pytest.mark.gpu

S_TOL = 1e-4      # SPEC.md:262 approximation tolerance (absolute, on s)
# What the fp32 pass achieves for UNflagged pairs: the subtile frames are
# watertight (vertices snapped to a common grid, exact in fp32 in every
# subtile) and near a surface R = v - p is formed from a double-single point,
# so every term is accurate to ~ulp of its own geometry; the worst pair over
# the FULL cfg2 mesh is 2.0e-6 (profiles/r02/diag_cfg2_strips_watertight.txt;
# 6.6e-5 before the watertight frames, diag_cfg2_before_watertight.txt).
S_EXPECT = 1e-5
TIE_EPS = 1e-9


def _compare_masks(m_gpu, m_ref, s_ref, T=0.5):
    K = s_ref.shape[1]
    bits = (np.arange(K, dtype=np.uint32))
    g = ((m_gpu[:, None] >> bits) & 1).astype(bool)
    r = ((m_ref[:, None] >> bits) & 1).astype(bool)
    tie = np.abs(s_ref - T) < TIE_EPS
    bad = (g != r) & ~tie
    return int(bad.sum()), int(tie.sum())


def test_cfg1_full_parity(ctx):
    cfg = synth.config(1)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    s_gpu, st = ctx.enclosure(nodes)
    m_ref, s_ref = oracle.label_nodes(nodes, S, want_s=True)
    assert np.max(np.abs(s_gpu - s_ref)) <= S_TOL
    assert np.max(np.abs(s_gpu - s_ref)) <= S_EXPECT
    labels, masks, st2 = ctx.label_mesh(nodes, tets, want_masks=True)
    bad, ties = _compare_masks(masks, m_ref, s_ref)
    assert bad == 0 and ties == 0
    assert int(m_ref.sum()) == 9795  # SURVEY.md §8d probe count for cfg1
    lab_ref = oracle.label_tets(tets, m_ref, S.label_ids)
    np.testing.assert_array_equal(labels, lab_ref)
    assert st2["evals"] == nodes.shape[0] * S.n_triangles


def test_cfg2_sample_parity(ctx):
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()
    rng = np.random.default_rng(2)
    idx = np.sort(rng.choice(nodes.shape[0], 20000, replace=False))
    pts = nodes[idx]
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    s_gpu, _ = ctx.enclosure(pts)
    m_ref, s_ref = oracle.label_nodes(pts, S, want_s=True)
    assert np.max(np.abs(s_gpu - s_ref)) <= S_EXPECT
    m_gpu, _ = ctx.label_nodes(pts)
    bad, ties = _compare_masks(m_gpu, m_ref, s_ref)
    assert bad == 0
    # full-mesh masks are independent of which subset is evaluated with it
    m_all, _ = ctx.label_nodes(nodes)
    np.testing.assert_array_equal(m_all[idx], m_gpu)


def test_near_surface_adversarial(ctx):
    """Points 1e-5..1e-8 mm off faces, edges and vertices of an icosphere at
    ~100 mm coordinates: fp32 alone gets some of these on the wrong side; the
    detector + fp64 fix-up must return the oracle's answer."""
    xyz, tri = synth.icosphere(100.0, 4, center=(3.0, -7.0, 11.0))
    S = synth.single_surface(xyz, tri)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    rng = np.random.default_rng(7)
    pts = []
    for t in rng.choice(tri.shape[0], 400, replace=False):
        a, b, c = xyz[tri[t]]
        n = np.cross(b - a, c - a)
        n /= np.linalg.norm(n)
        for eps in (1e-5, 1e-6, 1e-7, 1e-8):
            for sgn in (1, -1):
                w = rng.dirichlet([1, 1, 1])
                pts.append(w[0] * a + w[1] * b + w[2] * c + sgn * eps * n)       # near face
                pts.append(0.5 * (a + b) + sgn * eps * n)                            # near edge
                pts.append(a + sgn * eps * n)                                        # near vertex
    pts = np.array(pts)
    s_ref = oracle.enclosure(pts, S)
    m_ref = (s_ref[:, 0] >= 0.5).astype(np.uint32)
    m_gpu, st = ctx.label_nodes(pts)
    tie = np.abs(s_ref[:, 0] - 0.5) < TIE_EPS
    assert np.count_nonzero((m_gpu != m_ref) & ~tie) == 0
    assert st["flagged_points"] > 0


def test_spec_kats_gpu(ctx):
    # SPEC.md:231-233
    xyz, tri = synth.icosphere(1.0, 4)
    ctx.set_surfaces(xyz, tri, np.array([0, tri.shape[0]], np.uint32), np.array([1], np.int32))
    s, _ = ctx.enclosure(np.array([[0.0, 0, 0], [3.0, 0, 0]]))
    assert abs(s[0, 0] - 1.0) <= 1e-6 and abs(s[1, 0]) <= 1e-6
    bx, bt = synth.box_surface([0, 0, 0], [1, 1, 1])
    ctx.set_surfaces(bx, bt, np.array([0, 12], np.uint32), np.array([1], np.int32))
    s, st = ctx.enclosure(np.array([[0.0, 0, 0], [0.5, 0, 0], [0.5, 0.5, 0], [0.5, 0.5, 0.5]]))
    np.testing.assert_allclose(s[:, 0], [0.125, 0.25, 0.5, 1.0], atol=1e-6)


def test_empty_and_ragged(ctx):
    xyz, tri = synth.icosphere(10.0, 2)
    ctx.set_surfaces(xyz, tri, np.array([0, tri.shape[0]], np.uint32), np.array([3], np.int32))
    m, st = ctx.label_nodes(np.zeros((0, 3)))
    assert m.shape == (0,)
    for n in (1, 31, 33, 511, 513, 1025):
        pts = np.random.default_rng(n).uniform(-12, 12, (n, 3))
        m, _ = ctx.label_nodes(pts)
        np.testing.assert_array_equal(m, oracle.label_nodes(pts, synth.single_surface(xyz, tri)))


@pytest.mark.parametrize("layout", [1, 2])
def test_layouts_agree_with_oracle(layout):
    """Both tile layouts (independent triangles, strip segments) against the
    oracle on cfg3 (20 intersecting compartments) — a seeded node sample."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(3)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()
    idx = np.sort(np.random.default_rng(30 + layout).choice(nodes.shape[0], 3000, replace=False))
    pts = nodes[idx]
    with Context(0, layout=layout) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        assert c.surface_info()["layout"] == ("strips" if layout == 2 else "triangles")
        s_gpu, st = c.enclosure(pts)
        m_gpu, _ = c.label_nodes(pts)
    m_ref, s_ref = oracle.label_nodes(pts, S, want_s=True)
    assert np.max(np.abs(s_gpu - s_ref)) <= S_EXPECT
    bad, _ = _compare_masks(m_gpu, m_ref, s_ref)
    assert bad == 0


@pytest.mark.parametrize("div", [6, 10])
def test_relabel_matches_oracle(ctx, div):
    """nm_relabel (device frontier + relabel passes) == oracle relabel_recursive
    == initial labeling on the two-sphere fixture (acceptance #2)."""
    R = 30.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 3), synth.icosphere(R, 3)], labels=[1, 2])
    coarse = synth.concat_surfaces([synth.icosphere(0.6 * R, 1), synth.icosphere(R, 1)], labels=[1, 2])
    h = R / div
    n = int(np.ceil(2.6 * R / h))
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, h, (n, n, n))
    init = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
    prev = oracle.label_tets(tets, oracle.label_nodes(nodes, coarse), coarse.label_ids)
    lab_o, passes_o, conv_o, ev_o = oracle.relabel_recursive(nodes, tets, S, prev)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    lab, passes, conv, ev, st = ctx.relabel(nodes, tets, prev, want_evaluated=True)
    assert conv and conv_o and passes == passes_o
    np.testing.assert_array_equal(lab, lab_o)
    np.testing.assert_array_equal(lab, init)
    np.testing.assert_array_equal(ev, ev_o)
    assert st["points"] == int(ev.sum()) < nodes.shape[0]
    # converged input: one pass, nothing changes
    lab2, passes2, conv2, _, _ = ctx.relabel(nodes, tets, init)
    assert conv2 and passes2 == 1
    np.testing.assert_array_equal(lab2, init)


def test_refine_relabel_driver(ctx):
    """nm_refine_relabel (device straddle compaction + host refine + device
    evaluation of new nodes only) == oracle initial labeling of the refined
    mesh, two levels (cfg4 analogue on a nested two-sphere)."""
    R = 20.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 3), synth.icosphere(R, 3)], labels=[1, 2])
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, R / 6, (16, 16, 16))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    n2, t2, lab, masks, st = ctx.refine_relabel(nodes, tets, levels=2)
    assert t2.shape[0] > tets.shape[0]
    m_ref = oracle.label_nodes(n2, S)
    np.testing.assert_array_equal(masks, m_ref)
    np.testing.assert_array_equal(lab, oracle.label_tets(t2, m_ref, S.label_ids))
    # only new nodes were evaluated after the initial pass
    assert st["points"] == n2.shape[0]
    # same mesh as the host path driven by the oracle
    from paper_2203_10000_b200._native import refine
    m0 = oracle.label_nodes(nodes, S)
    l0 = oracle.label_tets(tets, m0, S.label_ids)
    a_n, a_t, a_l, _, _ = refine(nodes, tets, l0, oracle.flag_boundary(tets, m0))
    a_m = np.concatenate([m0, oracle.label_nodes(a_n[nodes.shape[0]:], S)])
    b_n, b_t, _, _, _ = refine(a_n, a_t, oracle.label_tets(a_t, a_m, S.label_ids), oracle.flag_boundary(a_t, a_m))
    np.testing.assert_array_equal(b_n, n2)
    np.testing.assert_array_equal(b_t, t2)


def test_device_refine_matches_host(ctx):
    """The device refinement inside nm_refine_relabel produces bit-identical
    nodes/tets/labels to the host nm_refine on the same selection (one level,
    random-ish selection through a perturbed surface)."""
    from paper_2203_10000_b200._native import refine
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 10.0, (22, 22, 22))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    n1, t1, l1, m1, st = ctx.refine_relabel(nodes, tets, levels=1)
    m0 = oracle.label_nodes(nodes, S)
    l0 = oracle.label_tets(tets, m0, S.label_ids)
    hn, ht, hl, _, n_old = refine(nodes, tets, l0, oracle.flag_boundary(tets, m0))
    np.testing.assert_array_equal(n1, hn)
    np.testing.assert_array_equal(t1, ht)
    m_ref = oracle.label_nodes(hn, S)
    np.testing.assert_array_equal(m1, m_ref)
    np.testing.assert_array_equal(l1, oracle.label_tets(ht, m_ref, S.label_ids))


def test_results_independent_of_point_set(ctx):
    """s (fp64, bitwise) for a point does not depend on which other points
    share its warp: a subset evaluated alone equals the same points evaluated
    inside the full set and inside a shuffled set (the sharding invariance of
    SPEC.md:265 at the finest level)."""
    cfg = synth.config(3)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()
    rng = np.random.default_rng(11)
    block = nodes[3_000_000:3_040_000]
    idx = np.sort(rng.choice(block.shape[0], 3000, replace=False))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    s_block, _ = ctx.enclosure(block)
    s_sub, _ = ctx.enclosure(block[idx])
    perm = rng.permutation(block.shape[0])
    s_perm, _ = ctx.enclosure(block[perm])
    np.testing.assert_array_equal(s_sub, s_block[idx])
    np.testing.assert_array_equal(s_perm, s_block[perm])


def test_max_compartments_and_limits():
    """32 compartments (the uint32 mask width, SPEC.md:96-103 allows many):
    masks and labels match the oracle; 33 are rejected with an error."""
    from paper_2203_10000_b200._native import Context, NativeError
    rng = np.random.default_rng(32)
    parts = [synth.icosphere(float(rng.uniform(2, 6)), 2, center=tuple(rng.uniform(-10, 10, 3))) for _ in range(32)]
    S = synth.concat_surfaces(parts, labels=list(range(100, 132)))
    pts = rng.uniform(-16, 16, (5000, 3))
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m, _ = c.label_nodes(pts)
        np.testing.assert_array_equal(m, oracle.label_nodes(pts, S))
        assert (m >> 31).any()
        S33 = synth.concat_surfaces(parts + [synth.icosphere(1.0, 1)])
        with pytest.raises(NativeError, match="32"):
            c.set_surfaces(S33.xyz, S33.tri, S33.comp_off, S33.label_ids)


def test_on_surface_ties_are_reported():
    """Lattice nodes lying exactly on a box surface (faces, edges, corners)
    have s = 1/2, 1/4, 1/8 — implementation-defined ties. The
    GPU must route them to the fp64 fix-up, agree with the oracle's s to
    1e-12 and report the tie pairs in nm_stats.ties."""
    from paper_2203_10000_b200._native import Context
    bx, bt = synth.box_surface([0, 0, 0], [4, 4, 4])
    S = synth.single_surface(bx, bt)
    nodes, _ = synth.lattice_mesh((-1.0, -1.0, -1.0), 1.0, (6, 6, 6))
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        s, st = c.enclosure(nodes)
    s_ref = oracle.enclosure(nodes, S)
    on_surface = (s_ref[:, 0] > 1e-9) & (s_ref[:, 0] < 1 - 1e-9)
    np.testing.assert_allclose(s[on_surface], s_ref[on_surface], atol=1e-12)   # fp64 fix-up
    np.testing.assert_allclose(s[~on_surface], s_ref[~on_surface], atol=S_EXPECT)
    on_face = np.isclose(s_ref[:, 0], 0.5, atol=1e-9)
    assert on_face.sum() > 0 and st["ties"] == int(on_face.sum())
    assert st["flagged_points"] >= int(np.count_nonzero((s_ref[:, 0] > 1e-9) & (s_ref[:, 0] < 1 - 1e-9)))


def test_centroid_mode(ctx):
    """nm_label_centroids (query points = tet centroids) == oracle on the
    centroids; on cfg1 it labels ~the sphere volume (cf. test_sphere_volume_kat)."""
    cfg = synth.config(1)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    lab, st = ctx.label_centroids(nodes, tets)
    a, b, c, d = (nodes[tets[:, i]] for i in range(4))
    cen = (a + b + c + d) * 0.25
    m = oracle.label_nodes(cen, S)
    ref = np.where(m != 0, S.label_ids[0], 0).astype(np.int32)
    np.testing.assert_array_equal(lab, ref)
    assert st["evals"] == tets.shape[0] * S.n_triangles


def test_extract_boundary_matches_reference(ctx):
    """Device compartment-boundary extraction == the UNMODIFIED reference
    extract_compartment_boundary / extract_region_boundary (mesh.hpp:100-155,
    compiled in oracle/_ref), triangles and nodes bit for bit."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 5.0, (44, 44, 44))
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    labels, _, _ = ctx.label_mesh(nodes, tets)
    for ls in ([1], [2], [4], [0], [1, 2], [2, 3, 4]):
        tri, nb = ctx.extract_boundary(tets, labels, ls)
        rtri, rnb = oracle.ref_boundary(tets, labels, ls)
        np.testing.assert_array_equal(tri, rtri)
        np.testing.assert_array_equal(nb, rnb)
    from paper_2203_10000_b200._native import NativeError
    with pytest.raises(NativeError, match="UnknownLabel"):
        ctx.extract_boundary(tets, labels, [77])


def test_device_lattice_bitwise(ctx):
    """nm_lattice_device == generate_lattice_mesh (via the pinned host
    generator) bit for bit; nm_label_lattice == nm_label_mesh on it."""
    import torch
    for (o, h, n) in [((-12.0, -12.0, -12.0), 0.75, (32, 32, 32)), ((-2.0, 1.0, 0.5), 1.25, (3, 4, 2)),
                      ((-107.5, -107.5, -107.5), 1.0, (60, 17, 33))]:
        nodes, tets = synth.lattice_mesh(o, h, n)
        dn = torch.empty(nodes.shape, dtype=torch.float64, device="cuda")
        dt = torch.empty(tets.shape, dtype=torch.int32, device="cuda")
        ctx.lattice_device(o, h, n, dn, dt)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(dn.cpu().numpy(), nodes)
        np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), tets)
    cfg = synth.config(1)
    S = cfg.surfaces
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    lab, masks, st = ctx.label_lattice(cfg.origin, cfg.h, cfg.n, want_masks=True)
    nodes, tets = cfg.lattice_mesh()
    ref, m_ref, _ = ctx.label_mesh(nodes, tets, want_masks=True)
    np.testing.assert_array_equal(lab, ref)
    np.testing.assert_array_equal(masks, m_ref)


def test_point_surface_distance_bitwise_vs_oracle(ctx):
    """quality.boundary_distance kernel: fp32 pass + fp64 refinement equals the
    fp64 oracle (min over all triangles) bit for bit; SPEC.md:431-432 KATs."""
    from paper_2203_10000_b200._native import sample_surface
    from paper_2203_10000_b200.quality import boundary_distance
    xyz, tri = synth.icosphere(10.0, 4, center=(30.0, -20.0, 5.0))
    rng = np.random.default_rng(5)
    pts = np.concatenate([rng.uniform(10, 50, (3000, 3)) * [1, -1, 0.3], sample_surface(xyz, tri, 2000, seed=3)])
    d, st = ctx.point_surface_distance(pts, xyz, tri)
    np.testing.assert_array_equal(d, oracle.point_surface_distance(pts, xyz, tri))
    assert np.all(d[3000:] < 1e-9)                       # identical surfaces -> < 1e-9 mm
    outer = synth.icosphere(11.0, 5, center=(30.0, -20.0, 5.0))
    r = boundary_distance(ctx, xyz, tri, *outer, samples=20000, seed=0)
    assert abs(r["median"] - 1.0) < 0.05                  # concentric spheres 10 and 11 mm


def test_far_from_origin_coordinates(ctx):
    """Scanner-frame coordinates (~1e3 mm offsets): the centred double-single
    frame keeps parity (masks bit-exact, s within 1e-5)."""
    cfg = synth.config(2)
    S = cfg.surfaces
    off = np.array([1234.5, -2047.25, 733.0])
    nodes = cfg.lattice_nodes()[::37] + off
    S2 = synth.SurfaceSet(S.xyz + off, S.tri, S.comp_off, S.label_ids, S.priorities, S.active, S.names)
    ctx.set_surfaces(S2.xyz, S2.tri, S2.comp_off, S2.label_ids)
    s, _ = ctx.enclosure(nodes)
    m_ref, s_ref = oracle.label_nodes(nodes, S2, want_s=True)
    assert np.max(np.abs(s - s_ref)) <= S_EXPECT
    m, _ = ctx.label_nodes(nodes)
    bad, _ = _compare_masks(m, m_ref, s_ref)
    assert bad == 0


def _tetra_soup(n, rng, scale=3.0):
    """n disjoint closed tetrahedra (4 outward triangles each): strips of <= 4
    triangles, the worst case for the strip layout."""
    parts = []
    for _ in range(n):
        c = rng.uniform(-20, 20, 3)
        v = c + rng.normal(size=(4, 3)) * scale
        a, b, cc, d = v
        if np.dot(b - a, np.cross(cc - a, d - a)) < 0:
            v[[2, 3]] = v[[3, 2]]
        tri = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]], np.uint32)  # outward (mesh.hpp:57-64)
        parts.append((v, tri))
    return parts


@pytest.mark.parametrize("layout", [0, 1, 2])
def test_poorly_stripifiable_surface(layout):
    """Many tiny closed surfaces + slivers in one compartment: auto layout
    falls back to independent triangles; every layout matches the oracle."""
    from paper_2203_10000_b200._native import Context
    rng = np.random.default_rng(9)
    parts = _tetra_soup(300, rng)
    xs, ts, vo = [], [], 0
    for v, t in parts:
        xs.append(v)
        ts.append(t + vo)
        vo += 4
    S = synth.single_surface(np.concatenate(xs), np.concatenate(ts))
    pts = rng.uniform(-25, 25, (4000, 3))
    with Context(0, layout=layout) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        info = c.surface_info()
        if layout == 0:
            assert info["layout"] == "triangles"
        s, _ = c.enclosure(pts)
        m, _ = c.label_nodes(pts)
    m_ref, s_ref = oracle.label_nodes(pts, S, want_s=True)
    assert np.max(np.abs(s - s_ref)) <= S_EXPECT
    bad, _ = _compare_masks(m, m_ref, s_ref)
    assert bad == 0


def _interface_tets(tets, labels, a, b):
    """Host restatement of the refine_boundary selection."""
    F = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])
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


def test_refine_boundary_device(ctx):
    """interface layers of a pair refined on both sides; a
    pair without a shared face leaves the mesh unchanged; bit-identical to
    host nm_refine on the same selection."""
    from paper_2203_10000_b200._native import refine
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (6, 6, 6))
    cen = (nodes[tets].mean(axis=1))
    labels = np.where(cen[:, 0] < 3.0, 1, 2).astype(np.int32)      # half-and-half cube
    labels[(cen[:, 0] > 5.5)] = 3
    n2, t2, l2, par, n_old = ctx.refine_boundary(nodes, tets, labels, 1, 2)
    sel = _interface_tets(tets, labels, 1, 2)
    assert sel.size > 0 and np.all(np.isin(labels[sel], [1, 2]))
    hn, ht, hl, hp, _ = refine(nodes, tets, labels, sel)
    np.testing.assert_array_equal(n2, hn)
    np.testing.assert_array_equal(t2, ht)
    np.testing.assert_array_equal(l2, hl)
    np.testing.assert_array_equal(par, hp)
    # 1 and 3 share no face -> identical mesh
    m2, u2, k2, _, _ = ctx.refine_boundary(nodes, tets, labels, 1, 3)
    np.testing.assert_array_equal(m2, nodes)
    np.testing.assert_array_equal(u2, tets)


def test_outside_culling_exact():
    """cull_outside: points outside a closed compartment's 13-DOP get
    s = 0 exactly; every other result is bit-identical to the full
    evaluation, masks/labels are unchanged, and the per-point decision keeps
    results independent of the point set."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(3)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()[2_000_000:2_060_000]
    with Context(0) as full, Context(0, cull_outside=1) as cull:
        for c in (full, cull):
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        s_full, _ = full.enclosure(nodes)
        s_cull, st = cull.enclosure(nodes)
        m_full, _ = full.label_nodes(nodes)
        m_cull, _ = cull.label_nodes(nodes)
        idx = np.arange(0, nodes.shape[0], 7)
        s_sub, _ = cull.enclosure(nodes[idx])
    np.testing.assert_array_equal(m_cull, m_full)
    culled = s_cull == 0.0
    assert culled.mean() > 0.2                       # nuclei: most points are outside their boxes
    np.testing.assert_array_equal(s_cull[~culled], s_full[~culled])
    assert np.max(np.abs(s_full[culled])) < 1e-5
    np.testing.assert_array_equal(s_sub, s_cull[idx])


@pytest.mark.parametrize("cfg_id,lo,hi", [(3, 2_000_000, 2_200_000), (2, 0, 1_300_000)])
def test_cell_culling_exact(cfg_id, lo, hi):
    """cull_outside=2 (certified cells): a pair resolved by a certified cell
    gets its exact winding number (0 or 1), every evaluated pair is
    bit-identical to the full evaluation, masks are unchanged, the fp64
    oracle agrees on a sample of resolved points, and results do not depend
    on the point set (a strided subset reproduces its rows bitwise)."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(cfg_id)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()[lo:hi]
    with Context(0) as full, Context(0, cull_outside=2) as cell:
        for c in (full, cell):
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        info0 = cell.cell_info()
        assert 0 < info0["certified"] <= info0["cells"]
        s_full, _ = full.enclosure(nodes)
        s_cell, _ = cell.enclosure(nodes)
        info = cell.cell_info()
        m_full, _ = full.label_nodes(nodes)
        m_cell, _ = cell.label_nodes(nodes)
        idx = np.arange(3, nodes.shape[0], 11)
        s_sub, _ = cell.enclosure(nodes[idx])
        m_sub, _ = cell.label_nodes(nodes[idx])
    np.testing.assert_array_equal(m_cell, m_full)
    np.testing.assert_array_equal(m_sub, m_full[idx])
    np.testing.assert_array_equal(s_sub, s_cell[idx])
    resolved = (s_cell == 0.0) | (s_cell == 1.0)
    assert info["last_pairs"] < 0.6 * s_full.size    # most pairs are resolved without evaluation
    diff = s_cell != s_full
    assert np.all(resolved[diff])                     # only resolved pairs may differ ...
    assert np.max(np.abs(s_full[diff] - s_cell[diff])) < 1e-5   # ... and only by fp32 rounding
    rng = np.random.default_rng(cfg_id)
    rows = np.unique(np.nonzero(diff)[0])
    pick = np.sort(rng.choice(rows, min(300, rows.size), replace=False))
    _, s_ref = oracle.label_nodes(nodes[pick], S, want_s=True)
    sel = diff[pick]
    np.testing.assert_allclose(s_cell[pick][sel], s_ref[sel], rtol=0, atol=1e-9)


@pytest.mark.parametrize("cfg_id,lo,hi", [(3, 3_000_000, 3_400_000), (5, 4_800_000, 5_200_000)])
def test_pair_resolve_exact(cfg_id, lo, hi, monkeypatch):
    """Pairs of uncertified children resolved through a surface-free ball
    to a certified neighbour (cells.cuh k_pair_resolve) get the exact winding
    number: masks identical to the pass without the step (NM_NO_RESOLVE=1),
    s identical except on newly resolved pairs, which are exactly 0 or 1 and
    agree with the fp64 oracle; far fewer pairs are left to evaluate."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(cfg_id)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()[lo:hi]
    out = {}
    for mode in ("off", "on"):
        if mode == "off":
            monkeypatch.setenv("NM_NO_RESOLVE", "1")
        else:
            monkeypatch.delenv("NM_NO_RESOLVE", raising=False)
        with Context(0, cull_outside=2) as c:
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
            s, _ = c.enclosure(nodes)
            pairs = c.cell_info()["last_pairs"]
            m, _ = c.label_nodes(nodes)
        out[mode] = (s, m, pairs)
    s_off, m_off, p_off = out["off"]
    s_on, m_on, p_on = out["on"]
    np.testing.assert_array_equal(m_on, m_off)
    assert p_on < 0.6 * p_off, (p_on, p_off)
    diff = s_on != s_off
    assert diff.any()
    assert np.all((s_on[diff] == 0.0) | (s_on[diff] == 1.0))
    assert np.max(np.abs(s_on[diff] - s_off[diff])) < 1e-5
    rng = np.random.default_rng(cfg_id)
    rows = np.unique(np.nonzero(diff)[0])
    pick = np.sort(rng.choice(rows, min(200, rows.size), replace=False))
    _, s_ref = oracle.label_nodes(nodes[pick], S, want_s=True)
    sel = diff[pick]
    np.testing.assert_allclose(s_on[pick][sel], s_ref[sel], rtol=0, atol=1e-9)


def test_cell_axis_changes_cost_not_results():
    """nm_options.cell_axis (certified-cell grid resolution) is performance
    only: coarser and finer grids certify different cells but give the same
    masks and the same s on every evaluated pair; out-of-range values fail."""
    from paper_2203_10000_b200._native import Context, NativeError
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()[::3]
    with Context(0) as full:
        full.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m_full, _ = full.label_nodes(nodes)
        s_full, _ = full.enclosure(nodes)
    infos = {}
    for axis in (48, 200):
        with Context(0, cull_outside=2, cell_axis=axis) as c:
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
            m, _ = c.label_nodes(nodes)
            s, _ = c.enclosure(nodes)
            infos[axis] = c.cell_info()
        np.testing.assert_array_equal(m, m_full)
        diff = s != s_full
        assert np.all((s[diff] == 0.0) | (s[diff] == 1.0))
        assert np.max(np.abs(s_full[diff] - s[diff]), initial=0.0) < 1e-5
    assert infos[200]["cells"] > infos[48]["cells"]
    assert infos[200]["last_pairs"] < infos[48]["last_pairs"]
    for bad in (4, 5000):
        with pytest.raises(NativeError, match="cell_axis"):
            Context(0, cull_outside=2, cell_axis=bad)


def test_cfg5_full_size_properties():
    """BASELINE configs[4] at full size (10,077,696 nodes x 983,040 triangles):
    size-independent properties over every node, the fp64 oracle on a seeded
    sample.
      * sample parity: masks bit-exact, |s - s_oracle| <= S_EXPECT;
      * nesting: the six shells are nested by construction, so shell j's
        inside bit implies shell j+1's for every node;
      * determinism: two half-mesh calls reproduce the full call bitwise
        (results independent of the point set);
      * exact outside culling (cull_outside=1) changes no bit;
      * tet labels = id[ffs(AND of the 4 node masks)] on a tet sample."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(5)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    c = Context(0)
    c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    m_all, st = c.label_nodes(nodes)
    assert st["ties"] == 0

    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(nodes.shape[0], 1500, replace=False))
    m_ref, s_ref = oracle.label_nodes(nodes[idx], S, want_s=True)
    bad, _ = _compare_masks(m_all[idx], m_ref, s_ref)
    assert bad == 0
    s_gpu, _ = c.enclosure(nodes[idx])
    assert np.max(np.abs(s_gpu - s_ref)) <= S_EXPECT
    # a 1,500-point call runs with the compartments split over 12 CTA rows,
    # the 10M-point call without: bitwise the same masks and s
    m_sub, _ = c.label_nodes(nodes[idx])
    np.testing.assert_array_equal(m_sub, m_all[idx])
    head = 4_000_000
    s_head, _ = c.enclosure(nodes[:head])
    sel = idx < head
    np.testing.assert_array_equal(s_gpu[sel], s_head[idx[sel]])
    del s_head

    shells = [k for k, name in enumerate(S.names) if name.startswith("shell")]
    assert len(shells) == 6
    for a, b in zip(shells, shells[1:]):
        inner = (m_all >> np.uint32(a)) & 1
        outer = (m_all >> np.uint32(b)) & 1
        assert np.all(outer >= inner)
    assert 0 < np.count_nonzero((m_all >> np.uint32(shells[0])) & 1) < nodes.shape[0]

    half = nodes.shape[0] // 2 + 12345
    m_a, _ = c.label_nodes(nodes[:half])
    m_b, _ = c.label_nodes(nodes[half:])
    np.testing.assert_array_equal(np.concatenate([m_a, m_b]), m_all)

    for mode in (1, 2):
        cc = Context(0, cull_outside=mode)
        cc.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m_cull, _ = cc.label_nodes(nodes)
        np.testing.assert_array_equal(m_cull, m_all)
        cc.close()

    labels, _, _ = c.label_mesh(nodes, tets)
    tidx = rng.choice(tets.shape[0], 200000, replace=False)
    conj = np.bitwise_and.reduce(m_all[tets[tidx]], axis=1)
    low = (conj & (~conj + np.uint32(1))).astype(np.float64)  # lowest set bit
    first = np.where(conj != 0, np.log2(np.maximum(low, 1.0)).astype(np.int64), -1)
    expect = np.where(first >= 0, S.label_ids[np.maximum(first, 0)], 0)
    np.testing.assert_array_equal(labels[tidx], expect)
    c.close()


def _torus(R, r, nu, nv, center=(0.0, 0.0, 0.0)):
    """Closed, outward torus (hole along z): nu x nv quads split in two."""
    u = np.arange(nu) * 2 * np.pi / nu
    v = np.arange(nv) * 2 * np.pi / nv
    U, V = np.meshgrid(u, v, indexing="ij")
    xyz = np.stack([(R + r * np.cos(V)) * np.cos(U), (R + r * np.cos(V)) * np.sin(U), r * np.sin(V)], -1)
    xyz = xyz.reshape(-1, 3) + np.asarray(center)
    idx = lambda i, j: (i % nu) * nv + (j % nv)
    tri = []
    for i in range(nu):
        for j in range(nv):
            a, b, c, d = idx(i, j), idx(i + 1, j), idx(i + 1, j + 1), idx(i, j + 1)
            tri += [(a, b, c), (a, c, d)]
    return xyz, np.array(tri, np.uint32)


def test_cell_culling_topology_and_thin_gaps():
    """cull_outside=2 on shapes that stress the run logic: a torus (the hole
    is inside the 13-DOP but outside the surface: runs through it need their
    own representative), two concentric spheres 0.2 mm apart (cells between
    them stay uncertified), a 1 mm sphere (tiny cells) and a sphere touching
    the lattice edge. Masks equal the brute-force pass; s of resolved pairs
    equals the fp64 oracle."""
    from paper_2203_10000_b200._native import Context
    tx, tt = _torus(20.0, 6.0, 96, 48)
    # sphere orientation from the synth generator (outward)
    s1 = synth.icosphere(15.0, 4, center=(0.0, 0.0, 30.0))
    s2 = synth.icosphere(15.2, 4, center=(0.0, 0.0, 30.0))
    s3 = synth.icosphere(1.0, 3, center=(0.3, -0.2, 0.1))
    s4 = synth.icosphere(8.0, 3, center=(-24.0, 24.0, -16.0))
    S = synth.concat_surfaces([(tx, tt), s1, s2, s3, s4])
    nodes = synth.lattice_nodes((-32.0, -32.0, -16.0), 0.37, (174, 174, 174))
    with Context(0) as full, Context(0, cull_outside=2) as cell:
        for c in (full, cell):
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m_full, _ = full.label_nodes(nodes)
        m_cell, _ = cell.label_nodes(nodes)
        info = cell.cell_info()
        rng = np.random.default_rng(11)
        idx = np.sort(rng.choice(nodes.shape[0], 4000, replace=False))
        s_cell, _ = cell.enclosure(nodes[idx])
    np.testing.assert_array_equal(m_cell, m_full)
    assert info["last_pairs"] < 0.25 * nodes.shape[0] * 5
    hole = (np.abs(nodes[:, 2]) < 2.0) & (np.hypot(nodes[:, 0], nodes[:, 1]) < 10.0)
    assert hole.any() and not np.any(m_full[hole] & 1)          # the hole is outside the torus
    _, s_ref = oracle.label_nodes(nodes[idx], S, want_s=True)
    resolved = (s_cell == 0.0) | (s_cell == 1.0)
    assert resolved.mean() > 0.5
    np.testing.assert_allclose(s_cell[resolved], s_ref[resolved], rtol=0, atol=1e-9)
    np.testing.assert_allclose(s_cell, s_ref, rtol=0, atol=S_EXPECT)


def test_cell_culling_small_and_empty_compartments():
    """cull_outside=2 with a 4-triangle tetrahedron surface (one cluster,
    fewer triangles than a cluster), an EMPTY compartment between two
    spheres, and points far outside every grid: masks equal the brute-force
    pass and s of resolved pairs equals the fp64 oracle."""
    from paper_2203_10000_b200._native import Context
    tet_xyz = np.array([[0, 0, 0], [4, 0, 0], [0, 4, 0], [0, 0, 4]], np.float64) + 1.0
    tet_tri = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.uint32)  # outward
    a = synth.icosphere(3.0, 2, center=(-6.0, 0.0, 0.0))
    b = synth.icosphere(9.0, 3)
    S = synth.concat_surfaces([(tet_xyz, tet_tri), a, (np.zeros((0, 3)), np.zeros((0, 3), np.uint32)), b])
    assert S.comp_off[2] == S.comp_off[3]
    rng = np.random.default_rng(3)
    pts = np.concatenate([rng.uniform(-12, 12, (200_000, 3)), rng.uniform(-1e3, 1e3, (2000, 3))])
    with Context(0) as full, Context(0, cull_outside=2) as cell:
        for c in (full, cell):
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m_full, _ = full.label_nodes(pts)
        m_cell, _ = cell.label_nodes(pts)
        s_cell, _ = cell.enclosure(pts[:3000])
    np.testing.assert_array_equal(m_cell, m_full)
    assert not np.any(m_full & np.uint32(1 << 2))                 # nothing is inside the empty compartment
    inside_tet = (pts[:, 0] > 1) & (pts[:, 1] > 1) & (pts[:, 2] > 1) & (pts.sum(axis=1) - 3 < 4)
    np.testing.assert_array_equal((m_full & 1).astype(bool), inside_tet)
    _, s_ref = oracle.label_nodes(pts[:3000], S, want_s=True)
    resolved = (s_cell == 0.0) | (s_cell == 1.0)
    np.testing.assert_allclose(s_cell[resolved], s_ref[resolved], rtol=0, atol=1e-9)
    np.testing.assert_allclose(s_cell, s_ref, rtol=0, atol=S_EXPECT)


def test_cell_culling_winding_number_two():
    """A compartment made of two overlapping closed spheres: the winding
    number is 2 in the overlap. Certified cells only accept winding numbers 0
    and 1, so the overlap stays evaluated: masks equal the brute-force pass
    and the oracle, s = 2 there."""
    from paper_2203_10000_b200._native import Context
    a = synth.icosphere(8.0, 3, center=(-3.0, 0.0, 0.0))
    b = synth.icosphere(8.0, 3, center=(3.0, 0.0, 0.0))
    two = (np.concatenate([a[0], b[0]]), np.concatenate([a[1], b[1] + np.uint32(a[0].shape[0])]))
    S = synth.concat_surfaces([two, synth.icosphere(14.0, 3)])
    rng = np.random.default_rng(9)
    pts = rng.uniform(-15, 15, (150_000, 3))
    with Context(0) as full, Context(0, cull_outside=2) as cell:
        for c in (full, cell):
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m_full, _ = full.label_nodes(pts)
        m_cell, _ = cell.label_nodes(pts)
        probe = np.array([[0.0, 0.0, 0.0], [-9.0, 0.0, 0.0], [0.0, 0.0, 12.0]])
        s_cell, _ = cell.enclosure(probe)
    np.testing.assert_array_equal(m_cell, m_full)
    _, s_ref = oracle.label_nodes(probe, S, want_s=True)
    np.testing.assert_allclose(s_cell, s_ref, rtol=0, atol=S_EXPECT)
    assert abs(s_cell[0, 0] - 2.0) < 1e-5 and abs(s_cell[1, 0] - 1.0) < 1e-5 and s_cell[2, 0] == 0.0


def test_cell_axis_memory_budget():
    """A certified-cell grid whose build would need more than the 8 GB host
    budget (cell_axis 1024 on a cube: ~1.1e9 cells) fails in nm_set_surfaces
    with a message, instead of exhausting host memory."""
    from paper_2203_10000_b200._native import Context, NativeError
    bx, bt = synth.box_surface([0, 0, 0], [10, 10, 10])
    with Context(0, cull_outside=2, cell_axis=1024) as c:
        with pytest.raises(NativeError, match="cell_axis"):
            c.set_surfaces(bx, bt, np.array([0, 12], np.uint32), np.array([1], np.int32))
    with Context(0, cull_outside=2, cell_axis=256) as c:   # ~0.3 GB: within budget
        c.set_surfaces(bx, bt, np.array([0, 12], np.uint32), np.array([1], np.int32))
        m, _ = c.label_nodes(np.array([[5.0, 5, 5], [20.0, 5, 5]]))
        np.testing.assert_array_equal(m, [1, 0])


@pytest.mark.parametrize("cfg_id", [2, 3, 5])
def test_device_cell_build_equals_host_build(cfg_id, monkeypatch):
    """The certified-cell build's run logic on the device (cells.cuh
    k_runs_* / k_rep_values / k_*_codes, the default) produces the SAME
    level-1 codes and child states, bit for bit, as the host restatement
    (NM_CELLS_HOST=1), and the same certified / representative counts."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(cfg_id)
    S = cfg.surfaces
    out = {}
    for mode in ("host", "device"):
        if mode == "host":
            monkeypatch.setenv("NM_CELLS_HOST", "1")
        else:
            monkeypatch.delenv("NM_CELLS_HOST", raising=False)
        with Context(0, cull_outside=2) as c:
            c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
            codes, ch = c.cell_dump()
            info = c.cell_info()
        out[mode] = (codes, ch, info)
    np.testing.assert_array_equal(out["device"][0], out["host"][0])
    np.testing.assert_array_equal(out["device"][1], out["host"][1])
    for k in ("cells", "certified", "reps"):
        assert out["device"][2][k] == out["host"][2][k], k
    assert (out["device"][0] == 2).any() and (out["device"][1] == 1).any()
