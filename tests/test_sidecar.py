"""Binary label / node-mask sidecar next to tetmesh v1 (
csrc/sidecar.cu). CPU tests: exact round trip, integrity checks, the mesh
fingerprint against an independent numpy restatement, and the sidecar beside
a tetmesh v1 file written and read back by the UNMODIFIED reference
save_tetmesh / load_tetmesh (mesh.hpp:238-289, oracle/_ref). GPU tests: the
lattice path (nm_label_lattice_sidecar) against nm_label_mesh + the host
fingerprint of the host-generated lattice."""
import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import NativeError, mesh_fingerprint, sidecar_read, sidecar_write

M64 = (1 << 64) - 1


def _mix64(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return z ^ (z >> np.uint64(31))


def _hash_words(buf: bytes, seed: int) -> int:
    if len(buf) % 8:
        buf = buf + b"\0" * (8 - len(buf) % 8)
    w = np.frombuffer(buf, np.uint64)
    i = np.arange(w.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix64(np.uint64(seed) ^ _mix64(i * np.uint64(0x9e3779b97f4a7c15) + w))
        return int(h.sum(dtype=np.uint64))


def _fingerprint(nodes, tets):
    """numpy restatement of nm_mesh_fingerprint (csrc/sidecar.cu)."""
    hn = _hash_words(np.ascontiguousarray(nodes, np.float64).tobytes(), 0x6e6f6465735f6e6d)
    ht = _hash_words(np.ascontiguousarray(tets, np.uint32).tobytes(), 0x746574735f5f6e6d)
    n, nt = nodes.shape[0], tets.shape[0]

    def mix(x):
        with np.errstate(over="ignore"):
            return int(_mix64(np.uint64(x & M64)))
    return mix(hn ^ mix(ht + 0x632be59bd9b4e019) ^ mix(n * 3 + 1) ^ mix(nt * 5 + 2))


def test_fingerprint_matches_restatement_and_detects_changes():
    nodes, tets = synth.lattice_mesh((-1.0, 2.0, 0.5), 0.75, (5, 4, 3))
    fp = mesh_fingerprint(nodes, tets)
    assert fp == _fingerprint(nodes, tets)
    n2 = nodes.copy()
    n2[7, 1] = np.nextafter(n2[7, 1], np.inf)          # one ulp of one coordinate
    assert mesh_fingerprint(n2, tets) != fp
    t2 = tets.copy()
    t2[[3, 4]] = t2[[4, 3]]                             # tet order matters
    assert mesh_fingerprint(nodes, t2) != fp
    assert mesh_fingerprint(nodes, tets) == fp          # deterministic


@pytest.mark.parametrize("with_masks", [True, False])
def test_round_trip_exact(tmp_path, with_masks):
    rng = np.random.default_rng(1)
    nodes, tets = synth.lattice_mesh((0.0, 0.0, 0.0), 1.0, (6, 5, 4))
    labels = rng.integers(-3, 40, tets.shape[0]).astype(np.int32)
    masks = rng.integers(0, 2**32, nodes.shape[0], dtype=np.uint64).astype(np.uint32)
    fp = mesh_fingerprint(nodes, tets)
    p = tmp_path / "m.tetmesh.nmlabels"
    sidecar_write(p, labels, masks if with_masks else None, n_nodes=nodes.shape[0], mesh_fingerprint=fp,
                  label_ids=[3, 9, 11], threshold=0.375)
    info, lab2, m2 = sidecar_read(p)
    np.testing.assert_array_equal(lab2, labels)
    if with_masks:
        np.testing.assert_array_equal(m2, masks)
    else:
        assert m2 is None
    assert info["mesh_fingerprint"] == fp and info["n_tets"] == tets.shape[0] and info["n_nodes"] == nodes.shape[0]
    assert info["label_ids"] == [3, 9, 11] and info["threshold"] == 0.375 and info["is_lattice"] == 0


def test_corruption_is_detected(tmp_path):
    labels = np.arange(1000, dtype=np.int32)
    p = tmp_path / "a.nmlabels"
    sidecar_write(p, labels, label_ids=[1])
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.nmlabels"
    raw2 = raw.copy()
    raw2[-100] ^= 0x10                                  # a label bit
    bad.write_bytes(bytes(raw2))
    with pytest.raises(NativeError, match="hash"):
        sidecar_read(bad)
    bad.write_bytes(bytes(raw[:-9]))                    # truncated
    with pytest.raises(NativeError, match="truncated"):
        sidecar_read(bad)
    bad.write_bytes(b"XXXXXXXX" + bytes(raw[8:]))       # not a sidecar
    with pytest.raises(NativeError, match="not a nestmesh label sidecar"):
        sidecar_read(bad)
    bad.write_bytes(bytes(raw) + b"\0")                 # trailing bytes
    with pytest.raises(NativeError, match="trailing"):
        sidecar_read(bad)


def test_sidecar_next_to_reference_tetmesh_v1(tmp_path):
    """The reference's own save_tetmesh writes the mesh (%.17g text); the
    sidecar beside it carries labels + masks; load_tetmesh reads the mesh
    back bit for bit, so its fingerprint matches the sidecar's and the
    labels apply."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    cfg = synth.config(1)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    nodes = nodes + np.random.default_rng(2).normal(scale=1e-3, size=nodes.shape)   # non-dyadic coordinates
    masks = oracle.label_nodes(nodes, S)
    labels = oracle.label_tets(tets, masks, S.label_ids)
    mesh = tmp_path / "head.tetmesh"
    oracle.ref_save_tetmesh(mesh, nodes, tets, np.zeros_like(labels))   # geometry only, labels 0
    sidecar_write(str(mesh) + ".nmlabels", labels, masks, n_nodes=nodes.shape[0],
                  mesh_fingerprint=mesh_fingerprint(nodes, tets), label_ids=S.label_ids)
    n2, t2, l2 = oracle.ref_load_tetmesh(mesh)
    np.testing.assert_array_equal(n2, nodes)
    info, lab, m = sidecar_read(str(mesh) + ".nmlabels")
    assert info["mesh_fingerprint"] == mesh_fingerprint(n2, t2)
    np.testing.assert_array_equal(lab, labels)
    np.testing.assert_array_equal(m, masks)


@pytest.mark.gpu
def test_label_lattice_sidecar_gpu(tmp_path):
    """nm_label_lattice_sidecar: device lattice -> labels -> sidecar; equals
    nm_label_mesh on the host-generated lattice; the device fingerprint equals
    the host fingerprint of generate_lattice_mesh's mesh."""
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    p = tmp_path / "cfg2.tetmesh.nmlabels"
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        info, st = c.label_lattice_sidecar(cfg.origin, cfg.h, cfg.n, p)
        ref_labels, ref_masks, _ = c.label_mesh(nodes, tets, want_masks=True)
    info2, lab, m = sidecar_read(p)
    assert info2 == info
    assert info["is_lattice"] == 1 and tuple(info["n"]) == tuple(cfg.n) and info["h"] == cfg.h
    np.testing.assert_array_equal(lab, ref_labels)
    np.testing.assert_array_equal(m, ref_masks)
    assert info["mesh_fingerprint"] == mesh_fingerprint(nodes, tets)
    assert info["label_ids"] == list(S.label_ids)
