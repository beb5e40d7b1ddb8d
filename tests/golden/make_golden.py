"""Regenerate the committed golden fixtures (run in the build container, where
/root/reference exists; the GPU box only reads the committed files).

  spec_kats.json      SPEC.md labeling examples (:231-233, :240-242) and the
                      analytic cube values, as (surface, point, expected, tol)
  ref_generators.json sha256 of the UNMODIFIED reference generators' outputs
                      (oracle/_ref: primitives.hpp icosphere/box_surface,
                      lattice.hpp generate_lattice_mesh) for the shapes the
                      configs use — pins csrc/synth.cpp on machines without
                      /root/reference
  oracle_cfg1.json    the oracle's cfg1 result (inside count, mask/label
                      hashes, s at 64 fixed nodes) — pins the oracle itself
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2203_10000_b200 import synth  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_icosphere(r, level, c=(0.0, 0.0, 0.0)):
    import ctypes
    R = oracle.ref()
    nv, nt = 10 * 4 ** level + 2, 20 * 4 ** level
    xyz = np.empty((nv, 3))
    tri = np.empty((nt, 3), np.uint32)
    cc = np.asarray(c, np.float64)
    R.ref_icosphere(r, level, cc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                    xyz.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                    tri.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    return xyz, tri


def ref_lattice(origin, h, n):
    import ctypes
    R = oracle.ref()
    nn = (n[0] + 1) * (n[1] + 1) * (n[2] + 1)
    nodes = np.empty((nn, 3))
    tets = np.empty((5 * n[0] * n[1] * n[2], 4), np.uint32)
    o = np.asarray(origin, np.float64)
    R.ref_lattice_mesh(o.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), h, n[0], n[1], n[2],
                       nodes.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                       tets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    return nodes, tets


def main():
    kats = {
        "source": "SPEC.md:231-233 (enclosure_ratio examples); analytic cube face/edge/corner/interior values",
        "cases": [
            {"surface": ["icosphere", 1.0, 4], "point": [0, 0, 0], "expect": 1.0, "tol": 1e-6, "ref": "SPEC.md:231"},
            {"surface": ["icosphere", 1.0, 4], "point": [3, 0, 0], "expect": 0.0, "tol": 1e-6, "ref": "SPEC.md:232"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [0, 0, 0], "expect": 0.125, "tol": 1e-6, "ref": "SPEC.md:233"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [1, 1, 1], "expect": 0.125, "tol": 1e-12, "ref": "octant symmetry"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [0.5, 0, 0], "expect": 0.25, "tol": 1e-12, "ref": "edge: quarter space"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [0.5, 0.5, 0], "expect": 0.5, "tol": 1e-12, "ref": "face: half space"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [0.5, 0.5, 0.5], "expect": 1.0, "tol": 1e-12, "ref": "interior"},
            {"surface": ["box", [0, 0, 0], [1, 1, 1]], "point": [2, 2, 2], "expect": 0.0, "tol": 1e-12, "ref": "exterior"},
            {"surface": ["icosphere", 10.0, 3], "point": [0, 0, 9.5], "expect": 1.0, "tol": 1e-9, "ref": "SPEC.md:231 near wall"},
            {"surface": ["icosphere", 10.0, 3], "point": [0, 0, 10.5], "expect": 0.0, "tol": 1e-9, "ref": "SPEC.md:232 near wall"},
        ],
    }
    (HERE / "spec_kats.json").write_text(json.dumps(kats, indent=1))

    gens = {"source": "oracle/_ref (unmodified reference headers): primitives.hpp:29-54, lattice.hpp:40-91"}
    if oracle.ref_available():
        for lvl in range(0, 7):
            x, t = ref_icosphere(1.0, lvl)
            gens[f"icosphere_1_L{lvl}"] = sha(x, t)
        x, t = ref_icosphere(10.0, 3)
        gens["icosphere_10_L3"] = sha(x, t)
        x, t = ref_icosphere(100.0, 4, (3.0, -7.0, 11.0))
        gens["icosphere_100_L4_off"] = sha(x, t)
        for (o, h, n) in [((-12.0, -12.0, -12.0), 0.75, (32, 32, 32)), ((-2.0, 1.0, 0.5), 1.25, (3, 4, 2)),
                          ((0.0, 0.0, 0.0), 1.0, (1, 1, 1))]:
            nodes, tets = ref_lattice(o, h, n)
            gens[f"lattice_{o}_{h}_{n}"] = sha(nodes, tets)
        (HERE / "ref_generators.json").write_text(json.dumps(gens, indent=1))

    cfg = synth.config(1)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    m, s = oracle.label_nodes(nodes, S, want_s=True)
    lab = oracle.label_tets(tets, m, S.label_ids)
    idx = np.linspace(0, nodes.shape[0] - 1, 64).astype(int)
    g = {"source": "oracle/labeling_oracle.cpp on cfg1 (icosphere(10,3), 32^3 lattice at h=0.75 from -12)",
         "inside_nodes": int(m.sum()), "labeled_tets": int((lab > 0).sum()), "mask_sha256": sha(m),
         "label_sha256": sha(lab), "s_idx": idx.tolist(), "s": s[idx, 0].tolist()}
    (HERE / "oracle_cfg1.json").write_text(json.dumps(g, indent=1))
    print("golden fixtures written")


if __name__ == "__main__":
    main()
