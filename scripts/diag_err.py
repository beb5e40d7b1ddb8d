import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg = synth.config(2)
S = cfg.surfaces
for off in (np.zeros(3), np.array([1234.5, -2047.25, 733.0])):
    nodes = cfg.lattice_nodes()[::37] + off
    S2 = synth.SurfaceSet(S.xyz + off, S.tri, S.comp_off, S.label_ids, S.priorities, S.active, S.names)
    with Context(0) as c:
        c.set_surfaces(S2.xyz, S2.tri, S2.comp_off, S2.label_ids)
        s, _ = c.enclosure(nodes)
    s_ref = oracle.enclosure(nodes, S2)
    err = np.abs(s - s_ref)
    idx = np.argsort(err.ravel())[::-1][:6]
    print("offset", off, "max", err.max(), "p99.99", np.quantile(err, 0.9999))
    for f in idx:
        i, k = divmod(f, S.K)
        x, t = S2.compartment(k)
        d = oracle.point_surface_distance(nodes[i:i + 1], x, t)[0]
        print(f"  pt {i} comp {k} err {err[i, k]:.3e} s_ref {s_ref[i, k]:.9f} dist {d:.4f} mm")
