"""Worst fp32-pass errors of s on a FULL config mesh vs the fp64 oracle
(diagnostic; not a test). Usage: python scripts/diag_err_full.py <cfg> [layout]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
layout = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
if len(sys.argv) > 3:
    nodes = nodes[::int(sys.argv[3])]
with Context(0, layout=layout) as c:
    c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    s, st = c.enclosure(nodes)
    print("layout", c.surface_info()["layout"], "flagged points", st["flagged_points"], "pairs", st["flagged_pairs"])
s_ref = oracle.enclosure(nodes, S)
err = np.abs(s - s_ref)
print(f"cfg{cfg_id} nodes {nodes.shape[0]} max {err.max():.3e} p99.99 {np.quantile(err, 0.9999):.3e} "
      f"p99.9999 {np.quantile(err, 0.999999):.3e} count>1e-5 {(err > 1e-5).sum()} >2e-5 {(err > 2e-5).sum()} >5e-5 {(err > 5e-5).sum()}")
idx = np.argsort(err.ravel())[::-1][:12]
for f in idx:
    i, k = divmod(int(f), S.K)
    x, t = S.compartment(k)
    d = oracle.point_surface_distance(nodes[i:i + 1], x, t)[0]
    # nearest triangle and its edge length
    cen = x[t].mean(axis=1)
    j = int(np.argmin(np.linalg.norm(cen - nodes[i], axis=1)))
    e = np.linalg.norm(x[t[j]][[1, 2, 0]] - x[t[j]], axis=1)
    print(f"  pt {i} {nodes[i]} comp {k} err {err[i, k]:.3e} s_ref {s_ref[i, k]:.9f} s_gpu {s[i, k]:.9f} "
          f"dist {d:.5f} mm nearest-tri edges {np.round(e, 3)}")
