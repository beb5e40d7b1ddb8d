"""One k_label launch on a cfg5 slab (for ncu; not a bench number)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 300000
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
mid = nodes.shape[0] // 2 - npts // 2
pts = nodes[mid:mid + npts]
ctx = Context(0)
ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
for _ in range(2):
    m, st = ctx.label_nodes(pts)
print({k: st[k] for k in ("evals", "ms_label", "ms_fixup", "flagged_points", "near_subtiles", "far_subtiles")},
      "evals/s %.3e" % (st["evals"] / st["ms_label"] * 1e3))
