"""k_label launches on a config's lattice for ncu captures (not a bench number).

    python scripts/ncu_label.py <cfg> <npts>        contiguous slab of npts nodes around the middle
    python scripts/ncu_label.py <cfg> stride:<s>    every s-th node of the whole lattice (the full
                                                    mesh's near/far and strip-chain mix)
    python scripts/ncu_label.py <cfg> full          every node (one full-mesh node pass)
Two node passes run; ncu filters the k_label launch it wants (-s / -c)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sel = sys.argv[2] if len(sys.argv) > 2 else "300000"
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
if sel == "full":
    pts = nodes
elif sel.startswith("stride:"):
    pts = np.ascontiguousarray(nodes[::int(sel.split(":")[1])])
else:
    npts = int(sel)
    mid = nodes.shape[0] // 2 - npts // 2
    pts = nodes[mid:mid + npts]
ctx = Context(0)
ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for _ in range(passes):
    m, st = ctx.label_nodes(pts)
print({k: st[k] for k in ("evals", "ms_label", "ms_fixup", "flagged_points", "near_subtiles", "far_subtiles")},
      "points", pts.shape[0], "evals/s %.3e" % (st["evals"] / st["ms_label"] * 1e3))
