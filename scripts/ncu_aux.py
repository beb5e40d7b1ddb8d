"""cfg5 full-mesh step for ncu captures of the auxiliary kernels (k_fixup, k_label_tets)."""
import sys
sys.path.insert(0, ".")
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
S = cfg.surfaces
nodes, tets = cfg.lattice_mesh()
ctx = Context(0)
ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
labels, masks, st = ctx.label_mesh(nodes, tets)
print({k: st[k] for k in ("ms_label", "ms_fixup", "ms_tets", "flagged_points")})
