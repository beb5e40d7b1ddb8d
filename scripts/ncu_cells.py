"""Certified-cell node pass on cfg5 (for an ncu launch list; not a bench number)."""
import sys
sys.path.insert(0, ".")
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
ctx = Context(0, cull_outside=2)
ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
for _ in range(3):
    m, st = ctx.label_nodes(nodes)
print(st["ms_total"], st["ms_label"], ctx.cell_info())
