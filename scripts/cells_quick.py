"""Certified-cell culling on a config: build time, resolved fraction, node-pass
time for cull_outside = 1 and 2, masks equal to cull 1 (not a bench number)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
res = {}
for mode in (1, 2, 2):
    ctx = Context(0, cull_outside=mode)
    t0 = time.perf_counter()
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    t_set = time.perf_counter() - t0
    ms = []
    for _ in range(3):
        m, st = ctx.label_nodes(nodes)
        ms.append(st["ms_total"])
    res[mode] = m
    info = ctx.cell_info() if mode == 2 else {}
    print({"mode": mode, "set_surfaces_s": round(t_set, 3), "ms_total": [round(x, 2) for x in ms],
           "ms_label": round(st["ms_label"], 2), "launches": st["launches"], **info}, flush=True)
    ctx.close()
print("masks equal:", bool(np.array_equal(res[1], res[2])))
