"""Certified-cell grid resolution vs cost (cfg id, axes...): set_surfaces
time (median of 3 fresh contexts), node pass time (median of 3), pairs left
to evaluate, masks equal to cell_axis 120. Not a bench number."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
axes = [int(a) for a in sys.argv[2:]] or [120, 144, 168, 200, 240]
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()
ref = None
for ax in axes:
    ts, tl = [], []
    for rep in range(3):
        ctx = Context(0, cull_outside=2, cell_axis=ax)
        t0 = time.perf_counter()
        ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ts.append(time.perf_counter() - t0)
        if rep == 2:
            for _ in range(3):
                m, st = ctx.label_nodes(nodes)
                tl.append(st["ms_total"])
            info = ctx.cell_info()
        ctx.close()
    if ref is None:
        ref = m
    print({"cell_axis": ax, "set_surfaces_ms": round(1e3 * sorted(ts)[1], 1), "node_pass_ms": round(sorted(tl)[1], 2),
           "pairs": info["last_pairs"], "reps": info["reps"], "cells": info["cells"],
           "masks_equal": bool(np.array_equal(m, ref))}, flush=True)
