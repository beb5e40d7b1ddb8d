"""nm_set_surfaces with certified cells (cull_outside = 2), repeated on fresh
contexts: wall time per call (NM_CELL_VERBOSE=1 prints the phases). Argv:
config id (default 5), repeats (default 3). Not a bench number."""
import sys
import time
sys.path.insert(0, ".")
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S = synth.config(cfg_id).surfaces
for i in range(reps):
    ctx = Context(0, cull_outside=2)
    t0 = time.perf_counter()
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    t = time.perf_counter() - t0
    print({"call": i, "set_surfaces_ms": round(1e3 * t, 1), **ctx.cell_info()}, flush=True)
    ctx.close()
