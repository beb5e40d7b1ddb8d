"""s of a config's points through the current library and NM_LABEL_LIB
(another build) written to .npy for a bitwise comparison (development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200._native import Context
cfg_id, out = int(sys.argv[1]), sys.argv[2]
cfg = synth.config(cfg_id)
S = cfg.surfaces
nodes = cfg.lattice_nodes()[::7]
with Context(0) as c:
    c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    s, _ = c.enclosure(nodes)
np.save(out, s)
