"""Phase timing of the C++ drop-in e2e (build/libdropin_bench.so) at cfg5
with certified cells; NM_TIMING=1 makes nm_label_mesh print its phases."""
import ctypes
import os
import sys
sys.path.insert(0, ".")
if not os.environ.get("NO_NM_TIMING"):
    os.environ["NM_TIMING"] = "1"
import numpy as np
from paper_2203_10000_b200 import synth
cfg = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
S = cfg.surfaces
nodes, tets = cfg.lattice_mesh()
L = ctypes.CDLL("build/libdropin_bench.so")
P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
sx, st, so, sid = (np.ascontiguousarray(S.xyz, np.float64), np.ascontiguousarray(S.tri, np.uint32),
                   np.ascontiguousarray(S.comp_off, np.uint32), np.ascontiguousarray(S.label_ids, np.int32))
out = np.zeros(6)
lab = np.empty(tets.shape[0], np.int32)
rc = L.dropin_bench(P(sx, ctypes.c_double), ctypes.c_size_t(sx.shape[0]), P(st, ctypes.c_uint32), P(so, ctypes.c_uint32),
                    ctypes.c_int(S.K), P(sid, ctypes.c_int), P(nodes, ctypes.c_double), ctypes.c_size_t(nodes.shape[0]),
                    P(tets, ctypes.c_uint32), ctypes.c_size_t(tets.shape[0]), ctypes.c_int(2), ctypes.c_int(2),
                    P(out, ctypes.c_double), P(lab, ctypes.c_int))
print("rc", rc, "build %.3f first %.3f by-value %.4f / %.4f into %.4f / %.4f s" % tuple(out))
