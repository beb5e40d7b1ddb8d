"""quality.boundary_distance on the B200.

Area-uniform samples (fixed seed) on a mesh compartment boundary — e.g. the
output of ``Context.extract_boundary`` (mesh.hpp:100-155 on the device) — and
their exact unsigned distance to the target segmentation surface, computed by
the same N-body tile loop as the labeling kernel with a min-reduction
(csrc/distance.cuh).
"""
from __future__ import annotations

import numpy as np

from ._native import sample_surface


def boundary_distance(ctx, mesh_nodes, boundary_tri, target_xyz, target_tri, samples: int = 20000, seed: int = 0):
    """Returns {"samples", "median", "q25", "q75", "stats"} (mm)."""
    if len(boundary_tri) == 0 or len(target_tri) == 0:
        raise ValueError("boundary_distance: both surfaces must be non-empty (SPEC.md:429)")
    pts = sample_surface(mesh_nodes, boundary_tri, samples, seed)
    d, st = ctx.point_surface_distance(pts, target_xyz, target_tri)
    q25, med, q75 = np.quantile(d, [0.25, 0.5, 0.75])
    return {"samples": d, "points": pts, "median": float(med), "q25": float(q25), "q75": float(q75), "stats": st}
