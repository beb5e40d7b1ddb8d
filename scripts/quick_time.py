"""Quick device timing of the node pass (development aid, not the bench)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2203_10000_b200 import synth  # noqa: E402
from paper_2203_10000_b200._native import Context  # noqa: E402


def run(cfg_id, max_points=None, reps=2, **opts):
    cfg = synth.config(cfg_id)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()
    if max_points and nodes.shape[0] > max_points:
        # a contiguous slab of k-planes keeps the spatial distribution realistic
        mid = nodes.shape[0] // 2 - max_points // 2
        nodes = nodes[mid:mid + max_points]
    ctx = Context(0, **opts)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    for r in range(reps):
        t = time.time()
        m, st = ctx.label_nodes(nodes)
        wall = time.time() - t
    ev = st["evals"]
    print(f"{opts} cfg{cfg_id}: n={nodes.shape[0]} T={S.n_triangles} K={S.K} evals={ev:.3e} "
          f"label {st['ms_label']:.1f} ms -> {ev / st['ms_label'] * 1e3:.3e} evals/s (frac57 {ev / st['ms_label'] * 1e3 / 6.53e11:.3f}); "
          f"fixup {st['ms_fixup']:.2f} ms flagged_pts={st['flagged_points']} pairs={st['flagged_pairs']} ties={st['ties']} "
          f"near/far subtiles={st['near_subtiles']}/{st['far_subtiles']} ({st['near_subtiles'] / max(1, st['near_subtiles'] + st['far_subtiles']):.4f}) "
          f"wall {wall:.2f}s inside={int(np.count_nonzero(m))}", flush=True)
    ctx.close()


if __name__ == "__main__":
    import os
    opts = {}
    if os.environ.get("NM_FAR_RATIO"):
        opts["far_ratio"] = float(os.environ["NM_FAR_RATIO"])
        opts["far_abs_mm"] = 0.0
    if os.environ.get("NM_LAYOUT"):
        opts["layout"] = int(os.environ["NM_LAYOUT"])
    if os.environ.get("NM_PAIRS"):
        opts["pairs_per_thread"] = int(os.environ["NM_PAIRS"])
    for a in sys.argv[1:]:
        cid, _, mp = a.partition(":")
        run(int(cid), int(mp) if mp else None, **opts)
