#!/usr/bin/env python
"""Bench: point-triangle solid-angle evaluations/s and full-mesh labeling time
on B200 (BASELINE.json `metric`), one process per GPU.

Workload (default `--config 5`, BASELINE.json configs[4], the config the
metric is quoted on at 1/2/4/8 B200): 12 compartments x icosphere L6
(983,040 triangles) over a 215^3-cell regular lattice (10,077,696 nodes,
49,691,875 tets), T = 0.5. One "step" = one full initial_label of that mesh:
Morton order -> fp32 solid-angle kernel -> flagged-point compaction -> fp64
fix-up -> NCCL all-gather of node masks (N > 1) -> tet labels.

  value      whole-job evals/s with nodes/tets resident in HBM
  e2e        same metric through the public host-buffer API (nm_label_mesh at
             N = 1; pinned host shards + H2D + label + D2H per rank at N > 1)
  roofline   the solid-angle kernel (k_label) against the FP32-pipe roofline
             148 SMs x 128 lanes x 1.965 GHz: achieved = evals/s x the FP32
             lane-ops per eval ncu counted on this build (stamped capture)
  cpu_baseline  the fp64 oracle (oracle/, a port of SPEC.md:225-237) on a
             seeded node sample with every host thread (rank 0, N = 1 only)

`--impl reference` times that CPU implementation alone (rank 0; other ranks
exit 0) on the same metric/config, each step a bounded node sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "point-triangle solid-angle evals/sec and full-mesh labeling time at 1/2/4/8 B200"
UNIT = "evals/s"
OPS_PER_EVAL = 57                      # canonical VOS cost (FP32-pipe ops per eval), for canonical_speedup
# FP32-pipe lane-ops the headline kernel issues per evaluation, MEASURED: ncu
# per-opcode thread-instruction counts of one k_label launch of the same build
# (scripts/ncu_opcounts.sh -> scripts/summarize_ncu.py opcounts), stamped with
# the SASS hash of k_label<1,true,0>; a capture of another build is refused.
# One pair per config (cfg5: scripts/gpu_ncu_r02.sh, cfg2/cfg3: gpu_r02bu.sh).
def opcount_file(cfg):
    return ROOT / "profiles" / "r02" / f"k_label_opcounts_cfg{cfg}.json"


def traffic_file(cfg):
    return ROOT / "profiles" / "r02" / f"k_label_traffic_cfg{cfg}.json"


def stamped(path, sass):
    """A committed ncu summary, only when it was captured on this build."""
    try:
        d = json.loads(path.read_text())
    except Exception:
        return None, f"{path.name} missing"
    if sass is None:
        return None, "cuobjdump unavailable: build hash unknown"
    if d.get("sass_sha16") != sass:
        return None, f"{path.name} was captured on build {d.get('sass_sha16')}, this build is {sass}"
    return d, None
FP32_LANES_PER_SM = 128
MY_KERNELS_PER_STEP = 7                # morton keys, k_label, 3x select, k_fixup, k_label_tets
CUB_KERNELS = 4                        # library radix-sort kernels counted in nm_stats.launches


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # a timed region shorter than nvidia-smi's start-up sees no sample:
        # then keep the first one taken right after it (flagged)
        in_region = len(self.rows)
        deadline = time.time() + 3.0
        while not self.rows and time.time() < deadline:
            time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except ValueError:
                continue
            for nm_, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm_)
        loaded = [v for v in sm if v > 500] or sm
        out = {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if in_region == 0 and sm:
            out["note"] = "timed region shorter than the first nvidia-smi sample; sampled right after it"
        return out


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, local, world


def cpu_baseline(nodes, surfaces, target_s=15.0, seed=0):
    """fp64 oracle (port of SPEC.md:225-237) on a seeded node sample, all threads."""
    import oracle
    cores = oracle.workers_default()
    T = surfaces.n_triangles
    rng = np.random.default_rng(seed)
    probe = nodes[rng.choice(nodes.shape[0], 16, replace=False)]
    t0 = time.perf_counter()
    oracle.label_nodes(probe, surfaces, workers=cores)
    rate = 16 * T / max(time.perf_counter() - t0, 1e-6)
    n_s = int(np.clip(rate * target_s / T, cores, 200000))
    sample = nodes[np.sort(rng.choice(nodes.shape[0], n_s, replace=False))]
    t0 = time.perf_counter()
    oracle.label_nodes(sample, surfaces, workers=cores)
    dt = time.perf_counter() - t0
    return {"value": n_s * T / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n_s} seeded-random lattice nodes x all {T} triangles "
                      f"({n_s / nodes.shape[0]:.2e} of the node set), fp64 VOS oracle, {dt:.1f} s"}


def run_reference(args):
    rank, local, world = dist_env()
    if rank != 0:
        return 0
    from paper_2203_10000_b200 import synth
    import oracle
    cfg = synth.config(args.config)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()
    cores = oracle.workers_default()
    T = S.n_triangles
    rng = np.random.default_rng(1)
    probe = nodes[rng.choice(nodes.shape[0], 16, replace=False)]
    t0 = time.perf_counter()
    oracle.label_nodes(probe, S, workers=cores)
    rate = 16 * T / max(time.perf_counter() - t0, 1e-6)
    n_s = int(np.clip(rate * args.ref_step_s / T, cores, 200000))
    samples = [nodes[np.sort(rng.choice(nodes.shape[0], n_s, replace=False))] for _ in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        oracle.label_nodes(samples[i], S, workers=cores)
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        oracle.label_nodes(samples[args.warmup + i], S, workers=cores)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = n_s * T / (ms / 1e3)
    sample = (f"{n_s} seeded-random lattice nodes x all {T} triangles per step "
              f"({n_s / nodes.shape[0]:.2e} of the node set), fp64 VOS oracle (port of SPEC.md:225-237), {cores} threads")
    full_s = nodes.shape[0] * T / value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": workload_config(cfg, nodes.shape[0], 5 * int(np.prod(cfg.n)), world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "full_mesh_labeling_time_s_extrapolated": full_s,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_recursive(args):
    """cfg4: the 20-compartment model with `levels` rounds of straddle-tet
    refinement, relabeling only the new nodes (nm_refine_relabel). Single GPU.
    value = evals of the new-node passes / their device time (CUDA events);
    the driver's wall time (host refinement included) is reported beside it."""
    import torch
    from paper_2203_10000_b200 import synth
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(4)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    ctx = Context(0)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    m0, st0 = ctx.label_nodes(nodes)
    runs = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        n2, t2, lab, masks, st = ctx.refine_relabel(nodes, tets, masks=m0, levels=args.levels)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            runs.append((wall, st))
    wall = sum(r[0] for r in runs) / len(runs)
    st = runs[-1][1]
    dev_ms = sum(r[1]["ms_label"] + r[1]["ms_fixup"] + r[1]["ms_tets"] for r in runs) / len(runs)
    host_ms = sum(r[1]["ms_host"] for r in runs) / len(runs)  # device refinement (CUDA events)
    evals = st["evals"]
    # check: the recursive result equals a full relabel of the refined mesh
    m_full, _ = ctx.label_nodes(n2)
    lab_full = ctx.label_tets(t2, m_full)
    line = {
        "metric": METRIC, "value": evals / (dev_ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"cfg4: cfg3 + {args.levels} levels of straddle-tet refinement, new nodes only",
                   "initial_nodes": int(nodes.shape[0]), "initial_tets": int(tets.shape[0]),
                   "refined_nodes": int(n2.shape[0]), "refined_tets": int(t2.shape[0]),
                   "new_nodes_evaluated": int(st["points"]), "triangles": S.n_triangles, "compartments": S.K},
        "driver_wall_ms": wall * 1e3, "refine_ms_device": host_ms, "device_ms": dev_ms,
        "initial_label_ms": st0["ms_total"],
        "recursive_equals_full_relabel": bool(np.array_equal(lab, lab_full) and np.array_equal(masks, m_full)),
        "labeling_stats_last_step": {k: st[k] for k in ("flagged_points", "ties", "near_subtiles", "far_subtiles")},
    }
    # the same driver with certified-cell culling (cull_outside=2, the C++
    # drop-in's default): initial labels + both refinement levels
    cc = Context(0, cull_outside=2)
    t0 = time.perf_counter()
    cc.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    t_set = time.perf_counter() - t0
    cw = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        mc, stc0 = cc.label_nodes(nodes)
        n2c, t2c, labc, masksc, stc = cc.refine_relabel(nodes, tets, masks=mc, levels=args.levels)
        if i >= args.warmup:
            cw.append(time.perf_counter() - t0)
    line["cull_outside_mode2"] = {
        "driver_wall_ms_incl_initial_label": sum(cw) / len(cw) * 1e3, "set_surfaces_s": t_set,
        "labels_identical": bool(np.array_equal(labc, lab) and np.array_equal(n2c, n2) and np.array_equal(t2c, t2)),
        "initial_label_ms": stc0["ms_total"]}
    cc.close()
    print(json.dumps(line), flush=True)
    ctx.close()
    del torch
    return 0


def run_recursive_dist(args):
    """cfg4 over N ranks (torchrun): the device-resident recursive driver
    (distributed.refine_relabel_device): every rank holds the mesh on its GPU,
    flags its tet range, the flag lists and the new-node masks are all-gathered
    (NCCL), every rank refines identically and evaluates its shard of the new
    nodes. value = evals of the new-node passes (all ranks) / the max-over-
    ranks device time of the whole driver (CUDA events); the result is checked
    against the single-GPU nm_refine_relabel on rank 0."""
    import torch
    import torch.distributed as dist
    from paper_2203_10000_b200 import synth
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import gather_labels, refine_relabel_device
    rank, local, world = dist_env()
    backend = os.environ.get("NM_DIST_BACKEND", "nccl")
    if os.environ.get("NM_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    cfg = synth.config(4)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    ctx = Context(local)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    d_nodes = torch.from_numpy(nodes).cuda()
    d_tets = torch.from_numpy(tets.view(np.int32)).cuda()
    d_m0 = torch.zeros(nodes.shape[0], dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    ctx.label_nodes_device(d_nodes, d_m0, stream=stream, stats=False)

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = None
    for _ in range(args.warmup):
        out = refine_relabel_device(ctx, d_nodes, d_tets, d_m0, args.levels, rank, world)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = refine_relabel_device(ctx, d_nodes, d_tets, d_m0, args.levels, rank, world)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = allmax(sum(times) / len(times))
    n2, t2, labels, tsh, masks = out
    new_nodes = int(n2.shape[0] - nodes.shape[0])
    evals = new_nodes * S.n_triangles
    full = gather_labels(labels, tsh)
    same = None
    if rank == 0:
        m2, t2r, labr, maskr, _ = ctx.refine_relabel(nodes, tets, masks=d_m0.cpu().numpy().view(np.uint32),
                                                     levels=args.levels)
        same = bool(np.array_equal(full.cpu().numpy(), labr) and np.array_equal(t2.cpu().numpy().view(np.uint32), t2r)
                    and np.array_equal(masks.cpu().numpy().view(np.uint32), maskr))
        line = {
            "metric": METRIC, "value": evals / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg4: cfg3 + {args.levels} levels of straddle-tet refinement, new nodes only, "
                                   f"{world} ranks (device-resident driver, NCCL exchange)",
                       "initial_nodes": int(nodes.shape[0]), "refined_nodes": int(n2.shape[0]),
                       "refined_tets": int(t2.shape[0]), "new_nodes_evaluated": new_nodes,
                       "triangles": S.n_triangles, "parallelism": f"dp{world}"},
            "recursive_equals_single_gpu_driver": same,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    ctx.close()
    return 0


def workload_config(cfg, n_nodes, n_tets, world):
    S = cfg.surfaces
    names = {1: "cfg1 icosphere L3 / 32^3 lattice", 2: "cfg2 4 nested perturbed spheres / 2 mm lattice",
             3: "cfg3 20-compartment head model / 1 mm lattice", 5: "cfg5 large sweep: 12 x icosphere L6 / 215^3 lattice"}
    return {"workload": names.get(cfg.id, f"cfg{cfg.id}"), "nodes": n_nodes, "tets": n_tets,
            "triangles": S.n_triangles, "compartments": S.K, "threshold": 0.5, "cell_mm": cfg.h,
            "parallelism": f"dp{world} (contiguous node shards, NCCL all-gather of uint32 node masks, tet shards)",
            "l2": "256 MiB L2 flush between steps; nodes+tets (1.04 GB at cfg5) exceed the 126 MB L2",
            "evals_per_step": n_nodes * S.n_triangles}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--levels", type=int, default=2, help="--config 4: recursive refinement levels")
    ap.add_argument("--quality", action="store_true", help="also time boundary extraction + boundary_distance")
    ap.add_argument("--no-cull", action="store_true", help="skip the opt-in exact-culling timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 4:
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            return run_recursive_dist(args)
        return run_recursive(args)

    import torch
    rank, local, world = dist_env()
    if world != args.gpus and rank == 0:
        print(f"[bench] note: WORLD_SIZE={world} but --gpus={args.gpus}; using WORLD_SIZE", file=sys.stderr)
    # NM_DIST_BACKEND=gloo + NM_SAME_DEVICE=1: every rank on cuda:0 with a
    # host-side collective — exercises the multi-rank path on a 1-GPU box
    # (the ranks' kernels never wait on one another). Default: NCCL, one GPU
    # per rank.
    backend = os.environ.get("NM_DIST_BACKEND", "nccl")
    if os.environ.get("NM_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    group = None
    use_dist = world > 1 or os.environ.get("NM_FORCE_DIST") == "1"
    if use_dist:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2203_10000_b200 import synth
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import all_gather_masks, shard

    def barrier():
        if use_dist:
            import torch.distributed as dist
            dist.barrier()

    def allmax(x):
        if not use_dist:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = synth.config(args.config)
    S = cfg.surfaces
    t0 = time.perf_counter()
    nodes, tets = cfg.lattice_mesh()
    gen_s = time.perf_counter() - t0
    n, nt = nodes.shape[0], tets.shape[0]
    T = S.n_triangles
    evals_total = n * T
    nsh, tsh = shard(n, world, rank), shard(nt, world, rank)

    ctx = Context(local)
    ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
    sinfo = ctx.surface_info()
    layout = sinfo["layout"]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    d_nodes = torch.from_numpy(nodes[nsh.lo:nsh.hi]).cuda()
    d_tets = torch.from_numpy(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32)).cuda()
    d_masks = torch.zeros(nsh.per, dtype=torch.int32, device="cuda")
    d_labels = torch.empty(tsh.size, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")  # 256 MiB > 126 MB L2

    last = {}

    def step():
        st = ctx.label_nodes_device(d_nodes, d_masks[: nsh.size], stream=sptr, stats=True)
        masks = all_gather_masks(d_masks, nsh, group)
        ctx.label_tets_device(d_tets, masks, d_labels, stream=sptr, stats=False)
        last.update(st)
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ms_label = []
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(i)
        ev[i][0].record(stream)
        st = step()
        ev[i][1].record(stream)
        ms_label.append(st["ms_label"])
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - w0
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_per_step = allmax(sum(step_ms) / len(step_ms))
    value = evals_total / (ms_per_step / 1e3)
    k_ms = sum(ms_label) / len(ms_label)
    achieved = nsh.size * T / (k_ms / 1e3)

    # ---- e2e through the public host-buffer API ------------------------------
    e2e = None
    if not args.no_e2e:
        h_nodes = torch.from_numpy(np.ascontiguousarray(nodes[nsh.lo:nsh.hi])).pin_memory()
        h_tets = torch.from_numpy(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32)).pin_memory()
        h_labels = torch.empty(tsh.size, dtype=torch.int32).pin_memory()
        if not use_dist:
            def e2e_step():
                labels, _, _ = ctx.label_mesh(h_nodes.numpy(), h_tets.numpy().view(np.uint32), out=h_labels.numpy())
                return labels
        else:
            def e2e_step():
                dn = h_nodes.cuda(non_blocking=True)
                dt = h_tets.cuda(non_blocking=True)
                dm = torch.zeros(nsh.per, dtype=torch.int32, device="cuda")
                ctx.label_nodes_device(dn, dm[: nsh.size], stream=sptr, stats=False)
                masks = all_gather_masks(dm, nsh, group)
                dl = torch.empty(tsh.size, dtype=torch.int32, device="cuda")
                ctx.label_tets_device(dt, masks, dl, stream=sptr, stats=False)
                h_labels.copy_(dl)
                return h_labels
        e2e_step()
        torch.cuda.synchronize()
        barrier()
        times = []
        for i in range(args.steps):
            flush.fill_(i)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        e_ms = allmax(1e3 * sum(times) / len(times))
        e2e = {"value": evals_total / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": n * 24 + nt * 16,
               "d2h_bytes_per_step": nt * 4, "ms_per_step": e_ms,
               "path": "nm_label_mesh (C ABI, host buffers)" if world == 1 else
                       "pinned host shards -> nm_label_nodes_device -> NCCL all-gather -> nm_label_tets_device -> D2H"}

    # Exact outside culling (nm_options.cull_outside, opt-in): the same step
    # with compartments skipped for points outside their 13-DOP (winding
    # number exactly 0 for a closed surface). Reported beside the headline,
    # which evaluates every pair.
    cull = None
    if rank == 0 and world == 1 and not args.no_cull:
        cull = {}
        notes = {1: "opt-in exact culling (nm_options.cull_outside=1): a compartment is skipped for points "
                    "outside its 13-DOP (winding number exactly 0 for a closed surface)",
                 2: "cull_outside=2: 13-DOP plus certified cells (per-compartment grid cells whose ball meets no "
                    "triangle carry their exact winding number 0/1; only the remaining (point, compartment) "
                    "pairs are evaluated, by the same k_label loop in sparse mode)"}
        for mode in (1, 2):
            # set_surfaces on fresh contexts: the first call of the process
            # (pinned staging buffers, device pool growth, lazy kernel loading)
            # and the faster of two more (what later contexts pay)
            t_sets = []
            for rep in range(3):
                if rep:
                    cctx.close()
                cctx = Context(local, cull_outside=mode)
                t_set = time.perf_counter()
                cctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
                t_sets.append(time.perf_counter() - t_set)
            t_set_first, t_set = t_sets[0], sorted(t_sets[1:])[0]
            cm = torch.zeros(nsh.per, dtype=torch.int32, device="cuda")
            cctx.label_nodes_device(d_nodes, cm[: nsh.size], stream=sptr, stats=True)
            cl = torch.empty(tsh.size, dtype=torch.int32, device="cuda")
            cms = []
            for i in range(args.steps):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                cctx.label_nodes_device(d_nodes, cm[: nsh.size], stream=sptr, stats=False)
                cctx.label_tets_device(d_tets, cm, cl, stream=sptr, stats=False)
                b.record(stream)
                torch.cuda.synchronize()
                cms.append(a.elapsed_time(b))
            same = bool(torch.equal(cl, d_labels))
            entry = {"full_mesh_labeling_time_s": sum(cms) / len(cms) / 1e3, "labels_identical": same,
                     "set_surfaces_s": t_set, "set_surfaces_first_call_s": t_set_first, "note": notes[mode]}
            if e2e is not None and not use_dist:
                # the same through the host-buffer C ABI (nm_label_mesh: H2D nodes + tets, D2H labels), wall clock
                hl, _, _ = cctx.label_mesh(h_nodes.numpy(), h_tets.numpy().view(np.uint32), out=h_labels.numpy())
                wt = []
                for i in range(args.steps):
                    flush.fill_(i)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    hl, _, _ = cctx.label_mesh(h_nodes.numpy(), h_tets.numpy().view(np.uint32), out=h_labels.numpy())
                    wt.append(time.perf_counter() - t0)
                entry["e2e_full_mesh_labeling_time_s"] = sum(wt) / len(wt)
                entry["e2e_labels_identical"] = bool(np.array_equal(hl, cl.cpu().numpy()))
            if mode == 2:
                ci = cctx.cell_info()
                entry.update({"cells": ci["cells"], "certified_cells": ci["certified"],
                              "representatives": ci["reps"], "cell_build_ms": ci["ms_build"],
                              "pairs_evaluated": ci["last_pairs"], "pairs_total": nsh.size * S.K,
                              "evals_performed": ci["last_evals"]})
            cull["mode%d" % mode] = entry
            cctx.close()
        cull["full_mesh_labeling_time_s"] = cull["mode2"]["full_mesh_labeling_time_s"]
        cull["labels_identical"] = cull["mode1"]["labels_identical"] and cull["mode2"]["labels_identical"]

    # The C++ drop-in end to end (include/nestmesh/labeling.hpp, persistent
    # nestmesh::Labeler; the mesh in the reference's own std::vector types, i.e.
    # pageable host memory): build/libdropin_bench.so, built with the
    # reference headers (tests/cpp/dropin_bench.cpp).
    cpp = None
    dl = ROOT / "build" / "libdropin_bench.so"
    if rank == 0 and world == 1 and not args.no_e2e and dl.exists():
        import ctypes
        L = ctypes.CDLL(str(dl))
        P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
        sx = np.ascontiguousarray(S.xyz, np.float64)
        st_ = np.ascontiguousarray(S.tri, np.uint32)
        so = np.ascontiguousarray(S.comp_off, np.uint32)
        sid = np.ascontiguousarray(S.label_ids, np.int32)
        ref_labels = d_labels.cpu().numpy()
        cpp = {"path": "nestmesh::Labeler::initial_label (C++, reference types, pageable std::vector buffers), "
                       "host clock per call: H2D nodes + tets, labeling, D2H labels"}
        for mode in (0, 2):
            out = np.zeros(6, np.float64)
            lab = np.empty(nt, np.int32)
            k = min(args.steps, 3) if mode == 0 else args.steps
            rc = L.dropin_bench(P(sx, ctypes.c_double), ctypes.c_size_t(sx.shape[0]), P(st_, ctypes.c_uint32),
                                P(so, ctypes.c_uint32), ctypes.c_int(S.K), P(sid, ctypes.c_int),
                                P(nodes, ctypes.c_double), ctypes.c_size_t(n), P(tets, ctypes.c_uint32),
                                ctypes.c_size_t(nt), ctypes.c_int(mode), ctypes.c_int(k), P(out, ctypes.c_double),
                                P(lab, ctypes.c_int))
            if rc != 0:
                cpp["cull%d" % mode] = {"error": "dropin_bench failed"}
                continue
            e = {"labeler_build_s": out[0], "first_call_s": out[1], "e2e_mean_s": out[2], "e2e_best_s": out[3],
                 "e2e_into_mesh_labels_mean_s": out[4], "e2e_into_mesh_labels_best_s": out[5],
                 "steps": k, "evals_per_s_e2e": evals_total / out[2] if out[2] else None,
                 "labels_identical": bool(np.array_equal(lab, ref_labels))}
            pinned = None
            if mode == 2 and cull and "e2e_full_mesh_labeling_time_s" in cull.get("mode2", {}):
                pinned = cull["mode2"]["e2e_full_mesh_labeling_time_s"]
            if mode == 0 and e2e:
                pinned = e2e["ms_per_step"] / 1e3
            if pinned:
                e["vs_python_pinned_e2e"] = out[2] / pinned
                e["into_vs_python_pinned_e2e"] = out[4] / pinned
            cpp["cull%d" % mode] = e

    # N > 1: the certified-cell pass split by COST over the ranks (every rank
    # holds all nodes, evaluates its share of the pair lists; the disjoint
    # partial masks merge in one all-reduce), then each rank's tet range.
    if use_dist and not args.no_cull:
        from paper_2203_10000_b200.distributed import merge_partial_masks
        cctx = Context(local, cull_outside=2)
        t_set = time.perf_counter()
        cctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        t_set = time.perf_counter() - t_set
        d_all = torch.from_numpy(nodes).cuda()
        part = torch.zeros(n, dtype=torch.int32, device="cuda")
        cl = torch.empty(tsh.size, dtype=torch.int32, device="cuda")

        def cstep():
            cctx.label_nodes_shard_device(d_all, part, rank, world, stream=sptr, stats=False)
            full = merge_partial_masks(part, group)
            cctx.label_tets_device(d_tets, full, cl, stream=sptr, stats=False)

        cstep()
        torch.cuda.synchronize()
        cms = []
        for i in range(args.steps):
            flush.fill_(i)
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cstep()
            b.record(stream)
            torch.cuda.synchronize()
            cms.append(a.elapsed_time(b))
        ci = cctx.cell_info()
        my_evals = float(ci["last_evals"])
        c_ms = allmax(sum(cms) / len(cms))
        max_evals = allmax(my_evals)
        same = allmax(0.0 if torch.equal(cl, d_labels) else 1.0) == 0.0
        cull = {"mode2_balanced": {
            "full_mesh_labeling_time_s": c_ms / 1e3, "labels_identical": same, "set_surfaces_s": t_set,
            "max_rank_evals_performed": max_evals, "ranks": world,
            "note": "cull_outside=2 over N ranks: each evaluates its cost-balanced share of the (point, compartment) "
                    "pair lists of all nodes (nm_label_nodes_shard_device); partial masks merged by one all-reduce"}}
        cull["full_mesh_labeling_time_s"] = c_ms / 1e3
        cull["labels_identical"] = same
        cctx.close()

    # §8(f) rows on the labeled mesh (not part of the headline): device
    # extraction of the region boundary of all compartments (the outer
    # surface, extract_region_boundary) and its boundary_distance to the
    # outermost segmentation surface, wall clock.
    quality = None
    if rank == 0 and world == 1 and args.quality:
        from paper_2203_10000_b200.quality import boundary_distance
        labels_h, _, _ = ctx.label_mesh(nodes, tets)
        t0 = time.perf_counter()
        btri, bnodes = ctx.extract_boundary(tets, labels_h, [int(x) for x in S.label_ids])
        t_first = time.perf_counter() - t0  # includes first-use device allocations
        t0 = time.perf_counter()
        btri, bnodes = ctx.extract_boundary(tets, labels_h, [int(x) for x in S.label_ids])
        t_ext = time.perf_counter() - t0
        tx, tt = S.compartment(S.K - 1)
        r = boundary_distance(ctx, nodes, btri, tx, tt, samples=20000, seed=0)  # warm-up
        t0 = time.perf_counter()
        r = boundary_distance(ctx, nodes, btri, tx, tt, samples=20000, seed=0)
        t_dist = time.perf_counter() - t0
        quality = {"region": "all compartments", "target": S.names[-1], "boundary_triangles": int(btri.shape[0]),
                   "extract_boundary_s": t_ext, "extract_boundary_first_call_s": t_first,
                   "boundary_distance_s": t_dist, "distance_cluster_visits": r["stats"]["far_subtiles"],
                   "distance_evals": r["stats"]["evals"], "median_mm": r["median"], "q25_mm": r["q25"],
                   "q75_mm": r["q75"], "fp64_candidates": r["stats"]["flagged_pairs"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(nodes, S, target_s=args.cpu_seconds)

    if rank == 0:
        peaks = measured_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        import torch as _t
        sms = _t.cuda.get_device_properties(local).multi_processor_count
        lane_peak = sms * FP32_LANES_PER_SM * sm_max * 1e6          # FP32 lane-ops/s of the whole GPU
        sys.path.insert(0, str(ROOT / "scripts"))
        from kernel_hash import sass_hash
        sass = sass_hash()
        OPCOUNT_FILE, TRAFFIC_FILE = opcount_file(args.config), traffic_file(args.config)
        ops, ops_why = stamped(OPCOUNT_FILE, sass)
        tr, tr_why = stamped(TRAFFIC_FILE, sass)
        strips = layout == "strips"
        ops_pe = ops["fp32_lane_ops_per_eval"] if (ops and strips) else None
        traffic = tr["traffic_bytes"] * (nsh.size / tr["points"]) if (tr and strips) else None
        roof = {
            "bound": "fp32", "kernel": f"k_label<1,{1 if strips else 0},0> (fp32x2 VOS tile loop, {layout} layout)",
            "achieved": achieved * ops_pe if ops_pe else None,
            "peak": lane_peak, "unit": "FP32 lane-ops/s",
            "frac": achieved * ops_pe / lane_peak if ops_pe else None,
            "traffic": traffic,
            # per point: fp64 xyz + evaluation order in, mask + flag out; plus
            # the triangle tiles once (48 B per padded triangle slot + the
            # 5-float4 subtile records)
            "algorithmic_bytes": nsh.size * (24 + 4 + 8) + sinfo["slots"] * 48
                                 + sinfo["slots"] // 32 * 80,
            "peak_basis": f"{sms} SMs x {FP32_LANES_PER_SM} FP32 lanes x {sm_max:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)",
            "evals_per_s": achieved,
            "fp32_lane_ops_per_eval": ops_pe,
            "ops_source": (f"{OPCOUNT_FILE.relative_to(ROOT)}: ncu sass__thread_inst_executed_true_per_opcode of one "
                           f"k_label launch on this build (sass {sass}), 2 x FFMA2/FADD2/FMUL2 + FFMA/FADD/FMUL"
                           if ops_pe else f"unavailable ({ops_why})"),
            "traffic_source": (f"{TRAFFIC_FILE.relative_to(ROOT)}: ncu dram__bytes_read.sum + dram__bytes_write.sum of "
                               f"one full-mesh k_label launch on this build" if traffic else f"unavailable ({tr_why})"),
            "kernel_ms_avg": k_ms, "kernel_share_of_step": k_ms / (sum(step_ms) / len(step_ms)),
            # the canonical formula's throughput (57 FP32 ops + 5 MUFU per eval), for
            # comparison with the paper-style count; NOT a roofline fraction
            "canonical_speedup": achieved / (lane_peak / OPS_PER_EVAL),
            "continued_segments": f"{sinfo.get('continued_segments', 0)} of {sinfo.get('segments', 0)}",
        }
        if clocks.get("sm_mhz") and ops_pe:
            roof["frac_at_measured_clock"] = achieved * ops_pe / (sms * FP32_LANES_PER_SM * clocks["sm_mhz"] * 1e6)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "dtype_note": "f32 arithmetic, f64 per-tile fold and f64 fix-up of flagged pairs",
            "data": "synthetic",
            "config": dict(workload_config(cfg, n, nt, world), distributed=use_dist),
            "full_mesh_labeling_time_s": ms_per_step / 1e3,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            # this repo's kernels per step: the node pass's launches minus the 4
            # CUB radix-sort kernels, plus k_label_tets
            "gpu_launches": (int(last.get("launches", MY_KERNELS_PER_STEP + 3)) - CUB_KERNELS + 1) * args.steps,
            "labeling_stats_last_step": {k: last[k] for k in ("flagged_points", "flagged_pairs", "ties", "near_subtiles",
                                                              "far_subtiles", "ms_label", "ms_fixup")},
            "lattice_generation_s": gen_s, "timed_wall_s": wall,
            "surface_layout": sinfo,
            "quality": quality,
            "cull_outside": cull,
            "cpp_dropin_e2e": cpp,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        import torch.distributed as dist
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
