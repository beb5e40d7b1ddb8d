"""GPU: the C++ drop-in (labeling.hpp over the reference types) and the NCCL
path of the partitioner (torchrun, one rank, real all_gather)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2203_10000_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_dropin_binary(tmp_path):
    exe = ROOT / "build" / "dropin_test"
    if not exe.exists():
        pytest.skip("build/dropin_test not built (needs the reference headers at build time)")
    out = tmp_path / "labels.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    labels = np.fromfile(out, dtype=np.int32)
    S = synth.concat_surfaces([synth.icosphere(6.0, 3), synth.icosphere(10.0, 3)], labels=[3, 9])
    nodes, tets = synth.lattice_mesh((-12.0, -12.0, -12.0), 0.75, (32, 32, 32))
    ref = oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids)
    np.testing.assert_array_equal(labels, ref)


def test_bench_nccl_path_one_rank(tmp_path):
    """bench.py under torchrun with --force-dist: the NCCL process group, the
    mask all-gather and max-over-ranks timing run for real (world size 1)."""
    env = dict(os.environ, NM_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29533", str(ROOT / "bench.py"), "--config", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["config"]["distributed"] is True


def _gpu_rank(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import gather_labels, label_mesh_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(2)
        S = cfg.surfaces
        nodes, tets = cfg.lattice_mesh()
        ctx = Context(0)
        ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)

        def node_fn(pts):
            m, _ = ctx.label_nodes(pts.numpy())
            return torch.from_numpy(m.view(np.int32))

        def tet_fn(t, masks):
            return torch.from_numpy(ctx.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32)))

        labels, tsh, masks = label_mesh_sharded(nodes, tets, node_fn, tet_fn, rank, world)
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, "labels.npy"), full.numpy())
        ctx.close()
    finally:
        dist.destroy_process_group()


def _gpu_rank_balanced(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import gather_labels, label_mesh_balanced
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(2)
        S = cfg.surfaces
        nodes, tets = cfg.lattice_mesh()
        ctx = Context(0, cull_outside=2)
        ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)

        def shard_fn(pts, r, w):
            d_pts = pts.cuda()
            d_m = torch.zeros(pts.shape[0], dtype=torch.int32, device="cuda")
            ctx.label_nodes_shard_device(d_pts, d_m, r, w)
            torch.cuda.synchronize()
            return d_m.cpu()

        def tet_fn(t, masks):
            return torch.from_numpy(ctx.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32)))

        labels, tsh, masks = label_mesh_balanced(nodes, tets, shard_fn, tet_fn, rank, world)
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, "labels.npy"), full.numpy())
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_balanced_cells_gpu_equals_single(tmp_path):
    """Certified-cell culling over two ranks: each evaluates its cost-balanced
    share of the pair lists (nm_label_nodes_shard_device), the disjoint partial
    masks merge with one all-reduce: labels equal the single-process
    brute-force labels bit for bit."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gpu_rank_balanced, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, _, _ = c.label_mesh(nodes, tets)
    np.testing.assert_array_equal(np.load(tmp_path / "labels.npy"), ref)


def test_two_ranks_sharded_gpu_equals_single(tmp_path):
    """Two ranks (processes) each label their node shard / tet range with the
    CUDA path, masks gathered over gloo: labels equal the single-process GPU
    labels bit for bit (the N>1 path with real kernels; the collective is
    host-side so the two ranks never wait on each other inside a kernel)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gpu_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, _, _ = c.label_mesh(nodes, tets)
    np.testing.assert_array_equal(np.load(tmp_path / "labels.npy"), ref)


@pytest.mark.parametrize("cull", [0, 2])
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_group_multi_context_bitwise(devices, cull):
    """nm_group (single-process multi-device API for C/C++ hosts): with 1, 2
    and 3 contexts (on the one GPU available) the labels and masks are
    bit-identical to a single context (acceptance #8) — with
    contiguous node shards (cull 0) and with the cost-balanced pair-list
    shards of certified-cell culling (cull 2)."""
    from paper_2203_10000_b200._native import Context, Group
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, mref, _ = c.label_mesh(nodes, tets, want_masks=True)
    with Group(devices, cull_outside=cull) as g:
        assert not g.uses_nccl                      # one GPU: peer copies between the contexts
        g.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        lab, m = g.label_mesh(nodes, tets)
    np.testing.assert_array_equal(lab, ref)
    np.testing.assert_array_equal(m, mref)


def test_group_nccl_exchange_one_device(monkeypatch):
    """The NCCL exchange of nm_group (ncclCommInitAll + ncclAllGather in
    place), forced on for a single device (NM_GROUP_NCCL=1): same labels and
    masks as a plain context. With distinct devices this is the path every
    multi-GPU group takes."""
    from paper_2203_10000_b200._native import Context, Group
    monkeypatch.setenv("NM_GROUP_NCCL", "1")
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, mref, _ = c.label_mesh(nodes, tets, want_masks=True)
    with Group([0]) as g:
        assert g.uses_nccl
        g.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        lab, m = g.label_mesh(nodes, tets)
    np.testing.assert_array_equal(lab, ref)
    np.testing.assert_array_equal(m, mref)


def test_label_mesh_chunked_tets_and_bad_index_in_last_chunk():
    """nm_label_mesh labels the tets chunk by chunk under their upload: the
    labels of a multi-chunk mesh (cfg3: 38M tets, five 8M-tet chunks) equal
    the device-buffer path's, and an out-of-range node id in the LAST chunk
    is still reported with its tet."""
    from paper_2203_10000_b200._native import Context, NativeError
    cfg = synth.config(3)
    S = cfg.surfaces
    nodes, tets = cfg.lattice_mesh()
    assert tets.shape[0] > 2 * (8 << 20)  # several 8M-tet chunks
    with Context(0, cull_outside=2) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        lab, _, _ = c.label_mesh(nodes, tets)
        m, _ = c.label_nodes(nodes)
        ref = c.label_tets(tets, m)
        np.testing.assert_array_equal(lab, ref)
        bad = tets.copy()
        bad[-3, 2] = nodes.shape[0]
        with pytest.raises(NativeError, match="references node"):
            c.label_mesh(nodes, bad)


def test_abi_input_validation():
    """The C ABI rejects malformed inputs with a message instead of faulting."""
    from paper_2203_10000_b200._native import Context, NativeError
    xyz, tri = synth.icosphere(5.0, 1)
    with Context(0) as c:
        with pytest.raises(NativeError, match="nm_set_surfaces has not been called"):
            c.label_nodes(np.zeros((4, 3)))
        with pytest.raises(NativeError, match="out of range"):
            c.set_surfaces(xyz, tri + 1000, np.array([0, tri.shape[0]], np.uint32), np.array([1], np.int32))
        with pytest.raises(NativeError, match="comp_tri_off"):
            c.set_surfaces(xyz, tri, np.array([0, 3], np.uint32), np.array([1], np.int32))
        with pytest.raises(NativeError, match="label ids must be > 0"):
            c.set_surfaces(xyz, tri, np.array([0, tri.shape[0]], np.uint32), np.array([0], np.int32))
        c.set_surfaces(xyz, tri, np.array([0, tri.shape[0]], np.uint32), np.array([1], np.int32))
        with pytest.raises(NativeError, match="threshold"):
            c.label_nodes(np.zeros((4, 3)), threshold=1.0)
        with pytest.raises(NativeError, match="references node"):
            c.label_mesh(np.zeros((4, 3)), np.array([[0, 1, 2, 9]], np.uint32))
        with pytest.raises(NativeError, match="references node"):
            c.refine_boundary(np.zeros((4, 3)), np.array([[0, 1, 2, 7]], np.uint32), np.array([1], np.int32), 1, 2)
        # device-side validation (k_max_index), host scan only for the message
        with pytest.raises(NativeError, match="tet 1 references node 4"):
            c.label_tets(np.array([[0, 1, 2, 3], [0, 1, 4, 3]], np.uint32), np.ones(4, np.uint32))
        with pytest.raises(NativeError, match="references node"):
            c.refine_relabel(np.zeros((4, 3)), np.array([[0, 1, 2, 5]], np.uint32), levels=1)
        with pytest.raises(NativeError, match="references node"):
            c.label_mesh(np.zeros((0, 3)), np.array([[0, 0, 0, 0]], np.uint32))
        big = np.tile(np.array([[0, 1, 2, 3]], np.uint32), (100000, 1))
        big[77777, 2] = 4
        with pytest.raises(NativeError, match="tet 77777 references node 4"):
            c.label_mesh(np.zeros((4, 3)), big)
        # still usable after errors
        m, _ = c.label_nodes(np.zeros((1, 3)))
        assert m[0] == 1


def _gpu_rank_recursive(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import gather_labels, refine_relabel_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(2)
        S = cfg.surfaces
        nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 5.0, (44, 44, 44))
        ctx = Context(0)
        ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        m0, _ = ctx.label_nodes(nodes)

        def node_fn(pts):
            m, _ = ctx.label_nodes(pts.numpy())
            return torch.from_numpy(m.view(np.int32))

        def flag_fn(t, masks):
            return torch.from_numpy(ctx.flag_boundary(t.numpy().view(np.uint32), masks.numpy().view(np.uint32))
                                    .astype(np.int32))

        def refine_fn(nd, tt, sel):
            n2, t2, _, _, n_old = ctx.refine_device(nd, tt, None, sel)
            return n2, t2, n_old

        def tet_fn(t, masks):
            return torch.from_numpy(ctx.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32)))

        n2, t2, labels, tsh, masks = refine_relabel_sharded(nodes, tets, torch.from_numpy(m0.view(np.int32)), 2,
                                                            node_fn, flag_fn, refine_fn, tet_fn, rank, world)
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, "labels.npy"), full.numpy())
            np.save(os.path.join(out_dir, "tets.npy"), t2)
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_recursive_driver_gpu(tmp_path):
    """The sharded recursive driver with real kernels on 2 ranks (flags and new
    masks gathered over a host collective) equals the single-process device
    driver nm_refine_relabel bit for bit."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gpu_rank_recursive, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 5.0, (44, 44, 44))
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        n2, t2, lab, masks, st = c.refine_relabel(nodes, tets, levels=2)
    np.testing.assert_array_equal(np.load(tmp_path / "tets.npy"), t2)
    np.testing.assert_array_equal(np.load(tmp_path / "labels.npy"), lab)


def _gpu_rank_recursive_device(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2203_10000_b200._native import Context
    from paper_2203_10000_b200.distributed import gather_labels, refine_relabel_device
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(2)
        S = cfg.surfaces
        nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 5.0, (44, 44, 44))
        ctx = Context(0)
        ctx.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        d_nodes = torch.from_numpy(nodes).cuda()
        d_tets = torch.from_numpy(tets.view(np.int32)).cuda()
        d_m = torch.zeros(nodes.shape[0], dtype=torch.int32, device="cuda")
        ctx.label_nodes_device(d_nodes, d_m, stream=torch.cuda.current_stream(), stats=False)
        n2, t2, labels, tsh, masks = refine_relabel_device(ctx, d_nodes, d_tets, d_m, 2, rank, world)
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, "labels.npy"), full.cpu().numpy())
            np.save(os.path.join(out_dir, "tets.npy"), t2.cpu().numpy().view(np.uint32))
            np.save(os.path.join(out_dir, "nodes.npy"), n2.cpu().numpy())
            np.save(os.path.join(out_dir, "masks.npy"), masks.cpu().numpy().view(np.uint32))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_recursive_driver_device_resident(tmp_path, world):
    """The device-resident multi-rank recursive driver (refine_relabel_device:
    flags, refinement, new-node masks all on the GPU; only counts reach the
    host) over 2 and 3 ranks equals the single-process nm_refine_relabel bit
    for bit (nodes, tets, masks, labels)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gpu_rank_recursive_device, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes, tets = synth.lattice_mesh((-110.0, -110.0, -110.0), 5.0, (44, 44, 44))
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        n2, t2, lab, masks, st = c.refine_relabel(nodes, tets, levels=2)
    np.testing.assert_array_equal(np.load(tmp_path / "nodes.npy"), n2)
    np.testing.assert_array_equal(np.load(tmp_path / "tets.npy"), t2)
    np.testing.assert_array_equal(np.load(tmp_path / "masks.npy"), masks)
    np.testing.assert_array_equal(np.load(tmp_path / "labels.npy"), lab)


def test_device_entry_points_follow_torch_stream():
    """Kernels launched through the *_device entry points with torch's default
    stream are ordered with torch work on it (cudaStreamLegacy mapping): a
    torch copy queued right after the node pass sees the finished masks."""
    import torch
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(2)
    S = cfg.surfaces
    nodes = torch.from_numpy(cfg.lattice_nodes()).cuda()
    with Context(0) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, _ = c.label_nodes(nodes.cpu().numpy())
        m = torch.zeros(nodes.shape[0], dtype=torch.int32, device="cuda")
        stream = torch.cuda.current_stream()
        for _ in range(3):
            m.zero_()
            c.label_nodes_device(nodes, m, stream=stream, stats=False)
            out = m.clone()                       # queued on the same (default) stream
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("world", [2, 3])
def test_bench_multi_rank_on_one_gpu(world):
    """bench.py under torchrun with `world` ranks sharing cuda:0 and a gloo
    (host) collective: the sharded step, the e2e leg and max-over-ranks timing
    run end to end and rank 0 prints one JSON line."""
    env = dict(os.environ, NM_DIST_BACKEND="gloo", NM_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + world}", str(ROOT / "bench.py"), "--gpus", str(world),
           "--config", "2", "--steps", "2", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["cpu_baseline"] is None
    bal = line["cull_outside"]["mode2_balanced"]      # cost-balanced certified-cell pass over the ranks
    assert bal["ranks"] == world and bal["labels_identical"] and bal["full_mesh_labeling_time_s"] > 0


def test_bench_cfg4_two_ranks_on_one_gpu():
    """bench.py --config 4 under torchrun (2 ranks sharing cuda:0, gloo host
    collective): the device-resident recursive driver runs end to end and
    equals the single-GPU nm_refine_relabel (nodes, tets, masks, labels)."""
    env = dict(os.environ, NM_DIST_BACKEND="gloo", NM_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29644", str(ROOT / "bench.py"), "--gpus", "2",
           "--config", "4", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["recursive_equals_single_gpu_driver"] is True


@pytest.mark.parametrize("cull", [0, 1, 2])
def test_shard_device_partials_are_disjoint_and_balanced(cull):
    """nm_label_nodes_shard_device: for 1, 2, 3 and 5 shards the partial masks
    are pairwise disjoint and OR to the single-pass masks (bit-identical), and
    the evaluated work is split evenly (pairs weighted by their compartment's
    tile count)."""
    import torch
    from paper_2203_10000_b200._native import Context
    cfg = synth.config(3)
    S = cfg.surfaces
    nodes = cfg.lattice_nodes()[1_500_000:1_800_000]
    with Context(0, cull_outside=cull) as c:
        c.set_surfaces(S.xyz, S.tri, S.comp_off, S.label_ids)
        ref, _ = c.label_nodes(nodes)
        d_pts = torch.from_numpy(nodes).cuda()
        for R in (1, 2, 3, 5):
            parts, evals = [], []
            for r in range(R):
                d_m = torch.zeros(nodes.shape[0], dtype=torch.int32, device="cuda")
                c.label_nodes_shard_device(d_pts, d_m, r, R)
                torch.cuda.synchronize()
                parts.append(d_m.cpu().numpy().view(np.uint32))
                evals.append(c.cell_info()["last_evals"])
            acc = np.zeros_like(ref)
            for p in parts:
                assert not np.any(acc & p)        # disjoint
                acc |= p
            np.testing.assert_array_equal(acc, ref)
            total = sum(np.uint64(p.astype(np.uint64)) for p in parts)
            np.testing.assert_array_equal(total.astype(np.uint32), ref)  # integer sum = OR (disjoint bits)
            assert max(evals) <= 1.01 * sum(evals) / R + 400_000     # balanced to one pair's weight
        with pytest.raises(RuntimeError):
            c.label_nodes_shard_device(d_pts, torch.zeros(nodes.shape[0], dtype=torch.int32, device="cuda"), 2, 2)
