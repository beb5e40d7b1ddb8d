"""The N>1 path on CPU: the point partitioner + mask all-gather of
paper_2203_10000_b200.distributed, run with world_size 2 and 3 over gloo, the
per-rank compute being the oracle (the checker). Labels must equal the
single-process labels bit for bit (acceptance #8)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2203_10000_b200 import synth
from paper_2203_10000_b200.distributed import gather_labels, label_mesh_balanced, label_mesh_sharded, shard


def test_shard_partition_properties():
    for n in (0, 1, 7, 35937, 10077696):
        for world in (1, 2, 3, 4, 8):
            parts = [shard(n, world, r) for r in range(world)]
            assert all(p.per == parts[0].per for p in parts)
            assert parts[0].lo == 0 and parts[-1].hi == n
            for a, b in zip(parts, parts[1:]):
                assert a.hi == b.lo
            assert sum(p.size for p in parts) == n
            assert parts[0].padded_total >= n and parts[0].padded_total - n < world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(1)
        S = cfg.surfaces
        nodes, tets = cfg.lattice_mesh()

        def node_fn(pts):
            m = oracle.label_nodes(pts.numpy(), S, workers=2)
            return torch.from_numpy(m.view(np.int32))

        def tet_fn(t, masks):
            lab = oracle.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32), S.label_ids)
            return torch.from_numpy(lab)

        labels, tsh, masks = label_mesh_sharded(nodes, tets, node_fn, tet_fn, rank, world)
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, f"labels_{world}.npy"), full.numpy())
            np.save(os.path.join(out_dir, f"masks_{world}.npy"), masks.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_labels_equal_single_process(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    cfg = synth.config(1)
    nodes, tets = cfg.lattice_mesh()
    m = oracle.label_nodes(nodes, cfg.surfaces)
    ref = oracle.label_tets(tets, m, cfg.surfaces.label_ids)
    np.testing.assert_array_equal(np.load(tmp_path / f"masks_{world}.npy").view(np.uint32), m)
    np.testing.assert_array_equal(np.load(tmp_path / f"labels_{world}.npy"), ref)


def _worker_recursive(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_10000_b200._native import refine
        from paper_2203_10000_b200.distributed import refine_relabel_sharded
        R = 10.0
        S = synth.concat_surfaces([synth.icosphere(0.6 * R, 2), synth.icosphere(R, 2)], labels=[1, 2])
        nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, R / 4, (11, 11, 11))
        m0 = torch.from_numpy(oracle.label_nodes(nodes, S).view(np.int32))

        def node_fn(pts):
            return torch.from_numpy(oracle.label_nodes(pts.numpy(), S, workers=1).view(np.int32))

        def flag_fn(t, masks):
            return torch.from_numpy(oracle.flag_boundary(t.numpy().view(np.uint32), masks.numpy().view(np.uint32))
                                    .astype(np.int32))

        def refine_fn(nd, tt, sel):
            n2, t2, _, _, n_old = refine(nd, tt, None, sel)
            return n2, t2, n_old

        def tet_fn(t, masks):
            return torch.from_numpy(oracle.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32),
                                                      S.label_ids))

        n2, t2, labels, tsh, masks = refine_relabel_sharded(nodes, tets, m0, 2, node_fn, flag_fn, refine_fn, tet_fn,
                                                            rank, world)
        from paper_2203_10000_b200.distributed import gather_labels
        full = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, "rec_labels.npy"), full.numpy())
            np.save(os.path.join(out_dir, "rec_nodes.npy"), n2)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_recursive_driver(tmp_path, world):
    """Refinement flags and new-node masks gathered across ranks: the sharded
    recursive driver equals the single-process driver (and the initial
    labeling of the refined mesh)."""
    mp.spawn(_worker_recursive, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_2203_10000_b200._native import refine
    R = 10.0
    S = synth.concat_surfaces([synth.icosphere(0.6 * R, 2), synth.icosphere(R, 2)], labels=[1, 2])
    nodes, tets = synth.lattice_mesh((-1.3 * R,) * 3, R / 4, (11, 11, 11))
    m = oracle.label_nodes(nodes, S)
    for _ in range(2):
        n2, t2, _, _, n_old = refine(nodes, tets, None, oracle.flag_boundary(tets, m))
        m = np.concatenate([m, oracle.label_nodes(n2[n_old:], S)])
        nodes, tets = n2, t2
    ref = oracle.label_tets(tets, m, S.label_ids)
    np.testing.assert_array_equal(np.load(tmp_path / "rec_nodes.npy"), nodes)
    np.testing.assert_array_equal(np.load(tmp_path / "rec_labels.npy"), ref)
    np.testing.assert_array_equal(ref, oracle.label_tets(tets, oracle.label_nodes(nodes, S), S.label_ids))


def _worker_balanced(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config(1)
        S = synth.concat_surfaces([synth.icosphere(6.0, 3), synth.icosphere(10.0, 3)])
        nodes, tets = cfg.lattice_mesh()
        full = oracle.label_nodes(nodes, S, workers=2)

        def shard_fn(pts, r, w):
            # disjoint ownership of (point, compartment) pairs, as the cost
            # split of nm_label_nodes_shard_device guarantees; the oracle is
            # the per-rank checker
            i = np.arange(pts.shape[0])[:, None]
            c = np.arange(2)[None, :]
            own = ((i + c) % w) == r
            bits = (((full[:, None] >> c.astype(np.uint32)) & 1) * own) << c.astype(np.uint32)
            return torch.from_numpy(bits.sum(axis=1).astype(np.uint32).view(np.int32))

        def tet_fn(t, masks):
            lab = oracle.label_tets(t.numpy().view(np.uint32), masks.numpy().view(np.uint32), S.label_ids)
            return torch.from_numpy(lab)

        labels, tsh, masks = label_mesh_balanced(nodes, tets, shard_fn, tet_fn, rank, world)
        out = gather_labels(labels, tsh)
        if rank == 0:
            np.save(os.path.join(out_dir, f"labels_{world}.npy"), out.numpy())
            np.save(os.path.join(out_dir, f"masks_{world}.npy"), masks.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_balanced_pair_shards_merge_to_single_process(tmp_path, world):
    """label_mesh_balanced: disjoint partial masks merged by one all-reduce
    equal the single-process masks and labels bit for bit."""
    mp.spawn(_worker_balanced, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    cfg = synth.config(1)
    S = synth.concat_surfaces([synth.icosphere(6.0, 3), synth.icosphere(10.0, 3)])
    nodes, tets = cfg.lattice_mesh()
    m = oracle.label_nodes(nodes, S)
    ref = oracle.label_tets(tets, m, S.label_ids)
    np.testing.assert_array_equal(np.load(tmp_path / f"masks_{world}.npy").view(np.uint32), m)
    np.testing.assert_array_equal(np.load(tmp_path / f"labels_{world}.npy"), ref)
