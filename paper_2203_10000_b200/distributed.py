"""Multi-GPU point partitioner: one process per GPU.

Query points (mesh nodes) are split into equal contiguous shards, one per
rank; the surface set is replicated on every rank. The single exchange step
is an all-gather of the per-node uint32 inside masks (NCCL over NVLink on the
GPU box, gloo in the CPU tests), after which every rank labels its own
contiguous range of tets. Because each node's result is a pure function of its
position the gathered masks, and hence the labels, are identical
for any world size.

With certified-cell culling the per-point work is far from uniform, so
``label_mesh_balanced`` instead gives every rank a cost-balanced share of the
(point, compartment) pairs of all nodes and merges the disjoint partial masks
with one all-reduce.

The per-rank compute is injected (``node_fn`` / ``tet_fn``) so the CPU tests
can exercise exactly this sharding + gather logic with the oracle as the
per-rank checker, while the GPU path plugs in the CUDA entry points.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n: int          # global item count
    per: int        # padded shard length (equal on every rank)
    lo: int         # first global item of this rank
    hi: int         # one past the last real item of this rank

    @property
    def size(self) -> int:
        return self.hi - self.lo

    @property
    def padded_total(self) -> int:
        return self.per * self.world


def shard(n: int, world: int, rank: int) -> Shard:
    """Equal contiguous shards; the tail rank(s) are padded so the all-gather
    moves equal-sized buffers."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = (n + world - 1) // world if n else 0
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return Shard(rank, world, n, per, lo, hi)


def all_gather_masks(local: "torch.Tensor", sh: Shard, group=None) -> "torch.Tensor":
    """Gather equal-length (padded) mask shards into one (n,) tensor."""
    import torch
    import torch.distributed as dist
    buf = local
    if local.shape[0] != sh.per:
        buf = torch.zeros(sh.per, dtype=local.dtype, device=local.device)
        buf[: local.shape[0]] = local
    out = torch.empty(sh.padded_total, dtype=local.dtype, device=local.device)
    if dist.is_available() and dist.is_initialized():
        if buf.is_cuda and dist.get_backend(group) == "gloo":
            # host-side collective (tests / single-GPU multi-rank runs)
            host = torch.empty(sh.padded_total, dtype=local.dtype)
            dist.all_gather_into_tensor(host, buf.cpu(), group=group)
            out.copy_(host)
        else:
            dist.all_gather_into_tensor(out, buf, group=group)
    else:
        out.copy_(buf)
    return out[: sh.n]


def label_mesh_sharded(nodes, tets, node_fn, tet_fn, rank: int, world: int, group=None, device="cpu"):
    """initial_label over `world` ranks.

    nodes: (N,3) float64 (host, every rank may hold the full array or only its
    shard — only rows [lo, hi) are read); tets: (T,4) uint32.
    node_fn(points (n,3) f64 torch) -> masks (n,) int32 torch on `device`.
    tet_fn(tets (t,4) torch, masks (N,) torch) -> labels (t,) int32 torch.
    Returns (labels of this rank's tet range, tet shard, full masks).
    """
    import torch
    n = nodes.shape[0]
    nsh = shard(n, world, rank)
    pts = torch.as_tensor(np.ascontiguousarray(nodes[nsh.lo:nsh.hi]), dtype=torch.float64, device=device)
    local = node_fn(pts)
    masks = all_gather_masks(local, nsh, group)
    tsh = shard(tets.shape[0], world, rank)
    t = torch.as_tensor(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32), device=device)
    labels = tet_fn(t, masks)
    return labels, tsh, masks


def merge_partial_masks(local: "torch.Tensor", group=None) -> "torch.Tensor":
    """Per-rank partial masks with pairwise DISJOINT bits (the cost-balanced
    pair-list shards of nm_label_nodes_shard_device) -> the full masks on
    every rank: one all-reduce SUM — disjoint bits add without carries, so
    the sum is the bitwise OR (NCCL has no OR reduction)."""
    import torch
    import torch.distributed as dist
    out = local.clone()
    if dist.is_available() and dist.is_initialized():
        if out.is_cuda and dist.get_backend(group) == "gloo":
            host = out.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            out.copy_(host)
        else:
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def label_mesh_balanced(nodes, tets, shard_fn, tet_fn, rank: int, world: int, group=None, device="cpu"):
    """initial_label with the node pass split by COST rather than by points
    (certified-cell culling leaves only the pairs near a surface, so equal
    point ranges would not be equal work). Every rank holds all nodes.

    shard_fn(points (N,3) f64 torch, rank, world) -> (N,) int32 partial masks
    whose bits are disjoint across ranks (nm_label_nodes_shard_device on the
    GPU); tet_fn as in label_mesh_sharded. Returns (labels of this rank's tet
    range, tet shard, full masks)."""
    import torch
    pts = torch.as_tensor(np.ascontiguousarray(nodes), dtype=torch.float64, device=device)
    masks = merge_partial_masks(shard_fn(pts, rank, world), group)
    tsh = shard(tets.shape[0], world, rank)
    t = torch.as_tensor(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32), device=device)
    return tet_fn(t, masks), tsh, masks


def gather_labels(labels: "torch.Tensor", sh: Shard, group=None) -> "torch.Tensor":
    """All-gather per-rank tet label ranges into the full (T,) label vector."""
    return all_gather_masks(labels, sh, group)


def _gather_into(out, buf, group):
    """all_gather_into_tensor; a host-side collective when the backend is gloo
    and the tensors live on the GPU (single-GPU multi-rank runs, tests)."""
    import torch
    import torch.distributed as dist
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, buf.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, buf, group=group)


def all_gather_varlen(local: "torch.Tensor", group=None) -> "torch.Tensor":
    """All-gather of variable-length 1-D tensors (rank order preserved):
    counts first, then equal padded buffers. Device tensors
    stay on the device with NCCL."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local.clone()
    world = dist.get_world_size(group)
    cnt = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    cnts = torch.empty(world, dtype=torch.int64, device=local.device)
    _gather_into(cnts, cnt, group)
    cl = [int(c) for c in cnts.tolist()]
    mx = max(cl) if cl else 0
    buf = torch.zeros(max(mx, 1), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = torch.empty(world * max(mx, 1), dtype=local.dtype, device=local.device)
    _gather_into(out, buf, group)
    parts = [out[r * max(mx, 1): r * max(mx, 1) + cl[r]] for r in range(world)]
    return torch.cat(parts) if parts else local[:0]


def refine_relabel_sharded(nodes, tets, masks, levels, node_fn, flag_fn, refine_fn, tet_fn, rank: int, world: int,
                           group=None, device="cpu"):
    """The recursive boundary driver over `world` ranks (PAPER.md:151,
    SPEC.md:294-297): per level, every rank flags the straddling tets of its
    tet range, the flag lists are all-gathered (refinement flags over NCCL on
    the GPU box), every rank refines the same mesh with the same selection
    (deterministic numbering -> identical meshes), evaluates only ITS shard of
    the new nodes and the new masks are all-gathered. Returns (nodes, tets,
    labels of this rank's tet range, tet shard, masks).

    node_fn(points (m,3) f64 torch) -> masks (m,) int32 torch
    flag_fn(tets (t,4) torch, masks (N,) torch) -> ascending local ids (int32 torch)
    refine_fn(nodes, tets, selected) -> (nodes2, tets2, n_old)   (host numpy)
    tet_fn(tets (t,4) torch, masks (N,) torch) -> labels (t,) int32 torch
    """
    import torch
    masks = masks.to(device)
    for _ in range(levels):
        tsh = shard(tets.shape[0], world, rank)
        t_local = torch.as_tensor(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32), device=device)
        ids = flag_fn(t_local, masks).to(torch.int64) + tsh.lo
        sel = all_gather_varlen(ids, group).cpu().numpy().astype(np.uint32)
        nodes2, tets2, n_old = refine_fn(nodes, tets, sel)
        new = nodes2[n_old:]
        nsh = shard(new.shape[0], world, rank)
        m_local = node_fn(torch.as_tensor(np.ascontiguousarray(new[nsh.lo:nsh.hi]), dtype=torch.float64,
                                          device=device))
        m_new = all_gather_masks(m_local, nsh, group)
        masks = torch.cat([masks, m_new])
        nodes, tets = nodes2, tets2
    tsh = shard(tets.shape[0], world, rank)
    t_local = torch.as_tensor(np.ascontiguousarray(tets[tsh.lo:tsh.hi]).view(np.int32), device=device)
    labels = tet_fn(t_local, masks)
    return nodes, tets, labels, tsh, masks


def refine_relabel_device(ctx, d_nodes, d_tets, d_masks, levels: int, rank: int, world: int, group=None,
                          active_mask: int = 0xFFFFFFFF):
    """The recursive boundary driver over `world` ranks with the mesh resident
    on every rank's GPU. Per level:
      1. each rank flags the straddling tets of ITS tet range on the device
         (nm_flag_boundary_device: ordered compaction);
      2. the flag lists are all-gathered (NCCL; ascending, so every rank gets
         the same global selection);
      3. every rank refines the same mesh with the same selection on its GPU
         (nm_refine_device_d; deterministic numbering -> identical meshes);
      4. each rank evaluates ITS shard of the new nodes and the new masks are
         all-gathered (NCCL).
    Nothing crosses to the host but counts. Returns (nodes, tets, labels of
    this rank's tet range, tet shard, masks), all device tensors; equal bit
    for bit to nm_refine_relabel on one GPU.

    ctx: a Context on this rank's device with the surfaces set; d_nodes
    (N,3) float64, d_tets (T,4) int32, d_masks (N,) int32 CUDA tensors."""
    import torch
    dev = d_nodes.device
    cs = torch.cuda.current_stream(dev)  # every kernel ordered with the torch collectives on this stream
    for _ in range(levels):
        tsh = shard(d_tets.shape[0], world, rank)
        ids = torch.empty(max(tsh.size, 1), dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        if tsh.size:
            ctx.flag_boundary_device(d_tets[tsh.lo:tsh.hi], d_masks, ids, cnt, active_mask=active_mask, stream=cs)
        k = int(cnt.item())
        sel = all_gather_varlen(ids[:k].to(torch.int64) + tsh.lo, group).to(torch.int32)
        nodes2, tets2, _, _, n_old = ctx.refine_device_tensors(d_nodes, d_tets, None, sel, stream=cs)
        new = nodes2[n_old:]
        nsh = shard(new.shape[0], world, rank)
        m_local = torch.zeros(max(nsh.per, 1), dtype=torch.int32, device=dev)
        if nsh.size:
            ctx.label_nodes_device(new[nsh.lo:nsh.hi], m_local[: nsh.size], stream=cs, stats=False)
        m_new = all_gather_masks(m_local[: nsh.per], nsh, group) if nsh.per else m_local[:0]
        d_masks = torch.cat([d_masks, m_new])
        d_nodes, d_tets = nodes2, tets2
    tsh = shard(d_tets.shape[0], world, rank)
    labels = torch.empty(max(tsh.size, 1), dtype=torch.int32, device=dev)[: tsh.size]
    if tsh.size:
        ctx.label_tets_device(d_tets[tsh.lo:tsh.hi], d_masks, labels, stream=cs, stats=False)
    return d_nodes, d_tets, labels, tsh, d_masks
