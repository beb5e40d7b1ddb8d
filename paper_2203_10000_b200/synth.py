"""Synthetic inputs (caller side of the labeling boundary).

Thin ctypes layer over libnestmesh_synth.so (csrc/synth.cpp): icosphere, box
surface, the regular 5-tet lattice (proj/include/nestmesh/lattice.hpp:40-91)
and the five BASELINE.json configurations.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._native import SYNTH_LIB, c_double_p, c_i32_p, c_u32_p, c_u8_p, ptr

_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not SYNTH_LIB.exists():
        raise ImportError(f"{SYNTH_LIB} is missing: run __graft_entry__.build()")
    lib = ctypes.CDLL(str(SYNTH_LIB))
    sz = ctypes.c_size_t
    lib.nm_icosphere_vertex_count.restype = sz
    lib.nm_icosphere_vertex_count.argtypes = [ctypes.c_int]
    lib.nm_icosphere_triangle_count.restype = sz
    lib.nm_icosphere_triangle_count.argtypes = [ctypes.c_int]
    lib.nm_icosphere.restype = None
    lib.nm_icosphere.argtypes = [ctypes.c_double, ctypes.c_int, c_double_p, c_double_p, c_u32_p]
    lib.nm_box_surface.restype = None
    lib.nm_box_surface.argtypes = [c_double_p, c_double_p, c_double_p, c_u32_p]
    lib.nm_lattice_node_count.restype = sz
    lib.nm_lattice_node_count.argtypes = [ctypes.c_int] * 3
    lib.nm_lattice_tet_count.restype = sz
    lib.nm_lattice_tet_count.argtypes = [ctypes.c_int] * 3
    lib.nm_lattice_nodes.restype = None
    lib.nm_lattice_nodes.argtypes = [c_double_p, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_double_p]
    lib.nm_lattice_tets.restype = None
    lib.nm_lattice_tets.argtypes = [c_double_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_u32_p]
    lib.nm_synth_config.restype = ctypes.c_void_p
    lib.nm_synth_config.argtypes = [ctypes.c_int]
    lib.nm_synth_free.restype = None
    lib.nm_synth_free.argtypes = [ctypes.c_void_p]
    lib.nm_synth_compartments.restype = ctypes.c_int
    lib.nm_synth_compartments.argtypes = [ctypes.c_void_p]
    lib.nm_synth_vertex_count.restype = sz
    lib.nm_synth_vertex_count.argtypes = [ctypes.c_void_p]
    lib.nm_synth_triangle_count.restype = sz
    lib.nm_synth_triangle_count.argtypes = [ctypes.c_void_p]
    lib.nm_synth_surfaces.restype = None
    lib.nm_synth_surfaces.argtypes = [ctypes.c_void_p, c_double_p, c_u32_p, c_u32_p, c_i32_p, c_i32_p, c_u8_p]
    lib.nm_synth_name.restype = ctypes.c_char_p
    lib.nm_synth_name.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.nm_synth_lattice.restype = None
    lib.nm_synth_lattice.argtypes = [ctypes.c_void_p, c_double_p, c_double_p, c_i32_p]
    _lib = lib
    return lib


def icosphere(radius: float, level: int, center=(0.0, 0.0, 0.0)):
    """(xyz (V,3) float64, tri (T,3) uint32) — primitives.hpp:29-54."""
    lib = _load()
    nv, nt = lib.nm_icosphere_vertex_count(level), lib.nm_icosphere_triangle_count(level)
    xyz = np.empty((nv, 3), np.float64)
    tri = np.empty((nt, 3), np.uint32)
    c = np.asarray(center, np.float64)
    lib.nm_icosphere(radius, level, ptr(c, ctypes.c_double), ptr(xyz, ctypes.c_double), ptr(tri, ctypes.c_uint32))
    return xyz, tri


def box_surface(lo, hi):
    """12 outward triangles — primitives.hpp:75-87."""
    lib = _load()
    xyz = np.empty((8, 3), np.float64)
    tri = np.empty((12, 3), np.uint32)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    lib.nm_box_surface(ptr(lo, ctypes.c_double), ptr(hi, ctypes.c_double), ptr(xyz, ctypes.c_double),
                       ptr(tri, ctypes.c_uint32))
    return xyz, tri


def lattice_nodes(origin, h, n):
    lib = _load()
    o = np.asarray(origin, np.float64)
    nodes = np.empty((lib.nm_lattice_node_count(*n), 3), np.float64)
    lib.nm_lattice_nodes(ptr(o, ctypes.c_double), h, n[0], n[1], n[2], ptr(nodes, ctypes.c_double))
    return nodes


def lattice_mesh(origin, h, n):
    """(nodes (N,3) float64, tets (T,4) uint32) — lattice.hpp:40-91."""
    lib = _load()
    nodes = lattice_nodes(origin, h, n)
    tets = np.empty((lib.nm_lattice_tet_count(*n), 4), np.uint32)
    lib.nm_lattice_tets(ptr(nodes, ctypes.c_double), n[0], n[1], n[2], ptr(tets, ctypes.c_uint32))
    return nodes, tets


@dataclass
class SurfaceSet:
    """Concatenated compartment surfaces, innermost (highest priority) first."""
    xyz: np.ndarray           # (V,3) float64
    tri: np.ndarray           # (T,3) uint32, global vertex ids
    comp_off: np.ndarray      # (K+1,) uint32 triangle offsets
    label_ids: np.ndarray     # (K,) int32
    priorities: np.ndarray    # (K,) int32
    active: np.ndarray        # (K,) uint8
    names: list = field(default_factory=list)

    @property
    def K(self) -> int:
        return len(self.label_ids)

    @property
    def n_triangles(self) -> int:
        return int(self.tri.shape[0])

    def compartment(self, k: int):
        """(xyz, tri) of compartment k with local vertex ids."""
        t = self.tri[self.comp_off[k]:self.comp_off[k + 1]]
        used = np.unique(t)
        remap = np.full(self.xyz.shape[0], -1, np.int64)
        remap[used] = np.arange(used.size)
        return self.xyz[used], remap[t].astype(np.uint32)


@dataclass
class Config:
    id: int
    surfaces: SurfaceSet
    origin: np.ndarray
    h: float
    n: tuple

    @property
    def n_nodes(self) -> int:
        return int(np.prod([v + 1 for v in self.n]))

    @property
    def n_tets(self) -> int:
        return 5 * int(np.prod(self.n))

    def lattice_nodes(self):
        return lattice_nodes(self.origin, self.h, self.n)

    def lattice_mesh(self):
        return lattice_mesh(self.origin, self.h, self.n)


def config(cfg_id: int) -> Config:
    """BASELINE.json configs[cfg_id-1] (cfg 4 shares cfg 3's surfaces/lattice)."""
    lib = _load()
    h = lib.nm_synth_config(cfg_id)
    if not h:
        raise ValueError(f"unknown config {cfg_id}")
    try:
        K = lib.nm_synth_compartments(h)
        nv, nt = lib.nm_synth_vertex_count(h), lib.nm_synth_triangle_count(h)
        xyz = np.empty((nv, 3), np.float64)
        tri = np.empty((nt, 3), np.uint32)
        off = np.empty(K + 1, np.uint32)
        ids = np.empty(K, np.int32)
        pri = np.empty(K, np.int32)
        act = np.empty(K, np.uint8)
        lib.nm_synth_surfaces(h, ptr(xyz, ctypes.c_double), ptr(tri, ctypes.c_uint32), ptr(off, ctypes.c_uint32),
                              ptr(ids, ctypes.c_int), ptr(pri, ctypes.c_int), ptr(act, ctypes.c_uint8))
        names = [lib.nm_synth_name(h, k).decode() for k in range(K)]
        o = np.empty(3, np.float64)
        hh = ctypes.c_double()
        n = np.empty(3, np.int32)
        lib.nm_synth_lattice(h, ptr(o, ctypes.c_double), ctypes.byref(hh), ptr(n, ctypes.c_int))
    finally:
        lib.nm_synth_free(h)
    return Config(cfg_id, SurfaceSet(xyz, tri, off, ids, pri, act, names), o, hh.value, tuple(int(v) for v in n))


def single_surface(xyz, tri, label=1) -> SurfaceSet:
    tri = np.asarray(tri, np.uint32).reshape(-1, 3)
    return SurfaceSet(np.asarray(xyz, np.float64).reshape(-1, 3), tri, np.array([0, tri.shape[0]], np.uint32),
                      np.array([label], np.int32), np.array([1], np.int32), np.array([1], np.uint8), ["surface"])


def concat_surfaces(parts, labels=None) -> SurfaceSet:
    """parts: list of (xyz, tri) innermost first."""
    xs, ts, off = [], [], [0]
    vo = 0
    for xyz, tri in parts:
        xs.append(np.asarray(xyz, np.float64).reshape(-1, 3))
        ts.append(np.asarray(tri, np.uint32).reshape(-1, 3) + np.uint32(vo))
        vo += xs[-1].shape[0]
        off.append(off[-1] + ts[-1].shape[0])
    K = len(parts)
    labels = np.arange(1, K + 1, dtype=np.int32) if labels is None else np.asarray(labels, np.int32)
    return SurfaceSet(np.concatenate(xs), np.concatenate(ts), np.array(off, np.uint32), labels,
                      np.arange(1, K + 1, dtype=np.int32), np.ones(K, np.uint8), [f"s{k}" for k in range(K)])
