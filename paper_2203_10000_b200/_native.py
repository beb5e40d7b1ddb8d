"""ctypes binding of libnestmesh_label.so (include/nestmesh_label.h).

The shared library is built in-tree by ``paper_2203_10000_b200.build`` and is
the only compute path: there is no CPU fallback. Loading fails loudly when the
library is missing; every compute call fails loudly without an sm_100 device.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
LABEL_LIB = Path(os.environ.get("NM_LABEL_LIB", LIB_DIR / "libnestmesh_label.so"))  # override: experiments only
SYNTH_LIB = LIB_DIR / "libnestmesh_synth.so"

c_double_p = ctypes.POINTER(ctypes.c_double)
c_u32_p = ctypes.POINTER(ctypes.c_uint32)
c_i32_p = ctypes.POINTER(ctypes.c_int)
c_u8_p = ctypes.POINTER(ctypes.c_uint8)
c_size_p = ctypes.POINTER(ctypes.c_size_t)


class NmOptions(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("tau", ctypes.c_float),
        ("delta_mm", ctypes.c_float),
        ("band", ctypes.c_double),
        ("tie_eps", ctypes.c_double),
        ("far_ratio", ctypes.c_float),
        ("far_abs_mm", ctypes.c_float),
        ("sort_points", ctypes.c_int),
        ("pairs_per_thread", ctypes.c_int),
        ("layout", ctypes.c_int),
        ("cull_outside", ctypes.c_int),
        ("cell_axis", ctypes.c_int),
    ]


class NmStats(ctypes.Structure):
    _fields_ = [
        ("points", ctypes.c_uint64),
        ("triangles", ctypes.c_uint64),
        ("evals", ctypes.c_uint64),
        ("flagged_points", ctypes.c_uint64),
        ("flagged_pairs", ctypes.c_uint64),
        ("ties", ctypes.c_uint64),
        ("near_subtiles", ctypes.c_uint64),
        ("far_subtiles", ctypes.c_uint64),
        ("launches", ctypes.c_uint64),
        ("ms_label", ctypes.c_float),
        ("ms_fixup", ctypes.c_float),
        ("ms_tets", ctypes.c_float),
        ("ms_total", ctypes.c_float),
        ("ms_host", ctypes.c_float),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class NmSidecarInfo(ctypes.Structure):
    _fields_ = [
        ("n_nodes", ctypes.c_uint64),
        ("n_tets", ctypes.c_uint64),
        ("mesh_fingerprint", ctypes.c_uint64),
        ("K", ctypes.c_int),
        ("has_masks", ctypes.c_int),
        ("is_lattice", ctypes.c_int),
        ("reserved", ctypes.c_int),
        ("label_ids", ctypes.c_int * 32),
        ("threshold", ctypes.c_double),
        ("origin", ctypes.c_double * 3),
        ("h", ctypes.c_double),
        ("n", ctypes.c_int * 3),
        ("reserved2", ctypes.c_int),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if not name.startswith("reserved")}
        d["label_ids"] = list(self.label_ids)[: self.K]
        d["origin"] = tuple(self.origin)
        d["n"] = tuple(self.n)
        return d


# name -> (restype, argtypes); mirrors include/nestmesh_label.h exactly.
LABEL_API = {
    "nm_abi_version": (ctypes.c_int, []),
    "nm_last_error": (ctypes.c_char_p, []),
    "nm_default_options": (None, [ctypes.POINTER(NmOptions)]),
    "nm_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(NmOptions)]),
    "nm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "nm_set_surfaces": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                       c_u32_p, ctypes.c_int, c_i32_p]),
    "nm_enclosure": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, ctypes.c_double, c_double_p,
                                    ctypes.POINTER(NmStats)]),
    "nm_label_nodes": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, ctypes.c_double, c_u32_p,
                                      ctypes.POINTER(NmStats)]),
    "nm_label_tets": (ctypes.c_int, [ctypes.c_void_p, c_u32_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t, c_i32_p,
                                     ctypes.POINTER(NmStats)]),
    "nm_label_mesh": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                     ctypes.c_double, c_i32_p, c_u32_p, ctypes.POINTER(NmStats)]),
    "nm_lattice_device": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_label_lattice": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_double, c_i32_p, c_u32_p, ctypes.POINTER(NmStats)]),
    "nm_label_centroids": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                          ctypes.c_double, c_i32_p, ctypes.POINTER(NmStats)]),
    "nm_flag_boundary": (ctypes.c_int, [ctypes.c_void_p, c_u32_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                        ctypes.c_uint32, c_u32_p, c_size_p]),
    "nm_relabel": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                  ctypes.c_double, ctypes.c_int, c_i32_p, c_i32_p, c_i32_p, c_u8_p,
                                  ctypes.POINTER(NmStats)]),
    "nm_label_nodes_shard_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double,
                                                   ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                   ctypes.POINTER(NmStats)]),
    "nm_label_nodes_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.POINTER(NmStats)]),
    "nm_label_tets_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(NmStats)]),
    "nm_flag_boundary_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                               ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_refine": (ctypes.c_int, [c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t, c_i32_p, c_u32_p,
                                 ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "nm_mesh_sizes": (ctypes.c_int, [ctypes.c_void_p, c_size_p, c_size_p, c_size_p]),
    "nm_mesh_copy": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_u32_p, c_i32_p, c_u32_p]),
    "nm_mesh_free": (None, [ctypes.c_void_p]),
    "nm_refine_last_error": (ctypes.c_char_p, []),
    "nm_mesh_masks": (ctypes.c_int, [ctypes.c_void_p, c_u32_p]),
    "nm_refine_device": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                        c_i32_p, c_u32_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "nm_refine_boundary": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                          c_i32_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "nm_refine_relabel": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                         c_u32_p, ctypes.c_double, ctypes.c_uint32, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(NmStats)]),
    "nm_extract_boundary": (ctypes.c_int, [ctypes.c_void_p, c_u32_p, ctypes.c_size_t, c_i32_p, c_i32_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "nm_boundary_sizes": (ctypes.c_int, [ctypes.c_void_p, c_size_p, c_size_p]),
    "nm_boundary_copy": (ctypes.c_int, [ctypes.c_void_p, c_u32_p, c_u32_p]),
    "nm_boundary_free": (None, [ctypes.c_void_p]),
    "nm_point_surface_distance": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_double_p,
                                                 ctypes.c_size_t, c_u32_p, ctypes.c_size_t, c_double_p,
                                                 ctypes.POINTER(NmStats)]),
    "nm_sample_surface": (ctypes.c_int, [c_double_p, c_u32_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64,
                                         c_double_p]),
    "nm_group_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, c_i32_p,
                                       ctypes.POINTER(NmOptions)]),
    "nm_group_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "nm_group_size": (ctypes.c_int, [ctypes.c_void_p]),
    "nm_group_set_surfaces": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                             c_u32_p, ctypes.c_int, c_i32_p]),
    "nm_group_label_mesh": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                           ctypes.c_double, c_i32_p, c_u32_p, ctypes.POINTER(NmStats)]),
    "nm_group_uses_nccl": (ctypes.c_int, [ctypes.c_void_p]),
    "nm_cell_dump": (ctypes.c_int, [ctypes.c_void_p, c_u32_p, ctypes.c_size_t, c_u8_p, ctypes.c_size_t, c_size_p,
                                    c_size_p]),
    "nm_refine_device_d": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "nm_mesh_copy_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "nm_surface_info": (ctypes.c_int, [ctypes.c_void_p, c_i32_p, c_size_p, c_size_p, c_i32_p]),
    "nm_surface_segments": (ctypes.c_int, [ctypes.c_void_p, c_size_p, c_size_p]),
    "nm_cell_info": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_uint64)] * 3
                     + [c_double_p] + [ctypes.POINTER(ctypes.c_uint64)] * 2),
    "nm_mesh_fingerprint": (ctypes.c_int, [c_double_p, ctypes.c_size_t, c_u32_p, ctypes.c_size_t,
                                           ctypes.POINTER(ctypes.c_uint64)]),
    "nm_mesh_fingerprint_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                                  ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]),
    "nm_sidecar_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(NmSidecarInfo), c_i32_p, c_u32_p]),
    "nm_sidecar_read_info": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(NmSidecarInfo)]),
    "nm_sidecar_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(NmSidecarInfo), c_i32_p, c_u32_p]),
    "nm_label_lattice_sidecar": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_double, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_char_p,
                                                ctypes.c_int, ctypes.POINTER(NmSidecarInfo), ctypes.POINTER(NmStats)]),
}

_lib = None


def load_label_lib() -> ctypes.CDLL:
    """Load the CUDA labeling library; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LABEL_LIB.exists():
        raise ImportError(
            f"{LABEL_LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the labeling path has no CPU fallback)")
    lib = ctypes.CDLL(str(LABEL_LIB))
    for name, (res, args) in LABEL_API.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class NativeError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc != 0:
        msg = load_label_lib().nm_last_error()
        raise NativeError(msg.decode() if msg else f"libnestmesh_label error {rc}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def default_options(**overrides) -> NmOptions:
    opt = NmOptions()
    load_label_lib().nm_default_options(ctypes.byref(opt))
    for k, v in overrides.items():
        setattr(opt, k, v)
    return opt


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream handle


def stream_handle(stream):
    """Map a caller stream to the ABI's void*: None -> the context's own
    stream; 0 (torch's default stream) -> cudaStreamLegacy, so the kernels are
    ordered with torch work on that stream; anything else as is."""
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    return CUDA_STREAM_LEGACY if int(stream) == 0 else int(stream)


class Context:
    """One device + one stream + the replicated surface set (nm_ctx)."""

    def __init__(self, device: int = 0, **options):
        self.lib = load_label_lib()
        opt = default_options(device=device, **options)
        h = ctypes.c_void_p()
        check(self.lib.nm_create(ctypes.byref(h), ctypes.byref(opt)))
        self.handle = h
        self.options = opt
        self.K = 0

    def close(self):
        if getattr(self, "handle", None):
            self.lib.nm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- surfaces ---------------------------------------------------------
    def set_surfaces(self, xyz, tri, comp_off, label_ids):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        tri = np.ascontiguousarray(tri, dtype=np.uint32).reshape(-1, 3)
        comp_off = np.ascontiguousarray(comp_off, dtype=np.uint32)
        label_ids = np.ascontiguousarray(label_ids, dtype=np.int32)
        K = len(label_ids)
        check(self.lib.nm_set_surfaces(self.handle, ptr(xyz, ctypes.c_double), xyz.shape[0], ptr(tri, ctypes.c_uint32),
                                       tri.shape[0], ptr(comp_off, ctypes.c_uint32), K, ptr(label_ids, ctypes.c_int)))
        self.K = K

    def surface_info(self):
        K = ctypes.c_int()
        t = ctypes.c_size_t()
        tp = ctypes.c_size_t()
        lay = ctypes.c_int()
        check(self.lib.nm_surface_info(self.handle, ctypes.byref(K), ctypes.byref(t), ctypes.byref(tp),
                                       ctypes.byref(lay)))
        segs, cont = ctypes.c_size_t(), ctypes.c_size_t()
        check(self.lib.nm_surface_segments(self.handle, ctypes.byref(segs), ctypes.byref(cont)))
        return {"K": K.value, "triangles": t.value, "slots": tp.value, "layout": "strips" if lay.value == 2 else "triangles",
                "segments": segs.value, "continued_segments": cont.value}

    def cell_dump(self):
        """(codes uint32 per level-1 cell, child states uint8) of the certified cells."""
        nc, nch = ctypes.c_size_t(), ctypes.c_size_t()
        check(self.lib.nm_cell_dump(self.handle, None, 0, None, 0, ctypes.byref(nc), ctypes.byref(nch)))
        codes = np.empty(nc.value, np.uint32)
        ch = np.empty(nch.value, np.uint8)
        check(self.lib.nm_cell_dump(self.handle, ptr(codes, ctypes.c_uint32), codes.size, ptr(ch, ctypes.c_uint8),
                                    ch.size, ctypes.byref(nc), ctypes.byref(nch)))
        return codes, ch

    def cell_info(self):
        """Certified-cell culling (cull_outside=2): grid size, certified cells,
        representative evaluations, build time, and the pairs / evaluations
        of the last node pass left to the sparse kernel."""
        v = [ctypes.c_uint64() for _ in range(5)]
        ms = ctypes.c_double()
        check(self.lib.nm_cell_info(self.handle, ctypes.byref(v[0]), ctypes.byref(v[1]), ctypes.byref(v[2]),
                                    ctypes.byref(ms), ctypes.byref(v[3]), ctypes.byref(v[4])))
        return {"cells": v[0].value, "certified": v[1].value, "reps": v[2].value, "ms_build": ms.value,
                "last_pairs": v[3].value, "last_evals": v[4].value}

    # -- host-buffer entry points ----------------------------------------
    def enclosure(self, pts, threshold=0.5):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        s = np.empty((pts.shape[0], self.K), dtype=np.float64)
        st = NmStats()
        check(self.lib.nm_enclosure(self.handle, ptr(pts, ctypes.c_double), pts.shape[0], threshold,
                                    ptr(s, ctypes.c_double), ctypes.byref(st)))
        return s, st.as_dict()

    def label_nodes(self, pts, threshold=0.5):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        m = np.empty(pts.shape[0], dtype=np.uint32)
        st = NmStats()
        check(self.lib.nm_label_nodes(self.handle, ptr(pts, ctypes.c_double), pts.shape[0], threshold,
                                      ptr(m, ctypes.c_uint32), ctypes.byref(st)))
        return m, st.as_dict()

    def label_tets(self, tets, masks):
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        masks = np.ascontiguousarray(masks, dtype=np.uint32)
        out = np.empty(tets.shape[0], dtype=np.int32)
        st = NmStats()
        check(self.lib.nm_label_tets(self.handle, ptr(tets, ctypes.c_uint32), tets.shape[0],
                                     ptr(masks, ctypes.c_uint32), masks.shape[0], ptr(out, ctypes.c_int),
                                     ctypes.byref(st)))
        return out

    def label_mesh(self, nodes, tets, threshold=0.5, want_masks=False, out=None):
        """out: optional int32 array of the tet count (e.g. a pinned buffer) for the labels."""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.empty(tets.shape[0], dtype=np.int32) if out is None else out
        if labels.dtype != np.int32 or labels.shape != (tets.shape[0],) or not labels.flags.c_contiguous:
            raise ValueError("out must be a contiguous int32 array with one entry per tet")
        masks = np.empty(nodes.shape[0], dtype=np.uint32) if want_masks else None
        st = NmStats()
        check(self.lib.nm_label_mesh(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                     ptr(tets, ctypes.c_uint32), tets.shape[0], threshold, ptr(labels, ctypes.c_int),
                                     ptr(masks, ctypes.c_uint32) if masks is not None else None, ctypes.byref(st)))
        return labels, masks, st.as_dict()

    def extract_boundary(self, tets, labels, label_set):
        """(triangles (m,3) uint32 outward + sorted, nodes sorted unique) of the
        region whose labels are in label_set (mesh.hpp:100-155)."""
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        ls = np.ascontiguousarray(np.atleast_1d(label_set), dtype=np.int32)
        h = ctypes.c_void_p()
        check(self.lib.nm_extract_boundary(self.handle, ptr(tets, ctypes.c_uint32), tets.shape[0],
                                           ptr(labels, ctypes.c_int), ptr(ls, ctypes.c_int), ls.size, ctypes.byref(h)))
        try:
            nt_, nn_ = ctypes.c_size_t(), ctypes.c_size_t()
            self.lib.nm_boundary_sizes(h, ctypes.byref(nt_), ctypes.byref(nn_))
            tri = np.empty((nt_.value, 3), np.uint32)
            nodes = np.empty(nn_.value, np.uint32)
            self.lib.nm_boundary_copy(h, ptr(tri, ctypes.c_uint32), ptr(nodes, ctypes.c_uint32))
        finally:
            self.lib.nm_boundary_free(h)
        return tri, nodes

    def point_surface_distance(self, pts, xyz, tri):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        tri = np.ascontiguousarray(tri, dtype=np.uint32).reshape(-1, 3)
        out = np.empty(pts.shape[0], np.float64)
        st = NmStats()
        check(self.lib.nm_point_surface_distance(self.handle, ptr(pts, ctypes.c_double), pts.shape[0],
                                                 ptr(xyz, ctypes.c_double), xyz.shape[0], ptr(tri, ctypes.c_uint32),
                                                 tri.shape[0], ptr(out, ctypes.c_double), ctypes.byref(st)))
        return out, st.as_dict()

    def label_lattice(self, origin, h, n, threshold=0.5, want_masks=False):
        """initial_label of a lattice generated on the device (no host mesh)."""
        o = np.ascontiguousarray(origin, dtype=np.float64)
        nt = 5 * n[0] * n[1] * n[2]
        labels = np.empty(nt, np.int32)
        masks = np.empty((n[0] + 1) * (n[1] + 1) * (n[2] + 1), np.uint32) if want_masks else None
        st = NmStats()
        check(self.lib.nm_label_lattice(self.handle, ptr(o, ctypes.c_double), h, n[0], n[1], n[2], threshold,
                                        ptr(labels, ctypes.c_int),
                                        ptr(masks, ctypes.c_uint32) if masks is not None else None, ctypes.byref(st)))
        return labels, masks, st.as_dict()

    def label_lattice_sidecar(self, origin, h, n, path, threshold=0.5, with_masks=True):
        """initial_label of a regular lattice written straight to a label
        sidecar (nm_label_lattice_sidecar): returns (info dict, stats)."""
        o = np.ascontiguousarray(origin, dtype=np.float64)
        info = NmSidecarInfo()
        st = NmStats()
        check(self.lib.nm_label_lattice_sidecar(self.handle, ptr(o, ctypes.c_double), float(h), int(n[0]), int(n[1]),
                                                int(n[2]), threshold, str(path).encode(), int(bool(with_masks)),
                                                ctypes.byref(info), ctypes.byref(st)))
        return info.as_dict(), st.as_dict()

    def mesh_fingerprint_device(self, d_nodes, d_tets, stream=None):
        fp = ctypes.c_uint64()
        check(self.lib.nm_mesh_fingerprint_device(self.handle, ctypes.c_void_p(d_nodes.data_ptr()), d_nodes.shape[0],
                                                  ctypes.c_void_p(d_tets.data_ptr()), d_tets.shape[0],
                                                  ctypes.byref(fp), stream_handle(stream)))
        return fp.value

    def lattice_device(self, origin, h, n, d_nodes, d_tets, stream=None):
        o = np.ascontiguousarray(origin, dtype=np.float64)
        check(self.lib.nm_lattice_device(self.handle, ptr(o, ctypes.c_double), h, n[0], n[1], n[2],
                                         d_nodes.data_ptr(), d_tets.data_ptr(), stream_handle(stream)))

    def label_centroids(self, nodes, tets, threshold=0.5):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.empty(tets.shape[0], dtype=np.int32)
        st = NmStats()
        check(self.lib.nm_label_centroids(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                          ptr(tets, ctypes.c_uint32), tets.shape[0], threshold,
                                          ptr(labels, ctypes.c_int), ctypes.byref(st)))
        return labels, st.as_dict()

    def flag_boundary(self, tets, masks, active_mask=0xFFFFFFFF):
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        masks = np.ascontiguousarray(masks, dtype=np.uint32)
        ids = np.empty(max(tets.shape[0], 1), dtype=np.uint32)
        cnt = ctypes.c_size_t()
        check(self.lib.nm_flag_boundary(self.handle, ptr(tets, ctypes.c_uint32), tets.shape[0],
                                        ptr(masks, ctypes.c_uint32), masks.shape[0], active_mask,
                                        ptr(ids, ctypes.c_uint32), ctypes.byref(cnt)))
        return ids[: cnt.value].copy()

    def relabel(self, nodes, tets, prev_labels, threshold=0.5, max_iters=64, want_evaluated=False):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.array(prev_labels, dtype=np.int32, copy=True)
        passes = ctypes.c_int()
        conv = ctypes.c_int()
        ev = np.zeros(nodes.shape[0], dtype=np.uint8) if want_evaluated else None
        st = NmStats()
        check(self.lib.nm_relabel(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                  ptr(tets, ctypes.c_uint32), tets.shape[0], threshold, max_iters,
                                  ptr(labels, ctypes.c_int), ctypes.byref(passes), ctypes.byref(conv),
                                  ptr(ev, ctypes.c_uint8) if ev is not None else None, ctypes.byref(st)))
        return labels, passes.value, bool(conv.value), ev, st.as_dict()

    def refine_device(self, nodes, tets, labels, selected):
        """refine_volume on the device: (nodes, tets, labels, parent, n_old)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        lab = np.ascontiguousarray(labels, dtype=np.int32) if labels is not None else None
        sel = np.ascontiguousarray(selected, dtype=np.uint32)
        h = ctypes.c_void_p()
        check(self.lib.nm_refine_device(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                        ptr(tets, ctypes.c_uint32), tets.shape[0],
                                        ptr(lab, ctypes.c_int) if lab is not None else None,
                                        ptr(sel, ctypes.c_uint32), sel.size, ctypes.byref(h)))
        return _take_mesh(self.lib, h)

    def refine_boundary(self, nodes, tets, labels, label_a, label_b):
        """refine_boundary on the device: (nodes, tets, labels, parent, n_old)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        h = ctypes.c_void_p()
        check(self.lib.nm_refine_boundary(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                          ptr(tets, ctypes.c_uint32), tets.shape[0], ptr(labels, ctypes.c_int),
                                          label_a, label_b, ctypes.byref(h)))
        try:
            nn, ntt, nold = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
            self.lib.nm_mesh_sizes(h, ctypes.byref(nn), ctypes.byref(ntt), ctypes.byref(nold))
            on = np.empty((nn.value, 3), np.float64)
            ot = np.empty((ntt.value, 4), np.uint32)
            ol = np.empty(ntt.value, np.int32)
            op = np.empty(ntt.value, np.uint32)
            self.lib.nm_mesh_copy(h, ptr(on, ctypes.c_double), ptr(ot, ctypes.c_uint32), ptr(ol, ctypes.c_int),
                                  ptr(op, ctypes.c_uint32))
        finally:
            self.lib.nm_mesh_free(h)
        return on, ot, ol, op, nold.value

    def refine_relabel(self, nodes, tets, masks=None, levels=2, active_mask=0xFFFFFFFF, threshold=0.5):
        """Recursive boundary driver: returns (nodes, tets, labels, masks, stats)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        m = np.ascontiguousarray(masks, dtype=np.uint32) if masks is not None else None
        h = ctypes.c_void_p()
        st = NmStats()
        check(self.lib.nm_refine_relabel(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                         ptr(tets, ctypes.c_uint32), tets.shape[0],
                                         ptr(m, ctypes.c_uint32) if m is not None else None, threshold, active_mask,
                                         levels, ctypes.byref(h), ctypes.byref(st)))
        try:
            nn, ntt, nold = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
            self.lib.nm_mesh_sizes(h, ctypes.byref(nn), ctypes.byref(ntt), ctypes.byref(nold))
            on = np.empty((nn.value, 3), np.float64)
            ot = np.empty((ntt.value, 4), np.uint32)
            ol = np.empty(ntt.value, np.int32)
            om = np.empty(nn.value, np.uint32)
            self.lib.nm_mesh_copy(h, ptr(on, ctypes.c_double), ptr(ot, ctypes.c_uint32), ptr(ol, ctypes.c_int), None)
            self.lib.nm_mesh_masks(h, ptr(om, ctypes.c_uint32))
        finally:
            self.lib.nm_mesh_free(h)
        return on, ot, ol, om, st.as_dict()

    # -- device-resident entry points (torch tensors) ---------------------
    def refine_device_tensors(self, d_nodes, d_tets, d_labels, d_sel, stream=None):
        """refine_volume on torch CUDA tensors (nm_refine_device_d): returns
        (nodes2, tets2, labels2, parent, n_old) as new tensors on the same
        device; nothing crosses to the host but a few counts."""
        import torch
        h = ctypes.c_void_p()
        check(self.lib.nm_refine_device_d(self.handle, d_nodes.data_ptr(), d_nodes.shape[0], d_tets.data_ptr(),
                                          d_tets.shape[0], d_labels.data_ptr() if d_labels is not None else None,
                                          d_sel.data_ptr(), d_sel.numel(), stream_handle(stream), ctypes.byref(h)))
        try:
            nn, ntt, nold = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
            self.lib.nm_mesh_sizes(h, ctypes.byref(nn), ctypes.byref(ntt), ctypes.byref(nold))
            dev = d_nodes.device
            on = torch.empty((nn.value, 3), dtype=torch.float64, device=dev)
            ot = torch.empty((ntt.value, 4), dtype=torch.int32, device=dev)
            ol = torch.empty(ntt.value, dtype=torch.int32, device=dev)
            op = torch.empty(ntt.value, dtype=torch.int32, device=dev)
            cs = stream if stream is not None else torch.cuda.current_stream(dev)
            check(self.lib.nm_mesh_copy_device(h, on.data_ptr(), ot.data_ptr(), ol.data_ptr(), op.data_ptr(),
                                               stream_handle(cs)))
            cs.synchronize()  # the handle's arrays are released below
        finally:
            self.lib.nm_mesh_free(h)
        return on, ot, ol, op, nold.value

    def label_nodes_device(self, d_pts, d_masks, threshold=0.5, d_s=None, stream=None, stats=True):
        """d_pts: CUDA float64 tensor (n,3); d_masks: CUDA uint32/int32 tensor (n,)."""
        st = NmStats() if stats else None
        check(self.lib.nm_label_nodes_device(self.handle, d_pts.data_ptr(), d_pts.shape[0], threshold,
                                             d_masks.data_ptr(), d_s.data_ptr() if d_s is not None else None,
                                             stream_handle(stream), ctypes.byref(st) if st is not None else None))
        return st.as_dict() if st is not None else None

    def label_nodes_shard_device(self, d_pts, d_masks, shard, nshards, threshold=0.5, stream=None, stats=True):
        """Cost-balanced share `shard` of `nshards` of the node pass over ALL points
        d_pts; the shards' d_masks OR (or add) to the full masks."""
        st = NmStats() if stats else None
        check(self.lib.nm_label_nodes_shard_device(self.handle, d_pts.data_ptr(), d_pts.shape[0], threshold,
                                                   d_masks.data_ptr(), shard, nshards, stream_handle(stream),
                                                   ctypes.byref(st) if st is not None else None))
        return st.as_dict() if st is not None else None

    def label_tets_device(self, d_tets, d_masks, d_labels, stream=None, stats=True):
        st = NmStats() if stats else None
        check(self.lib.nm_label_tets_device(self.handle, d_tets.data_ptr(), d_tets.shape[0], d_masks.data_ptr(),
                                            d_labels.data_ptr(), stream_handle(stream),
                                            ctypes.byref(st) if st is not None else None))
        return st.as_dict() if st is not None else None

    def flag_boundary_device(self, d_tets, d_masks, d_ids, d_count, active_mask=0xFFFFFFFF, stream=None):
        check(self.lib.nm_flag_boundary_device(self.handle, d_tets.data_ptr(), d_tets.shape[0], d_masks.data_ptr(),
                                               active_mask, d_ids.data_ptr(), d_count.data_ptr(),
                                               stream_handle(stream)))


def _take_mesh(lib, h):
    try:
        nn, ntt, nold = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        lib.nm_mesh_sizes(h, ctypes.byref(nn), ctypes.byref(ntt), ctypes.byref(nold))
        on = np.empty((nn.value, 3), np.float64)
        ot = np.empty((ntt.value, 4), np.uint32)
        ol = np.empty(ntt.value, np.int32)
        op = np.empty(ntt.value, np.uint32)
        lib.nm_mesh_copy(h, ptr(on, ctypes.c_double), ptr(ot, ctypes.c_uint32), ptr(ol, ctypes.c_int),
                         ptr(op, ctypes.c_uint32))
    finally:
        lib.nm_mesh_free(h)
    return on, ot, ol, op, nold.value


class Group:
    """Single-process multi-GPU group (nm_group): devices may repeat."""

    def __init__(self, devices, **options):
        self.lib = load_label_lib()
        devs = np.ascontiguousarray(devices, dtype=np.int32)
        opt = default_options(**options)
        h = ctypes.c_void_p()
        check(self.lib.nm_group_create(ctypes.byref(h), devs.size, ptr(devs, ctypes.c_int), ctypes.byref(opt)))
        self.handle = h

    @property
    def uses_nccl(self) -> bool:
        """Masks exchanged by NCCL (distinct devices) rather than peer copies."""
        return bool(self.lib.nm_group_uses_nccl(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self.lib.nm_group_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_surfaces(self, xyz, tri, comp_off, label_ids):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        tri = np.ascontiguousarray(tri, dtype=np.uint32).reshape(-1, 3)
        comp_off = np.ascontiguousarray(comp_off, dtype=np.uint32)
        label_ids = np.ascontiguousarray(label_ids, dtype=np.int32)
        check(self.lib.nm_group_set_surfaces(self.handle, ptr(xyz, ctypes.c_double), xyz.shape[0],
                                             ptr(tri, ctypes.c_uint32), tri.shape[0], ptr(comp_off, ctypes.c_uint32),
                                             len(label_ids), ptr(label_ids, ctypes.c_int)))

    def label_mesh(self, nodes, tets, threshold=0.5):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
        labels = np.empty(tets.shape[0], np.int32)
        masks = np.empty(nodes.shape[0], np.uint32)
        check(self.lib.nm_group_label_mesh(self.handle, ptr(nodes, ctypes.c_double), nodes.shape[0],
                                           ptr(tets, ctypes.c_uint32), tets.shape[0], threshold,
                                           ptr(labels, ctypes.c_int), ptr(masks, ctypes.c_uint32), None))
        return labels, masks


def refine(nodes, tets, labels, selected):
    """refine_volume on the host. Returns (nodes, tets,
    labels, parent, n_old_nodes); new nodes are appended after the old ones."""
    lib = load_label_lib()
    nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
    tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
    labels = np.ascontiguousarray(labels, dtype=np.int32) if labels is not None else None
    sel = np.ascontiguousarray(selected, dtype=np.uint32)
    h = ctypes.c_void_p()
    rc = lib.nm_refine(ptr(nodes, ctypes.c_double), nodes.shape[0], ptr(tets, ctypes.c_uint32), tets.shape[0],
                       ptr(labels, ctypes.c_int) if labels is not None else None, ptr(sel, ctypes.c_uint32), sel.size,
                       ctypes.byref(h))
    if rc != 0:
        raise NativeError(lib.nm_refine_last_error().decode())
    try:
        nn, ntt, nold = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        lib.nm_mesh_sizes(h, ctypes.byref(nn), ctypes.byref(ntt), ctypes.byref(nold))
        on = np.empty((nn.value, 3), np.float64)
        ot = np.empty((ntt.value, 4), np.uint32)
        ol = np.empty(ntt.value, np.int32)
        op = np.empty(ntt.value, np.uint32)
        lib.nm_mesh_copy(h, ptr(on, ctypes.c_double), ptr(ot, ctypes.c_uint32), ptr(ol, ctypes.c_int),
                         ptr(op, ctypes.c_uint32))
    finally:
        lib.nm_mesh_free(h)
    return on, ot, ol, op, nold.value


def sample_surface(xyz, tri, count, seed=0):
    """Area-uniform samples, splitmix64(seed)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    tri = np.ascontiguousarray(tri, dtype=np.uint32).reshape(-1, 3)
    out = np.empty((count, 3), np.float64)
    if load_label_lib().nm_sample_surface(ptr(xyz, ctypes.c_double), ptr(tri, ctypes.c_uint32), tri.shape[0], count,
                                          seed, ptr(out, ctypes.c_double)) != 0:
        raise NativeError("empty surface")
    return out


def mesh_fingerprint(nodes, tets) -> int:
    """nm_mesh_fingerprint (host): order-independent 64-bit mesh fingerprint."""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
    tets = np.ascontiguousarray(tets, dtype=np.uint32).reshape(-1, 4)
    fp = ctypes.c_uint64()
    check(load_label_lib().nm_mesh_fingerprint(ptr(nodes, ctypes.c_double), nodes.shape[0],
                                               ptr(tets, ctypes.c_uint32), tets.shape[0], ctypes.byref(fp)))
    return fp.value


def sidecar_write(path, labels, masks=None, *, n_nodes=None, mesh_fingerprint=0, label_ids=(), threshold=0.5,
                  lattice=None):
    """Write a label sidecar. lattice = (origin, h, (nx, ny, nz)) marks a
    generate_lattice_mesh mesh."""
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    info = NmSidecarInfo()
    info.n_tets = labels.shape[0]
    info.n_nodes = n_nodes if n_nodes is not None else (0 if masks is None else len(masks))
    info.mesh_fingerprint = mesh_fingerprint
    info.K = len(label_ids)
    for k, v in enumerate(label_ids):
        info.label_ids[k] = int(v)
    info.threshold = threshold
    m = None
    if masks is not None:
        m = np.ascontiguousarray(masks, dtype=np.uint32)
        if m.shape[0] != info.n_nodes:
            raise ValueError("masks length != n_nodes")
        info.has_masks = 1
    if lattice is not None:
        (o, h, n) = lattice
        info.is_lattice = 1
        for a in range(3):
            info.origin[a] = float(o[a])
            info.n[a] = int(n[a])
        info.h = float(h)
    check(load_label_lib().nm_sidecar_write(str(path).encode(), ctypes.byref(info), ptr(labels, ctypes.c_int),
                                            ptr(m, ctypes.c_uint32) if m is not None else None))


def sidecar_read(path):
    """(info dict, labels int32, masks uint32 or None)."""
    lib = load_label_lib()
    info = NmSidecarInfo()
    check(lib.nm_sidecar_read_info(str(path).encode(), ctypes.byref(info)))
    labels = np.empty(info.n_tets, np.int32)
    masks = np.empty(info.n_nodes, np.uint32) if info.has_masks else None
    check(lib.nm_sidecar_read(str(path).encode(), ctypes.byref(info), ptr(labels, ctypes.c_int),
                              ptr(masks, ctypes.c_uint32) if masks is not None else None))
    return info.as_dict(), labels, masks


def exported_symbols(path=LABEL_LIB) -> set:
    """Dynamic symbols exported by a shared library (for the ABI test)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def cuda_device_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return os.path.exists("/dev/nvidia0")
