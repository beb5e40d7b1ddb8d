"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the fp64 CPU oracle
(oracle/labeling_oracle.cpp) and of the reference-header shim (oracle/_ref).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package. The product path never does.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "build" / "liblabel_oracle.so"
REF_LIB = HERE / "_ref" / "libnestmesh_ref.so"

_d = ctypes.POINTER(ctypes.c_double)
_u32 = ctypes.POINTER(ctypes.c_uint32)
_i32 = ctypes.POINTER(ctypes.c_int)
_u8 = ctypes.POINTER(ctypes.c_uint8)
_sz = ctypes.c_size_t

_lib = None
_ref = None


def _p(a, t):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def lib():
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            raise ImportError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(ORACLE_LIB))
        L.oracle_enclosure.argtypes = [_d, _sz, _d, _u32, _u32, ctypes.c_int, ctypes.c_int, _d]
        L.oracle_label_nodes.argtypes = [_d, _sz, _d, _u32, _u32, ctypes.c_int, ctypes.c_double, ctypes.c_int, _u32, _d]
        L.oracle_label_tets.argtypes = [_u32, _sz, _u32, _i32, ctypes.c_int, _i32]
        L.oracle_flag_boundary.argtypes = [_u32, _sz, _u32, ctypes.c_uint32, _u32]
        L.oracle_flag_boundary.restype = _sz
        L.oracle_relabel_recursive.argtypes = [_d, _sz, _u32, _sz, _d, _u32, _u32, _i32, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int, ctypes.c_int, _i32, _i32, _u8, ctypes.POINTER(_sz)]
        L.oracle_point_surface_distance.argtypes = [_d, _sz, _d, _u32, _sz, ctypes.c_int, _d]
        L.oracle_lhuilier_solid_angle.argtypes = [_d, _d, _d, _d]
        L.oracle_lhuilier_solid_angle.restype = ctypes.c_double
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_LIB.exists()


def ref():
    """The unmodified reference headers behind oracle/ref_shim.cpp."""
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise ImportError(f"{REF_LIB} missing (built only where /root/reference exists)")
        R = ctypes.CDLL(str(REF_LIB))
        R.ref_icosphere.argtypes = [ctypes.c_double, ctypes.c_int, _d, _d, _u32]
        R.ref_box_surface.argtypes = [_d, _d, _d, _u32]
        R.ref_lattice_mesh.argtypes = [_d, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d, _u32]
        R.ref_lattice_covering.argtypes = [_d, _d, ctypes.c_double, _d, _i32]
        R.ref_validate_closed.argtypes = [_d, _sz, _u32, _sz]
        R.ref_validate_closed.restype = ctypes.c_int
        R.ref_signed_volume.argtypes = [_d, _sz, _u32, _sz]
        R.ref_signed_volume.restype = ctypes.c_double
        R.ref_compartment_boundary_size.argtypes = [_d, _sz, _u32, _sz, _i32, ctypes.c_int]
        R.ref_compartment_boundary_size.restype = ctypes.c_long
        R.ref_boundary.argtypes = [_u32, _sz, _i32, _i32, ctypes.c_int, _u32, _sz, _u32, _sz, ctypes.POINTER(_sz)]
        R.ref_boundary.restype = ctypes.c_long
        R.ref_validate_mesh_ok.argtypes = [_d, _sz, _u32, _sz]
        R.ref_validate_mesh_ok.restype = ctypes.c_int
        R.ref_save_tetmesh.argtypes = [ctypes.c_char_p, _d, _sz, _u32, _i32, _sz]
        R.ref_load_tetmesh.argtypes = [ctypes.c_char_p, ctypes.POINTER(_sz), ctypes.POINTER(_sz), _d, _u32, _i32]
        _ref = R
    return _ref


def ref_boundary(tets, labels, label_set):
    """The UNMODIFIED reference extract_compartment_boundary / extract_region_boundary."""
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    labels = np.ascontiguousarray(labels, np.int32)
    ls = np.ascontiguousarray(np.atleast_1d(label_set), np.int32)
    cap = 4 * tets.shape[0]
    tri = np.empty((max(cap, 1), 3), np.uint32)
    nodes = np.empty(max(4 * tets.shape[0], 1), np.uint32)
    nn = ctypes.c_size_t()
    c = ref().ref_boundary(_p(tets, ctypes.c_uint32), tets.shape[0], _p(labels, ctypes.c_int), _p(ls, ctypes.c_int),
                           ls.size, _p(tri, ctypes.c_uint32), cap, _p(nodes, ctypes.c_uint32), nodes.size,
                           ctypes.byref(nn))
    if c < 0:
        raise KeyError(f"UnknownLabel {label_set}")
    return tri[:c].copy(), nodes[:nn.value].copy()


def ref_save_tetmesh(path, nodes, tets, labels):
    """The UNMODIFIED reference save_tetmesh (tetmesh v1 text, mesh.hpp:238-289)."""
    nodes = np.ascontiguousarray(nodes, np.float64).reshape(-1, 3)
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    labels = np.ascontiguousarray(labels, np.int32)
    assert ref().ref_save_tetmesh(str(path).encode(), _p(nodes, ctypes.c_double), nodes.shape[0],
                                  _p(tets, ctypes.c_uint32), _p(labels, ctypes.c_int), tets.shape[0]) == 0


def ref_load_tetmesh(path):
    R = ref()
    nn, nt = _sz(), _sz()
    assert R.ref_load_tetmesh(str(path).encode(), ctypes.byref(nn), ctypes.byref(nt), None, None, None) == 0
    nodes = np.empty((nn.value, 3), np.float64)
    tets = np.empty((nt.value, 4), np.uint32)
    labels = np.empty(nt.value, np.int32)
    assert R.ref_load_tetmesh(str(path).encode(), ctypes.byref(nn), ctypes.byref(nt), _p(nodes, ctypes.c_double),
                              _p(tets, ctypes.c_uint32), _p(labels, ctypes.c_int)) == 0
    return nodes, tets, labels


def workers_default() -> int:
    return os.cpu_count() or 1


def _surf(surfaces):
    xyz = np.ascontiguousarray(surfaces.xyz, np.float64)
    tri = np.ascontiguousarray(surfaces.tri, np.uint32)
    off = np.ascontiguousarray(surfaces.comp_off, np.uint32)
    return xyz, tri, off


def enclosure(pts, surfaces, workers=0):
    """s[i,k] in fp64."""
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    xyz, tri, off = _surf(surfaces)
    K = len(off) - 1
    s = np.empty((pts.shape[0], K), np.float64)
    lib().oracle_enclosure(_p(pts, ctypes.c_double), pts.shape[0], _p(xyz, ctypes.c_double), _p(tri, ctypes.c_uint32),
                           _p(off, ctypes.c_uint32), K, workers, _p(s, ctypes.c_double))
    return s


def label_nodes(pts, surfaces, T=0.5, workers=0, want_s=False):
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    xyz, tri, off = _surf(surfaces)
    K = len(off) - 1
    m = np.empty(pts.shape[0], np.uint32)
    s = np.empty((pts.shape[0], K), np.float64) if want_s else None
    rc = lib().oracle_label_nodes(_p(pts, ctypes.c_double), pts.shape[0], _p(xyz, ctypes.c_double),
                                  _p(tri, ctypes.c_uint32), _p(off, ctypes.c_uint32), K, T, workers,
                                  _p(m, ctypes.c_uint32), _p(s, ctypes.c_double))
    assert rc == 0
    return (m, s) if want_s else m


def label_tets(tets, masks, label_ids):
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    masks = np.ascontiguousarray(masks, np.uint32)
    ids = np.ascontiguousarray(label_ids, np.int32)
    out = np.empty(tets.shape[0], np.int32)
    lib().oracle_label_tets(_p(tets, ctypes.c_uint32), tets.shape[0], _p(masks, ctypes.c_uint32),
                            _p(ids, ctypes.c_int), len(ids), _p(out, ctypes.c_int))
    return out


def flag_boundary(tets, masks, active_mask=0xFFFFFFFF):
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    masks = np.ascontiguousarray(masks, np.uint32)
    out = np.empty(max(tets.shape[0], 1), np.uint32)
    c = lib().oracle_flag_boundary(_p(tets, ctypes.c_uint32), tets.shape[0], _p(masks, ctypes.c_uint32),
                                   active_mask, _p(out, ctypes.c_uint32))
    return out[:c].copy()


def relabel_recursive(nodes, tets, surfaces, prev_labels, T=0.5, max_iters=64, workers=0):
    nodes = np.ascontiguousarray(nodes, np.float64).reshape(-1, 3)
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    xyz, tri, off = _surf(surfaces)
    ids = np.ascontiguousarray(surfaces.label_ids, np.int32)
    labels = np.array(prev_labels, np.int32, copy=True)
    conv = ctypes.c_int()
    ev = np.zeros(nodes.shape[0], np.uint8)
    nev = ctypes.c_size_t()
    passes = lib().oracle_relabel_recursive(
        _p(nodes, ctypes.c_double), nodes.shape[0], _p(tets, ctypes.c_uint32), tets.shape[0],
        _p(xyz, ctypes.c_double), _p(tri, ctypes.c_uint32), _p(off, ctypes.c_uint32), _p(ids, ctypes.c_int),
        len(ids), T, max_iters, workers, _p(labels, ctypes.c_int), ctypes.byref(conv), _p(ev, ctypes.c_uint8),
        ctypes.byref(nev))
    return labels, passes, bool(conv.value), ev


def point_surface_distance(pts, xyz, tri, workers=0):
    """quality.boundary_distance restatement, fp64."""
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
    tri = np.ascontiguousarray(tri, np.uint32).reshape(-1, 3)
    out = np.empty(pts.shape[0], np.float64)
    lib().oracle_point_surface_distance(_p(pts, ctypes.c_double), pts.shape[0], _p(xyz, ctypes.c_double),
                                        _p(tri, ctypes.c_uint32), tri.shape[0], workers, _p(out, ctypes.c_double))
    return out


def lhuilier(p, a, b, c):
    arr = [np.ascontiguousarray(x, np.float64) for x in (p, a, b, c)]
    return lib().oracle_lhuilier_solid_angle(*[_p(x, ctypes.c_double) for x in arr])


REFINE_LIB = HERE / "build" / "librefine_oracle.so"
_rlib = None


def _refine_lib():
    global _rlib
    if _rlib is None:
        if not REFINE_LIB.exists():
            raise ImportError(f"{REFINE_LIB} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(REFINE_LIB))
        L.oracle_refine.argtypes = [_d, _sz, _u32, _sz, _i32, _u32, _sz]
        L.oracle_refine.restype = ctypes.c_void_p
        L.oracle_refine_sizes.argtypes = [ctypes.c_void_p, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]
        L.oracle_refine_copy.argtypes = [ctypes.c_void_p, _d, _u32, _i32, _u32]
        L.oracle_refine_free.argtypes = [ctypes.c_void_p]
        L.oracle_refine_last_error.restype = ctypes.c_char_p
        _rlib = L
    return _rlib


def refine_volume(nodes, tets, labels, selected):
    """refine_volume restatement (oracle/refine_oracle.cpp, SPEC.md:285-293,
    311-312, 321): returns nodes, tets, labels, parent (children in an
    oracle-chosen order inside each parent; compare with canonical_children)."""
    L = _refine_lib()
    nodes = np.ascontiguousarray(nodes, np.float64).reshape(-1, 3)
    tets = np.ascontiguousarray(tets, np.uint32).reshape(-1, 4)
    lab = None if labels is None else np.ascontiguousarray(labels, np.int32)
    sel = np.ascontiguousarray(np.asarray(selected, np.uint32).reshape(-1))
    h = L.oracle_refine(_p(nodes, ctypes.c_double), nodes.shape[0], _p(tets, ctypes.c_uint32), tets.shape[0],
                        _p(lab, ctypes.c_int), _p(sel, ctypes.c_uint32), sel.size)
    if not h:
        raise ValueError(L.oracle_refine_last_error().decode())
    nn, nt = _sz(), _sz()
    L.oracle_refine_sizes(h, ctypes.byref(nn), ctypes.byref(nt))
    on = np.empty((nn.value, 3), np.float64)
    ot = np.empty((nt.value, 4), np.uint32)
    ol = np.empty(nt.value, np.int32)
    op = np.empty(nt.value, np.uint32)
    L.oracle_refine_copy(h, _p(on, ctypes.c_double), _p(ot, ctypes.c_uint32), _p(ol, ctypes.c_int),
                         _p(op, ctypes.c_uint32))
    L.oracle_refine_free(h)
    return on, ot, ol, op


def canonical_children(tets, labels, parent):
    """Children as a sorted table of (parent, sorted node ids, label): the
    comparison key for refinements whose within-parent child order differs."""
    t = np.sort(np.asarray(tets, np.int64).reshape(-1, 4), axis=1)
    rows = np.column_stack([np.asarray(parent, np.int64), t, np.asarray(labels, np.int64)])
    return rows[np.lexsort(rows.T[::-1])]
