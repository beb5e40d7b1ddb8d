"""The drop-in boundary: libnestmesh_label.so loads, exports exactly what
include/nestmesh_label.h declares, carries sm_100a code, and fails loudly
(no CPU fallback) when there is no device. CPU only — no compute calls."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2203_10000_b200 import _native

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "nestmesh_label.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(nm_[a-z_]+)\s*\(", text))


def test_header_symbols_exported():
    declared = header_functions()
    assert {"nm_create", "nm_set_surfaces", "nm_label_nodes", "nm_label_tets", "nm_label_mesh", "nm_enclosure",
            "nm_flag_boundary", "nm_relabel", "nm_last_error"} <= declared
    exported = _native.exported_symbols()
    missing = declared - exported
    assert not missing, missing


def test_python_binding_mirrors_header():
    assert set(_native.LABEL_API) == header_functions()
    lib = _native.load_label_lib()
    assert lib.nm_abi_version() == 2


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LABEL_LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LABEL_LIB)], capture_output=True, text=True).stdout
    assert "k_label" in sass and "FFMA2" in sass and "MUFU.SQRT" in sass


def test_default_options():
    o = _native.default_options()
    assert o.device == 0 and abs(o.tau - 1e-2) < 1e-9 and abs(o.band - 1e-3) < 1e-15 and o.sort_points == 1
    assert o.cull_outside == 0 and o.cell_axis == 120


def test_no_cpu_fallback_without_device(has_gpu):
    if has_gpu:
        pytest.skip("a device is present")
    lib = _native.load_label_lib()
    h = ctypes.c_void_p()
    rc = lib.nm_create(ctypes.byref(h), None)
    assert rc != 0
    assert b"no CUDA device" in lib.nm_last_error()
    with pytest.raises(_native.NativeError, match="no CUDA device"):
        _native.Context(0)


def test_null_context_errors():
    lib = _native.load_label_lib()
    rc = lib.nm_label_nodes(None, None, 0, 0.5, None, None)
    assert rc != 0 and b"null context" in lib.nm_last_error()


def test_cpp_dropin_header_compiles(tmp_path):
    """include/nestmesh/labeling.hpp (SPEC signatures over the reference types)
    compiles against the unmodified reference headers and links the C ABI."""
    ref_inc = Path("/root/reference/proj/include")
    if not ref_inc.exists():
        pytest.skip("reference headers not present on this machine")
    src = tmp_path / "t.cpp"
    src.write_text('#include "nestmesh/labeling.hpp"\nint main() { return nestmesh::labeling_abi_version() == 2 ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", f"-I{ref_inc}", f"-I{ROOT / 'include'}",
                        str(src), "-o", str(tmp_path / "t"), f"-L{_native.LIB_DIR}", "-lnestmesh_label",
                        f"-Wl,-rpath,{_native.LIB_DIR}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0
