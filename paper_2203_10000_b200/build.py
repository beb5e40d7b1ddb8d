"""In-tree build of the native libraries (sm_100a only).

    libnestmesh_label.so   CUDA kernels + C ABI (include/nestmesh_label.h)
    libnestmesh_synth.so   synthetic-input generators (caller side)

plus the oracle (test infrastructure, oracle/Makefile). Outputs stay in the
repo tree so they travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-shared", f"-I{ROOT / 'include'}",
              "-Xptxas", "-v"]


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}")
    if log is not None:
        log.write_text(r.stdout + r.stderr)
    return r


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def LABEL_SOURCES():
    """CUDA translation units of libnestmesh_label.so (context.cuh is shared)."""
    return [str(CSRC / f) for f in ("nestmesh_label.cu", "cell_build.cu", "group.cu", "mesh_ops.cu", "sidecar.cu")]


def compile_label_lib(out: Path, defs=(), log=None):
    """Compile the translation units in parallel (one nvcc per source), then link."""
    from concurrent.futures import ThreadPoolExecutor

    objdir = out.parent / f".obj_{out.stem}"
    objdir.mkdir(parents=True, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defs]
    srcs = LABEL_SOURCES() + [str(CSRC / "refine.cpp")]
    objs = [objdir / (Path(s).stem + ".o") for s in srcs]
    with ThreadPoolExecutor(len(srcs)) as ex:
        rs = list(ex.map(lambda so: _run([NVCC, *ARCH, *cflags, "-c", so[0], "-o", str(so[1])]), zip(srcs, objs)))
    _run([NVCC, *ARCH, "-shared", *map(str, objs), "-o", str(out)])
    text = "".join(r.stdout + r.stderr for r in rs)
    if log is not None:
        log.write_text(text)
    return text


def build_label_lib(force=False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libnestmesh_label.so"
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [CSRC / "refine.cpp", ROOT / "include" / "nestmesh_label.h"]
    if force or _stale(out, deps):
        compile_label_lib(out, log=LIB / "ptxas_label.log")
    return out


def build_checked_lib(force=False) -> Path:
    """lib/checked/libnestmesh_label.so: the same sources with NM_CHECKED
    (device-side bounds checks, csrc/check.cuh) for tests/test_gpu_checked.py."""
    out = LIB / "checked" / "libnestmesh_label.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [CSRC / "refine.cpp", ROOT / "include" / "nestmesh_label.h"]
    if force or _stale(out, deps):
        compile_label_lib(out, defs=("NM_CHECKED",), log=out.parent / "ptxas_checked.log")
    return out


def build_synth_lib(force=False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libnestmesh_synth.so"
    src = CSRC / "synth.cpp"
    if force or _stale(out, [src]):
        _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-Wextra",
              str(src), "-o", str(out)])
    return out


def build_oracle() -> None:
    """Test infrastructure: the fp64 oracle and, when /root/reference exists, oracle/_ref."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def build_cpp_dropin_test(force=False):
    """tests/cpp/dropin_test.cpp against the unmodified reference headers
    (only where /root/reference exists; the binary travels to the GPU box)."""
    ref_inc = Path("/root/reference/proj/include")
    if not ref_inc.exists():
        return None
    out = ROOT / "build" / "dropin_test"
    src = ROOT / "tests" / "cpp" / "dropin_test.cpp"
    deps = [src, ROOT / "include" / "nestmesh" / "labeling.hpp", ROOT / "include" / "nestmesh" / "label_sidecar.hpp",
            ROOT / "include" / "nestmesh_label.h", LIB / "libnestmesh_label.so"]
    if force or _stale(out, deps):
        out.parent.mkdir(exist_ok=True)
        _run([CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ref_inc}", f"-I{ROOT / 'include'}", str(src),
              "-o", str(out), f"-L{LIB}", "-lnestmesh_label", "-Wl,-rpath,$ORIGIN/../paper_2203_10000_b200/lib"])
    return out


def build_cpp_dropin_bench(force=False):
    """tests/cpp/dropin_bench.cpp -> build/libdropin_bench.so: the C++ drop-in's
    end-to-end leg of bench.py (reference types, pageable buffers)."""
    ref_inc = Path("/root/reference/proj/include")
    if not ref_inc.exists():
        return None
    out = ROOT / "build" / "libdropin_bench.so"
    src = ROOT / "tests" / "cpp" / "dropin_bench.cpp"
    deps = [src, ROOT / "include" / "nestmesh" / "labeling.hpp", ROOT / "include" / "nestmesh_label.h",
            LIB / "libnestmesh_label.so"]
    if force or _stale(out, deps):
        out.parent.mkdir(exist_ok=True)
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{ref_inc}", f"-I{ROOT / 'include'}",
              str(src), "-o", str(out), f"-L{LIB}", "-lnestmesh_label",
              "-Wl,-rpath,$ORIGIN/../paper_2203_10000_b200/lib"])
    return out


def build_all(force=False) -> None:
    build_synth_lib(force)
    build_label_lib(force)
    build_checked_lib(force)
    build_oracle()
    build_cpp_dropin_test(force)
    build_cpp_dropin_bench(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", *sorted(p.name for p in LIB.glob("*.so")))
