"""sha256 (first 16 hex) of the SASS of the headline kernel k_label<1,true,0>
in the built libnestmesh_label.so: stamps committed ncu summaries so bench.py
can refuse a capture of a different build."""
import hashlib
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2203_10000_b200" / "lib" / "libnestmesh_label.so"
KERNEL = "_ZN2nm7k_labelILi1ELb1ELi0EEEvNS_11LabelParamsE"


def sass_hash(lib=LIB, kernel=KERNEL):
    try:
        out = subprocess.run(["cuobjdump", "-sass", "-fun", kernel, str(lib)], capture_output=True, text=True,
                             timeout=120).stdout
    except Exception:
        return None
    body = [l for l in out.splitlines() if "/*" in l]
    if not body:
        return None
    return hashlib.sha256("\n".join(body).encode()).hexdigest()[:16]


if __name__ == "__main__":
    print(sass_hash(Path(sys.argv[1]) if len(sys.argv) > 1 else LIB))
