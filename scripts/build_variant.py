"""Build an experimental variant of libnestmesh_label.so with extra -D flags
into paper_2203_10000_b200/lib/variants/<name>.so (development aid; select
with NM_LABEL_LIB=... for scripts/quick_time.py)."""
import sys
sys.path.insert(0, ".")
from paper_2203_10000_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.LIB / "variants" / f"{name}.so"
out.parent.mkdir(parents=True, exist_ok=True)
lines = b.compile_label_lib(out, defs).splitlines()
for i, l in enumerate(lines):
    if "Function properties for _ZN2nm7k_labelILi1ELb1ELi0EE" in l:
        print(name, lines[i + 1].strip(), "|", lines[i + 2].strip())
        break
