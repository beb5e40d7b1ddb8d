#!/bin/bash
# nm_label_mesh tet chunking x staging chunk A/B through the C++ drop-in (pageable) and the Python pinned path
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ay
mkdir -p $O
for rep in 1 2; do
for v in base one one16 c16 t2m t8m; do
  d=/tmp/vlib_$v; mkdir -p $d; ln -sf $GRAFT_REPO_ROOT/paper_2203_10000_b200/lib/variants/$v.so $d/libnestmesh_label.so
  for c in 5 3 2; do
    echo "== rep $rep $v cfg$c $(NO_NM_TIMING=1 LD_LIBRARY_PATH=$d python scripts/cpp_e2e_timing.py $c 2>&1 | tail -1)" >> $O/ab.txt
  done
done
done
cat $O/ab.txt
