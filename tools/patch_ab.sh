#!/bin/bash
# A/B of library builds on the patch-kernel workloads: C2 closed loops
# (tools/c2_ab.py) and step-0 solves of C4 cells at N=1000 (tools/c4_quick.py),
# alternated twice: tools/patch_ab.sh lib1.so lib2.so ...
cells=${CELLS:-"2:5 3:10 4:20 5:20 6:10 3:30"}
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $(basename $lib)"
    DLMPC_LIB=$lib timeout 300 python tools/c2_ab.py
    DLMPC_LIB=$lib timeout 600 python tools/c4_quick.py $cells
  done
done
