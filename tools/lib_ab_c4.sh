#!/bin/bash
# A/B of library builds on C4 cells (tools/c4_quick.py, step-0 solve, best of 5),
# alternated twice: tools/lib_ab_c4.sh "d:T d:T" lib1.so lib2.so ...
cells=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $(basename $lib)"
    DLMPC_LIB=$lib timeout 600 python tools/c4_quick.py $cells
  done
done
