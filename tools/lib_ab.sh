#!/bin/bash
# A/B of library builds on fixed-iteration device time (tools/iter_time.py),
# alternated: tools/lib_ab.sh "N1 N2" lib1.so lib2.so ...
ns=$1; shift
for rep in 1 2; do
  for n in $ns; do
    for lib in "$@"; do
      echo -n "$(basename $lib) "
      DLMPC_LIB=$lib timeout 300 python tools/iter_time.py $n 200
    done
  done
done
