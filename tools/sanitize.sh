#!/bin/bash
# compute-sanitizer over the persistent kernels (run on the GPU box):
#   bash tools/sanitize.sh [tool ...]      (default: memcheck racecheck synccheck)
# One process per (tool, case), each under its own timeout; logs and a
# summary line per run go to gpurun_out/sanitize_<tool>_<case>.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
tools=${@:-memcheck racecheck synccheck}
for tool in $tools; do
  for case in c1 c2 stream twophase sched; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 600 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_case.py $case > gpurun_out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  done
done
