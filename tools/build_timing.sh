#!/bin/bash
# Profiling build of the library with per-phase timers (-DDLMPC_PHASE_TIMING).
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -DDLMPC_PHASE_TIMING -o paper_2103_14990_b200/libdlmpc_timing.so \
  paper_2103_14990_b200/csrc/dlmpc.cu paper_2103_14990_b200/csrc/dlmpc_multi.cu
