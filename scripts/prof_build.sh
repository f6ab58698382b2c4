#!/usr/bin/env bash
# Profiling build of the evaluator (-DARROW_PROF: serial-step cycles by
# event kind, burst/round selection vs execution) and its C2 breakdown.
#   bash scripts/prof_build.sh [c2|c5 [sample]]     (on the GPU box)
set -e
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_2505_11916_b200/csrc --shared -DARROW_PROF \
  -o /tmp/libarrow_prof.so paper_2505_11916_b200/csrc/arrow_sim.cu paper_2505_11916_b200/csrc/traces.cu \
  paper_2505_11916_b200/csrc/stats.cu
ARROW_SIM_LIB=/tmp/libarrow_prof.so python scripts/prof_serial.py "$@"
