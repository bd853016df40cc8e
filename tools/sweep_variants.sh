#!/bin/bash
# Build librp with each compile-time variant and time the sweep kernel on the bench workload.
# Usage (on the GPU box): bash tools/sweep_variants.sh "-DRP_SWEEP_MINB=4" "-DRP_SWEEP_MINB=5" ...
for v in "$@"; do
  touch paper_1911_02373_b200/csrc/rp_sweep.cu paper_1911_02373_b200/csrc/rp_decide.cu
  make -s -C paper_1911_02373_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  echo "$v: $(timeout 120 python tools/prof_kernels.py sweep --reps 5)"
done
touch paper_1911_02373_b200/csrc/rp_sweep.cu
make -s -C paper_1911_02373_b200/csrc > /dev/null 2>&1
