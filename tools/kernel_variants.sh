#!/bin/bash
# Build librp with each compile-time variant and time one kernel on its bench workload.
# Usage (on the GPU box): bash tools/kernel_variants.sh sweep|gram|solve|svd "-DFLAG=1" "-DFLAG=2" ...
which=$1; shift
for v in "$@"; do
  touch paper_1911_02373_b200/csrc/*.cu
  make -s -C paper_1911_02373_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  echo "$v: $(timeout 300 python tools/prof_kernels.py $which --reps 3 2>&1 | tail -1)"
done
touch paper_1911_02373_b200/csrc/*.cu
make -s -C paper_1911_02373_b200/csrc > /dev/null 2>&1
