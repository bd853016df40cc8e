#!/bin/bash
# Build librp variants (compile-time knobs) under paper_1911_02373_b200/variants/.
#   bash tools/sweep_variants.sh NAME "-DKNOB=1 ..." [NAME2 "..."]...
# On the GPU box: for f in paper_1911_02373_b200/variants/*.so; do RP_LIBRP=$f python tools/sweep_variant_time.py $(basename $f .so); done
set -e
root="$(cd "$(dirname "$0")/.." && pwd)"
mkdir -p $root/paper_1911_02373_b200/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=/tmp/rpvar_$name; rm -rf $d; mkdir -p $d
  cp $root/paper_1911_02373_b200/csrc/*.cu $root/paper_1911_02373_b200/csrc/*.cuh $root/paper_1911_02373_b200/csrc/Makefile $d/
  make -s -C $d -j8 EXTRA="$flags" INC=$root/include OUT=$root/paper_1911_02373_b200/variants/librp_$name.so 2>&1 | grep -E "error" || true
  echo "built $name ($flags)"
done
