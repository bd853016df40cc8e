#!/bin/bash
# GPU box: time the default build and every variant under paper_1911_02373_b200/variants/
mkdir -p gpurun_out
out=gpurun_out/${1:-variants}.jsonl
: > $out
for rep in 1 2; do
  timeout 300 python tools/${2:-sweep}_variant_time.py default >> $out 2>>gpurun_out/variants.err
  for f in paper_1911_02373_b200/variants/*.so; do
    RP_LIBRP=$f timeout 300 python tools/${2:-sweep}_variant_time.py $(basename $f .so) >> $out 2>>gpurun_out/variants.err
  done
done
cat $out
