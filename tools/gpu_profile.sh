#!/bin/bash
# One GPU round: bench (clean), launch list under ncu, full ncu captures of k_sweep and k_gram.
# Usage (from the repo root, under gpurun): bash tools/gpu_profile.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 -o gpurun_out/prof_sweep_$TAG \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sweep_$TAG.log 2>&1
echo "ncu sweep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_gram$' -s 3 -c 1 -o gpurun_out/prof_gram_$TAG \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gram_$TAG.log 2>&1
echo "ncu gram rc=$?"
