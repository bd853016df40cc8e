#!/bin/bash
# compute-sanitizer passes over tools/sanitize_workload.py (GPU box).  Logs: gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_workload.py all > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}.log
done
for part in sweep gram svd decide tc; do
  timeout 1200 $CS --tool racecheck --racecheck-report all --error-exitcode 9 --print-limit 50 python tools/sanitize_workload.py $part > gpurun_out/sanitize_racecheck_${part}.log 2>&1
  echo "racecheck $part rc=$?" >> gpurun_out/sanitize_racecheck_${part}.log
done
timeout 900 $CS --tool initcheck --error-exitcode 9 --print-limit 50 python tools/sanitize_workload.py sweep > gpurun_out/sanitize_initcheck.log 2>&1
echo "initcheck rc=$?" >> gpurun_out/sanitize_initcheck.log
tail -n 4 gpurun_out/sanitize_*.log
