#!/bin/bash
# round-2 GPU pass: selected tests, bench, ncu launch list + full captures of k_sweep and k_refine
# usage: gpurun -- 'bash tools/r02_check.sh TAG "<pytest -k expression>|all" [full]'
TAG=${1:-x}
SEL=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "$SEL" = "all" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
elif [ -n "$SEL" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -rf -k "$SEL" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
timeout 400 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "$3" = "full" ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launches.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 -o gpurun_out/${TAG}_sweep \
    python tools/prof_kernels.py sweep --reps 5 > gpurun_out/${TAG}_ncu_sweep.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refine -s 3 -c 1 -o gpurun_out/${TAG}_refine \
    python tools/prof_kernels.py sweep --reps 5 > gpurun_out/${TAG}_ncu_refine.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_ws -s 2 -c 1 -o gpurun_out/${TAG}_gram \
    python tools/gram_variant_time.py ncu > gpurun_out/${TAG}_ncu_gram.log 2>&1
fi
tail -5 gpurun_out/${TAG}_pytest.log 2>/dev/null
head -c 600 gpurun_out/${TAG}_bench.json
