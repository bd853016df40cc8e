# Round-end style GPU pass: full -m gpu suite, smoke, bench (default K/W), ncu launch list of the
# bench command, ncu --set full of k_sweep (bench workload launch) and k_gram_mom, bench_configs.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_final.sh TAG'
T=${1:-fin}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=15 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 -o gpurun_out/${T}_sweep \
  python tools/sweep_variant_time.py ncu > gpurun_out/${T}_ncu_sweep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_mom -s 2 -c 1 -o gpurun_out/${T}_gram \
  python tools/gram_variant_time.py ncu > gpurun_out/${T}_ncu_gram.log 2>&1
timeout 300 python tools/bench_configs.py > gpurun_out/${T}_configs.json 2> gpurun_out/${T}_configs.err
tail -3 gpurun_out/${T}_pytest.log; tail -1 gpurun_out/${T}_smoke.log
head -c 400 gpurun_out/${T}_bench.json; echo; head -c 300 gpurun_out/${T}_bench_ref.json
