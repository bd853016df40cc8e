mkdir -p gpurun_out
T=${1:-g5}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 400 python bench.py --steps 20 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -3 gpurun_out/${T}_pytest.log; cat gpurun_out/${T}_smoke.log | tail -1; head -c 1500 gpurun_out/${T}_bench.json
