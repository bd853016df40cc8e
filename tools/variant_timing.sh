# A/B timing of librp variants on the bench's fitted sweep (tools/sweep_variant_time.py):
# default build, dense-only plan, then every paper_1911_02373_b200/variants/*.so
mkdir -p gpurun_out
T=${1:-var}
python tools/sweep_variant_time.py default > gpurun_out/${T}_time.jsonl 2>gpurun_out/${T}_time.err
for f in paper_1911_02373_b200/variants/*.so; do RP_LIBRP=$f python tools/sweep_variant_time.py $(basename $f .so) >> gpurun_out/${T}_time.jsonl 2>>gpurun_out/${T}_time.err; done
python tools/sweep_variant_time.py default >> gpurun_out/${T}_time.jsonl 2>>gpurun_out/${T}_time.err
cat gpurun_out/${T}_time.jsonl
