"""Run a randomised GPU parity test of tests/test_gpu_parity.py over a range of seeds.

  python tools/sweep_stress.py FIRST LAST [test_name]   (default: test_sweep_randomised_programs)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_parity as T  # noqa: E402

fn = getattr(T, sys.argv[3] if len(sys.argv) > 3 else "test_sweep_randomised_programs")
bad = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    try:
        fn(seed)
    except Exception as e:  # report and continue
        bad += 1
        print("seed", seed, "FAILED:", repr(e)[:300])
print("done, failures:", bad)
