import sys, os, traceback
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_gpu_parity as T
bad = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    try:
        T.test_sweep_randomised_programs(seed)
    except Exception as e:
        bad += 1
        print("seed", seed, "FAILED:", repr(e)[:300])
print("done, failures:", bad)
