"""CPU oracle throughput per BASELINE config on the host cores (1 thread and all threads), for
BASELINE.md §3.  Bounded samples: `large` on 2,000 D x 1,024 F, `fitheavy` on 20,000 rows.

  python tools/oracle_configs.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import synth

cores = len(os.sched_getaffinity(0))
out = {"cores": cores}


def rate(fn, units):
    t = time.perf_counter()
    fn()
    return units / (time.perf_counter() - t)


for name, case, nd in (("tiny", synth.tiny_sweep(), None), ("polybench", synth.polybench_sweep(), 2000),
                       ("multikernel", synth.multikernel_sweep(), 1000), ("large", synth.large_sweep(nD=2000), None)):
    D = case.D if nd is None else case.D[:nd]
    spec = case.programs[0]
    pairs = len(D) * len(case.F)
    out[name] = {"sample": f"{len(D)} D x {len(case.F)} F, program 0",
                 "evals_per_s_1core": rate(lambda: oracle.sweep(spec, D, case.F, nthreads=1), pairs),
                 "evals_per_s_all": rate(lambda: oracle.sweep(spec, D, case.F, nthreads=cores), pairs)}

fc = synth.fitheavy(K=20_000)
V = np.asarray(oracle.program_metrics(fc.truths[0], fc.X)[0], dtype=np.float64)
out["fitheavy"] = {"sample": "20,000 rows, 1 metric (140 columns)",
                   "rows_per_s_1core": rate(lambda: oracle.fit(fc.X, V, fc.num_exp, fc.den_exp, nthreads=1), len(V)),
                   "rows_per_s_all": rate(lambda: oracle.fit(fc.X, V, fc.num_exp, fc.den_exp, nthreads=cores), len(V))}
print(json.dumps(out))
