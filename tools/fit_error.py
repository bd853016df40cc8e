"""Coefficient error of the device fit against the oracle on fitheavy (noise-free and 1% noise):
the margin of the 1e-9 gate of tests/test_gpu_parity.py::test_fit_fitheavy_full_size."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_02373_b200 as rp, synth, oracle
for sigma in (0.0, 0.01):
    fc = synth.fitheavy(sigma=sigma)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
    if fc.noise is not None:
        V = V * fc.noise
    coef, (c, e), infos = rp.fit(torch.from_numpy(fc.X).cuda(), torch.from_numpy(V).cuda(), fc.num_exp, fc.den_exp)
    for i in range(len(V)):
        r = oracle.fit(fc.X, V[i], fc.num_exp, fc.den_exp, nthreads=16)
        want = np.asarray(r["coef"], dtype=np.float64)
        print(f"sigma {sigma} metric {i}: coef err {np.max(np.abs(coef[i] - want)) / np.max(np.abs(want)):.3e}, "
              f"min pivot {infos[i]['min_pivot']:.3e}, cond est {infos[i]['cond_est']:.3e}")
