"""Device time of rp_fit_svd on the fitheavy sample (3 metrics, K = 10^6, 1% noise) and its
coefficients' gap to the normal-equation fit; one JSON line (RP_SVD_R=tsqr selects the TSQR R).
  python tools/svd_time.py [tag]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_02373_b200 as rp
import synth

tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("RP_SVD_R", "default")
dev = torch.device("cuda:0")
fc = synth.fitheavy(sigma=0.01)
X = torch.from_numpy(fc.X).to(dev)
V = (rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)).contiguous()
coef, sigma, _, infos = rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
ms = []
for _ in range(5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
cne, _, _ = rp.fit(X, V, fc.num_exp, fc.den_exp)
gap = [float(np.max(np.abs(np.asarray(coef[i]) - np.asarray(cne[i].cpu() if hasattr(cne[i], "cpu") else cne[i]))))
       for i in range(3)]
print(json.dumps({"variant": tag, "fit_svd_ms": statistics.median(ms), "sigma_min": [float(np.min(np.asarray(s))) for s in sigma],
                  "sigma_max": [float(np.max(np.asarray(s))) for s in sigma], "coef_gap_vs_normal_eq": gap}))
