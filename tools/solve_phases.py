"""Phase timestamps of k_solve (build with EXTRA=-DRP_SOLVE_TS: coef[0][1..6] carry clock64
deltas: load, factorisation, first solve pair, residual, second solve pair, resid2) and the
device time of the solve on the fitheavy Gram (3 metrics, n_c = 140).
  RP_LIBRP=paper_1911_02373_b200/variants/librp_ts.so python tools/solve_phases.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_02373_b200 as rp
import synth

dev = torch.device("cuda:0")
fc = synth.fitheavy(sigma=0.01)
X = torch.from_numpy(fc.X).to(dev)
V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
coef, xf, _ = rp.fit_dev(X, V, fc.num_exp, fc.den_exp)
c, e = rp.xform_from_box(*rp.minmax(X))
G = rp.gram(X, V, fc.num_exp, fc.den_exp, c, e)
cf = torch.empty_like(coef)
info = torch.empty((3, 5), dtype=torch.float64, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    rp.solve_dev(G, fc.num_exp, fc.den_exp, coef=cf, info=info)
torch.cuda.synchronize()
ev[0].record()
for _ in range(20):
    rp.solve_dev(G, fc.num_exp, fc.den_exp, coef=cf, info=info)
ev[1].record()
torch.cuda.synchronize()
out = {"variant": os.environ.get("RP_LIBRP", "default"), "solve_us": 1e3 * ev[0].elapsed_time(ev[1]) / 20}
if "ts" in out["variant"]:
    out["phases_cycles"] = dict(zip(["load", "factor", "solve1", "resid", "solve2", "resid2"],
                                    cf[0, 1:7].cpu().numpy().tolist()))
print(json.dumps(out))
