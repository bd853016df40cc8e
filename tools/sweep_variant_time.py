"""Time k_sweep / k_refine of the bench's own launch (fitted program of the noisy fitheavy sample,
`large` D and F) with the librp the RP_LIBRP environment variable names; one JSON line.

  RP_LIBRP=paper_1911_02373_b200/variants/librp_X.so python tools/sweep_variant_time.py X
Winner checksum and E sum let variants be compared with the default build."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1911_02373_b200 as rp

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
reps = 10
dev = torch.device("cuda:0")
inp = bench.workload_inputs()
X = torch.from_numpy(inp["X"]).to(dev)
V = rp.eval_metrics(inp["truth"], X) * torch.from_numpy(inp["noise"]).to(dev)
coef, xf, _ = rp.fit_dev(X, V, inp["num"], inp["den"])
plan = rp.Plan([inp["truth"]], torch.from_numpy(inp["F"]).to(dev))
plan.update(coef, xf)
plan.enable_timing()
D = torch.from_numpy(inp["D"]).to(dev)
idx, E, _ = plan.eval(D, second=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ks, rf = [], []
for _ in range(reps):
    flush.zero_()
    torch.cuda.synchronize()
    plan.eval(D, out=(idx, E, None), second=False)
    t = plan.last_timing()
    ks.append(t["sweep_ms"])
    rf.append(t["refine_ms"])
i = idx.cpu().numpy().ravel()
e = E.cpu().numpy().ravel()
print(json.dumps({"variant": tag, "sweep_ms": statistics.median(ks), "refine_ms": statistics.median(rf),
                  "idx_sum": int(i.astype(np.int64).sum()), "n_neg": int((i < 0).sum()),
                  "E_sum": float(np.sum(e[np.isfinite(e)]))}), flush=True)
