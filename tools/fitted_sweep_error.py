"""The bench's own sweep (the FITTED program of the bench step) against the oracle on a subsample:
max relative E error, its ratio to R31's kappa-aware bound, and winner agreement where the oracle's
margin exceeds 1e-9 (analysis; prints one JSON line).

  python tools/fitted_sweep_error.py [every]"""
import copy
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle  # noqa: E402
import paper_1911_02373_b200 as rp  # noqa: E402
import synth  # noqa: E402


def main():
    every = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    inp = bench.workload_inputs()
    dev = torch.device("cuda:0")
    X = torch.from_numpy(inp["X"]).to(dev)
    V = (rp.eval_metrics(inp["truth"], X) * torch.from_numpy(inp["noise"]).to(dev)).contiguous()
    coef, (c, e), _ = rp.fit(X, V, inp["num"], inp["den"])
    spec = copy.deepcopy(inp["truth"])
    spec.coef = [np.asarray(coef[i]) for i in range(3)]
    spec.xform_c, spec.xform_e = list(c), list(e)
    idx, E, _ = rp.eval_argmin(spec, torch.from_numpy(inp["D"]).to(dev), torch.from_numpy(inp["F"]).to(dev),
                               second=False)
    idx, E = idx.cpu().numpy().ravel(), E.cpu().numpy().ravel()
    sel = synth.large_subsample_index(len(inp["D"]), every=every)
    ref = oracle.sweep(spec, inp["D"][sel], inp["F"])
    feas = ref["idx"] >= 0
    rel = np.abs(E[sel][feas] - ref["best"][feas]) / ref["best"][feas]
    kap = ref["kappa"][feas]
    bound = np.maximum(1e-12, 1024 * 2.0 ** -53 * kap)
    with np.errstate(invalid="ignore"):
        margin = (ref["second"] - ref["best"]) / ref["best"]
    strict = feas & (margin > 1e-9)
    print(json.dumps({"sample": int(len(sel)), "feasible": int(feas.sum()),
                      "max_rel_E": float(rel.max()), "p99_rel_E": float(np.percentile(rel, 99)),
                      "frac_rel_gt_1e-12": float(np.mean(rel > 1e-12)),
                      "kappa_p50_p99_max": [float(np.percentile(kap, 50)), float(np.percentile(kap, 99)), float(kap.max())],
                      "max_rel_over_R31_bound": float(np.max(rel / bound)),
                      "winners_equal_where_margin_gt_1e-9": bool(np.array_equal(idx[sel][strict], ref["idx"][strict])),
                      "n_margin_gt_1e-9": int(strict.sum())}))


if __name__ == "__main__":
    main()
