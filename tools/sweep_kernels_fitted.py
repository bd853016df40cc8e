"""Every sweep kernel variant on the bench's own launch (the FITTED program of the bench step,
1e6 D x 1,024 F, second=False): CUDA-event time and winners against the default k_sweep.

  python tools/sweep_kernels_fitted.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1911_02373_b200 as rp  # noqa: E402


def main():
    inp = bench.workload_inputs()
    dev = torch.device("cuda:0")
    X = torch.from_numpy(inp["X"]).to(dev)
    V = (rp.eval_metrics(inp["truth"], X) * torch.from_numpy(inp["noise"]).to(dev)).contiguous()
    coef, xf, _ = rp.fit_dev(X, V, inp["num"], inp["den"])
    plan = rp.Plan([inp["truth"]], torch.from_numpy(inp["F"]).to(dev))
    plan.update(coef, xf)
    D = torch.from_numpy(inp["D"]).to(dev)
    out = {}
    ref = None
    for name, env in (("k_sweep", {}), ("k_sweep_ws", {"RP_SWEEP_KERNEL": "ws"}), ("k_sweep_tc", {"RP_SWEEP_KERNEL": "tc"}),
                      ("k_sweep + refine", {"RP_SWEEP_REFINE": "1"})):
        for k in ("RP_SWEEP_KERNEL", "RP_SWEEP_REFINE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        idx, E, _ = plan.eval(D, second=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.eval(D, out=(idx, E, None), second=False)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        if ref is None:
            ref = idx.clone()
        out[name] = {"ms": sorted(ts)[2], "winners_equal_default": bool(torch.equal(idx, ref))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
