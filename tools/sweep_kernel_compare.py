"""Compare a sweep kernel variant (RP_SWEEP_KERNEL=<name>) with the default k_sweep at `large`
(10^6 D x 1,024 F, the bench's second=False launch): winners, E, and CUDA-event time of each.

  python tools/sweep_kernel_compare.py tc [nD]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_02373_b200 as rp  # noqa: E402
import synth  # noqa: E402


def run(kernel, plan, D, reps=5):
    if kernel:
        os.environ["RP_SWEEP_KERNEL"] = kernel
    else:
        os.environ.pop("RP_SWEEP_KERNEL", None)
    idx, E, _ = plan.eval(D, second=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.eval(D, out=(idx, E, None), second=False)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return idx.clone(), E.clone(), float(np.median(ts))


def main():
    kern = sys.argv[1]
    nD = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    case = synth.large_sweep(nD=nD)
    dev = torch.device("cuda:0")
    plan = rp.Plan(case.programs, torch.from_numpy(case.F).to(dev))
    D = torch.from_numpy(case.D).to(dev)
    i0, e0, t0 = run(None, plan, D)
    i1, e1, t1 = run(kern, plan, D)
    os.environ.pop("RP_SWEEP_KERNEL", None)
    i0, e0, i1, e1 = (x.cpu().numpy().ravel() for x in (i0, e0, i1, e1))
    fin = np.isfinite(e0)
    rel = np.abs(e1[fin] - e0[fin]) / e0[fin]
    print(json.dumps({"nD": nD, "kernel": kern, "ms_default": t0, "ms_variant": t1,
                      "idx_mismatch": int(np.sum(i0 != i1)), "max_rel_E_diff": float(rel.max()) if rel.size else 0.0,
                      "inf_mismatch": int(np.sum(np.isfinite(e0) != np.isfinite(e1)))}))


if __name__ == "__main__":
    main()
