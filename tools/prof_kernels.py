"""Launch the two hot kernels on the bench workload for ncu / timing (no oracle).

  python tools/prof_kernels.py sweep|gram [--reps N]
Prints the CUDA-event time per launch.  Under ncu use -k regex:k_sweep / 'regex:k_gram$'."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_02373_b200 as rp
import synth

which = sys.argv[1]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
dev = torch.device("cuda:0")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
if which == "sweep":
    case = synth.large_sweep()
    plan = rp.Plan(case.programs, torch.from_numpy(case.F).to(dev))
    D = torch.from_numpy(case.D).to(dev)
    out = plan.eval(D, second=False)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        plan.eval(D, out=out, second=False)
    ev[1].record()
elif which == "jit":
    case = synth.large_sweep()
    jit = rp.Jit(case.programs[0])
    D = torch.from_numpy(case.D).to(dev)
    F = torch.from_numpy(case.F).to(dev)
    out = jit.eval(D, F, second=False)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        jit.eval(D, F, second=False, out=out)
    ev[1].record()
elif which == "svd":
    fc = synth.fitheavy(sigma=0.01)
    X = torch.from_numpy(fc.X).to(dev)
    V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
    _, sig, _, infos = rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    print("jacobi sweeps / cond:", [(i["iters"], i["cond_est"]) for i in infos])
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    ev[1].record()
elif which == "solve":
    fc = synth.fitheavy(sigma=0.01)
    X = torch.from_numpy(fc.X).to(dev)
    V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
    c, e = rp.xform_from_box(*rp.minmax(X))
    G = rp.gram(X, V, fc.num_exp, fc.den_exp, c, e)
    coef, info = rp.solve_dev(G, fc.num_exp, fc.den_exp)
    print("info:", info.cpu().numpy().tolist())
    print("coef[0][:8]:", coef[0, :8].cpu().numpy().tolist())
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        rp.solve_dev(G, fc.num_exp, fc.den_exp, coef=coef, info=info)
    ev[1].record()
else:
    fc = synth.fitheavy(sigma=0.01)
    X = torch.from_numpy(fc.X).to(dev)
    V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
    c, e = rp.xform_from_box(*rp.minmax(X))
    G = rp.gram(X, V, fc.num_exp, fc.den_exp, c, e)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        rp.gram(X, V, fc.num_exp, fc.den_exp, c, e, out=G)
    ev[1].record()
torch.cuda.synchronize()
print(f"{which}: {ev[0].elapsed_time(ev[1]) / reps:.3f} ms per launch")
