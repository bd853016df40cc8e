import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1911_02373_b200 as rp, synth
dev = torch.device("cuda:0")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
case = synth.large_sweep()
plan = rp.Plan(case.programs, torch.from_numpy(case.F).to(dev))
fc = synth.fitheavy(sigma=0.01)
X = torch.from_numpy(fc.X).to(dev)
V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
for frac in (1, 2, 4, 8):
    nD = 1_000_000 // frac
    D = torch.from_numpy(case.D[:nD]).to(dev)
    out = plan.eval(D, second=False)
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(5): plan.eval(D, out=out, second=False)
    ev[1].record(); torch.cuda.synchronize()
    ts = ev[0].elapsed_time(ev[1]) / 5
    K = 1_000_000 // frac
    Xs, Vs = X[:K].contiguous(), V[:, :K].contiguous()
    coef, xf, info = rp.fit_dev(Xs, Vs, fc.num_exp, fc.den_exp)
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(5): rp.fit_dev(Xs, Vs, fc.num_exp, fc.den_exp)
    ev[1].record(); torch.cuda.synchronize()
    tf = ev[0].elapsed_time(ev[1]) / 5
    print(f"1/{frac}: sweep {ts:.3f} ms (x{frac} = {ts*frac:.3f}), fit {tf:.3f} ms (x{frac} = {tf*frac:.3f})")
