"""A small workload that launches every librp kernel once or twice, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Sizes are small (racecheck is slow) but cover
ragged tiles.  python tools/sanitize_workload.py [part]   part in {all, sweep, gram, svd, decide, tc, jit}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_02373_b200 as rp
import synth

part = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def want(p):
    return part in ("all", p)


if want("sweep"):
    case = synth.tiny_sweep()
    rp.eval_argmin(case.programs[0], cu(case.D), cu(case.F))                 # k_sweep SECOND + k_refine
    pb = synth.polybench_sweep(nD=300)
    rp.eval_argmin_batched(pb.programs, cu(pb.D), cu(pb.F), second=False)    # batched, 4 programs
    lg = synth.large_sweep(nD=5000)                                          # D1 buckets (nD >= 4096)
    plan = rp.Plan(lg.programs, cu(lg.F))
    plan.eval(cu(lg.D), second=False)
    plan.eval(cu(lg.D[:37]), second=True)
    fc = synth.fitheavy(K=3000)
    X = cu(fc.X)
    V = rp.eval_metrics(fc.truths[0], X)
    coef, xf, _ = rp.fit_dev(X, V, fc.num_exp, fc.den_exp)
    plan.update(coef, xf)                                                    # k_plan_refresh
    plan.eval(cu(lg.D), second=False)
if want("gram"):
    fc = synth.polybench_fit_box(K=700)
    V = rp.eval_metrics(fc.truths[0], cu(fc.X))
    rp.fit(cu(fc.X), V, fc.num_exp, fc.den_exp)                              # minmax, xform, k_gram_mom (TMA ring), solve
    rp.fit(cu(fc.X[:699]), V[:, :699].contiguous(), fc.num_exp, fc.den_exp)  # odd K: the plain-load producer path
    os.environ["RP_MOM_GENERIC"] = "1"
    rp.fit(cu(fc.X), V, fc.num_exp, fc.den_exp)                              # the generic monomial step
    os.environ.pop("RP_MOM_GENERIC")
    for kern in ("ws", "fused"):                                             # the outer-product kernels
        os.environ["RP_GRAM_KERNEL"] = kern
        rp.fit(cu(fc.X), V, fc.num_exp, fc.den_exp)
        os.environ.pop("RP_GRAM_KERNEL")
    rp.fit_sk(cu(fc.X), V, fc.num_exp, fc.den_exp, iters=2, raise_on_degenerate=False)  # weighted moments (WT = 2)
if want("svd"):
    fc = synth.tiny_fit_box()
    V = rp.eval_metrics(fc.truths[0], cu(fc.X))
    rp.fit_svd(cu(fc.X), V, fc.num_exp, fc.den_exp, raise_on_degenerate=False)  # k_tsqr (K < 4 n_c), k_svd_gk
    pf = synth.polybench_fit_box(K=700)
    Vp = rp.eval_metrics(pf.truths[0], cu(pf.X))
    rp.fit_svd(cu(pf.X), Vp, pf.num_exp, pf.den_exp, raise_on_degenerate=False)  # k_vabsmax, k_gram_dd, k_chol_dd
if want("decide"):
    pb = synth.polybench_sweep(nD=20)
    plan = rp.Plan(pb.programs[:1], cu(pb.F))
    plan.decide(pb.D, prog=0, margin=0.01)
    plan.enable_history(0, 8, 0.01)
    plan.decide(pb.D, prog=0, margin=0.01)
    plan.decide(pb.D, prog=0, margin=0.01)
    dc = rp.Decider(plan, prog=0, margin=0.01)
    for d in pb.D[:4]:
        dc(d)
    dc.close()
if want("tc"):
    os.environ["RP_SWEEP_KERNEL"] = "tc"
    lg = synth.large_sweep(nD=300)
    rp.eval_argmin(lg.programs[0], cu(lg.D), cu(lg.F), second=False)        # k_tc_pack, k_sweep_tc
    os.environ.pop("RP_SWEEP_KERNEL")
if want("jit"):
    case = synth.tiny_sweep()
    j = rp.Jit(case.programs[0])
    j.eval(cu(case.D), cu(case.F))
torch.cuda.synchronize()
print("sanitize workload", part, "done")
