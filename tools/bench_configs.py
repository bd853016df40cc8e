"""Throughput / latency of every BASELINE config on one GPU (device-resident inputs, CUDA events,
L2 flushed between timed repetitions).  Prints one JSON object; used to fill BASELINE.md §2.

  python tools/bench_configs.py [--reps N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_02373_b200 as rp
import synth

reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 10
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=reps, flush_l2=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush_l2:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {"gpu": torch.cuda.get_device_name(0)}

# tiny: latency of one rp_eval_argmin call (plan + sweep), and of a sweep on a prepared plan
tiny = synth.tiny_sweep()
Dt, Ft = torch.from_numpy(tiny.D).to(dev), torch.from_numpy(tiny.F).to(dev)
ms = timed(lambda: rp.eval_argmin(tiny.programs[0], Dt, Ft, second=False), flush_l2=False)
plan = rp.Plan(tiny.programs, Ft)
res = plan.eval(Dt, second=False)
ms_plan = timed(lambda: plan.eval(Dt, out=res, second=False), flush_l2=False)
t0 = time.perf_counter()
for _ in range(200):
    plan.eval(Dt, out=res, second=False)
torch.cuda.synchronize()
out["tiny"] = {"pairs": int(len(tiny.D) * len(tiny.F)), "eval_argmin_us": 1e3 * ms,
               "plan_eval_device_us": 1e3 * ms_plan,
               "plan_eval_host_wall_us": 1e6 * (time.perf_counter() - t0) / 200}

# f2: single-decision latency through the DecisionService (host wall per call: rp_decider's
# mapped-memory graph launch and synchronisation included), fresh decisions and history hits
case = synth.polybench_sweep(nD=2000)
plan = rp.Plan(case.programs[:1], torch.from_numpy(case.F).to(dev))
svc = rp.DecisionService(plan, prog=0, margin=0.01, history_log2=16)
for d in case.D[:50]:
    svc(d)
t0 = time.perf_counter()
for d in case.D[50:1050]:
    svc(d)
fresh_us = 1e6 * (time.perf_counter() - t0) / 1000
t0 = time.perf_counter()
for d in case.D[50:1050]:
    svc(d)
memo_us = 1e6 * (time.perf_counter() - t0) / 1000
svc.memo = None  # device-history hits only
t0 = time.perf_counter()
for d in case.D[50:1050]:
    svc(d)
hit_us = 1e6 * (time.perf_counter() - t0) / 1000
stats = plan.history_stats()
svc.decider.close()
plan2 = rp.Plan(case.programs[:1], torch.from_numpy(case.F).to(dev))
dc = rp.Decider(plan2, prog=0, margin=0.01)  # no history, no memo: every call a full decision
for d in case.D[:50]:
    dc(d)
t0 = time.perf_counter()
for d in case.D[50:1050]:
    dc(d)
nohist_us = 1e6 * (time.perf_counter() - t0) / 1000
# the paper's own placement of the decision (host CPU, one D at a time):
# the oracle's orc_decide on one core, program marshalled once, the same 1,000 tuples
import ctypes as C
import numpy as np
import oracle
h = oracle._ProgramHolder(case.programs[0])
Fa = np.ascontiguousarray(case.F, dtype=np.int32)
Eh, six, gap = np.zeros(1), np.zeros(6, dtype=np.int32), np.zeros(1)
Ds = [np.ascontiguousarray(d, dtype=np.int32).ravel() for d in case.D[50:1050]]
t0 = time.perf_counter()
for d in Ds:
    oracle.lib().orc_decide(C.byref(h.pr), oracle._p(d), oracle._p(Fa), len(Fa), 0.01, oracle._p(Eh), oracle._p(six),
                            oracle._p(gap))
host_us = 1e6 * (time.perf_counter() - t0) / len(Ds)
out["decision_service"] = {"program": "polybench gemm, 266 configs", "path": "rp_decider (mapped memory + graph)",
                           "fresh_decision_us": fresh_us, "device_history_hit_us": hit_us,
                           "host_memo_hit_us": memo_us, "no_history_decision_us": nohist_us,
                           "history": stats,
                           "host_oracle_decision_us": host_us,
                           "host_oracle_note": "orc_decide (x87 long double, 1 core, the same 1,000 tuples and margin): "
                                               "the paper's host-side placement of the decision, as a reference point"}

for name, case in (("polybench", synth.polybench_sweep()), ("multikernel", synth.multikernel_sweep())):
    D, F = torch.from_numpy(case.D).to(dev), torch.from_numpy(case.F).to(dev)
    plan = rp.Plan(case.programs, F)
    res = plan.eval(D, second=False)
    ms = timed(lambda: plan.eval(D, out=res, second=False))
    pairs = len(case.programs) * len(case.D) * len(case.F)
    out[name] = {"programs": len(case.programs), "nD": len(case.D), "nF": len(case.F), "pairs": pairs,
                 "sweep_ms": ms, "evals_per_s": pairs / (ms * 1e-3)}

case = synth.large_sweep()
D, F = torch.from_numpy(case.D).to(dev), torch.from_numpy(case.F).to(dev)
plan = rp.Plan(case.programs, F)
res = plan.eval(D, second=False)
ms = timed(lambda: plan.eval(D, out=res, second=False))
out["large"] = {"nD": len(case.D), "nF": len(case.F), "pairs": len(case.D) * len(case.F), "sweep_ms": ms,
                "evals_per_s": len(case.D) * len(case.F) / (ms * 1e-3),
                "static_feasible": plan.static_feasible()}

fc = synth.fitheavy(sigma=0.01)
X = torch.from_numpy(fc.X).to(dev)
V = rp.eval_metrics(fc.truths[0], X) * torch.from_numpy(fc.noise).to(dev)
ms = timed(lambda: rp.fit(X, V, fc.num_exp, fc.den_exp))
c, e = rp.xform_from_box(*rp.minmax(X))
G = rp.gram(X, V, fc.num_exp, fc.den_exp, c, e)
ms_g = timed(lambda: rp.gram(X, V, fc.num_exp, fc.den_exp, c, e, out=G))
ms_s = timed(lambda: rp.solve_normal(G, fc.num_exp, fc.den_exp), flush_l2=False)
out["fitheavy"] = {"K": len(fc.X), "metrics": 3, "n_c": 140, "fit_ms": ms, "rows_per_s": len(fc.X) / (ms * 1e-3),
                   "gram_ms": ms_g, "solve_ms": ms_s}
print(json.dumps(out))
