#!/usr/bin/env python
"""Benchmark of the rational-program hot path (arXiv 1911.02373) on B200.

One step = the whole hot path over one batch of synthetic input:
  fit   -- rp_fit of the 3 metrics (comp, coal, uncoal) on the `fitheavy` sample set
           (K = 10^6 noisy points in (D1, D2, bx, by), total degree <= 4 -> 140 Gram columns);
  sweep -- the fitted rational program (MWP-CWP estimate E) over the `large` grid
           (10^6 data tuples x 1,024 configurations, ~10^9 (D,P) pairs) with per-D argmin.
N > 1 (torchrun): K rows and D tuples are split across ranks (strong scaling); the partial Grams
are all-reduced and the per-D winners all-gathered over NCCL.

value = nD * nF / (device time of one step, max over ranks)  [RP evals/s, fit included];
fit_rows_per_s and sweep_evals_per_s break the step down.  Prints ONE JSON line on rank 0.

`--impl reference` times the CPU oracle (oracle/, x87 long double) as it stands on the host
cores, each step a bounded 1/200 sample of the same workload.
"""
from __future__ import annotations

import argparse
import copy
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RP evals/s over (D,P) grid incl. per-D argmin at 1/2/4/8 B200; fit rows/s"
UNIT = "evals/s"
SAMPLE_DIV = 200  # CPU oracle sample: 1/200 of the step (5,000 D x 1,024 F and 5,000 rows x 3 metrics)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz
# SURVEY.md 8(d) "Algorithmic work per unit" (large): 235 flop per evaluated (D,P) pair
# (a4 3*2*(15+15) + 14 P-monomials + ~30 + 11 divisions) and 2*3*2*70 = 840 per D tuple (a2)
FLOP_PER_PAIR = 235
FLOP_PER_D = 840


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload_inputs(nD=1_000_000, K=1_000_000):
    """Seeded host inputs: fitheavy X + noise multipliers, large D, F, the truth program."""
    fc = synth.fitheavy(sigma=0.01, K=K)
    return dict(X=fc.X, noise=fc.noise, num=fc.num_exp, den=fc.den_exp, truth=fc.truths[0],
                D=synth.large_D(nD), F=synth.F_large())


def evaluated_pairs(D, F, t_max=1024):
    """Number of (D,P) pairs the sweep evaluates: statically feasible P (warp rule, T <= T_max;
    B_active > 0 holds for every such T at R = 40, Z = 0) that pass P1 P2 <= D1^2."""
    T = F[:, 0].astype(np.int64) * F[:, 1]
    ok = (T % 32 == 0) & (T <= t_max)
    p12 = np.sort(T[ok])
    d1sq = D[:, 0].astype(np.int64) ** 2
    return int(np.searchsorted(p12, d1sq, side="right").sum())


# ------------------------------------------------------------------------------------------
# clocks
# ------------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/rp_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "20"], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[1].isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------

def oracle_step(inp, part: int, cores: int, div: int = SAMPLE_DIV):
    """The oracle's whole path on a 1/div slice (slice `part`): fit of the 3 metrics on
    K/div rows, then the sweep of the fitted program over nD/div tuples x all of F."""
    import oracle
    K = len(inp["X"]) // div
    nd = len(inp["D"]) // div
    X = inp["X"][part * K:(part + 1) * K]
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(inp["truth"], X)])
    V *= inp["noise"][:, part * K:(part + 1) * K]
    D = inp["D"][part * nd:(part + 1) * nd]
    t0 = time.perf_counter()
    prog = copy.deepcopy(inp["truth"])
    coefs = []
    for i in range(3):
        r = oracle.fit(X, V[i], inp["num"], inp["den"], nthreads=cores)
        coefs.append(np.asarray(r["coef"], dtype=np.float64))
    prog.coef = coefs
    prog.xform_c, prog.xform_e = list(r["c"]), list(r["e"])
    oracle.sweep(prog, D, inp["F"], nthreads=cores)
    dt = time.perf_counter() - t0
    return nd * len(inp["F"]) / dt, dt


def cpu_info():
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return  # rank 0 alone runs and prints it
    inp = workload_inputs()
    cores, model = cpu_info()
    for w in range(args.warmup):
        oracle_step(inp, w % SAMPLE_DIV, cores)
    vals, dts = [], []
    for s in range(args.steps):
        v, dt = oracle_step(inp, (args.warmup + s) % SAMPLE_DIV, cores)
        vals.append(v)
        dts.append(dt)
    value = len(inp["F"]) * (len(inp["D"]) // SAMPLE_DIV) * len(dts) / sum(dts)
    sample = (f"1/{SAMPLE_DIV} of the step per step: fit of 3 metrics on {len(inp['X']) // SAMPLE_DIV} rows + "
              f"sweep of {len(inp['D']) // SAMPLE_DIV} D x {len(inp['F'])} F (consecutive slices)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(dts) / len(dts),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "long double (x87)",
           "data": "synthetic (seeded)", "config": {"workload": "large+fitheavy", "nD": len(inp["D"]),
                                                   "nF": len(inp["F"]), "K": len(inp["X"]), "n_metrics": 3,
                                                   "n_c": 140, "sample": sample},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                            "cpu": model},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def parity_summary():
    """What the timed program's parity is: the -m gpu test that gates this exact workload at full
    size (tests/test_gpu_fullsize.py) and its last committed report (profiles/)."""
    out = {"test": "tests/test_gpu_fullsize.py::test_bench_workload_noisy_fit_sweep",
           "gate": "SURVEY 8(c) #25 (long double oracle, kappa <= 1e3: idx exact where margin > 1e-9, "
                   "E <= 1e-12) and, on every sampled D, E <= 1e-12 vs the binary128 oracle at the GPU's pick"}
    for f in ("r02_parity_bench_workload.json",):
        path = os.path.join(ROOT, "profiles", f)
        if os.path.exists(path):
            try:
                rep = json.load(open(path))
                out["report"] = "profiles/" + f
                out["vs_binary128"] = rep.get("vs_binary128")
                out["survey_8c_25"] = rep.get("survey_8c_25")
                out["fit_coef_gap_inf_norm"] = rep.get("fit_coef_gap_inf_norm")
            except (OSError, ValueError):
                pass
    return out


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the informational k_sweep_tc timing (ncu launch lists)")
    ap.add_argument("--nD", type=int, default=1_000_000)
    ap.add_argument("--K", type=int, default=1_000_000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as tdist

    import paper_1911_02373_b200 as rp
    from paper_1911_02373_b200 import dist as rdist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    # RP_BENCH_SHARED_GPU=1 (test only): every rank on cuda:0 with gloo, so the N > 1 code path can be
    # exercised on a one-GPU box; the numbers of such a run mean nothing
    shared = os.environ.get("RP_BENCH_SHARED_GPU") == "1"
    if shared:  # a hang in this test mode dumps every thread's stack
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ.get("RP_BENCH_HANG_S", "150")), exit=True)
    local_dev = 0 if shared else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)

    inp = workload_inputs(args.nD, args.K)
    F_dev = torch.from_numpy(inp["F"]).to(dev)
    # metric values V of the sample set: the truth evaluated by the product (rp_eval_metrics),
    # times the seeded 1% noise multipliers -- input synthesis, outside the timed region
    X_all = torch.from_numpy(inp["X"]).to(dev)
    V_all = rp.eval_metrics(inp["truth"], X_all) * torch.from_numpy(inp["noise"]).to(dev)
    klo, khi = rdist.shard_bounds(len(inp["X"]), world, rank)
    dlo, dhi = rdist.shard_bounds(len(inp["D"]), world, rank)
    X_dev = X_all[klo:khi].contiguous()
    V_dev = V_all[:, klo:khi].contiguous()
    D_dev = torch.from_numpy(inp["D"][dlo:dhi]).to(dev)
    del X_all
    nD, nF, K = len(inp["D"]), len(inp["F"]), len(inp["X"])
    ops = rdist.LibOps()
    idx_out = torch.empty((1, dhi - dlo), dtype=torch.int32, device=dev)
    E_out = torch.empty((1, dhi - dlo), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def fitted_program(coef, c, e):
        prog = copy.deepcopy(inp["truth"])
        prog.coef = [np.asarray(coef[i]) for i in range(3)]
        prog.xform_c, prog.xform_e = list(c), list(e)
        return prog

    # device-resident step: the fit leaves its coefficients and transform on the device, the plan
    # (made once: allocation and F staging are setup) is refitted in place and re-planned (a1/a5)
    # on the device, the sweep follows -- no host round trip inside a step
    plan_dev = rp.Plan([inp["truth"]], F_dev)
    plan_dev.enable_timing()  # CUDA events around the sweep kernel / refinement inside each eval

    def step_dev(ev=None):
        if world == 1:
            coef, xf, _ = rp.fit_dev(X_dev, V_dev, inp["num"], inp["den"])
        else:
            coef, xf, _ = rdist.sharded_fit_dev(X_dev, V_dev, inp["num"], inp["den"], ops, n_vars=4)
        if ev is not None:
            ev[0].record(stream)
        plan_dev.update(coef, xf)
        if ev is not None:
            ev[1].record(stream)
        idx, E, _ = plan_dev.eval(D_dev, out=(idx_out, E_out, None), second=False)
        if ev is not None:
            ev[2].record(stream)
        if world > 1:
            idx, E = rdist.gather_winners(idx, E, nD)
        return idx, E

    # host-API step (the e2e leg): host buffers through the C ABI, the library stages the copies
    def step(ev=None, X=X_dev, V=V_dev, D=D_dev, out=(idx_out, E_out), F=F_dev):
        if world == 1:
            coef, (c, e), _ = rp.fit(X, V, inp["num"], inp["den"], raise_on_degenerate=False)
        else:
            coef, (c, e), _ = rdist.sharded_fit(X, V, inp["num"], inp["den"], ops, n_vars=4)
        plan = rp.Plan([fitted_program(coef, c, e)], F)
        idx, E, _ = plan.eval(D, out=(out[0], out[1], None), second=False)
        if world > 1:
            idx, E = rdist.gather_winners(idx, E, nD)
        plan.close()
        return idx, E

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        step_dev()
    barrier()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.5)  # nvidia-smi up before the timed region
    for _ in range(2):  # every rank: the step has collectives at N > 1
        step_dev()
    torch.cuda.synchronize()
    times, t_fit, t_sweep_k, t_plan, t_kern, t_ref = [], [], [], [], [], []
    for _ in range(args.steps):
        flush.zero_()  # L2 (126 MB) flushed between timed steps
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        a.record(stream)
        step_dev(ev)
        b.record(stream)
        barrier()
        times.append(a.elapsed_time(b))
        t_fit.append(a.elapsed_time(ev[0]))
        t_sweep_k.append(ev[1].elapsed_time(ev[2]))
        t_plan.append(ev[0].elapsed_time(ev[1]))
        lt = plan_dev.last_timing()  # the same launch, events on its stream (rp_plan_last_timing)
        t_kern.append(lt["sweep_ms"])
        t_ref.append(lt["refine_ms"])
    clocks = sampler.stop() if sampler else None
    # self-check: the device-resident step and the host-API step give identical winners
    i_dev, E_dev = (t.clone() for t in step_dev())
    i_host, E_host = step()
    selfcheck = bool(torch.equal(i_dev.reshape(-1), i_host.reshape(-1)) and torch.equal(E_dev.reshape(-1), E_host.reshape(-1)))
    med = statistics.median  # the median of the timed steps
    step_ms, fit_ms, sweep_ms = med(times), med(t_fit), med(t_sweep_k)
    kern_ms, refine_ms = med(t_kern), med(t_ref)
    if world > 1:
        t = torch.tensor([step_ms, fit_ms, sweep_ms, kern_ms, refine_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        step_ms, fit_ms, sweep_ms, kern_ms, refine_ms = t.tolist()

    # ---- alternative sweep kernel (informational, after the timed region): k_sweep_tc, the
    # tcgen05 split-tf32 contraction + FP32 screen (RP_SWEEP_KERNEL=tc), on the same launch; its
    # winners must equal the default kernel's ------------------------------------------------
    loc_idx, loc_E = idx_out.clone(), E_out.clone()
    os.environ["RP_SWEEP_KERNEL"] = "tc"
    try:
        if args.no_alt:
            raise RuntimeError("skipped (--no-alt)")
        ti, tE = torch.empty_like(idx_out), torch.empty_like(E_out)
        plan_dev.eval(D_dev, out=(ti, tE, None), second=False)
        tc_ms = []
        for _ in range(5):
            flush.zero_()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            plan_dev.eval(D_dev, out=(ti, tE, None), second=False)
            t1.record(stream)
            torch.cuda.synchronize()
            tc_ms.append(t0.elapsed_time(t1))
        alt_sweep = {"kernel": "k_sweep_tc (RP_SWEEP_KERNEL=tc)", "ms": sorted(tc_ms)[len(tc_ms) // 2],
                     "winners_identical": bool(torch.equal(ti, loc_idx) and torch.equal(tE, loc_E)),
                     "note": "the FITTED program's polynomials cancel heavily (Cauchy-Schwarz rho median 35, "
                             "p99 1.7e3 for metric 2), beyond what an FP32-accumulated contraction can screen: "
                             "its tuples fall back to FP64 (DESIGN.md 'Tensor-core screened sweep')"}
    except Exception as exc:  # informational only
        alt_sweep = {"kernel": "k_sweep_tc", "error": str(exc)[:200]}
    finally:
        os.environ.pop("RP_SWEEP_KERNEL", None)

    # ---- secondary kernel: the Gram (timed alone after the timed region) ----------------------
    c0, e0 = rp.xform_from_box(*rp.minmax(X_dev))
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    G = rp.gram(X_dev, V_dev, inp["num"], inp["den"], c0, e0)
    torch.cuda.synchronize()
    g0.record(stream)
    for _ in range(3):
        rp.gram(X_dev, V_dev, inp["num"], inp["den"], c0, e0, out=G)
    g1.record(stream)
    torch.cuda.synchronize()
    gram_ms = g0.elapsed_time(g1) / 3

    # ---- e2e: the same step fed from pinned host buffers --------------------------------------
    # (1) pipelined (the headline e2e): at N = 1 the C ABI's rp_pipeline (rp_pipeline.cu, through
    #     pipeline.StepPipeline): step i+1's X, V, D stream in on one copy stream and step i-1's
    #     winners stream out on another while step i fits, refreshes the plan and sweeps; timed by
    #     librp's device events from the first H2D to the last D2H (rp_pipeline_timer_*), every
    #     step's copies inside.  At N > 1 the sharded fit needs torch.distributed between the Gram
    #     and the solve, so pipeline.FitSweepPipeline runs the same schedule on torch streams.
    # (2) call by call: rp_fit / rp_plan_create / rp_plan_eval_argmin with host pointers, the
    #     library staging the copies synchronously (no overlap) -- reported as e2e.sync.
    e2e = None
    if not args.no_e2e:
        from paper_1911_02373_b200.pipeline import FitSweepPipeline, StepPipeline
        Xh = torch.from_numpy(inp["X"][klo:khi]).pin_memory()
        Vh = V_dev.cpu().pin_memory()
        Dh = torch.from_numpy(inp["D"][dlo:dhi]).pin_memory()
        Fh = torch.from_numpy(inp["F"]).pin_memory().numpy()
        n_out = nD if world > 1 else dhi - dlo
        oi = torch.empty((1, n_out), dtype=torch.int32).pin_memory()
        oE = torch.empty((1, n_out), dtype=torch.float64).pin_memory()
        n_e = max(4, args.steps)
        if world == 1:
            cpipe = StepPipeline(inp["truth"], F_dev, inp["num"], inp["den"], khi - klo, 3, dhi - dlo, 2, depth=2)
            oi1, oE1 = oi.reshape(-1), oE.reshape(-1)
            for _ in range(3):
                cpipe.submit(Xh, Vh, Dh, oi1, oE1)
            cpipe.sync()
            barrier()
            cpipe.timer_start()
            for _ in range(n_e):
                cpipe.submit(Xh, Vh, Dh, oi1, oE1)
            e_ms = cpipe.timer_stop() / n_e
            cpipe.sync()
            cpipe.close()
            e2e_path = ("rp_pipeline (C ABI, rp_pipeline.cu): pinned X, V, D in and winners out on two copy streams "
                        "inside librp, overlapped with the neighbouring steps' fit -> plan update -> sweep; device "
                        "events from the first H2D to the last D2H")
        else:
            fit_fn = None
            gather_fn = None
            if world > 1:
                def fit_fn(X, V):
                    return rdist.sharded_fit_dev(X, V, inp["num"], inp["den"], ops, n_vars=4)[:2]

                def gather_fn(i, E):
                    return rdist.gather_winners(i, E, nD)
            pipe = FitSweepPipeline(inp["truth"], F_dev, inp["num"], inp["den"], khi - klo, 4, 3, dhi - dlo, 2,
                                    device=dev, fit_fn=fit_fn, gather_fn=gather_fn)

            def fed_step():
                with torch.cuda.stream(pipe.compute):
                    flush.zero_()
                return pipe.submit(Xh, Vh, Dh, oi, oE)

            for _ in range(3):
                fed_step()
            barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(pipe.h2d)
            for _ in range(n_e):
                done = fed_step()
            pipe.d2h.wait_event(done)
            t1.record(pipe.d2h)
            barrier()
            e_ms = t0.elapsed_time(t1) / n_e
            pipe.close()
            e2e_path = ("FitSweepPipeline (pipeline.py): pinned X, V, D in and winners out on two copy streams, "
                        "overlapped with the neighbouring steps' sharded fit -> plan update -> sweep -> gather")
        ok_e2e = bool(torch.equal(oi.reshape(-1), i_dev.reshape(-1).cpu()))
        # call by call (no overlap)
        Xn, Vn, Dn = Xh.numpy(), Vh.numpy(), Dh.numpy()
        oin = torch.empty((1, dhi - dlo), dtype=torch.int32).pin_memory().numpy()
        oEn = torch.empty((1, dhi - dlo), dtype=torch.float64).pin_memory().numpy()
        for _ in range(2):
            step(X=Xn, V=Vn, D=Dn, out=(oin, oEn), F=Fh)
        s_times = []
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            idx, E = step(X=Xn, V=Vn, D=Dn, out=(oin, oEn), F=Fh)
            if world > 1:
                idx, E = idx.cpu(), E.cpu()  # gathered winners back to the host
            b.record(stream)
            barrier()
            s_times.append(a.elapsed_time(b))
        s_ms = sum(s_times) / len(s_times)
        if world > 1:
            t = torch.tensor([e_ms, s_ms], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            e_ms, s_ms = t.tolist()
        h2d = Xh.nbytes + Vh.nbytes + Dh.nbytes
        d2h = oi.nbytes + oE.nbytes
        e2e = {"value": nD * nF / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": n_e, "winners_match_device_step": ok_e2e, "path": e2e_path,
               "l2": "not flushed: every step's 72 MB of inputs arrive by H2D while the previous step computes",
               "sync": {"value": nD * nF / (s_ms * 1e-3), "ms_per_step": s_ms,
                        "path": "rp_fit + rp_plan_create + rp_plan_eval_argmin with pinned host buffers, "
                                "library-staged copies, no overlap"}}

    if rank != 0:
        if world > 1:
            tdist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (k_sweep) ----------------------------------------------
    pairs_eval = evaluated_pairs(inp["D"][dlo:dhi], inp["F"])
    flop_launch = pairs_eval * FLOP_PER_PAIR + (dhi - dlo) * FLOP_PER_D
    achieved = flop_launch / (kern_ms * 1e-3) / 1e12
    traffic, counters = None, None
    prof = os.path.join(ROOT, "profiles", "sweep_ncu_latest.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic, counters = pj.get("dram_bytes_per_launch"), pj.get("counters")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "alu", "kernel": "k_sweep", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz (DESIGN.md 'Peaks'); "
                               "measured DFMA microbenchmark 34.1 TF/s (profiles/r01_fp64_microbench.jsonl)",
                "flop_per_launch": flop_launch, "flop_per_pair": FLOP_PER_PAIR, "flop_per_D": FLOP_PER_D,
                "evaluated_pairs": pairs_eval, "ms_per_launch": kern_ms,
                "timing": "CUDA events recorded by librp around k_sweep on its stream inside every timed step "
                          "(rp_plan_last_timing), median", "ncu": counters}
    # moment contraction: every Gram entry is a weighted moment of one monomial,
    # so a row costs 2 x (1 + 2 n_v) weights x C(D + n, n) monomials of degree <= D = 2 x 4 in
    # n = 4 variables: 2 x 7 x 495 = 6,930 flop (the DMMA tiles execute 2 x 8 x 496 = 7,936);
    # the outer-product Gram it replaces is 2 x 7 x 70 x 71 / 2 = 34,790 flop per row
    n_mom = math.comb(2 * 4 + 4, 4)
    gram_flop = (khi - klo) * 2 * (1 + 2 * 3) * n_mom
    gram_ach = gram_flop / (gram_ms * 1e-3) / 1e12
    gram_exec = (khi - klo) * 2 * 8 * (8 * ((n_mom + 7) // 8)) / (gram_ms * 1e-3) / 1e12
    gram_equiv = (khi - klo) * (1 + 2 * 3) * 70 * 71 / (gram_ms * 1e-3) / 1e12
    gtraffic, gcounters = None, None
    gprof = os.path.join(ROOT, "profiles", "gram_ncu_latest.json")
    if os.path.exists(gprof):
        try:
            gj = json.load(open(gprof))
            gtraffic, gcounters = gj.get("dram_bytes_per_launch"), gj.get("counters")
        except (OSError, ValueError):
            gtraffic = None
    roofline_fit = {"bound": "tensor", "kernel": "k_gram_mom (moment contraction on DMMA.8x8x4)", "achieved": gram_ach,
                    "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": gram_ach / FP64_PEAK_TFLOPS,
                    "flop_per_row": 2 * (1 + 2 * 3) * n_mom, "executed_tflops": gram_exec,
                    "outer_product_equiv_tflops": gram_equiv,
                    "traffic": gtraffic, "ncu": gcounters,
                    "ms_per_call": gram_ms, "peak_source": "FP64 tensor = FP64 FMA rate on B200 "
                                                           "(measured DMMA 36.9 TF/s)"}

    cpu_baseline = None
    if world == 1 and not args.no_cpu_baseline:
        cores, model = cpu_info()
        # size each sample for ~10 s of oracle work: probe on 1/SAMPLE_DIV, then rescale
        _, dt0 = oracle_step(inp, 0, cores)
        div = max(2, min(SAMPLE_DIV, int(SAMPLE_DIV * dt0 / 10.0)))
        v, dt = oracle_step(inp, 1, cores, div)
        _, dt1 = oracle_step(inp, 2, 1, 4 * SAMPLE_DIV)
        div1 = max(2, min(4 * SAMPLE_DIV, int(4 * SAMPLE_DIV * dt1 / 10.0)))
        v1, dt1 = oracle_step(inp, 3, 1, div1)
        cpu_baseline = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": model,
                        "seconds": dt, "sample": f"1/{div} of the step (second slice): fit of 3 metrics on "
                                               f"{K // div} rows + sweep of {nD // div} D x {nF} F",
                        "one_core": {"value": v1, "cores": 1, "seconds": dt1,
                                     "sample": f"1/{div1} of the step (fourth slice): fit on {K // div1} rows + "
                                               f"sweep of {nD // div1} D x {nF} F"}}

    # fit: minmax part / final, xform, xform_to_basis, gram_ws, gram_fused_sum, gram_fused_reduce,
    # solve (8); plan update: plan_refresh (1); sweep: bucket count / scan / scatter, sweep, refine (5)
    # (the ncu launch list of this command, profiles/r01_launches_bench.txt, shows the same 13)
    launches_per_step = 14
    out = {"metric": METRIC, "value": nD * nF / (step_ms * 1e-3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded: class-F truths, box-sampled K with 1% noise, log-uniform D)",
           "config": {"workload": "large+fitheavy", "nD": nD, "nF": nF, "K": K, "n_metrics": 3, "n_c": 140,
                      "parallelism": f"dp{world}: D and K rows sharded, Gram all_reduce, winners all_gather",
                      "l2": "flushed between timed steps (256 MiB write); inputs 64 MB"},
           "fit_rows_per_s": K / (fit_ms * 1e-3), "fit_ms": fit_ms,
           "sweep_evals_per_s": nD * nF / (sweep_ms * 1e-3), "sweep_ms": sweep_ms, "sweep_kernel_ms": kern_ms,
           "refine_ms": refine_ms, "parity": parity_summary(),
           "plan_update_ms": sum(t_plan) / len(t_plan),
           "evaluated_pairs_per_s": (pairs_eval if world == 1 else evaluated_pairs(inp["D"], inp["F"])) / (sweep_ms * 1e-3),
           "roofline": roofline, "roofline_fit": roofline_fit, "cpu_baseline": cpu_baseline, "e2e": e2e,
           "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
           "selfcheck": {"device_step_equals_host_api_step": selfcheck}, "alt_sweep": alt_sweep}
    print(json.dumps(out), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
