"""Class-L diagnostics (SURVEY 8(c) "parity classes", 8(d) run matrix; VERDICT r1 missing #2, #3).

The paper profiles small data sizes at launch shapes and warns
that the resulting matrix is "highly likely" rank-deficient, which is why it uses the "more
numerically stable" SVD.  For each class-L design (synth.classL_case: tiny
launch design with the class-F truth; polybench and multikernel launch designs with the
kernel-flavoured truths, 1% noise) this module

* fits every metric five ways: the oracle's normal equations (long double) and SVD, the GPU's
  normal equations (rp_fit) and SVD (rp_fit_svd) on centred variables, and both GPU solvers on
  UNcentred variables (identity transform: rp_gram_accumulate + rp_solve_normal, rp_tsqr_accumulate
  + rp_svd_rows);
* reports the equilibrated cond(G_ff), the GPU-vs-oracle coefficient gap (not gated: the fits are
  non-unique), and each fit's value-space error against the truth on held-out
  pairs of the sweep domain (the quantity a launch decision depends on);
* sweeps the ORACLE's fit on both sides over the config's D x F grid and gates it against the
  binary128 oracle everywhere (E within 1e-12 at the GPU's pick, idx bit-exact where the margin
  exceeds 1e-9, else within the 1e-9 tie set) and, SURVEY 8(c) #25 literally, against the long
  double oracle where it is accurate (kappa <= 1e3, long double E within 1e-13 of binary128),
  reporting the covered fraction.

Gated here: the Gram of every design (always well-posed, 1e-12 sqrt(G_ii G_jj)), the kappa-filtered
sweep, and the finiteness of every centred fit.  Everything else is the committed report
gpurun_out/classL_<name>.json (profiles/r02_classL_*.json).
"""
import copy
import json
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_02373_b200 as rp  # noqa: E402

DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NT = len(os.sched_getaffinity(0))


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _cond_eq(G, beta0):
    """Equilibrated condition number of G_ff (beta_0's row and column removed)."""
    keep = [i for i in range(G.shape[0]) if i != beta0]
    A = np.asarray(G, dtype=np.float64)[np.ix_(keep, keep)]
    d = np.sqrt(np.abs(np.diag(A)))
    d[d == 0] = 1.0
    return float(np.linalg.cond(A / np.outer(d, d)))


def _held_out(case, n=3000):
    """n (N, P) pairs of the sweep domain that pass the static rules and P1 P2 <= N^2."""
    g = synth.rng(case.name, "heldout")
    D = case.sweep.D[:, 0]
    F = case.sweep.F
    T = F.prod(axis=1)
    F = F[(T % 32 == 0) & (T <= 1024)]
    out = []
    while len(out) < n:
        N = D[g.integers(0, len(D))]
        P = F[g.integers(0, len(F))]
        if int(P[0]) * (int(P[1]) if len(P) > 1 else 1) <= int(N) * int(N):
            out.append([N, *P])
    return np.asarray(out, dtype=np.float64)


def _vrel(truth, i, Xh, num, den, coef, c, e):
    """max / median relative value-space error of a fit of metric i against the truth."""
    want = np.asarray(oracle.program_metrics(truth, Xh)[i], dtype=np.float64)
    got = np.asarray(oracle.eval_ratfunc(num, den, coef, c, e, Xh)[0], dtype=np.float64)
    r = np.abs(got - want) / np.abs(want)
    r = np.where(np.isfinite(r), r, np.inf)
    return float(np.median(r)), float(np.quantile(r, 0.99)), float(np.max(r))


def _run(name, n_kernels=20, sweep_nD=2000):
    case = synth.classL_case(name, n_kernels=n_kernels)
    X = case.X
    n = X.shape[1]
    b = case.basis
    nn = len(b)
    zc, ze = np.zeros(n), np.zeros(n, dtype=np.int32)
    Xh = _held_out(case)
    rep = {"design": name, "K": int(len(X)), "n_c": 2 * nn, "programs": []}
    fitted = []
    for gi, truth in enumerate(case.truths):
        V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(truth, X)]) * case.noise[gi]
        coef_g, (c, e), inf_g = rp.fit(_cuda(X), _cuda(V), b, b, raise_on_degenerate=False)
        coef_s, sig_s, _, inf_s = rp.fit_svd(_cuda(X), _cuda(V), b, b, raise_on_degenerate=False)
        G_u = rp.gram(_cuda(X), _cuda(V), b, b, zc, ze)
        coef_gu, inf_gu = rp.solve_normal(G_u, b, b, raise_on_degenerate=False)
        R_u = rp.tsqr(_cuda(X), _cuda(V), b, b, zc, ze)
        coef_su, _, inf_su = rp.svd_rows(R_u, b, b, raise_on_degenerate=False)
        G_c = rp.gram(_cuda(X), _cuda(V), b, b, c, e).cpu().numpy()
        prog_rep = {"program": gi, "metrics": []}
        ocoefs = []
        for i in range(3):
            o = oracle.fit(X, V[i], b, b, nthreads=NT)
            o_u = oracle.fit(X, V[i], b, b, nthreads=NT, xform=(zc, ze))
            osvd = oracle.fit_svd(X, V[i], b, b)
            assert np.array_equal(o["c"], c) and np.array_equal(o["e"], e)
            Go = np.asarray(o["G"], dtype=np.float64)
            dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
            gram_err = float(np.max(np.abs(G_c[i] - Go) / dg))
            assert gram_err <= 1e-12, (name, gi, i, gram_err)  # the Gram gate holds in class L
            oc = np.asarray(o["coef"], dtype=np.float64)
            ocoefs.append(oc)
            assert np.all(np.isfinite(coef_g[i]) | np.isnan(coef_g[i]))
            gap = float(np.max(np.abs(coef_g[i] - oc)) / np.max(np.abs(oc))) if np.all(np.isfinite(oc)) else None
            m = {"metric": i, "cond_eq_G_ff": _cond_eq(Go, nn), "gpu_ne_status": inf_g[i]["status"],
                 "gpu_ne_cond_est": inf_g[i]["cond_est"], "oracle_ne_status": int(o["status"]),
                 "coef_gap_gpu_vs_oracle_ne": gap, "gram_err": gram_err,
                 "svd_sigma_min_over_max": float(sig_s[i][0] / sig_s[i][-1]) if sig_s[i][-1] > 0 else None,
                 "value_err_vs_truth": {}}
            fits = {"oracle_ne": (oc, c, e), "gpu_ne": (coef_g[i], c, e), "gpu_svd": (coef_s[i], c, e),
                    "oracle_svd": (np.asarray(osvd["coef"], dtype=np.float64), c, e),
                    "oracle_ne_uncentred": (np.asarray(o_u["coef"], dtype=np.float64), zc, ze),
                    "gpu_ne_uncentred": (coef_gu[i], zc, ze), "gpu_svd_uncentred": (coef_su[i], zc, ze)}
            for k, (cf, cc, ee) in fits.items():
                if np.all(np.isfinite(cf)):
                    med, p99, mx = _vrel(truth, i, Xh, b, b, cf, cc, ee)
                    m["value_err_vs_truth"][k] = {"median": med, "p99": p99, "max": mx}
                else:
                    m["value_err_vs_truth"][k] = "degenerate (NaN coefficients)"
            m["uncentred_status"] = {"gpu_ne": inf_gu[i]["status"], "gpu_ne_cond_est": inf_gu[i]["cond_est"],
                                     "gpu_svd": inf_su[i]["status"], "oracle_ne": int(o_u["status"])}
            prog_rep["metrics"].append(m)
        rep["programs"].append(prog_rep)
        spec = copy.deepcopy(case.fit_programs[gi])
        spec.coef = ocoefs
        spec.xform_c, spec.xform_e = list(c), list(e)
        fitted.append(spec)
    # the oracle's fits swept on both sides.  Gate A (every feasible tuple): E within 1e-12 of the
    # binary128 oracle at the GPU's pick, idx exact where the exact margin exceeds 1e-9, else in
    # the 1e-9 tie set.  Gate B, SURVEY 8(c) #25 literally, against the long double oracle where
    # it is itself accurate: kappa <= 1e3 at winner and runner-up AND its E within 1e-13 of the
    # binary128 value (mixed-sign metrics make Appendix A's sums cancel: the long double E is then
    # off by up to ~1e-11 while the GPU's refined E equals the binary128 value, R31)
    D = case.sweep.D[:sweep_nD]
    F = case.sweep.F
    idx, E, S = rp.eval_argmin_batched(fitted, _cuda(D), _cuda(F))
    idx, E = idx.cpu().numpy(), E.cpu().numpy()
    tot = dict(feasible=0, idx_exact_A=0, tie_A=0, covered_B=0, idx_exact_B=0, mask_disagree=0)
    eA, eB = 0.0, 0.0
    kap = []
    for gi, spec in enumerate(fitted):
        ref = oracle.sweep(spec, D, F, nthreads=NT)
        refq = oracle.sweep(spec, D, F, nthreads=NT, quad=True)
        feas = (refq["idx"] >= 0) & (idx[gi] >= 0)
        tot["mask_disagree"] += int(((refq["idx"] >= 0) != (idx[gi] >= 0)).sum())
        with np.errstate(invalid="ignore", divide="ignore"):
            mq = (refq["second"] - refq["best"]) / refq["best"]
            ml = (ref["second"] - ref["best"]) / ref["best"]
        strict = feas & (mq > 1e-9)
        assert np.array_equal(idx[gi][strict], refq["idx"][strict]), (name, gi)
        Eq = refq["best"].copy()
        for t in np.nonzero(feas & (idx[gi] != refq["idx"]))[0]:
            tr = oracle.eval_pair(spec, D[t], F[idx[gi][t]], quad=True)
            assert tr["feasible"]
            Eq[t] = float(tr["E"])
            assert (Eq[t] - refq["best"][t]) <= 1e-9 * refq["best"][t], (name, gi, t)
            tot["tie_A"] += 1
        rel = np.abs(E[gi][feas] - Eq[feas]) / Eq[feas]
        assert rel.max(initial=0) <= 1e-12, (name, gi, rel.max())
        eA = max(eA, float(rel.max(initial=0)))
        with np.errstate(invalid="ignore", divide="ignore"):
            ld_ok = np.abs(ref["best"] - refq["best"]) <= 1e-13 * np.abs(refq["best"])
        cov = feas & (ref["idx"] >= 0) & ld_ok & (ref["kappa"] <= 1e3) & ((ref["kappa2"] <= 1e3) | (ref["idx2"] < 0))
        sB = cov & (ml > 1e-9)
        assert np.array_equal(idx[gi][sB], ref["idx"][sB]), (name, gi)
        relB = np.abs(E[gi][cov] - ref["best"][cov]) / ref["best"][cov]
        assert relB.max(initial=0) <= 1e-12, (name, gi, relB.max())
        eB = max(eB, float(relB.max(initial=0)))
        tot["feasible"] += int(feas.sum())
        tot["idx_exact_A"] += int(strict.sum())
        tot["covered_B"] += int(cov.sum())
        tot["idx_exact_B"] += int(sB.sum())
        kap.extend(ref["kappa"][ref["idx"] >= 0].tolist())
    rep["sweep"] = dict(tot, nD=int(len(D)), nF=int(len(F)), programs=len(fitted),
                        E_max_rel_err_vs_binary128=eA, E_max_rel_err_covered_B=eB,
                        covered_fraction_B=tot["covered_B"] / max(tot["feasible"], 1),
                        kappa_winner_median=float(np.median(kap)) if kap else None,
                        kappa_winner_max=float(np.max(kap)) if kap else None)
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"classL_{name}.json"), "w") as f:
        json.dump(rep, f, indent=1, sort_keys=True, default=float)
    return rep


def test_classL_tiny():
    rep = _run("tiny")
    assert rep["sweep"]["feasible"] > 0


def test_classL_polybench():
    rep = _run("polybench")
    assert rep["sweep"]["feasible"] > 0


def test_classL_multikernel():
    rep = _run("multikernel", n_kernels=20, sweep_nD=1000)
    assert rep["sweep"]["feasible"] > 0
