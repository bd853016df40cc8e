"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on the same seeded inputs.

Tolerances (BASELINE.json north_star): argmin config index bit-exact wherever the oracle's
(second - best)/best margin exceeds 1e-9; E within 1e-12 relative; fitted coefficients within
1e-9 relative (inf-norm, after beta_0 = 1); Gram entries within
1e-12 * sqrt(G_ii G_jj).  Near ties (margin <= 1e-9) must pick a config inside the oracle's
epsilon-tie set (reading R20).
"""
import copy

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


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def subset(ref, sel):
    """The oracle sweep's per-D arrays restricted to `sel` (counters dropped)."""
    return {k: v[sel] for k, v in ref.items() if isinstance(v, np.ndarray)}


def check_sweep(idx, E, S, ref, spec=None, D=None, F=None, tag=""):
    idx = np.asarray(idx.cpu() if hasattr(idx, "cpu") else idx)
    E = np.asarray(E.cpu() if hasattr(E, "cpu") else E)
    feas = ref["idx"] >= 0
    assert np.array_equal(idx < 0, ~feas), tag
    assert np.all(np.isinf(E[~feas])), tag
    b = ref["best"][feas]
    rel = np.abs(E[feas] - b) / b
    tol = 1e-12
    assert np.all(rel <= tol), (tag, rel.max())
    with np.errstate(invalid="ignore"):
        margin = (ref["second"] - ref["best"]) / ref["best"]
    strict = feas & (margin > 1e-9)
    assert np.array_equal(idx[strict], ref["idx"][strict]), tag
    # near ties: the GPU winner's oracle E must be within the tie margin of the best
    for i in np.nonzero(feas & ~(margin > 1e-9))[0]:
        if idx[i] != ref["idx"][i]:
            tr = oracle.eval_pair(spec, D[i], F[idx[i]])
            assert tr["feasible"] and abs(float(tr["E"]) - ref["best"][i]) <= 1e-9 * ref["best"][i], (tag, i)
    if S is not None:
        S = np.asarray(S.cpu() if hasattr(S, "cpu") else S)
        fin = np.isfinite(ref["second"])
        assert np.array_equal(np.isfinite(S), fin), tag
        r2 = np.abs(S[fin] - ref["second"][fin]) / ref["second"][fin]
        assert r2.max(initial=0) <= 1e-12, (tag, r2.max())
    return int(strict.sum()), int(feas.sum())


def test_sweep_tiny():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    ref = oracle.sweep(spec, D, case.F)
    idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(case.F))
    check_sweep(idx, E, S, ref, spec, D, case.F, "tiny")


def test_sweep_tiny_host_pointers():
    """The same call with host (numpy) buffers: the library stages them itself."""
    case = synth.tiny_sweep()
    spec = case.programs[0]
    ref = oracle.sweep(spec, case.D, case.F)
    idx, E, S = rp.eval_argmin(spec, case.D, case.F)
    assert isinstance(idx, np.ndarray)
    check_sweep(idx, E, S, ref, spec, case.D, case.F, "tiny-host")


def test_sweep_g1_template_all_tie():
    """SPEC.md:492 example through the GPU: E = N^2/(bx*by), N = 64 -> lowest T=1024 index."""
    from helpers import ratfunc_program
    F = synth.F_pow2_2d()
    spec = ratfunc_program(synth.HW_GTX1080TI, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2, R=16)
    D = np.array([[64], [8], [1000]], dtype=np.int32)
    ref = oracle.sweep(spec, D, F)
    idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(F))
    assert np.array_equal(idx.cpu().numpy(), ref["idx"])
    assert np.array_equal(E.cpu().numpy(), ref["best"])


@pytest.mark.parametrize("which", ["polybench", "multikernel"])
def test_sweep_batched(which):
    case = synth.polybench_sweep() if which == "polybench" else synth.multikernel_sweep()
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    idx, E, S = rp.eval_argmin_batched(case.programs, _cuda(D), _cuda(case.F))
    for g, spec in enumerate(case.programs):
        ref = oracle.sweep(spec, D, case.F)
        check_sweep(idx[g], E[g], S[g], ref, spec, D, case.F, f"{which}[{g}]")


def test_sweep_large_full_size_sampled():
    """The bench's launch configuration: all 10^6 D x 1,024 F on the GPU (through a plan, as
    bench.py does), compared on the oracle's subsample (every 100th D + first/last 100)."""
    case = synth.large_sweep()
    spec = case.programs[0]
    plan = rp.Plan([spec], _cuda(case.F))
    assert plan.static_feasible() == 464
    idx, E, S = plan.eval(_cuda(case.D))
    # the bench times the runner-up-free template: identical winners and estimates
    idx2, E2, _ = plan.eval(_cuda(case.D), second=False)
    assert torch.equal(idx2, idx) and torch.equal(E2, E)
    sub = synth.large_subsample_index(len(case.D))
    ref = oracle.sweep(spec, case.D[sub], case.F)
    strict, feas = check_sweep(idx[0][sub], E[0][sub], S[0][sub], ref, spec, case.D[sub], case.F, "large")
    assert feas == len(sub) and strict >= 0.99 * feas
    c = ref["counters"]
    assert c["case1"] > 0 and c["case2"] > 0 and c["case3"] > 0


def test_eval_metrics():
    fc = synth.fitheavy(K=5000)
    spec = fc.truths[0]
    got = rp.eval_metrics(spec, _cuda(fc.X)).cpu().numpy()
    want = np.asarray(oracle.program_metrics(spec, fc.X), dtype=np.float64)
    assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-13


def _fit_parity(fc, sigma_noise=None, gram_check=True, cached=None):
    if cached is not None:
        fc, V, oref = cached
    else:
        truth = fc.truths[0]
        V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(truth, fc.X)])
        if fc.noise is not None:
            V = V * fc.noise
        oref = [oracle.fit(fc.X, V[i], fc.num_exp, fc.den_exp, nthreads=8) for i in range(len(V))]
    coef, (c, e), infos = rp.fit(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    worst = 0.0
    for i in range(len(V)):
        r = oref[i]
        assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
        want = np.asarray(r["coef"], dtype=np.float64)
        err = np.max(np.abs(coef[i] - want)) / np.max(np.abs(want))
        worst = max(worst, err)
        assert err <= 1e-9, (fc.name, i, err, infos[i])
        if gram_check:
            G = rp.gram(_cuda(fc.X), _cuda(V[i:i + 1]), fc.num_exp, fc.den_exp, c, e)[0].cpu().numpy()
            Go = np.asarray(r["G"], dtype=np.float64)
            dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
            assert np.max(np.abs(G - Go) / dg) <= 1e-12, (fc.name, i)
    return worst


def test_fit_tiny_box():
    _fit_parity(synth.tiny_fit_box())
    _fit_parity(synth.tiny_fit_box(sigma=0.01))


def test_fit_polybench_box():
    _fit_parity(synth.polybench_fit_box(sigma=0.01))


def test_fit_fitheavy_full_size():
    """The north star's 10^6-row Gram fit (noise-free and 1% noise, 3 metrics, 140 columns)."""
    from conftest import oracle_fitheavy_fit
    _fit_parity(None, gram_check=False, cached=oracle_fitheavy_fit(0.0))
    _fit_parity(None, gram_check=True, cached=oracle_fitheavy_fit(0.01))


def test_fit_host_pointers_and_gram_edge_cases():
    fc = synth.tiny_fit_box()
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
    coef_h, xf_h, _ = rp.fit(fc.X, V, fc.num_exp, fc.den_exp)  # host buffers
    coef_d, xf_d, _ = rp.fit(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    assert np.array_equal(coef_h, coef_d)
    c, e = xf_d
    # K = 0: G = 0; ragged K (not a multiple of the 64-row tile, odd)
    G0 = rp.gram(np.zeros((0, 3)), np.zeros((1, 0)), fc.num_exp, fc.den_exp, c, e)
    assert np.all(G0 == 0)
    for K in (1, 3, 63, 65, 127):
        X = fc.X[:K]
        Gk = rp.gram(_cuda(X), _cuda(V[:1, :K]), fc.num_exp, fc.den_exp, c, e)[0].cpu().numpy()
        Go = np.asarray(oracle.gram(X, V[0, :K], fc.num_exp, fc.den_exp, c, e), dtype=np.float64)
        dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
        assert np.max(np.abs(Gk - Go) / dg) <= 1e-13, K


@pytest.mark.parametrize("kernel", ["mom", "mom_generic", "ws", "fused"])
@pytest.mark.parametrize("basis", ["tree", "no_tree"])
def test_gram_fused_kernels(kernel, basis, monkeypatch):
    """The Gram kernels -- the moment contraction (default), the warp-specialised and the
    single-role outer-product kernels -- on a basis that is closed under parents (monomial-tree
    staging) and on one that is not (power-table staging), at ragged row counts, against the
    oracle's plain sum of outer products."""
    monkeypatch.setenv("RP_GRAM_KERNEL", kernel.split("_")[0])
    if kernel == "mom_generic":  # the runtime monomial step instead of the specialised one
        monkeypatch.setenv("RP_MOM_GENERIC", "1")
    fc = synth.polybench_fit_box()
    if basis == "tree":
        num = fc.num_exp
    else:  # 12 monomials, most without their parent in the list (e.g. x0^2 without x0)
        num = np.array([[0, 0, 0, 0], [2, 0, 0, 0], [0, 2, 0, 0], [0, 0, 1, 1], [2, 2, 0, 0], [1, 1, 1, 0],
                        [0, 0, 0, 3], [3, 0, 0, 0], [0, 1, 2, 0], [2, 0, 0, 1], [1, 0, 1, 1], [0, 3, 0, 0]],
                       dtype=np.int16)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
    lo, hi = fc.X.min(axis=0), fc.X.max(axis=0)
    c, e = rp.xform_from_box(lo, hi)
    for K in (1, 31, 33, 517, 2000):
        X = fc.X[:K]
        G = rp.gram(_cuda(X), _cuda(V[:, :K]), num, num, c, e).cpu().numpy()
        for i in range(len(V)):
            Go = np.asarray(oracle.gram(X, V[i, :K], num, num, c, e), dtype=np.float64)
            dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
            assert np.max(np.abs(G[i] - Go) / dg) <= 1e-12, (kernel, basis, K, i)


def test_fit_degenerate():
    X = np.ones((10, 1))
    V = np.full((1, 10), 3.0)
    b = np.array([[0], [1]], dtype=np.int16)
    with pytest.raises(rp.RPError) as ei:
        rp.fit(_cuda(X), _cuda(V), b, b)
    assert ei.value.status == 3


def test_end_to_end_fit_then_sweep():
    """fitheavy noise-free fit (GPU) -> large sweep (GPU) vs the same chain on the oracle, on a
    subsample; the fitted program recovers the truth to ~1e-13 so both agree."""
    import copy
    fc = synth.fitheavy(K=200_000)
    truth = fc.truths[0]
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(truth, fc.X)])
    coef, (c, e), _ = rp.fit(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    fitted = copy.deepcopy(truth)
    fitted.coef = [coef[i] for i in range(3)]
    fitted.xform_c, fitted.xform_e = list(c), list(e)
    D = synth.large_D(2000)
    F = synth.F_large()
    idx, E, S = rp.eval_argmin(fitted, _cuda(D), _cuda(F))
    ref = oracle.sweep(fitted, D, F)
    check_sweep(idx, E, S, ref, fitted, D, F, "e2e")


def test_determinism_bitwise():
    """Same inputs, same launch configuration -> bit-identical outputs (no atomics in the
    sweep's argmin, fixed-order Gram partial sums)."""
    case = synth.polybench_sweep(nD=3000)
    D, F = _cuda(case.D), _cuda(case.F)
    a = rp.eval_argmin_batched(case.programs, D, F)
    b = rp.eval_argmin_batched(case.programs, D, F)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    fc = synth.fitheavy(K=50_000)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
    c, e = oracle.xform_from_box(*oracle.minmax(fc.X))
    G1 = rp.gram(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp, c, e)
    G2 = rp.gram(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp, c, e)
    assert torch.equal(G1, G2)


def test_sweep_without_second_and_single_tuple():
    case = synth.large_sweep(nD=1)
    spec = case.programs[0]
    D = synth.large_D(4001)[3990:]
    ref = oracle.sweep(spec, D, case.F)
    idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(case.F), second=False)
    assert S is None
    check_sweep(idx, E, None, ref, spec, D, case.F, "no-second")
    idx1, E1, _ = rp.eval_argmin(spec, _cuda(D[:1]), _cuda(case.F))
    assert idx1.item() == idx[0].item() and E1.item() == E[0].item()


def test_sweep_one_dimensional_blocks():
    """p = 1 (1-D thread blocks): the D rule is P1 <= D1^2, grid gx = ceil(N / bx)."""
    n = 2
    basis = synth.basis_total_degree(n, 3)
    g = synth.rng("tests", "p1")
    coefs = [synth.classf_coefficients(g, basis, s) for s in synth.METRIC_SCALES]
    spec = synth.ProgramSpec(d=1, p=1, num_exp=[basis] * 3, den_exp=[basis] * 3, coef=coefs,
                             hw=dict(synth.HW_GTX1080TI), R=32, Z0=0, Z1=0, grid_map=(0, -1, -1),
                             box_lo=[2, 1], box_hi=[4096, 1024])
    F = np.array([[b] for b in (1, 16, 32, 48, 64, 96, 128, 256, 512, 768, 1024)], dtype=np.int32)
    D = np.array([[2], [4], [5], [6], [10], [31], [32], [100], [1000], [4096]], dtype=np.int32)
    ref = oracle.sweep(spec, D, F)
    idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(F))
    check_sweep(idx, E, S, ref, spec, D, F, "p=1")


def test_sweep_batch_of_mixed_bases():
    """Programs of different degree (different staged shapes) in one batched launch."""
    base = synth.polybench_sweep(nD=500)
    p2 = synth.classf_program("mixed", 1, 3, 2, *synth.POLY_BOX, hw=synth.HW_GTX1080TI, R=64, Z0=1024, Z1=1,
                              grid_map=(0, 0, -1))
    progs = [base.programs[0], p2, base.programs[3]]
    idx, E, S = rp.eval_argmin_batched(progs, _cuda(base.D), _cuda(base.F))
    for g, spec in enumerate(progs):
        ref = oracle.sweep(spec, base.D, base.F)
        check_sweep(idx[g], E[g], S[g], ref, spec, base.D, base.F, f"mixed[{g}]")


def test_unsupported_sizes_rejected():
    b = synth.basis_total_degree(4, 5)  # 126 monomials -> n_c = 252 > 176
    X = np.ones((10, 4))
    with pytest.raises(rp.RPError) as ei:
        rp.gram(_cuda(X), _cuda(np.ones((1, 10))), b, b, [0.0] * 4, [0] * 4)
    assert ei.value.status == 5


def test_fit_sk_parity():
    """NEXT row f4: Sanathanan-Koerner refit, GPU vs oracle (1e-9 coefficients).  Gated where the
    previous denominator stays away from zero on the sample (reading R29): noisy tiny / polybench
    and noise-free fitheavy (exact recovery is a fixed point).  fitheavy with 1% noise has a plain
    fit whose q changes sign on the sample, which makes the weights 1/q unbounded; its gap is
    reported, not gated."""
    fh = synth.fitheavy(K=50_000)
    for fc, iters, noisy in ((synth.tiny_fit_box(sigma=0.01), 3, True), (synth.polybench_fit_box(sigma=0.01), 3, True),
                             (fh, 2, False)):
        truth = fc.truths[0]
        V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(truth, fc.X)])
        if noisy:
            V = V * fc.noise
        coef, (c, e), infos = rp.fit_sk(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp, iters=iters)
        for i in range(len(V)):
            r = oracle.fit_sk(fc.X, V[i], fc.num_exp, fc.den_exp, iters=iters, nthreads=8)
            assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
            want = np.asarray(r["coef"], dtype=np.float64)
            err = np.max(np.abs(coef[i] - want)) / np.max(np.abs(want))
            assert err <= 1e-9, (fc.name, i, err)
    # diagnostic: the ill-posed case runs and returns finite coefficients
    fn = synth.fitheavy(sigma=0.01, K=50_000)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fn.truths[0], fn.X)]) * fn.noise
    coef, _, _ = rp.fit_sk(_cuda(fn.X), _cuda(V), fn.num_exp, fn.den_exp, iters=2, raise_on_degenerate=False)
    assert np.all(np.isfinite(coef) | np.isnan(coef))


def test_gram_weighted_vs_oracle_rows():
    """The weighted Gram equals sum_r s_r^2 a_r a_r^T (oracle design rows)."""
    fc = synth.tiny_fit_box()
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
    S = synth.rng("tests", "weights").uniform(0.5, 2.0, size=V.shape)
    c, e = oracle.xform_from_box(*oracle.minmax(fc.X))
    G = rp.gram_weighted(_cuda(fc.X), _cuda(V), _cuda(S), fc.num_exp, fc.den_exp, c, e).cpu().numpy()
    for i in range(3):
        A = np.stack([oracle.design_row(fc.num_exp, fc.den_exp, c, e, x, v) for x, v in zip(fc.X, V[i])])
        A = A * S[i][:, None].astype(np.longdouble)
        Go = np.asarray(A.T @ A, dtype=np.float64)
        dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
        assert np.max(np.abs(G[i] - Go) / dg) <= 1e-13


def test_device_resident_fit_and_plan_update():
    """rp_fit_dev == rp_fit (same kernels, bit for bit); rp_plan_update_program on a plan made
    from another program gives the same sweep as a fresh plan of the fitted program."""
    import copy
    fc = synth.polybench_fit_box(sigma=0.01, K=2000)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)]) * fc.noise
    X, Vd = _cuda(fc.X), _cuda(V)
    coef, (c, e), infos = rp.fit(X, Vd, fc.num_exp, fc.den_exp)
    cd, xf, info = rp.fit_dev(X, Vd, fc.num_exp, fc.den_exp)
    assert np.array_equal(cd.cpu().numpy(), coef)
    assert np.array_equal(xf.cpu().numpy()[:, 0], c) and np.array_equal(xf.cpu().numpy()[:, 1], e)
    assert np.all(info.cpu().numpy()[:, 0] == 0)
    # a plan of the truth program, then updated in place to the fitted coefficients / transform
    case = synth.polybench_sweep(nD=3000)
    truth = case.programs[0]
    fitted = copy.deepcopy(truth)
    fitted.coef = [coef[i] for i in range(3)]
    fitted.xform_c, fitted.xform_e = list(c), list(e)
    D, F = _cuda(case.D), _cuda(case.F)
    plan = rp.Plan([truth], F)
    plan.update(cd, xf)
    i1, E1, S1 = plan.eval(D)
    i2, E2, S2 = rp.eval_argmin(fitted, D, F)
    assert torch.equal(i1[0], i2) and torch.equal(E1[0], E2) and torch.equal(S1[0], S2)
    plan.close()
    # a batched plan: updating program 2 in place changes program 2 only
    progs = case.programs[:3]
    bplan = rp.Plan(progs, F)
    before = bplan.eval(D)
    bplan.update(cd, xf, prog=2)
    after = bplan.eval(D)
    for g in (0, 1):
        assert torch.equal(after[0][g], before[0][g]) and torch.equal(after[1][g], before[1][g])
    assert torch.equal(after[0][2], i2) and torch.equal(after[1][2], E2) and torch.equal(after[2][2], S2)
    bplan.close()


def test_sweep_tensor_core_screen(monkeypatch):
    """RP_SWEEP_KERNEL=tc: the tcgen05 screened sweep (split-tf32 contraction in TMEM, FP32 screen
    with a per-pair bound, FP64 for the candidates, FP64 re-sweep of flagged tuples) under the
    default kernel's gates on tiny, polybench and a `large` subsample; and at the bench's full
    `large` launch, winners identical to the default kernel's."""
    monkeypatch.setenv("RP_SWEEP_KERNEL", "tc")
    for case in (synth.tiny_sweep(), synth.polybench_sweep(nD=2000)):
        idx, E, _ = rp.eval_argmin_batched(case.programs, _cuda(case.D), _cuda(case.F), second=False)
        for g, spec in enumerate(case.programs):
            ref = oracle.sweep(spec, case.D, case.F)
            check_sweep(idx[g], E[g], None, ref, spec, case.D, case.F, tag=case.name)
    case = synth.large_sweep(nD=1_000_000)
    spec = case.programs[0]
    sel = synth.large_subsample_index(1_000_000, every=500)
    plan = rp.Plan([spec], _cuda(case.F))
    D = _cuda(case.D)
    idx, E, _ = plan.eval(D, second=False)
    ref = oracle.sweep(spec, case.D[sel], case.F)
    check_sweep(np.asarray(idx.cpu()).ravel()[sel], np.asarray(E.cpu()).ravel()[sel], None, ref, spec,
                case.D[sel], case.F, tag="large")
    monkeypatch.delenv("RP_SWEEP_KERNEL")
    idx0, E0, _ = plan.eval(D, second=False)
    plan.close()
    assert torch.equal(idx.cpu(), idx0.cpu())
    fin = torch.isfinite(E0)
    assert torch.equal(fin, torch.isfinite(E))
    rel = ((E - E0).abs()[fin] / E0[fin]).max().item() if bool(fin.any()) else 0.0
    assert rel <= 1e-12, rel


@pytest.mark.parametrize("shape", ["p1_d1_deg3", "p2_d3_deg2", "p3_d1_deg4"])
def test_sweep_other_program_shapes(shape):
    """Program shapes the BASELINE configs do not use: one program variable (a 1-D block, grid
    rule on one dimension), three data parameters, and 35 program-part monomials (the NPE = 36
    kernel), each against the oracle on the full grid."""
    g = np.random.default_rng(20260 + len(shape))
    if shape == "p1_d1_deg3":
        spec = synth.classf_program("shape_p1", 1, 1, 3, [8, 1], [8192, 1024], synth.HW_GTX1080TI, R=32,
                                    Z0=0, Z1=0, grid_map=(0, -1, -1))
        F = np.concatenate([np.arange(32, 1025, 32), [1, 16, 48, 100, 2048]]).astype(np.int32)[:, None]
        D = synth.log_uniform_ints(g, 8, 8192, (3000, 1)).astype(np.int32)
    elif shape == "p2_d3_deg2":
        spec = synth.classf_program("shape_d3", 3, 2, 2, [8, 8, 8, 1, 1], [4096, 4096, 512, 1024, 1024],
                                    synth.HW_B200, R=40, Z0=1024, Z1=1, grid_map=(1, 0, -1))
        F = synth.F_pow2_2d()
        D = synth.log_uniform_ints(g, 8, 4096, (3000, 3)).astype(np.int32)
        D[:, 2] = np.minimum(D[:, 2], 512)
    else:
        spec = synth.classf_program("shape_p3", 1, 3, 4, [8, 1, 1, 1], [16384, 1024, 1024, 64],
                                    synth.HW_GTX1080TI, R=24, Z0=0, Z1=0, grid_map=(0, 0, -1))
        F = synth.F_pow2_3d()
        D = synth.log_uniform_ints(g, 8, 16384, (2000, 1)).astype(np.int32)
    ref = oracle.sweep(spec, D, F)
    for second in (True, False):
        idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=second)
        strict, feas = check_sweep(idx, E, S if second else None, ref, spec, D, F, tag=shape)
        assert feas > 0 and strict >= 0.95 * feas


def test_fit_different_numerator_denominator_bases():
    """Numerator and denominator bases that differ (degree 3 over degree 1, and a box basis over a
    total-degree one): the generic Gram kernel (not the fused symmetric-block one), its Gram and
    coefficients against the oracle, at ragged K."""
    fc = synth.polybench_fit_box(sigma=0.01)
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)]) * fc.noise
    bases = [(synth.basis_total_degree(4, 3), synth.basis_total_degree(4, 1)),
             (synth.basis_box([1, 2, 1, 1]), synth.basis_total_degree(4, 2))]
    for num, den in bases:
        for K in (97, 2000):
            X = fc.X[:K]
            coef, (c, e), infos = rp.fit(_cuda(X), _cuda(V[:, :K]), num, den)
            for i in range(len(V)):
                r = oracle.fit(X, V[i, :K], num, den, nthreads=8)
                assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
                want = np.asarray(r["coef"], dtype=np.float64)
                err = np.max(np.abs(coef[i] - want)) / np.max(np.abs(want))
                assert err <= 1e-9, (len(num), len(den), K, i, err)
                G = rp.gram(_cuda(X), _cuda(V[i:i + 1, :K]), num, den, c, e)[0].cpu().numpy()
                Go = np.asarray(r["G"], dtype=np.float64)
                dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
                assert np.max(np.abs(G - Go) / dg) <= 1e-12, (len(num), len(den), K, i)


@pytest.mark.parametrize("seed", range(6))
def test_sweep_randomised_programs(seed):
    """Randomised stress: class-F programs with random hardware fixtures (SM count, warp / block /
    register / shared-memory limits), kernel resources (R, Z0, Z1) and a random subset of F with
    odd shapes, against the oracle on the full grid (both templates)."""
    g = np.random.default_rng(7000 + seed)
    hw = dict(synth.HW_GTX1080TI)
    hw.update(n_sm=int(g.integers(1, 200)), w_max=int(g.choice([32, 48, 64])), b_max=int(g.choice([8, 16, 32])),
              t_max=int(g.choice([512, 1024])), r_max=int(g.choice([32768, 65536])),
              z_max=int(g.choice([12288, 24576, 49152])))
    p = int(g.integers(1, 4))
    lo = [8] + [1] * p
    hi = [int(g.choice([2048, 16384]))] + [1024] * p
    spec = synth.classf_program(f"rand{seed}", 1, p, int(g.integers(1, 4)), lo, hi, hw,
                                R=int(g.integers(8, 256)), Z0=int(g.choice([0, 512, 4096])), Z1=int(g.integers(0, 3)),
                                grid_map=tuple([0] * p + [-1] * (3 - p)), stream=f"s{seed}")
    nF = int(g.integers(40, 400))
    F = np.stack([g.choice([1, 2, 3, 4, 8, 16, 24, 32, 48, 64, 96, 128, 256, 512, 1024], nF) for _ in range(p)], 1)
    F = F.astype(np.int32)
    D = synth.log_uniform_ints(g, 1, hi[0], (1500, 1)).astype(np.int32)
    ref = oracle.sweep(spec, D, F)
    for second in (True, False):
        idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=second)
        check_sweep(idx, E, S if second else None, ref, spec, D, F, tag=f"rand{seed}")


@pytest.mark.parametrize("seed", range(6))
def test_gram_randomised_bases(seed):
    """Randomised stress of the Gram kernels: random variable counts, exponent lists (equal
    numerator / denominator lists of 16, 40 or 72 monomials take the fused warp-specialised path,
    others the generic one), row counts and metric values, against the oracle's plain sum of outer
    products at 1e-12 sqrt(G_ii G_jj)."""
    g = np.random.default_rng(9100 + seed)
    n = int(g.integers(1, 6))
    full = synth.basis_total_degree(n, 6 if n <= 2 else (4 if n <= 4 else 3))
    def pick(m):
        m = min(m, len(full))
        idx = np.sort(g.choice(len(full), m, replace=False))
        if 0 not in idx:
            idx[0] = 0
        return np.ascontiguousarray(full[np.unique(idx)])
    if g.random() < 0.5:
        num = pick(int(g.choice([16, 40, 72])))
        den = num.copy()
    else:
        num, den = pick(int(g.integers(3, 40))), pick(int(g.integers(2, 30)))
    K = int(g.integers(1, 5000))
    X = g.uniform(-50, 800, (K, n)).round()
    V = g.uniform(0.1, 100.0, (2, K))
    lo, hi = X.min(axis=0), X.max(axis=0)
    c, e = rp.xform_from_box(lo, hi)
    G = rp.gram(_cuda(X), _cuda(V), num, den, c, e).cpu().numpy()
    for i in range(2):
        Go = np.asarray(oracle.gram(X, V[i], num, den, c, e), dtype=np.float64)
        dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
        assert np.max(np.abs(G[i] - Go) / dg) <= 1e-12, (seed, n, len(num), len(den), K, i)


@pytest.mark.parametrize("seed", range(6))
def test_fit_randomised(seed):
    """Randomised fits: class-F truths with random data / program dimensions (d, p in 1..2), total
    degree 1..3, box, K (from 3 n_c to 20,000) and noise (0 or 1%); the GPU fit of all l metrics
    (symmetric-block Gram, equilibrated Cholesky + refinement) against the oracle's
    (long double Gauss with partial pivoting): same transform, coefficients within 1e-9."""
    g = np.random.default_rng(9100 + seed)
    d, p, deg = int(g.integers(1, 3)), int(g.integers(1, 3)), int(g.integers(1, 4))
    lo = [int(g.choice([1, 8, 32]))] * d + [1] * p
    hi = [int(g.choice([2048, 16384]))] * d + [int(g.choice([64, 1024]))] * p
    spec = synth.classf_program(f"fitrand{seed}", d, p, deg, lo, hi, synth.HW_GTX1080TI, R=32, Z0=0, Z1=0,
                                grid_map=tuple([0] * p + [-1] * (3 - p)), stream=f"f{seed}")
    n_c = 2 * len(spec.num_exp[0])
    K = int(g.integers(3 * n_c, 20_000))
    X = synth.box_random_design(g, lo, hi, K)
    sigma = float(g.choice([0.0, 0.01]))
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(spec, X)])
    if sigma:
        V = V * np.stack([synth.noise_multipliers(g, K, sigma) for _ in range(len(V))])
    num = den = spec.num_exp[0]
    coef, (c, e), _ = rp.fit(_cuda(X), _cuda(V), num, den)
    for i in range(len(V)):
        r = oracle.fit(X, V[i], num, den, nthreads=8)
        assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
        want = np.asarray(r["coef"], dtype=np.float64)
        err = np.max(np.abs(coef[i] - want)) / np.max(np.abs(want))
        assert err <= 1e-9, (seed, d, p, deg, K, sigma, i, err)


def test_sweep_tensor_core_fitted_program(monkeypatch):
    """k_sweep_tc on a FITTED program (noisy fitheavy samples, 70-term bases): its polynomials
    cancel heavily, the FP32 screen flags most pairs and the FP64 fallback decides; winners and E
    must still equal the default kernel's and meet the oracle's gates."""
    fc = synth.fitheavy(sigma=0.01, K=20_000)
    prog = fc.truths[0]
    X = _cuda(fc.X)
    V = (rp.eval_metrics(prog, X) * _cuda(fc.noise)).contiguous()
    coef, (c, e), _ = rp.fit(X, V, fc.num_exp, fc.den_exp)
    spec = copy.deepcopy(prog)
    spec.coef = [np.asarray(coef[i]) for i in range(3)]
    spec.xform_c, spec.xform_e = list(c), list(e)
    D = synth.large_D(3000)
    F = synth.F_large()
    idx0, E0, _ = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=False)
    monkeypatch.setenv("RP_SWEEP_KERNEL", "tc")
    idx1, E1, _ = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=False)
    assert torch.equal(idx0.cpu(), idx1.cpu())
    assert torch.equal(E0.cpu(), E1.cpu())
    sel = np.arange(0, 3000, 10)
    ref = oracle.sweep(spec, D[sel], F)
    check_sweep(np.asarray(idx1.cpu()).ravel()[sel], np.asarray(E1.cpu()).ravel()[sel], None, ref, spec, D[sel], F,
                tag="fitted")


def _fitted_program(K=20_000):
    fc = synth.fitheavy(sigma=0.01, K=K)
    prog = fc.truths[0]
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(prog, fc.X)]) * fc.noise
    spec = copy.deepcopy(prog)
    coefs = []
    for i in range(3):  # the oracle's fit (class-L style: both sides sweep the same program)
        r = oracle.fit(fc.X, V[i], fc.num_exp, fc.den_exp, nthreads=8)
        coefs.append(np.asarray(r["coef"], dtype=np.float64))
    spec.coef = coefs
    spec.xform_c, spec.xform_e = list(r["c"]), list(r["e"])
    return spec


@pytest.mark.parametrize("second", [False, True])
def test_sweep_refined_winners_fitted_program(second, monkeypatch):
    """The winner refinement (default on; reading R31) on a FITTED, ill-conditioned program
    (noisy fitheavy samples, kappa up to ~1e6): E within 1e-12 of the binary128 oracle's value at
    the chosen pair for every tuple, winners as the unrefined sweep's, the runner-up refined too
    (best <= second) and re-ranked on the exact key."""
    spec = _fitted_program()
    D = synth.large_D(3000)
    F = synth.F_large()
    monkeypatch.setenv("RP_SWEEP_REFINE", "0")
    idx0, E0, S0 = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=second)
    monkeypatch.delenv("RP_SWEEP_REFINE")
    idx1, E1, S1 = rp.eval_argmin(spec, _cuda(D), _cuda(F), second=second)
    i0, i1 = idx0.cpu().numpy(), idx1.cpu().numpy()
    e0, e1 = E0.cpu().numpy(), E1.cpu().numpy()
    sel = np.arange(0, 3000, 10)
    errs0, errs1 = [], []
    for t in sel:
        if i1[t] < 0:
            assert i0[t] < 0
            continue
        tq = oracle.eval_pair(spec, D[t], F[i1[t]], quad=True)
        assert tq["feasible"]
        Eq = float(tq["E"])
        errs1.append(abs(e1[t] - Eq) / Eq)
        if i0[t] == i1[t]:
            errs0.append(abs(e0[t] - Eq) / Eq)
    assert max(errs1) <= 1e-12, max(errs1)
    assert np.mean(i0 == i1) >= 0.999  # re-ranking moves only near-ties of the runner-up
    if second:
        s1 = S1.cpu().numpy()
        fin = np.isfinite(s1)
        assert np.all(e1[fin] <= s1[fin])
    ref = oracle.sweep(spec, D[sel], F)
    # the long double oracle is itself accurate to ~1e-12 only where kappa <= 1e3
    cov = (ref["kappa"] <= 1e3) & (ref["kappa2"] <= 1e3) & (ref["idx"] >= 0)
    sub = np.nonzero(cov)[0]
    check_sweep(i1[sel][sub], e1[sel][sub], None, subset(ref, sub), spec, D[sel][sub], F, tag="fitted-refined")
    print("refine: max rel E err vs binary128: unrefined %.2e refined %.2e; kappa<=1e3 covers %.1f%%"
          % (max(errs0), max(errs1), 100 * cov.mean()))


def test_refine_g1_template_three_metrics():
    """the refinement picks the E formula from the template, not from the number of
    polynomials: a RP_TEMPLATE_G1 program with 3 metrics gets E = p_0/q_0 refined (was the
    MWP-CWP estimate)."""
    case = synth.polybench_sweep(nD=500)
    spec = copy.deepcopy(case.programs[0])
    spec.template = "g1"
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    ref = oracle.sweep(spec, D, case.F)
    for second in (False, True):
        idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(case.F), second=second)
        check_sweep(idx, E, S, ref, spec, D, case.F, "g1x3")


def test_sweep_nonpositive_data_and_huge_blocks():
    """Reading R32: tuples with some D_k < 1 have no meaningful configuration, and
    configurations whose product P1 P2 P3 would wrap around in 64 bits are masked (T > T_max)
    instead of passing the warp rule as T = 0.  GPU sweep, decide and JIT against the oracle."""
    case = synth.polybench_sweep(nD=50)
    spec = case.programs[0]
    F = np.concatenate([case.F, np.array([[1 << 30, 1 << 30, 16], [2147483647, 2147483647, 2147483647],
                                          [0, 32, 1], [-32, -1, 1], [64, 1 << 28, 1 << 4]], dtype=np.int32)])
    D = np.concatenate([np.array([[0], [-1], [-2147483647], [1]], dtype=np.int32), case.D])
    ref = oracle.sweep(spec, D, F)
    assert ref["idx"][:3].tolist() == [-1, -1, -1]
    idx, E, S = rp.eval_argmin(spec, _cuda(D), _cuda(F))
    check_sweep(idx, E, S, ref, spec, D, F, "R32")
    plan = rp.Plan([spec], _cuda(F))
    assert plan.static_feasible() == int(np.sum([oracle.eval_pair(spec, np.array([16384], np.int32), P)["mask"]
                                                 not in (1, 2, 4) for P in F]))
    dec = plan.decide(D, prog=0, margin=0.0)
    assert np.array_equal(dec["idx"], ref["idx"])
    jit = rp.Jit(spec)
    ji, jE, _ = jit.eval(_cuda(D), _cuda(F))
    assert np.array_equal(ji.cpu().numpy().ravel(), ref["idx"])


def test_factored_tiles_match_dense_and_oracle():
    """The factored contraction (k_plan_groups: configurations sharing every P_k but one, one
    DMMA pair per polynomial and tile) against the dense one (RP_SWEEP_GROUPS=0) and the
    oracle: `large` truth program on a 20,000-tuple slice plus edge tuples (small D1 exercises
    the a3 exit inside groups), and a p = 3 program whose groups fall back to dense."""
    import os
    for name, spec, F, D in (
            ("large", synth.large_program(), synth.F_large(),
             np.concatenate([synth.random_D_edge_cases(2), synth.large_D(20_000)])),
            ("polybench", synth.polybench_sweep(nD=8).programs[0], synth.F_pow2_3d(),
             synth.polybench_sweep(nD=3000).D),
            # p = 3 at degree 2: every Horner variable's lists fit, so 3-D groups form
            ("p3deg2", synth.classf_program("p3deg2", 1, 3, 2, [8, 1, 1, 1], [16384, 1024, 1024, 64],
                                            synth.HW_GTX1080TI, R=32, Z0=0, Z1=0, grid_map=(0, 0, -1),
                                            stream="p3deg2"),
             synth.F_pow2_3d(), synth.polybench_sweep(nD=3000).D)):
        outs = []
        for groups in ("1", "0"):
            os.environ["RP_SWEEP_GROUPS"] = groups
            try:
                plan = rp.Plan([spec], _cuda(F))
            finally:
                os.environ.pop("RP_SWEEP_GROUPS", None)
            outs.append([t.cpu().numpy() for t in plan.eval(_cuda(D), second=True)])
        (i1, e1, s1), (i0, e0, s0) = outs
        assert np.array_equal(i1, i0), name
        fin = np.isfinite(e0)
        assert np.array_equal(fin, np.isfinite(e1)), name
        assert np.max(np.abs(e1[fin] - e0[fin]) / e0[fin], initial=0) <= 1e-12, name
        sel = np.arange(0, len(D), 7)
        ref = oracle.sweep(spec, D[sel], F)
        check_sweep(i1[0][sel], e1[0][sel], s1[0][sel], ref, spec, D[sel], F, name)


def test_sweep_beyond_sort_limit():
    """A plan with more than 8,192 statically feasible configurations keeps index order (no
    P1 P2 sort, no a3 early exit, no groups): parity with the oracle, and rp_plan_decide
    refuses it (its per-CTA candidate limit)."""
    hw = dict(synth.HW_GTX1080TI)
    hw.update(t_max=16384, w_max=1024, b_max=32, r_max=1 << 40, z_max=1 << 40)
    spec = synth.classf_program("bigF", 1, 3, 2, [8, 1, 1, 1], [4096, 64, 64, 64], hw, R=16, Z0=0, Z1=0,
                                grid_map=(0, 0, 0), stream="bigF")
    F = np.array([(a, b, c) for a in range(1, 65) for b in range(1, 65) for c in range(1, 65)
                  if (a * b * c) % 32 == 0], dtype=np.int32)
    plan = rp.Plan([spec], _cuda(F))
    assert plan.static_feasible() > 8192
    D = np.concatenate([synth.random_D_edge_cases(1),
                        synth.log_uniform_ints(np.random.default_rng(5), 1, 4096, (120, 1))]).astype(np.int32)
    idx, E, S = plan.eval(_cuda(D), second=True)
    ref = oracle.sweep(spec, D, F)
    check_sweep(idx[0], E[0], S[0], ref, spec, D, F, "bigF")
    with pytest.raises(rp.RPError):
        plan.decide(D[:2])


def test_gram_sum_ordered_bitwise():
    """rp_gram_sum_ordered (a13, deterministic form) equals the rank-ordered sum bit for bit."""
    g = np.random.default_rng(11)
    for n_parts in (1, 2, 3, 8):
        parts = g.standard_normal((n_parts, 3, 140, 140)) * 10.0 ** g.integers(-3, 8, (n_parts, 1, 1, 1))
        want = parts[0].copy()
        for p in parts[1:]:
            want = want + p
        got = rp.gram_sum_ordered(_cuda(parts)).cpu().numpy()
        assert got.tobytes() == want.tobytes(), n_parts


def _total_degree_exps(n, deg):
    out = []

    def rec(prefix, left):
        if len(prefix) == n:
            out.append(list(prefix))
            return
        for e in range(left + 1):
            rec(prefix + [e], left - e)
    rec([], deg)
    out.sort(key=lambda v: (sum(v), v))
    return np.array(out, dtype=np.int16)


@pytest.mark.parametrize("n,deg,diff_den", [(1, 3, False), (1, 7, True), (2, 2, False), (2, 4, True), (3, 3, False),
                                            (5, 2, True), (6, 1, False)])
def test_gram_moments_variable_counts(n, deg, diff_den):
    """The moment Gram (generic monomial step: every (n, D) other than the BASELINE ones) for 1 to 6
    variables, identical and differing numerator / denominator bases, 1 and 3 metrics, ragged K, on
    the TMA and plain-load paths, against the oracle's sum of outer products."""
    rng = np.random.default_rng(1000 + 10 * n + deg)
    num = _total_degree_exps(n, deg)
    den = _total_degree_exps(n, max(deg - 1, 0)) if diff_den else num
    for K in (37, 1000):
        X = rng.integers(1, 500, size=(K, n)).astype(np.float64)
        V = rng.uniform(0.5, 3.0, size=(3, K))
        c, e = rp.xform_from_box(X.min(axis=0), X.max(axis=0))
        G = rp.gram(_cuda(X), _cuda(V), num, den, c, e).cpu().numpy()
        for i in range(3):
            Go = np.asarray(oracle.gram(X, V[i], num, den, c, e), dtype=np.float64)
            dg = np.sqrt(np.outer(np.diag(Go), np.diag(Go))) + 1e-300
            assert np.max(np.abs(G[i] - Go) / dg) <= 1e-12, (n, deg, diff_den, K, i)
