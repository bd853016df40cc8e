"""FitSweepPipeline (pipeline.py): host-fed steps overlapped on copy streams give, step by step,
exactly the winners of the same librp calls made one after another (different inputs per step,
more steps than in-flight slots, so a slot mix-up or a missing event dependency shows)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_02373_b200 as rp  # noqa: E402
from paper_1911_02373_b200.pipeline import FitSweepPipeline  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_pipeline_matches_sequential_calls(depth):
    K, nD, steps = 20_000, 5_000, 5
    fc = synth.fitheavy(sigma=0.01, K=K * steps)
    prog = fc.truths[0]
    V_all = (rp.eval_metrics(prog, torch.from_numpy(fc.X).to(DEV)) * torch.from_numpy(fc.noise).to(DEV)).cpu()
    D_all = synth.large_D(nD * steps)
    F = synth.F_large()
    Xs = [torch.from_numpy(fc.X[i * K:(i + 1) * K]).pin_memory() for i in range(steps)]
    Vs = [V_all[:, i * K:(i + 1) * K].contiguous().pin_memory() for i in range(steps)]
    Ds = [torch.from_numpy(D_all[i * nD:(i + 1) * nD]).pin_memory() for i in range(steps)]
    outs = [(torch.empty((1, nD), dtype=torch.int32).pin_memory(),
             torch.empty((1, nD), dtype=torch.float64).pin_memory()) for _ in range(steps)]
    pipe = FitSweepPipeline(prog, F, fc.num_exp, fc.den_exp, K, 4, 3, nD, 2, device=DEV, depth=depth)
    done = [pipe.submit(Xs[i], Vs[i], Ds[i], *outs[i]) for i in range(steps)]
    for ev in done:
        ev.synchronize()
    pipe.close()
    plan = rp.Plan([prog], torch.from_numpy(F).to(DEV))
    for i in range(steps):
        coef, xf, _ = rp.fit_dev(Xs[i].to(DEV), Vs[i].to(DEV), fc.num_exp, fc.den_exp)
        plan.update(coef, xf)
        idx, E, _ = plan.eval(Ds[i].to(DEV), second=False)
        assert torch.equal(outs[i][0], idx.cpu()), i
        assert torch.equal(outs[i][1], E.cpu()), i
    plan.close()


@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("pinned", [True, False])
def test_c_abi_step_pipeline_matches_sequential_calls(depth, pinned):
    """rp_pipeline (the C ABI's host-fed pipeline, rp_pipeline.cu): every step's winners equal the
    same librp calls made one by one; pinned and pageable host buffers."""
    from paper_1911_02373_b200.pipeline import StepPipeline
    K, nD, steps = 20_000, 5_000, 5
    fc = synth.fitheavy(sigma=0.01, K=K * steps)
    prog = fc.truths[0]
    V_all = (rp.eval_metrics(prog, torch.from_numpy(fc.X).to(DEV)) * torch.from_numpy(fc.noise).to(DEV)).cpu()
    D_all = synth.large_D(nD * steps)
    F = synth.F_large()
    pin = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    Xs = [pin(torch.from_numpy(fc.X[i * K:(i + 1) * K].copy())) for i in range(steps)]
    Vs = [pin(V_all[:, i * K:(i + 1) * K].contiguous()) for i in range(steps)]
    Ds = [pin(torch.from_numpy(D_all[i * nD:(i + 1) * nD].copy())) for i in range(steps)]
    outs = [(pin(torch.empty(nD, dtype=torch.int32)), pin(torch.empty(nD, dtype=torch.float64)))
            for _ in range(steps)]
    pipe = StepPipeline(prog, torch.from_numpy(F).to(DEV), fc.num_exp, fc.den_exp, K, 3, nD, 2, depth=depth)
    for i in range(steps):
        pipe.submit(Xs[i], Vs[i], Ds[i], *outs[i])
    pipe.sync()
    pipe.close()
    plan = rp.Plan([prog], torch.from_numpy(F).to(DEV))
    for i in range(steps):
        coef, xf, _ = rp.fit_dev(Xs[i].to(DEV), Vs[i].to(DEV), fc.num_exp, fc.den_exp)
        plan.update(coef, xf)
        idx, E, _ = plan.eval(Ds[i].to(DEV), second=False)
        assert torch.equal(outs[i][0], idx.cpu().reshape(-1)), i
        assert torch.equal(outs[i][1], E.cpu().reshape(-1)), i
    plan.close()


def test_c_abi_step_pipeline_rejects_bad_shapes():
    from paper_1911_02373_b200.pipeline import StepPipeline
    fc = synth.fitheavy(K=100)
    case = synth.polybench_sweep(nD=10)
    F = torch.from_numpy(synth.F_large()).to(DEV)
    with pytest.raises(rp.RPError):  # d = 3 but the program has d = 2
        StepPipeline(fc.truths[0], F, fc.num_exp, fc.den_exp, 100, 3, 10, 3)
    with pytest.raises(rp.RPError):  # a multi-program plan
        from paper_1911_02373_b200 import _check, _lib
        import ctypes as C
        plan = rp.Plan(case.programs, torch.from_numpy(case.F).to(DEV))
        b = rp.Basis(fc.num_exp, fc.den_exp)
        h = C.c_void_p()
        _check(_lib.rp_pipeline_create(plan.handle, 0, C.byref(b.c), 3, 100, 1, 10, 2, C.byref(h)))
