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
