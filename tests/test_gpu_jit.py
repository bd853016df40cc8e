"""Parity of the f3 path -- the rational program generated as CUDA source (rp_codegen), compiled
by NVRTC for sm_100a (rp_jit_create) and searched exhaustively (rp_jit_eval_argmin) -- with the
CPU oracle on the same seeded programs and inputs, under the sweep gates of the north star:
idx bit-exact where the oracle's margin exceeds 1e-9, E within 1e-12 relative, near ties inside
the oracle's epsilon-tie set (reading R20); and agreement with the data-driven sweep."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_02373_b200 as rp  # noqa: E402
from test_gpu_parity import check_sweep  # noqa: E402

DEV = torch.device("cuda:0")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_jit_tiny():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    jit = rp.Jit(spec)
    idx, E, S = jit.eval(_cuda(D), _cuda(case.F))
    ref = oracle.sweep(spec, D, case.F)
    check_sweep(idx, E, S, ref, spec, D, case.F, "jit-tiny")
    jit.close()


@pytest.mark.parametrize("g", [0, 1, 2, 3])
def test_jit_polybench(g):
    case = synth.polybench_sweep(nD=2000)
    spec = case.programs[g]
    jit = rp.Jit(spec)
    idx, E, S = jit.eval(_cuda(case.D), _cuda(case.F))
    ref = oracle.sweep(spec, case.D, case.F)
    check_sweep(idx, E, S, ref, spec, case.D, case.F, f"jit-polybench-{g}")


def test_jit_multikernel_resources():
    """Register- and shared-memory-limited occupancy branches and B_active = 0 masks."""
    case = synth.multikernel_sweep(nD=500)
    for g in (0, 5, 11, 19):
        spec = case.programs[g]
        idx, E, S = rp.Jit(spec).eval(_cuda(case.D), _cuda(case.F))
        ref = oracle.sweep(spec, case.D, case.F)
        check_sweep(idx, E, S, ref, spec, case.D, case.F, f"jit-multikernel-{g}")


def test_jit_large_sampled_and_vs_plan():
    """`large` program (n = 4, degree 4, 1,024 configurations incl. T > 1024 and T mod 32 != 0)
    on the oracle's subsample; the full batch agrees with the data-driven sweep."""
    case = synth.large_sweep(nD=200_000)
    spec = case.programs[0]
    sub = synth.large_subsample_index(len(case.D), every=100, edge=50)
    jit = rp.Jit(spec)
    idx, E, S = jit.eval(_cuda(case.D), _cuda(case.F))
    ref = oracle.sweep(spec, case.D[sub], case.F)
    check_sweep(idx.cpu()[sub], E.cpu()[sub], S.cpu()[sub], ref, spec, case.D[sub], case.F, "jit-large")
    pi, pE, _ = rp.eval_argmin(spec, _cuda(case.D), _cuda(case.F))
    pi, pE, idx, E = (x.cpu().numpy() for x in (pi, pE, idx, E))
    ok = pi >= 0
    assert np.array_equal(pi < 0, idx < 0)
    assert np.max(np.abs(pE[ok] - E[ok]) / E[ok]) <= 2e-12
    assert np.mean(pi == idx) > 0.999


def test_jit_g1_all_tie_and_host_pointers():
    """E = N^2 / (bx by) at N = 64 ties every T = 1024 configuration: the lowest
    index wins; host inputs and outputs go through the library's staging."""
    from helpers import ratfunc_program
    F = synth.F_pow2_2d()
    spec = ratfunc_program(synth.HW_GTX1080TI, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2, R=16)
    D = np.array([[64], [8], [1000]], dtype=np.int32)
    ref = oracle.sweep(spec, D, F)
    idx, E, S = rp.Jit(spec).eval(D, F)
    assert np.array_equal(idx, ref["idx"])
    assert np.array_equal(E, ref["best"])


def test_codegen_deterministic():
    spec = synth.polybench_sweep(nD=10).programs[2]
    assert rp.codegen(spec) == rp.codegen(spec)
