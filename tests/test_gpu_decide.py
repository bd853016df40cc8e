"""Parity of the runtime decision service (NEXT row f2, rp_plan_decide) with the oracle's
orc_decide, and the runtime history."""
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
from helpers import golden, ratfunc_program  # noqa: E402

DEV = torch.device("cuda:0")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_spec_decision_example_on_gpu():
    ex, grid_ex = golden("spec_worked.json")["decision"]
    F = synth.F_pow2_2d()
    spec = ratfunc_program(synth.HW_GTX1080TI, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2, R=16)
    plan = rp.Plan([spec], _cuda(F))
    r = plan.decide(np.array([[ex["N"]]], dtype=np.int32), margin=1e-9)[0]
    assert tuple(F[r["idx"]]) == tuple(ex["block"]) and tuple(r["launch"]) == tuple(ex["launch"])
    assert r["E"] == 4.0 and r["from_history"] == 0
    plan1 = rp.Plan([spec], _cuda(np.array([grid_ex["block"]], dtype=np.int32)))
    r = plan1.decide(np.array([[grid_ex["N"]]], dtype=np.int32))[0]
    assert tuple(r["launch"][:3]) == tuple(grid_ex["grid"])


@pytest.mark.parametrize("which", ["tiny", "polybench", "multikernel"])
def test_decide_parity(which):
    case = {"tiny": synth.tiny_sweep, "polybench": lambda: synth.polybench_sweep(nD=150),
            "multikernel": lambda: synth.multikernel_sweep(nD=60)}[which]()
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    plan = rp.Plan(case.programs, _cuda(case.F))
    checked = 0
    for g, spec in enumerate(case.programs[:4]):
        ref_sweep = oracle.sweep(spec, D, case.F)
        for margin in (0.0, 0.05, 1e300):
            got = plan.decide(D, prog=g, margin=margin)
            for i, d in enumerate(D):
                ref = oracle.decide(spec, d, case.F, margin=margin)
                if ref["idx"] < 0:
                    assert got[i]["idx"] == -1 and np.isinf(got[i]["E"]) and tuple(got[i]["launch"]) == (0,) * 6
                    continue
                if margin == 0.0:
                    gap = (ref_sweep["second"][i] - ref_sweep["best"][i]) / ref_sweep["best"][i]
                    if not gap > 1e-9:
                        continue  # near tie (reading R20)
                elif not ref["boundary"] > 1e-10:
                    continue  # a candidate within rounding of the margin boundary (reading R28)
                assert got[i]["idx"] == ref["idx"], (which, g, margin, i)
                assert tuple(got[i]["launch"]) == ref["launch"]
                assert abs(got[i]["E"] - ref["E"]) <= 1e-12 * ref["E"]
                checked += 1
    assert checked > 0.9 * len(D) * min(4, len(case.programs)) * 3 * 0.6


def test_decide_matches_sweep_at_margin_zero():
    case = synth.large_sweep(nD=1)
    D = synth.large_D(3000)
    plan = rp.Plan(case.programs, _cuda(case.F))
    idx, E, S = plan.eval(_cuda(D))
    dec = rp.decisions_from_device(plan.decide(_cuda(D)))
    idx, E, S = idx[0].cpu().numpy(), E[0].cpu().numpy(), S[0].cpu().numpy()
    strict = (S - E) / E > 1e-9
    assert np.array_equal(dec["idx"][strict], idx[strict])
    assert np.max(np.abs(dec["E"][strict] - E[strict]) / E[strict]) <= 1e-13


def test_runtime_history():
    case = synth.polybench_sweep(nD=64)
    D = np.concatenate([case.D, case.D[:16]])  # 16 repeated tuples in the batch
    plan = rp.Plan(case.programs, _cuda(case.F))
    fresh = plan.decide(D, prog=2, margin=0.02)
    plan.enable_history(prog=2, log2_capacity=10, margin=0.02)
    first = plan.decide(D, prog=2, margin=0.02)
    st = plan.history_stats()
    assert st["hits"] + st["misses"] == len(D) and st["entries"] == len(np.unique(case.D))
    again = plan.decide(D, prog=2, margin=0.02)
    assert np.all(again["from_history"] == 1)
    for f in ("idx", "E", "launch"):
        assert np.array_equal(again[f], first[f]) and np.array_equal(first[f], fresh[f])
    assert plan.history_stats()["hits"] == st["hits"] + len(D)
    with pytest.raises(rp.RPError):
        plan.decide(D, prog=1, margin=0.02)  # the history belongs to program 2
    plan.clear_history()
    assert plan.history_stats() == {"hits": 0, "misses": 0, "entries": 0}
    assert np.all(plan.decide(D[:5], prog=2, margin=0.02)["from_history"] == 0)


def test_decision_service_graph():
    case = synth.polybench_sweep(nD=40)
    plan = rp.Plan(case.programs[:1], _cuda(case.F))
    ref = plan.decide(case.D, prog=0, margin=0.01)
    for memo in (0, 1 << 10):
        svc = rp.DecisionService(plan, prog=0, margin=0.01, history_log2=12, host_memo=memo)
        for i in range(len(case.D)):
            r = svc(case.D[i])
            assert r["idx"] == ref[i]["idx"] and r["E"] == ref[i]["E"]
            assert tuple(r["launch"]) == tuple(ref[i]["launch"])
        r = svc(case.D[3])
        assert r["idx"] == ref[3]["idx"]
        if memo == 0:
            assert r["from_history"] == 1  # served by the device history
        else:
            assert len(svc.memo) == len(np.unique(case.D))  # served by the host memo


@pytest.mark.parametrize("history", [False, True])
def test_decider_matches_batched_decide(history):
    """rp_decider (mapped memory + captured graph) returns, tuple by tuple, the decisions of the
    batched rp_plan_decide; with the history on, repeats come from the table."""
    case = synth.polybench_sweep(nD=64)
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    plan = rp.Plan(case.programs, _cuda(case.F))
    want = plan.decide(D, prog=1, margin=0.02)
    if history:
        plan.enable_history(1, 10, 0.02)
    dc = rp.Decider(plan, prog=1, margin=0.02)
    for rep in range(2 if history else 1):
        for i, d in enumerate(D):
            r = dc(d)
            assert r["idx"] == want[i]["idx"] and r["E"] == want[i]["E"], (rep, i)
            assert tuple(r["launch"]) == tuple(want[i]["launch"]), (rep, i)
            if history and rep == 1 and want[i]["idx"] >= 0:
                assert r["from_history"] == 1
    dc.close()
    with pytest.raises(rp.RPError):  # a history for another program/margin is refused
        plan.enable_history(0, 8, 0.0)
        rp.Decider(plan, prog=1, margin=0.02)


def test_history_reenable_keeps_live_deciders_valid():
    """re-enabling the history must not free the table a live decider's graph holds.
    Same capacity: cleared in place, the decider keeps answering; another capacity: refused."""
    case = synth.polybench_sweep(nD=16)
    plan = rp.Plan(case.programs[:1], _cuda(case.F))
    want = plan.decide(case.D, prog=0, margin=0.0)
    svc1 = rp.DecisionService(plan, prog=0, margin=0.0, history_log2=10, host_memo=0)
    svc2 = rp.DecisionService(plan, prog=0, margin=0.0, history_log2=10, host_memo=0)
    plan.enable_history(0, 10, 0.0)  # same capacity: in place
    for i in range(len(case.D)):
        assert svc1(case.D[i])["idx"] == want[i]["idx"]
        assert svc2(case.D[i])["idx"] == want[i]["idx"]
    with pytest.raises(rp.RPError):  # reallocation while deciders live
        plan.enable_history(0, 11, 0.0)
    with pytest.raises(rp.RPError):  # another margin while deciders live
        plan.enable_history(0, 10, 0.5)
    svc1.decider.close()
    svc2.decider.close()
    plan.enable_history(0, 11, 0.0)  # no decider left: allowed


def test_decision_service_memo_invalidated_by_update():
    """Plan.update (a refit) invalidates the service's host memo, so the next call
    decides with the new program instead of serving the pre-refit decision."""
    case = synth.polybench_sweep(nD=8)
    progs = case.programs
    plan = rp.Plan(progs[:1], _cuda(case.F))
    svc = rp.DecisionService(plan, prog=0, margin=0.0, history_log2=None, host_memo=1 << 10)
    d = case.D[0]
    before = svc(d)
    # refit: program 0's coefficients replaced by program 3's (same bases and transform box);
    # the resources (R, Z) stay program 0's
    refit = copy.deepcopy(progs[0])
    refit.coef = [np.asarray(c, dtype=np.float64) for c in progs[3].coef]
    plan.update(torch.from_numpy(np.stack(refit.coef)).to(DEV))
    ref = rp.Plan([refit], _cuda(case.F)).decide(case.D[:1], prog=0, margin=0.0)
    after = svc(d)
    assert after["idx"] == ref[0]["idx"] and after["E"] == ref[0]["E"]
    assert len(svc.memo) == 1 and svc.memo[tuple(int(v) for v in d)]["E"] == ref[0]["E"]
    assert before["E"] != after["E"]


def test_history_save_load_across_plans():
    """rp_plan_history_save / _load: a saved runtime history serves the next run's decisions as
    hits and is refused by a plan whose program or F differs."""
    case = synth.polybench_sweep(nD=200)
    D = case.D
    plan = rp.Plan(case.programs, _cuda(case.F))
    plan.enable_history(prog=1, log2_capacity=12, margin=0.01)
    first = plan.decide(D, prog=1, margin=0.01)
    blob = plan.save_history()
    assert blob == plan.save_history()  # deterministic (slot order)
    n_entries = plan.history_stats()["entries"]
    assert n_entries == len(np.unique(D, axis=0))

    plan2 = rp.Plan(case.programs, _cuda(case.F))
    plan2.enable_history(prog=1, log2_capacity=12, margin=0.01)
    plan2.load_history(blob)
    assert plan2.history_stats()["entries"] == n_entries
    again = plan2.decide(D, prog=1, margin=0.01)
    assert np.all(again["from_history"] == 1)
    for f in ("idx", "E", "launch"):
        assert np.array_equal(again[f], first[f])
    # another capacity: the entries re-hash into the new table
    plan3 = rp.Plan(case.programs, _cuda(case.F))
    plan3.enable_history(prog=1, log2_capacity=9, margin=0.01)
    plan3.load_history(blob)
    assert np.all(plan3.decide(D, prog=1, margin=0.01)["from_history"] == 1)
    # refused: other margin, other program index, other coefficients, other F, refit, tampering
    plan4 = rp.Plan(case.programs, _cuda(case.F))
    plan4.enable_history(prog=1, log2_capacity=12, margin=0.02)
    with pytest.raises(rp.RPError):
        plan4.load_history(blob)
    other = copy.deepcopy(case.programs)
    other[1].coef[0] = other[1].coef[0] * (1 + 2.0 ** -40)
    plan5 = rp.Plan(other, _cuda(case.F))
    plan5.enable_history(prog=1, log2_capacity=12, margin=0.01)
    with pytest.raises(rp.RPError):
        plan5.load_history(blob)
    plan6 = rp.Plan(case.programs, _cuda(case.F[:-1]))
    plan6.enable_history(prog=1, log2_capacity=12, margin=0.01)
    with pytest.raises(rp.RPError):
        plan6.load_history(blob)
    coef = _cuda(np.stack([np.asarray(c, dtype=np.float64) for c in case.programs[1].coef]))
    plan2.update(coef, prog=1)  # same values, but a refit clears the history
    assert plan2.history_stats()["entries"] == 0
    bad = bytearray(blob)
    bad[40] ^= 1
    with pytest.raises(rp.RPError):
        plan3.load_history(bytes(bad))
