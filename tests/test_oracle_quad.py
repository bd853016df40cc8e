"""Pins for the oracle's condition number kappa and for its binary128 instance.

kappa (orc_trace.kappa, the sweep's kappa / kappa2): max over the 2l polynomials of
sum |c m| / |sum c m| at the pair (reading R19; SURVEY 8(c) #25 gates on it).  Pinned by
hand-computed cases with exact small-integer terms.

orc_eval_pair_q / orc_sweep_q: the same transcription (oracle/rp_oracle_pair.inc) in IEEE
binary128.  Pinned by the exact-rational worked examples of tests/golden/mwpcwp_worked.json (to
the double the trace is read back in), by a cancellation that long double cannot resolve and
binary128 must (2^70 + N - 2^65 bx at bx = 32 is exactly N), and by agreement with the long
double instance on well-conditioned class-F sweeps.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from helpers import const_program, frac, golden, ratfunc_program

HW = synth.HW_GTX1080TI


def _exact(x) -> Fraction:
    return Fraction(*np.longdouble(x).as_integer_ratio())


def test_kappa_hand_computed():
    # p = N^2 - 4 bx by + 1 at (N, bx, by) = (64, 32, 32): terms 4096, -4096, 1 -> p = 1,
    # sum |terms| = 8193; q = 1 -> kappa = 8193 (every term exact in long double)
    spec = ratfunc_program(HW, [[0, 0, 0], [2, 0, 0], [0, 1, 1]], [[0, 0, 0]], [1.0, 1.0, -4.0, 1.0], d=1, p=2)
    tr = oracle.eval_pair(spec, [64], [32, 32])
    assert tr["feasible"] and _exact(tr["E"]) == 1
    assert _exact(tr["kappa"]) == 8193
    # p = N (kappa 1); q = 3 + bx - 2 by at (64, 16): terms 3, 64, -32 -> q = 35, sum 99 ->
    # kappa = max(1, 99/35)
    spec = ratfunc_program(HW, [[1, 0, 0]], [[0, 0, 0], [0, 1, 0], [0, 0, 1]], [1.0, 3.0, 1.0, -2.0], d=1, p=2)
    tr = oracle.eval_pair(spec, [64], [64, 16])
    assert tr["feasible"]
    assert abs(_exact(tr["kappa"]) - Fraction(99, 35)) <= Fraction(99, 35) * Fraction(1, 10**15)
    assert abs(_exact(tr["E"]) - Fraction(64, 35)) <= Fraction(64, 35) * Fraction(1, 10**15)
    # the sweep reports the same kappa at its winner and runner-up
    F = np.array([[64, 16], [32, 32]], dtype=np.int32)
    r = oracle.sweep(spec, np.array([[64]], dtype=np.int32), F)
    tr2 = oracle.eval_pair(spec, [64], [32, 32])  # q = 3 + 32 - 64 = -29 -> E < 0, masked
    assert not tr2["feasible"]
    assert r["idx"][0] == 0 and r["idx2"][0] == -1
    assert abs(Fraction(r["kappa"][0]) - Fraction(99, 35)) <= Fraction(99, 35) * Fraction(1, 10**15)


def test_sweep_runner_up_index():
    """idx2 is the index of the second-smallest (E, index) key: on an exact tie the next index."""
    spec = ratfunc_program(HW, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2)  # E = N^2 / (bx by)
    F = synth.F_pow2_2d()
    r = oracle.sweep(spec, np.array([[64]], dtype=np.int32), F)
    T = F[:, 0] * F[:, 1]
    ties = np.nonzero(T == 1024)[0]  # all T = 1024 configurations tie
    assert r["idx"][0] == ties[0] and r["idx2"][0] == ties[1] and r["best"][0] == r["second"][0] == 4.0


@pytest.mark.parametrize("ex", golden("mwpcwp_worked.json")["examples"], ids=lambda e: e["name"])
def test_quad_worked_examples(ex):
    W = golden("mwpcwp_worked.json")
    hw = dict(W["hw"])
    hw.update(ex.get("hw_override", {}))
    pr = dict(W["program"])
    pr.update(ex.get("program_override", {}))
    spec = const_program(hw, ex["g"], d=pr["d"], p=pr["p"], R=pr["R"], Z0=pr["Z0"], Z1=pr["Z1"],
                         grid_map=pr["grid_map"])
    tq = oracle.eval_pair(spec, ex["D"], ex["P"], quad=True)
    tl = oracle.eval_pair(spec, ex["D"], ex["P"])
    for k in ("feasible", "mask", "branch", "B_active", "W_active", "blocks", "sm_active", "mwp_case"):
        assert tq[k] == tl[k], k
    if "mask" in ex:
        return
    exact = frac(ex["E"])
    # binary128 to ~1e-30; ctypes hands trace values back as doubles (relative 2^-53)
    assert abs(_exact(tq["E"]) - exact) <= exact * Fraction(12, 10**17)


def test_quad_resolves_what_long_double_cannot():
    # p = 2^70 + N - 2^65 bx, q = 1, at N = 63, bx = 32: exactly 63.  In basis order the long
    # double sum 2^70 + 63 rounds to 2^70 (ulp 128), so p = 0 and E = 0 is masked (R17).
    spec = ratfunc_program(HW, [[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 0]],
                           [2.0 ** 70, 1.0, -(2.0 ** 65), 1.0], d=1, p=2)
    tl = oracle.eval_pair(spec, [63], [32, 1])
    tq = oracle.eval_pair(spec, [63], [32, 1], quad=True)
    assert not tl["feasible"] and tl["mask"] == 5
    assert tq["feasible"] and _exact(tq["E"]) == 63
    # kappa = (2^70 + 63 + 2^70) / 63
    want = Fraction(2 ** 71 + 63, 63)
    assert abs(_exact(tq["kappa"]) - want) <= want * Fraction(12, 10**17)


def test_quad_sweep_agrees_with_long_double_on_class_f():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    rl = oracle.sweep(spec, case.D, case.F)
    rq = oracle.sweep(spec, case.D, case.F, quad=True)
    assert np.array_equal(rl["idx"], rq["idx"]) and np.array_equal(rl["idx2"], rq["idx2"])
    feas = rl["idx"] >= 0
    assert np.max(np.abs(rl["best"][feas] - rq["best"][feas]) / rq["best"][feas]) <= 1e-16
    assert rl["counters"] == rq["counters"]
