"""Pins for the oracle's occupancy program (a5) -- Fig. occupancysimpleflowchart
 and Eq. (1).

Pinned by: SPEC.md's hand-derived worked examples; the paper's structural counts (n = 8 inputs,
5 terminating nodes: PAPER.md:1973-1977); the closed form floor(min(B_max, 32 W_max / T,
R_max/(R T), Z_max/Z)) that the four diamonds encode ("this limit is minimal");
monotonicity in R and Z.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from helpers import golden, frac


def test_spec_worked_examples():
    hw = synth.HW_SPEC_OCC
    for ex in golden("spec_worked.json")["occupancy"]:
        B, branch = oracle.active_blocks(hw, ex["r"], ex["z"], ex["t"])
        W = oracle.active_warps(hw, ex["r"], ex["z"], ex["t"])
        assert B == ex["B_active"], ex
        assert W == ex["W_active"], ex
        assert Fraction(W, hw["w_max"]) == frac(ex["occupancy"]), ex


def _closed_form(hw, R, Z, T):
    lims = [Fraction(hw["b_max"]), Fraction(32 * hw["w_max"], T)]
    if R > 0:
        lims.append(Fraction(hw["r_max"], R * T))
    if Z > 0:
        lims.append(Fraction(hw["z_max"], Z))
    m = min(lims)
    return m.numerator // m.denominator


@pytest.mark.parametrize("hw", [synth.HW_SPEC_OCC, synth.HW_GTX1080TI, synth.HW_B200])
def test_flowchart_equals_min_formula(hw):
    g = synth.rng("tests", "occupancy-fuzz")
    n = 100_000 if hw is synth.HW_SPEC_OCC else 20_000
    T = g.integers(1, hw["t_max"] + 1, size=n)
    R = g.integers(0, 256, size=n)
    Z = np.where(g.random(n) < 0.3, 0, g.integers(0, 2 * hw["z_max"], size=n))
    branches = set()
    for t, r, z in zip(T.tolist(), R.tolist(), Z.tolist()):
        B, br = oracle.active_blocks(hw, r, z, t)
        branches.add(br)
        assert B == _closed_form(hw, r, z, t), (t, r, z, B, br)
    # 4 decision diamonds + "Failure to Launch": at most 5 terminating nodes;
    # branch 5 is unreachable for non-negative inputs (reading R7)
    assert branches <= {1, 2, 3, 4}
    assert branches == {1, 2, 3, 4}


def test_structure_counts():
    """n = 8 inputs: R_max, Z_max, T_max, B_max, W_max, R, Z, T; 5 terminal
    nodes.  The oracle's flowchart exposes exactly the branch ids 1..5."""
    hw = dict(synth.HW_SPEC_OCC)
    inputs = {"r_max", "z_max", "t_max", "b_max", "w_max"}
    assert inputs <= set(hw)
    # crafted inputs reaching each of the four Yes-terminals
    cases = {1: (32, 16, 0), 2: (256, 32, 0), 3: (128, 256, 0), 4: (32, 1, 12289)}
    for br, (t, r, z) in cases.items():
        assert oracle.active_blocks(hw, r, z, t)[1] == br


def test_monotone_in_R_and_Z():
    hw = synth.HW_GTX1080TI
    for T in (32, 64, 96, 128, 256, 512, 1024):
        prevR = None
        for R in range(0, 256, 3):
            B = oracle.active_blocks(hw, R, 0, T)[0]
            assert prevR is None or B <= prevR
            prevR = B
        prevZ = None
        for Z in range(0, 30000, 97):
            B = oracle.active_blocks(hw, 32, Z, T)[0]
            assert prevZ is None or B <= prevZ
            prevZ = B


def test_eq1_active_warps():
    hw = synth.HW_GTX1080TI
    for T in (32, 64, 128, 1024):
        for R in (16, 32, 64, 128):
            B = oracle.active_blocks(hw, R, 0, T)[0]
            assert oracle.active_warps(hw, R, 0, T) == min((B * T) // 32, hw["w_max"])
