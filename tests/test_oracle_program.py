"""Pins for the oracle's per-pair program: transform (a10), g_i evaluation (a4), masks (a1, a3),
grid (a6) and the MWP-CWP estimate E (a7, DESIGN.md Appendix A).

Pinned by: hand-derived worked examples (tests/golden/mwpcwp_worked.json; each derivation written
out there), SPEC.md worked examples (tests/golden/spec_worked.json), closed forms of the
transform, and invariance of E when numerator and denominator are scaled together (the north
star's named invariant; bit-exact for powers of two).
"""
import copy
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from helpers import const_program, frac, golden, scaled_program


def _worked():
    return golden("mwpcwp_worked.json")


@pytest.mark.parametrize("ex", _worked()["examples"], ids=lambda e: e["name"])
def test_mwpcwp_worked_examples(ex):
    W = _worked()
    hw = dict(W["hw"])
    hw.update(ex.get("hw_override", {}))
    pr = dict(W["program"])
    pr.update(ex.get("program_override", {}))
    spec = const_program(hw, ex["g"], d=pr["d"], p=pr["p"], R=pr["R"], Z0=pr["Z0"], Z1=pr["Z1"],
                         grid_map=pr["grid_map"])
    tr = oracle.eval_pair(spec, ex["D"], ex["P"])
    if "mask" in ex:
        assert not tr["feasible"]
        assert tr["mask"] == ex["mask"]
        if "branch" in ex:
            assert tr["branch"] == ex["branch"]
        return
    assert tr["feasible"] == 1
    assert tr["B_active"] == ex["B_active"]
    assert tr["branch"] == ex["branch"]
    assert tr["W_active"] == ex["W_active"]
    assert tr["blocks"] == ex["blocks"]
    assert tr["sm_active"] == ex["sm_active"]
    assert tr["mwp_case"] == ex["case"]
    exact = frac(ex["E"])
    got = Fraction(float(tr["E"]))  # long double -> nearest double, compared to the exact value
    assert abs(got - exact) <= exact * Fraction(1, 10**15), (float(tr["E"]), float(exact))


def test_ratfunc_spec_examples():
    for ex in golden("spec_worked.json")["ratfunc"]:
        v, _ = oracle.eval_ratfunc(ex["num"], ex["den"], ex["coef"], [0.0], [0], np.array([ex["x"]], dtype=float))
        exact = frac(ex["value"])
        assert abs(Fraction(float(v[0])) - exact) <= abs(exact) * Fraction(1, 10**15)


def test_design_row_spec_examples():
    for ex in golden("spec_worked.json")["design_row"]:
        row = oracle.design_row(ex["num"], ex["den"], [0.0], [0], ex["x"], ex["v"])
        assert [float(r) for r in row] == [float(r) for r in ex["row"]]


@pytest.mark.parametrize("lo,hi,c,e", [(8, 16384, 8196.0, 13), (1, 1024, 512.5, 9), (1, 64, 32.5, 5),
                                       (5, 5, 5.0, 0), (0, 4, 2.0, 1), (32, 256, 144.0, 7), (8, 1536, 772.0, 10)])
def test_transform_closed_form(lo, hi, c, e):
    cc, ee = oracle.xform_from_box([lo], [hi])
    assert cc[0] == c and ee[0] == e
    # u = (x-c) 2^-e maps the box into [-1,1] and e is the least such exponent (h > 2^(e-1))
    h = max((hi - lo) / 2, 1)
    assert 2.0 ** e >= h and (e == 0 or 2.0 ** (e - 1) < h)


def test_masks_and_grid_rule():
    hw = synth.HW_GTX1080TI
    spec = const_program(hw, [100, 50, 1], R=32)
    # footnote rule P1 P2 <= D1^2, non-strict (reading R6)
    assert oracle.eval_pair(spec, [32], [32, 32])["feasible"] == 1  # 1024 <= 1024
    assert oracle.eval_pair(spec, [31], [32, 32])["mask"] == 3
    # grid rule gx = ceil(N/bx), gy = ceil(N/by)
    tr = oracle.eval_pair(spec, [100], [32, 8])
    assert tr["blocks"] == 4 * 13  # SPEC.md:406 example (4, 13, 1)
    spec3 = const_program(hw, [100, 50, 1], d=1, p=3, grid_map=(0, 0, -1))
    tr = oracle.eval_pair(spec3, [100], [8, 4, 2])
    assert tr["blocks"] == 13 * 25 and tr["T"] == 64


def test_E_invariant_to_scaling_p_and_q_together():
    """ĝ = p/q is unchanged when p and q are multiplied by the same c, so E
    is too: bit-exact for c = 2^k, within 1e-15 otherwise."""
    case = synth.tiny_sweep()
    spec = case.programs[0]
    for factors, exact in [((2.0, 0.25, 1024.0), True), ((3.0, 7.0, 0.1), False)]:
        s2 = scaled_program(spec, factors)
        for D in case.D[::3]:
            for P in case.F[::5]:
                a = oracle.eval_pair(spec, D, P)
                b = oracle.eval_pair(s2, D, P)
                assert a["feasible"] == b["feasible"] and a["mwp_case"] == b["mwp_case"]
                if not a["feasible"]:
                    continue
                if exact:
                    assert a["E"] == b["E"]
                else:
                    assert abs(a["E"] - b["E"]) <= 1e-15 * abs(a["E"])


def test_classf_program_is_well_conditioned():
    """Class-F programs keep q in [0.5, 1.5], p >= 1 on the box, so kappa is small (SURVEY
    §8(d)); this is what makes float64 parity at 1e-12 meaningful (reading R19)."""
    case = synth.tiny_sweep()
    res = oracle.sweep(case.programs[0], case.D, case.F)
    assert np.all(res["kappa"][res["idx"] >= 0] < 20)
