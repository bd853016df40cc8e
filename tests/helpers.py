"""Small shared helpers for the tests (no method arithmetic here)."""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def frac(s) -> Fraction:
    return Fraction(str(s))


def const_program(hw: dict, g, d: int = 1, p: int = 2, R: int = 16, Z0: int = 0, Z1: int = 0,
                  grid_map=(0, 0, -1), template: str = "mwpcwp") -> synth.ProgramSpec:
    """Program whose metrics are the constants g_i (numerator and denominator basis {1},
    beta_0 = 1) with the identity transform (c = 0, e = 0)."""
    n = d + p
    zero = np.zeros((1, n), dtype=np.int16)
    coef = [np.array([float(gi), 1.0]) for gi in g]
    return synth.ProgramSpec(d=d, p=p, num_exp=[zero] * len(g), den_exp=[zero] * len(g), coef=coef,
                             hw=dict(hw), R=R, Z0=Z0, Z1=Z1, grid_map=tuple(grid_map), template=template,
                             xform_c=[0.0] * n, xform_e=[0] * n)


def ratfunc_program(hw: dict, num_exp, den_exp, coef, d: int, p: int, R: int = 16, Z0: int = 0,
                    Z1: int = 0, grid_map=(0, 0, -1), template: str = "g1") -> synth.ProgramSpec:
    """One-metric program E := g_1 = p/q with the identity transform."""
    n = d + p
    return synth.ProgramSpec(d=d, p=p, num_exp=[np.asarray(num_exp, dtype=np.int16)],
                             den_exp=[np.asarray(den_exp, dtype=np.int16)], coef=[np.asarray(coef, dtype=np.float64)],
                             hw=dict(hw), R=R, Z0=Z0, Z1=Z1, grid_map=tuple(grid_map), template=template,
                             xform_c=[0.0] * n, xform_e=[0] * n)


def scaled_program(spec: synth.ProgramSpec, factors) -> synth.ProgramSpec:
    """Same program with numerator AND denominator of metric i multiplied by factors[i]."""
    import copy
    s = copy.deepcopy(spec)
    s.coef = [np.asarray(c) * f for c, f in zip(spec.coef, factors)]
    return s


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
