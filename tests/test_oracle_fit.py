"""Pins for the oracle's least-squares fit (a10-a14): PAPER.md:2558-2615 (rational function
estimation by linear least squares), step 2 PAPER.md:2222-2235.

Pinned by: SPEC.md's worked fit ((2x+1)/(x+1) -> 21/11 at x = 10) and its closed-form
coefficients in the centred variable; exact recovery of known full-degree truths from noise-free
samples ("if the values of V_i were known exactly ... g_i could be determined exactly",
PAPER.md:2227-2230); the polynomial special case against numpy.linalg.lstsq; invariances
(V scaling, row permutation); degenerate systems.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from helpers import frac, golden

LD = np.longdouble


def _V(truth, i, X, noise=None):
    v = np.asarray(oracle.program_metrics(truth, X)[i], dtype=np.float64)
    return v if noise is None else v * noise


def test_spec_fit_example():
    ex = golden("spec_worked.json")["fit"][0]
    X = np.array(ex["x"], dtype=float).reshape(-1, 1)
    V = np.array([(2 * x + 1) / (x + 1) for x in ex["x"]], dtype=float)  # SPEC.md:321 samples
    basis = np.array(ex["basis"], dtype=np.int16)
    r = oracle.fit(X, V, basis, basis)
    assert r["status"] == 0
    # transform of the sample box [0,4]: c = 2, e = 1  ->  x = 2 + 2u; (2x+1)/(x+1) =
    # (5 + 4u)/(3 + 2u) = (5/3 + 4/3 u)/(1 + 2/3 u) with beta_0 = 1 (closed form)
    assert r["c"][0] == 2.0 and r["e"][0] == 1
    expect = [Fraction(5, 3), Fraction(4, 3), Fraction(1), Fraction(2, 3)]
    for got, want in zip(r["coef"], expect):
        assert abs(float(got) - float(want)) <= 1e-15 * float(abs(want) + 1)
    val, _ = oracle.eval_ratfunc(basis, basis, np.asarray(r["coef"], dtype=np.float64), r["c"], r["e"],
                                 np.array([[ex["eval_at"]]], dtype=float))
    assert abs(float(val[0]) - float(frac(ex["value"]))) <= 1e-14


@pytest.mark.parametrize("which", ["tiny", "polybench", "fitheavy"])
def test_exact_recovery_classf(which):
    """Noise-free V from a known in-basis truth gives back the truth's coefficients."""
    if which == "tiny":
        case = synth.tiny_fit_box()
        tol = 1e-13
    elif which == "polybench":
        case = synth.polybench_fit_box()
        tol = 1e-12
    else:
        case = synth.fitheavy(K=20_000)
        tol = 1e-11
    truth = case.truths[0]
    for i in range(truth.n_metrics):
        V = _V(truth, i, case.X)
        r = oracle.fit(case.X, V, case.num_exp, case.den_exp, nthreads=8)
        assert r["status"] == 0
        # the sample contains both box corners, so the fit's transform is the truth's
        c, e = oracle.program_xform(truth)
        assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
        want = truth.coef[i]
        err = np.max(np.abs(np.asarray(r["coef"], dtype=np.float64) - want)) / np.max(np.abs(want))
        assert err < tol, (which, i, err)
        scale = float(np.sum(V.astype(LD) ** 2))
        assert float(r["resid2"]) <= 1e-16 * scale  # cancellation floor of c^T G c in long double


def test_polynomial_special_case_matches_lstsq():
    """Denominator basis {1}: the fit is ordinary polynomial least squares (numpy lstsq)."""
    g = synth.rng("tests", "poly-lstsq")
    X = g.uniform(-3, 5, size=(400, 2))
    V = 1 + X[:, 0] - 2 * X[:, 1] ** 2 + 0.3 * X[:, 0] * X[:, 1] + 0.01 * g.standard_normal(400)
    num = synth.basis_total_degree(2, 2)
    den = np.zeros((1, 2), dtype=np.int16)
    r = oracle.fit(X, V, num, den)
    c, e = r["c"], r["e"]
    U = (X - c) / (2.0 ** e)
    M = np.stack([np.prod(U ** ex, axis=1) for ex in num], axis=1)
    ref = np.linalg.lstsq(M, V, rcond=None)[0]
    got = np.asarray(r["coef"][: len(num)], dtype=np.float64)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-12)
    assert r["coef"][len(num)] == 1


def test_scaling_and_permutation_invariance():
    case = synth.tiny_fit_box(sigma=0.01)
    truth = case.truths[0]
    V = _V(truth, 1, case.X, case.noise[1])
    r1 = oracle.fit(case.X, V, case.num_exp, case.den_exp)
    r7 = oracle.fit(case.X, 7 * V, case.num_exp, case.den_exp)
    m = len(case.num_exp)
    a1 = np.asarray(r1["coef"], dtype=np.float64)
    a7 = np.asarray(r7["coef"], dtype=np.float64)
    np.testing.assert_allclose(a7[:m], 7 * a1[:m], rtol=1e-13, atol=1e-13 * np.abs(a1).max())
    np.testing.assert_allclose(a7[m:], a1[m:], rtol=1e-13, atol=1e-14)
    perm = synth.rng("tests", "perm").permutation(len(V))
    rp = oracle.fit(case.X[perm], V[perm], case.num_exp, case.den_exp)
    np.testing.assert_allclose(np.asarray(rp["coef"], dtype=np.float64), a1, rtol=1e-14, atol=1e-14 * np.abs(a1).max())


def test_gram_is_sum_of_outer_products():
    """G equals the brute-force sum of a_r a_r^T over the rows, is symmetric and PSD."""
    case = synth.tiny_fit_box()
    V = _V(case.truths[0], 0, case.X)
    c, e = oracle.xform_from_box(*oracle.minmax(case.X))
    G = oracle.gram(case.X, V, case.num_exp, case.den_exp, c, e, nthreads=3)
    A = np.stack([oracle.design_row(case.num_exp, case.den_exp, c, e, x, v) for x, v in zip(case.X, V)])
    Gb = A.T @ A
    assert np.max(np.abs(G - Gb)) <= 1e-16 * np.max(np.abs(Gb))
    assert np.array_equal(G, G.T)
    w = np.linalg.eigvalsh(np.asarray(G, dtype=np.float64))
    assert w.min() > -1e-9 * w.max()


def test_degenerate_system():
    """Rank deficiency: identical rows cannot determine 4 unknowns."""
    X = np.ones((10, 1))
    V = np.full(10, 3.0)
    b = np.array([[0], [1]], dtype=np.int16)
    r = oracle.fit(X, V, b, b)
    assert r["status"] == 3
