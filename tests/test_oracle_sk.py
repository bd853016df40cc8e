"""Pins for the oracle's Sanathanan-Koerner refit (NEXT row f4, reading R29): one solve is the
plain fit; noise-free in-basis data stay exactly recovered at every iteration;
a constant denominator basis makes every weight 1 (plain least squares); V x 7 scales alpha only;
on noisy data the reweighted solves lower the value-space error sum (p/q - V)^2 it is meant to
approximate."""
import numpy as np

import oracle
import synth


def _V(truth, i, X):
    return np.asarray(oracle.program_metrics(truth, X)[i], dtype=np.float64)


def test_one_iteration_is_plain_fit():
    fc = synth.tiny_fit_box(sigma=0.01)
    V = _V(fc.truths[0], 0, fc.X) * fc.noise[0]
    a = oracle.fit(fc.X, V, fc.num_exp, fc.den_exp)
    b = oracle.fit_sk(fc.X, V, fc.num_exp, fc.den_exp, iters=1)
    assert np.array_equal(a["coef"], b["coef"])


def test_exact_recovery_every_iteration():
    fc = synth.polybench_fit_box()
    V = _V(fc.truths[0], 1, fc.X)
    want = fc.truths[0].coef[1]
    for it in (2, 4):
        r = oracle.fit_sk(fc.X, V, fc.num_exp, fc.den_exp, iters=it)
        got = np.asarray(r["coef"], dtype=np.float64)
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


def test_constant_denominator_is_plain_least_squares():
    g = synth.rng("tests", "sk-poly")
    X = g.uniform(-3, 5, size=(300, 2))
    V = 1 + X[:, 0] - 0.5 * X[:, 1] ** 2 + 0.02 * g.standard_normal(300)
    num = synth.basis_total_degree(2, 2)
    den = np.zeros((1, 2), dtype=np.int16)
    a = oracle.fit(X, V, num, den)
    b = oracle.fit_sk(X, V, num, den, iters=3)
    np.testing.assert_allclose(np.asarray(b["coef"], dtype=float), np.asarray(a["coef"], dtype=float), rtol=1e-14, atol=1e-15)


def test_scaling_invariance():
    fc = synth.tiny_fit_box(sigma=0.02)
    V = _V(fc.truths[0], 2, fc.X) * fc.noise[2]
    m = len(fc.num_exp)
    a = np.asarray(oracle.fit_sk(fc.X, V, fc.num_exp, fc.den_exp, iters=3)["coef"], dtype=float)
    b = np.asarray(oracle.fit_sk(fc.X, 7 * V, fc.num_exp, fc.den_exp, iters=3)["coef"], dtype=float)
    np.testing.assert_allclose(b[:m], 7 * a[:m], rtol=1e-12, atol=1e-12 * np.abs(a).max())
    np.testing.assert_allclose(b[m:], a[m:], rtol=1e-12, atol=1e-13)


def test_reduces_value_error_and_converges():
    fc = synth.polybench_fit_box(sigma=0.05)
    g = synth.rng("tests", "sk-noise")
    truth = fc.truths[0]
    V = _V(truth, 0, fc.X) * (1 + 0.05 * g.standard_normal(len(fc.X)))

    def value_err(r):
        f = np.asarray(oracle.eval_ratfunc(fc.num_exp, fc.den_exp, np.asarray(r["coef"], dtype=float),
                                           r["c"], r["e"], fc.X)[0], dtype=float)
        return float(np.sum((f - V) ** 2))

    e1 = value_err(oracle.fit_sk(fc.X, V, fc.num_exp, fc.den_exp, iters=1))
    # the linearised fit weighs rows by q(x); near-poles of the plain fit make its value error
    # large, and every reweighted solve brings it down by orders of magnitude (SK need not be
    # monotone from one iteration to the next, so no convergence claim)
    for it in (2, 3, 4, 5):
        assert value_err(oracle.fit_sk(fc.X, V, fc.num_exp, fc.den_exp, iters=it)) < 0.01 * e1
