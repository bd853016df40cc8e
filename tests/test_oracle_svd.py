"""Pins for the oracle's homogeneous SVD fit (NEXT row f1): "the method of singular value
decomposition" on the homogeneous system (draft PAPER.md:2595-2598).
Pinned by SPEC.md:331's hand-derived null space, exact recovery of in-basis truths
(PAPER.md:2227-2230), numpy.linalg.svd on small well-conditioned problems, and optimality of the
Rayleigh quotient ||A c|| / ||c|| against the beta_0 = 1 least-squares solution."""
import numpy as np

import oracle
import synth


def test_spec_null_space_example():
    """A = [[1, -1]] (one sample y = 1 of a constant model) -> v ~ (1, 1)/sqrt(2)."""
    r = oracle.fit_svd(np.array([[0.0]]), np.array([1.0]), [[0]], [[0]])
    assert [float(x) for x in r["coef"]] == [1.0, 1.0]
    assert float(r["sigma"][0]) == 0.0 and abs(float(r["sigma"][1]) - np.sqrt(2)) < 1e-18


def test_exact_recovery():
    for fc, i in ((synth.tiny_fit_box(), 0), (synth.polybench_fit_box(K=1500), 1), (synth.fitheavy(K=1500), 2)):
        V = np.asarray(oracle.program_metrics(fc.truths[0], fc.X)[i], dtype=np.float64)
        r = oracle.fit_svd(fc.X, V, fc.num_exp, fc.den_exp)
        want = fc.truths[0].coef[i]
        got = np.asarray(r["coef"], dtype=np.float64)
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12
        assert float(r["sigma"][0]) <= 1e-12 * float(r["sigma"][-1])


def _design(fc, V, c, e):
    return np.stack([oracle.design_row(fc.num_exp, fc.den_exp, c, e, x, v) for x, v in zip(fc.X, V)])


def test_matches_numpy_svd():
    fc = synth.tiny_fit_box(sigma=0.05)
    V = np.asarray(oracle.program_metrics(fc.truths[0], fc.X)[0], dtype=np.float64) * fc.noise[0]
    r = oracle.fit_svd(fc.X, V, fc.num_exp, fc.den_exp)
    A = np.asarray(_design(fc, V, r["c"], r["e"]), dtype=np.float64)
    U, s, Vt = np.linalg.svd(A)
    np.testing.assert_allclose(np.asarray(r["sigma"], dtype=float), s[::-1], rtol=1e-10)
    v = Vt[-1] / Vt[-1][len(fc.num_exp)]
    np.testing.assert_allclose(np.asarray(r["coef"], dtype=float), v, rtol=1e-8, atol=1e-10 * np.abs(v).max())


def test_rayleigh_quotient_optimal():
    fc = synth.polybench_fit_box(sigma=0.02, K=800)
    V = np.asarray(oracle.program_metrics(fc.truths[0], fc.X)[2], dtype=np.float64) * fc.noise[2]
    r = oracle.fit_svd(fc.X, V, fc.num_exp, fc.den_exp)
    ls = oracle.fit(fc.X, V, fc.num_exp, fc.den_exp)
    A = _design(fc, V, r["c"], r["e"])

    def rq(cf):
        cf = np.asarray(cf, dtype=np.longdouble)
        return float(np.linalg.norm(np.asarray(A @ cf, dtype=float)) / np.linalg.norm(np.asarray(cf, dtype=float)))

    assert rq(r["coef"]) <= rq(ls["coef"]) * (1 + 1e-12)
    assert abs(rq(r["coef"]) - float(r["sigma"][0])) <= 1e-9 * float(r["sigma"][-1])


def test_svd_rows_matches_numpy_and_row_stacking():
    """orc_svd_rows on an explicit matrix: numpy.linalg.svd's singular values and smallest right
    singular vector; zero rows and row order change nothing (A^T A is what matters)."""
    g = np.random.default_rng(7)
    A = g.standard_normal((40, 9))
    A[:, 3] = A[:, 0] - 2 * A[:, 5] + 0.5 * A[:, 8]  # a (near) null vector
    A += 1e-6 * g.standard_normal(A.shape)
    r = oracle.svd_rows(A, 0)  # beta_0 slot = column 0 (a large component of the null vector)
    U, s, Vt = np.linalg.svd(A)
    np.testing.assert_allclose(np.asarray(r["sigma"], dtype=float), s[::-1], rtol=1e-9)
    v = Vt[-1] / Vt[-1][0]
    np.testing.assert_allclose(np.asarray(r["coef"], dtype=float), v, rtol=1e-8, atol=1e-12)
    r2 = oracle.svd_rows(np.concatenate([A[20:], np.zeros((5, 9)), A[:20]]), 0)
    np.testing.assert_allclose(np.asarray(r2["coef"], dtype=float), np.asarray(r["coef"], dtype=float), rtol=1e-12,
                               atol=1e-16)


def test_fit_svd_equals_svd_of_design_rows():
    fc = synth.tiny_fit_box(sigma=0.05)
    V = np.asarray(oracle.program_metrics(fc.truths[0], fc.X)[1], dtype=np.float64) * fc.noise[1]
    r = oracle.fit_svd(fc.X, V, fc.num_exp, fc.den_exp)
    A = np.stack([oracle.design_row(fc.num_exp, fc.den_exp, r["c"], r["e"], x, v) for x, v in zip(fc.X, V)])
    r2 = oracle.svd_rows(A, len(fc.num_exp))
    assert np.array_equal(r["coef"], r2["coef"]) and np.array_equal(r["sigma"], r2["sigma"])
