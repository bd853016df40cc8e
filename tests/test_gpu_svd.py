"""Parity of the f1 SVD path (rp_fit_svd / rp_tsqr_accumulate / rp_svd_rows, through the C ABI)
with the CPU oracle's one-sided Jacobi SVD (oracle.fit_svd, long double) on the same seeded inputs.

Gates: coefficients within 1e-9 relative (inf-norm after beta_0 = 1, the north star's fit
tolerance); singular values within 1e-12 * sigma_max (the TSQR + fp64 Jacobi is backward
stable: errors ~ n_c eps ||A||); at full size (K = 10^6, where the O(K n_c^2 sweeps) oracle cannot
run) exact recovery of the class-F truths and R^T R = the oracle's Gram.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_02373_b200 as rp  # noqa: E402

DEV = torch.device("cuda:0")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _metrics(fc, X=None):
    X = fc.X if X is None else X
    V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], X)])
    if fc.noise is not None:
        V = V * fc.noise[:, :len(X)]
    return V


def _coef_err(got, want):
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got) - want)) / np.max(np.abs(want)))


def _check_vs_oracle(fc, X, V, metrics, tag):
    coef, sigma, (c, e), infos = rp.fit_svd(_cuda(X), _cuda(V), fc.num_exp, fc.den_exp)
    for i in metrics:
        r = oracle.fit_svd(X, V[i], fc.num_exp, fc.den_exp)
        assert r["status"] == 0
        np.testing.assert_array_equal(c, r["c"])
        np.testing.assert_array_equal(e, r["e"])
        err = _coef_err(coef[i], r["coef"])
        assert err <= 1e-9, (tag, i, err)
        s_ref = np.asarray(r["sigma"], dtype=np.float64)
        assert np.max(np.abs(sigma[i] - s_ref)) <= 1e-12 * s_ref[-1], (tag, i)
        assert np.all(np.diff(sigma[i]) >= 0)
        assert infos[i]["status"] == 0
        assert abs(infos[i]["min_pivot"] - s_ref[0]) <= 1e-12 * s_ref[-1]
    return coef, sigma


def test_svd_tiny_box_noisy():
    fc = synth.tiny_fit_box(sigma=0.01)
    V = _metrics(fc)
    _check_vs_oracle(fc, fc.X, V, range(3), "tiny")


def test_svd_tiny_exact_recovery():
    fc = synth.tiny_fit_box()
    V = _metrics(fc)
    coef, sigma, _, infos = rp.fit_svd(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    for i in range(3):
        assert _coef_err(coef[i], fc.truths[0].coef[i]) <= 1e-10
        assert sigma[i][0] <= 1e-12 * sigma[i][-1]


def test_svd_polybench_box_noisy():
    fc = synth.polybench_fit_box(sigma=0.01, K=2000)
    V = _metrics(fc)
    _check_vs_oracle(fc, fc.X, V, range(3), "polybench")


def test_svd_fitheavy_subsample_noisy():
    """fitheavy basis (n_c = 140: TSQR chunk tails, several leaves and a merge tree)."""
    fc = synth.fitheavy(sigma=0.01, K=3000)
    V = _metrics(fc)
    _check_vs_oracle(fc, fc.X, V, [0], "fitheavy-3000")


@pytest.mark.parametrize("K", [97, 96 * 3 + 1, 1000, 96 * 11])
def test_svd_ragged_K(K):
    """Chunk tails (K mod 96 != 0), one leaf, odd leaf counts with pass-through tree nodes."""
    fc = synth.polybench_fit_box(sigma=0.02, K=K)
    V = _metrics(fc)
    _check_vs_oracle(fc, fc.X, V, [1], f"K={K}")


def test_svd_fewer_rows_than_columns():
    """K = 12 < n_c = 20: rank K and an 8-dimensional null space (the paper's rank deficiency,
    PAPER.md:2609-2611).  Any null vector is a least-squares solution: the chosen one solves
    A v = 0 to rounding, or -- when its beta_0 vanishes -- the call reports DEGENERATE."""
    fc = synth.tiny_fit_box(sigma=0.01)
    X, V = fc.X[:12], _metrics(fc)[:, :12]
    coef, sigma, (c, e), infos = rp.fit_svd(_cuda(X), _cuda(V), fc.num_exp, fc.den_exp, raise_on_degenerate=False)
    for i in range(3):
        assert infos[i]["rank"] == 12
        assert np.all(sigma[i][:8] <= 1e-13 * sigma[i][-1])
        if infos[i]["status"] == 3:
            assert np.all(np.isnan(coef[i]))
            continue
        assert infos[i]["status"] == 0
        A = np.stack([np.asarray(oracle.design_row(fc.num_exp, fc.den_exp, c, e, x, v), dtype=np.float64)
                      for x, v in zip(X, V[i])])
        assert np.linalg.norm(A @ coef[i]) <= 1e-12 * np.linalg.norm(A) * np.linalg.norm(coef[i])


def test_svd_host_pointers_and_determinism():
    fc = synth.polybench_fit_box(sigma=0.01, K=2000)
    V = _metrics(fc)
    a = rp.fit_svd(fc.X, V, fc.num_exp, fc.den_exp)
    b = rp.fit_svd(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    c = rp.fit_svd(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(b[0], c[0])
    assert np.array_equal(a[1], b[1])


def test_tsqr_split_form_and_stacked_rows():
    """R^T R equals the oracle's Gram; the SVD of the stacked factors of two shards equals the
    one-call fit (the K-sharded path of dist.sharded_fit_svd)."""
    fc = synth.polybench_fit_box(sigma=0.01, K=2000)
    V = _metrics(fc)
    c, e = oracle.xform_from_box(*oracle.minmax(fc.X))
    R = rp.tsqr(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp, c, e).cpu().numpy()
    for i in range(3):
        G = np.asarray(oracle.gram(fc.X, V[i], fc.num_exp, fc.den_exp, c, e), dtype=np.float64)
        assert np.allclose(np.tril(R[i], -1), 0.0)
        d = np.sqrt(np.outer(np.diag(G), np.diag(G)))
        assert np.max(np.abs(R[i].T @ R[i] - G) / d) <= 1e-12
    h = len(fc.X) // 2
    R0 = rp.tsqr(_cuda(fc.X[:h]), _cuda(V[:, :h]), fc.num_exp, fc.den_exp, c, e)
    R1 = rp.tsqr(_cuda(fc.X[h:]), _cuda(V[:, h:]), fc.num_exp, fc.den_exp, c, e)
    coef, sigma, _ = rp.svd_rows(torch.cat([R0, R1], dim=1), fc.num_exp, fc.den_exp)
    ref, sref, _, _ = rp.fit_svd(_cuda(fc.X), _cuda(V), fc.num_exp, fc.den_exp)
    for i in range(3):
        assert _coef_err(coef[i], ref[i]) <= 1e-10
        assert np.max(np.abs(sigma[i] - sref[i])) <= 1e-12 * sref[i][-1]
    # empty shard: R = 0
    Z = rp.tsqr(_cuda(fc.X[:0]), _cuda(V[:, :0]), fc.num_exp, fc.den_exp, c, e)
    assert float(Z.abs().max()) == 0.0


def test_svd_fitheavy_full_size_exact_recovery():
    """K = 10^6 noise-free rows of the class-F truths: the smallest right singular vector is the
    truth -- a property that holds at any size."""
    fc = synth.fitheavy()
    X = _cuda(fc.X)
    V = rp.eval_metrics(fc.truths[0], X)
    coef, sigma, _, infos = rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    for i in range(3):
        assert _coef_err(coef[i], fc.truths[0].coef[i]) <= 1e-9, i
        assert sigma[i][0] <= 1e-8 * sigma[i][1]
        assert infos[i]["rank"] == 139


@pytest.mark.parametrize("r_path", ["dd", "tsqr"])
def test_svd_both_r_paths_vs_oracle(r_path, monkeypatch):
    """The SVD's R from the double-double Gram (default for K >= 4 n_c, reading R34) and from the
    Householder TSQR (RP_SVD_R=tsqr), each against the oracle's one-sided Jacobi SVD of A on the
    same polybench sample (K = 2,000 >= 4 n_c = 280), at the file's gates."""
    if r_path == "tsqr":
        monkeypatch.setenv("RP_SVD_R", "tsqr")
    fc = synth.polybench_fit_box(sigma=0.01)
    V = _metrics(fc)
    _check_vs_oracle(fc, fc.X, V, range(len(V)), r_path)


def test_svd_r_paths_agree_full_size():
    """At K = 10^6 (fitheavy, 1% noise) the two R paths give the same singular values (within
    1e-12 sigma_max) and coefficients (within 1e-9)."""
    import os
    fc = synth.fitheavy(sigma=0.01)
    X = _cuda(fc.X)
    V = (rp.eval_metrics(fc.truths[0], X) * _cuda(fc.noise)).contiguous()
    c_dd, s_dd, _, _ = rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    os.environ["RP_SVD_R"] = "tsqr"
    try:
        c_ts, s_ts, _, _ = rp.fit_svd(X, V, fc.num_exp, fc.den_exp)
    finally:
        del os.environ["RP_SVD_R"]
    for i in range(3):
        s1, s2 = np.asarray(s_dd[i]), np.asarray(s_ts[i])
        assert np.max(np.abs(s1 - s2)) <= 1e-12 * s2[-1], i
        assert _coef_err(c_dd[i], c_ts[i]) <= 1e-9, i
