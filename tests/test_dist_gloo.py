"""The N > 1 sharding / collective logic of paper_1911_02373_b200.dist on CPU with gloo,
world_size 2 (and 3: a rank with an empty shard).  The per-shard compute is the oracle, so this
checks exactly the host-side partitioning, the min/max and Gram reductions and the winner gather:
the sharded sweep must equal the unsharded one bit for bit, the sharded fit must equal the
unsharded fit within rounding of the Gram summation order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


class OracleOps:
    def minmax(self, X):
        return oracle.minmax(np.asarray(X))

    def xform(self, lo, hi):
        return oracle.xform_from_box(lo, hi)

    def gram(self, X, V, num, den, c, e):
        X = np.asarray(X)
        V = np.atleast_2d(np.asarray(V))
        nc = len(num) + len(den)
        if X.shape[0] == 0:
            return np.zeros((V.shape[0], nc, nc))
        return np.stack([np.asarray(oracle.gram(X, V[i], num, den, c, e), dtype=np.float64) for i in range(V.shape[0])])

    def solve(self, G, num, den):
        G = np.asarray(G.cpu() if hasattr(G, "cpu") else G)
        out = [oracle.solve(G[i].astype(np.longdouble), len(num)) for i in range(G.shape[0])]
        return np.stack([np.asarray(r["coef"], dtype=np.float64) for r in out]), out

    # device-resident forms (here: CPU tensors through the oracle)
    def minmax_dev(self, X):
        lo, hi = oracle.minmax(np.asarray(X))
        return torch.from_numpy(np.stack([lo, hi], 1))

    def xform_dev(self, lohi):
        lohi = lohi.numpy()
        c, e = oracle.xform_from_box(lohi[:, 0], lohi[:, 1])
        return torch.from_numpy(np.stack([c, e.astype(np.float64)], 1))

    def gram_dev(self, X, V, num, den, xf):
        xf = xf.numpy()
        return torch.from_numpy(self.gram(X, V, num, den, xf[:, 0], xf[:, 1].astype(np.int32)))

    def solve_dev(self, G, num, den):
        coef, out = self.solve(G, num, den)
        return torch.from_numpy(coef), out

    def gram_sum(self, parts):
        """Rank-ordered sum of the gathered partials (what rp_gram_sum_ordered computes)."""
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        return acc

    def tsqr(self, X, V, num, den, c, e):
        """Any B with B^T B = A^T A serves: the shard's design rows themselves."""
        X = np.asarray(X)
        V = np.atleast_2d(np.asarray(V))
        nc = len(num) + len(den)
        return np.stack([np.asarray([oracle.design_row(num, den, c, e, x, v) for x, v in zip(X, V[i])],
                                    dtype=np.float64).reshape(len(X), nc) for i in range(V.shape[0])])

    def svd_rows(self, rows, num, den):
        rows = np.asarray(rows.cpu() if hasattr(rows, "cpu") else rows)
        out = [oracle.svd_rows(rows[i], len(num)) for i in range(rows.shape[0])]
        return (np.stack([np.asarray(r["coef"], dtype=np.float64) for r in out]),
                np.stack([np.asarray(r["sigma"], dtype=np.float64) for r in out]), out)

    def sweep(self, progs, D, F):
        res = [oracle.sweep(p, np.asarray(D), F) for p in progs]
        return (torch.from_numpy(np.stack([r["idx"] for r in res])),
                torch.from_numpy(np.stack([r["best"] for r in res])))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, deterministic):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_02373_b200_dist_shim import dist_mod
        ops = OracleOps()
        # sweep: polybench programs over a D batch (ragged split)
        case = synth.polybench_sweep(nD=203)
        D = np.concatenate([synth.random_D_edge_cases(1), case.D])
        idx, E = dist_mod.sharded_sweep(case.programs[:2], D, case.F, ops)
        for g, spec in enumerate(case.programs[:2]):
            ref = oracle.sweep(spec, D, case.F)
            assert np.array_equal(idx[g].numpy(), ref["idx"])
            assert np.array_equal(E[g].numpy(), ref["best"])
        # fit: tiny box design, 3 metrics, rows split across ranks
        fc = synth.tiny_fit_box(sigma=0.01)
        V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)]) * fc.noise
        lo, hi = dist_mod.shard_bounds(len(fc.X), world, rank)
        coef, (c, e), _ = dist_mod.sharded_fit(fc.X[lo:hi], V[:, lo:hi], fc.num_exp, fc.den_exp, ops, n_vars=3,
                                               deterministic=deterministic)
        for i in range(3):
            r = oracle.fit(fc.X, V[i], fc.num_exp, fc.den_exp)
            assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
            want = np.asarray(r["coef"], dtype=np.float64)
            assert np.max(np.abs(coef[i] - want)) / np.max(np.abs(want)) < 1e-12
        # every rank holds the same coefficients
        t = torch.from_numpy(np.ascontiguousarray(coef))
        t0 = t.clone()
        dist.broadcast(t0, 0)
        assert torch.equal(t, t0)
        # the device-resident form of the same fit
        coef_d, xf_d, _ = dist_mod.sharded_fit_dev(fc.X[lo:hi], V[:, lo:hi], fc.num_exp, fc.den_exp, ops, n_vars=3)
        assert np.array_equal(xf_d.numpy()[:, 0], c) and np.array_equal(xf_d.numpy()[:, 1], e)
        assert np.max(np.abs(coef_d.numpy() - coef)) <= 1e-12 * np.max(np.abs(coef))
        # f1: SVD of the stacked shard factors == SVD of all rows (zero-padded shards included)
        coef, sigma, (c, e), _ = dist_mod.sharded_fit_svd(fc.X[lo:hi], V[:, lo:hi], fc.num_exp, fc.den_exp, ops,
                                                          n_vars=3)
        for i in range(3):
            r = oracle.fit_svd(fc.X, V[i], fc.num_exp, fc.den_exp)
            assert np.array_equal(r["c"], c) and np.array_equal(r["e"], e)
            want = np.asarray(r["coef"], dtype=np.float64)
            assert np.max(np.abs(coef[i] - want)) / np.max(np.abs(want)) < 1e-12
            sref = np.asarray(r["sigma"], dtype=np.float64)
            assert np.max(np.abs(sigma[i] - sref)) <= 1e-13 * sref[-1]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,deterministic", [(2, False), (2, True), (3, True)])
def test_sharded_sweep_and_fit_gloo(world, deterministic, tmp_path, monkeypatch):
    # make the dist module importable in spawned workers without importing the CUDA binding
    shim = tmp_path / "paper_1911_02373_b200_dist_shim.py"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    shim.write_text(
        "import importlib.util, os\n"
        f"spec = importlib.util.spec_from_file_location('rp_dist', os.path.join({root!r}, 'paper_1911_02373_b200', 'dist.py'))\n"
        "dist_mod = importlib.util.module_from_spec(spec)\n"
        "spec.loader.exec_module(dist_mod)\n")
    monkeypatch.setenv("PYTHONPATH", os.pathsep.join([str(tmp_path), root, os.path.join(root, "tests"),
                                                      os.environ.get("PYTHONPATH", "")]))
    import sys
    sys.path.insert(0, str(tmp_path))
    mp.spawn(_worker, args=(world, _free_port(), deterministic), nprocs=world, join=True)


def test_shard_bounds():
    from importlib.util import module_from_spec, spec_from_file_location
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = spec_from_file_location("rp_dist", os.path.join(root, "paper_1911_02373_b200", "dist.py"))
    m = module_from_spec(spec)
    spec.loader.exec_module(m)
    for n in (0, 1, 7, 8, 1000001):
        for w in (1, 2, 3, 8):
            b = [m.shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
