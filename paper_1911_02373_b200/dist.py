"""Rank sharding of the hot path over the GPUs of one node.

* Sweep (a1-a9): the D batch is split into contiguous shards, each rank sweeps its shard with
  the replicated program and F, and the per-D winners (idx int32, E float64) are gathered with
  ``all_gather_into_tensor`` (NCCL over NVLink).  D rows are independent, so the gathered result
  is bit-identical to the 1-GPU result.
* Fit (a10-a14): the K rows are split into contiguous shards.  The transform needs the global
  box: per-variable (-lo, hi) is all-reduced with MAX first.  Each rank accumulates the partial
  Gram of its rows on device, the partials are combined (``all_reduce`` SUM, or -- with
  ``deterministic=True`` -- ``all_gather`` followed by a rank-ordered sum, bit-reproducible),
  and every rank solves the same small system.

The per-shard compute is injected (``Ops``): on GPUs it is librp; the CPU ``gloo`` tests inject
the oracle to exercise exactly this sharding / collective logic.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous ceil-split [lo, hi) of n items; trailing ranks may get fewer (or zero)."""
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


class LibOps:
    """Per-shard compute through librp (device tensors on the rank's GPU)."""

    def __init__(self):
        import paper_1911_02373_b200 as rp
        self.rp = rp

    def minmax(self, X):
        return self.rp.minmax(X)

    def xform(self, lo, hi):
        return self.rp.xform_from_box(lo, hi)

    def gram(self, X, V, num, den, c, e):
        return self.rp.gram(X, V, num, den, c, e)

    def solve(self, G, num, den):
        return self.rp.solve_normal(G, num, den)

    def minmax_dev(self, X):
        return self.rp.minmax_dev(X)

    def xform_dev(self, lohi):
        return self.rp.xform_dev(lohi)

    def gram_dev(self, X, V, num, den, xf):
        return self.rp.gram_dev(X, V, num, den, xf)

    def solve_dev(self, G, num, den):
        return self.rp.solve_dev(G, num, den)

    def gram_sum(self, parts):
        return self.rp.gram_sum_ordered(parts)

    def tsqr(self, X, V, num, den, c, e):
        return self.rp.tsqr(X, V, num, den, c, e)

    def svd_rows(self, rows, num, den):
        return self.rp.svd_rows(rows, num, den)

    def sweep(self, plan_or_progs, D, F=None):
        if isinstance(plan_or_progs, self.rp.Plan):
            return plan_or_progs.eval(D, second=False)[:2]
        return self.rp.eval_argmin_batched(plan_or_progs, D, F, second=False)[:2]


def _comm_device(group=None):
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def sharded_fit(X_local, V_local, num, den, ops, n_vars: int, group=None, deterministic: bool = False):
    """Fit n_v metrics whose K rows are split across the ranks of `group`.  X_local [K_r][n],
    V_local [n_v][K_r] (K_r may be 0).  Returns (coef [n_v][n_c], (c, e), infos), identical on
    every rank."""
    dev = _comm_device(group)
    K_r = X_local.shape[0]
    if K_r > 0:
        lo, hi = ops.minmax(X_local)
    else:
        lo, hi = np.full(n_vars, np.inf), np.full(n_vars, -np.inf)
    box = torch.tensor(np.concatenate([-np.asarray(lo), np.asarray(hi)]), dtype=torch.float64, device=dev)
    dist.all_reduce(box, op=dist.ReduceOp.MAX, group=group)
    box = box.cpu().numpy()
    lo, hi = -box[:n_vars], box[n_vars:]
    c, e = ops.xform(lo, hi)
    G = ops.gram(X_local, V_local, num, den, c, e)
    G = G if isinstance(G, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(G, dtype=np.float64))
    G = G.to(dev)
    if deterministic:  # all_gather, then the rank-ordered sum on the device (ops.gram_sum)
        world = dist.get_world_size(group)
        parts = torch.empty((world * G.shape[0],) + tuple(G.shape[1:]), dtype=G.dtype, device=G.device)
        dist.all_gather_into_tensor(parts, G.contiguous(), group=group)
        G = ops.gram_sum(parts.view((world,) + tuple(G.shape)))
    else:
        dist.all_reduce(G, op=dist.ReduceOp.SUM, group=group)
    coef, infos = ops.solve(G, num, den)
    return coef, (c, e), infos


def sharded_fit_dev(X_local, V_local, num, den, ops, n_vars: int, group=None):
    """sharded_fit without a host round trip (the bench's N > 1 step): per-rank (min, max) on the
    device, one all_reduce(MAX) of (-lo, hi), the transform on the device, the partial Gram,
    all_reduce(SUM), the solve into device coefficients.  Returns device tensors (coef [n_v][n_c],
    xf [n][2], info [n_v][5]); every rank holds the same values.  A rank with K_r = 0 contributes
    (+inf, -inf) bounds and a zero Gram."""
    K_r = X_local.shape[0]
    if K_r > 0:
        lohi = ops.minmax_dev(X_local)
    else:
        lohi = torch.stack([torch.full((n_vars,), float("inf"), dtype=torch.float64),
                            torch.full((n_vars,), float("-inf"), dtype=torch.float64)], 1)
        lohi = lohi.to(X_local.device if isinstance(X_local, torch.Tensor) else "cpu")
    box = torch.stack([-lohi[:, 0], lohi[:, 1]], 1).contiguous()
    dist.all_reduce(box, op=dist.ReduceOp.MAX, group=group)
    lohi = torch.stack([-box[:, 0], box[:, 1]], 1).contiguous()
    xf = ops.xform_dev(lohi)
    G = ops.gram_dev(X_local, V_local, num, den, xf)
    dist.all_reduce(G, op=dist.ReduceOp.SUM, group=group)
    coef, info = ops.solve_dev(G, num, den)
    return coef, xf, info


def sharded_fit_svd(X_local, V_local, num, den, ops, n_vars: int, group=None):
    """NEXT row f1 sharded over K: agree the transform (all_reduce MAX of (-lo, hi)), factor this
    rank's rows (TSQR: R_r with R_r^T R_r = A_r^T A_r, or any B_r with that property), all_gather
    the factors in rank order and take the SVD of the stacked [R_0; R_1; ...] -- the same
    singular vectors as the SVD of all K rows.  Returns (coef, sigma, (c, e), infos), identical
    on every rank (deterministic: fixed stacking order)."""
    dev = _comm_device(group)
    K_r = X_local.shape[0]
    if K_r > 0:
        lo, hi = ops.minmax(X_local)
    else:
        lo, hi = np.full(n_vars, np.inf), np.full(n_vars, -np.inf)
    box = torch.tensor(np.concatenate([-np.asarray(lo), np.asarray(hi)]), dtype=torch.float64, device=dev)
    dist.all_reduce(box, op=dist.ReduceOp.MAX, group=group)
    box = box.cpu().numpy()
    lo, hi = -box[:n_vars], box[n_vars:]
    c, e = ops.xform(lo, hi)
    R = ops.tsqr(X_local, V_local, num, den, c, e)
    R = R if isinstance(R, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(R, dtype=np.float64))
    R = R.to(dev).contiguous()
    # factors may have different row counts per rank (a generic B_r): gather the counts first
    world = dist.get_world_size(group)
    cnt = torch.tensor([R.shape[1]], dtype=torch.int64, device=dev)
    cnts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    m = max(int(x.item()) for x in cnts)
    if R.shape[1] < m:  # zero rows change nothing (A^T A is unchanged)
        R = torch.cat([R, torch.zeros((R.shape[0], m - R.shape[1], R.shape[2]), dtype=R.dtype, device=dev)], 1)
    parts = [torch.empty_like(R) for _ in range(world)]
    dist.all_gather(parts, R, group=group)
    rows = torch.cat(parts, dim=1)
    coef, sigma, infos = ops.svd_rows(rows, num, den)
    return coef, sigma, (c, e), infos


def gather_winners(idx_local, E_local, nD: int, group=None):
    """all_gather the per-D winners of contiguous shards into full [n_prog][nD] arrays."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    idx_local = torch.as_tensor(idx_local).to(dev)
    E_local = torch.as_tensor(E_local).to(dev)
    n_prog = idx_local.shape[0]
    per = (nD + world - 1) // world
    pad = per - idx_local.shape[1]
    if pad:
        idx_local = torch.cat([idx_local, torch.full((n_prog, pad), -1, dtype=idx_local.dtype, device=dev)], 1)
        E_local = torch.cat([E_local, torch.full((n_prog, pad), float("inf"), dtype=E_local.dtype, device=dev)], 1)
    # shard-major gather buffers [world][n_prog][per], then transposed back to [n_prog][nD]
    gi = torch.empty((world * n_prog, per), dtype=idx_local.dtype, device=dev)
    gE = torch.empty((world * n_prog, per), dtype=E_local.dtype, device=dev)
    dist.all_gather_into_tensor(gi, idx_local.contiguous(), group=group)
    dist.all_gather_into_tensor(gE, E_local.contiguous(), group=group)
    idx = gi.view(world, n_prog, per).permute(1, 0, 2).reshape(n_prog, world * per)[:, :nD]
    E = gE.view(world, n_prog, per).permute(1, 0, 2).reshape(n_prog, world * per)[:, :nD]
    return idx, E


def sharded_sweep(plan_or_progs, D_full, F, ops, group=None, gather: bool = True):
    """Each rank sweeps its contiguous shard of D; winners are all-gathered if `gather`."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nD = D_full.shape[0]
    lo, hi = shard_bounds(nD, world, rank)
    idx, E = ops.sweep(plan_or_progs, D_full[lo:hi], F)
    if not gather:
        return idx, E
    return gather_winners(idx, E, nD, group)
