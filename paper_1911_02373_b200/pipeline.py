"""Host-fed fit -> plan update -> sweep, pipelined over steps (plumbing only).

`StepPipeline` is the C ABI's rp_pipeline (rp_pipeline.cu): the copies and the event ordering run
inside librp.  `FitSweepPipeline` below is the same schedule written with torch streams, for the
multi-rank case, whose fit needs the torch.distributed all-reduce between the Gram and the solve.

A user who tunes many launches feeds batches from host memory: sampled points X, measured metrics
V and data tuples D in, the per-D winners out.  `FitSweepPipeline` overlaps those copies with the
computation of the neighbouring steps: the inputs of step i+1 stream in on one copy stream and the
winners of step i-1 stream out on another while step i computes.  Everything it does itself is
copies and event ordering; every computation is a librp call through the binding (`fit_dev` or a
caller-supplied sharded fit, `Plan.update` = rp_plan_update_program, `Plan.eval` =
rp_plan_eval_argmin).  Device buffers are allocated once per in-flight slot.

Ordering per slot s (depth slots in flight):
  h2d:     wait out_done[s] (the previous user of s is fully retired), copy X, V, D -> s, in_ready[s]
  compute: wait in_ready[s], fit, update, sweep (+ gather), comp_done[s]
  d2h:     wait comp_done[s], copy winners -> the caller's pinned host arrays, out_done[s]
"""
from __future__ import annotations

import numpy as np

import ctypes as C

from . import Basis, Plan, _check, _lib, _ptr, fit_dev


class StepPipeline:
    """rp_pipeline: submit(X, V, D, idx_out, E_out) with host arrays (pinned for overlap) enqueues
    one fit -> plan update -> sweep step and returns at once; sync() waits for every step."""

    def __init__(self, program, F, num_exp, den_exp, K: int, n_v: int, nD: int, d: int, depth: int = 2):
        self.plan = Plan([program], F)
        self.basis = Basis(num_exp, den_exp)
        self.h = C.c_void_p()
        _check(_lib.rp_pipeline_create(self.plan.handle, 0, C.byref(self.basis.c), n_v, K, d, nD, depth,
                                       C.byref(self.h)))
        self.keep = []  # host buffers of steps in flight

    def submit(self, X, V, D, idx_out, E_out):
        self.keep.append((X, V, D, idx_out, E_out))
        _check(_lib.rp_pipeline_submit(self.h, _ptr(X), _ptr(V), _ptr(D), _ptr(idx_out), _ptr(E_out)))

    def sync(self):
        _check(_lib.rp_pipeline_sync(self.h))
        self.keep.clear()

    def timer_start(self):
        _check(_lib.rp_pipeline_timer_start(self.h))

    def timer_stop(self) -> float:
        """ms from timer_start to the D2H of the last submitted step (device events)."""
        ms = C.c_float()
        _check(_lib.rp_pipeline_timer_stop(self.h, C.byref(ms)))
        return float(ms.value)

    def close(self):
        if self.h:
            _lib.rp_pipeline_destroy(self.h)
            self.h = C.c_void_p()
            self.plan.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FitSweepPipeline:
    def __init__(self, program, F, num_exp, den_exp, K: int, n_vars: int, n_v: int, nD: int, d: int,
                 device=None, depth: int = 2, fit_fn=None, gather_fn=None):
        import torch

        self.torch = torch
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.num_exp, self.den_exp = num_exp, den_exp
        self.depth = depth
        self.fit_fn = fit_fn or (lambda X, V: fit_dev(X, V, num_exp, den_exp)[:2])
        self.gather_fn = gather_fn
        self.compute = torch.cuda.current_stream(self.dev)
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        Fd = F if isinstance(F, torch.Tensor) and F.is_cuda else torch.from_numpy(np.ascontiguousarray(F)).to(self.dev)
        self.plan = Plan([program], Fd)
        f64, i32 = torch.float64, torch.int32
        self.X = [torch.empty((K, n_vars), dtype=f64, device=self.dev) for _ in range(depth)]
        self.V = [torch.empty((n_v, K), dtype=f64, device=self.dev) for _ in range(depth)]
        self.D = [torch.empty((nD, d), dtype=i32, device=self.dev) for _ in range(depth)]
        self.idx = [torch.empty((1, nD), dtype=i32, device=self.dev) for _ in range(depth)]
        self.E = [torch.empty((1, nD), dtype=f64, device=self.dev) for _ in range(depth)]
        self.in_ready = [torch.cuda.Event() for _ in range(depth)]
        self.comp_done = [torch.cuda.Event() for _ in range(depth)]
        self.out_done = [torch.cuda.Event() for _ in range(depth)]
        self.used = [False] * depth
        self.n = 0

    def submit(self, X_h, V_h, D_h, idx_h, E_h):
        """Enqueue one step; X_h, V_h, D_h, idx_h, E_h are pinned host tensors (idx_h / E_h of the
        gathered size when a gather_fn is given).  Returns the event that completes when the
        winners are in idx_h / E_h."""
        torch = self.torch
        s = self.n % self.depth
        self.n += 1
        with torch.cuda.stream(self.h2d):
            if self.used[s]:
                self.h2d.wait_event(self.out_done[s])
            self.X[s].copy_(X_h, non_blocking=True)
            self.V[s].copy_(V_h, non_blocking=True)
            self.D[s].copy_(D_h, non_blocking=True)
            self.in_ready[s].record(self.h2d)
        self.used[s] = True
        with torch.cuda.stream(self.compute):
            self.compute.wait_event(self.in_ready[s])
            coef, xf = self.fit_fn(self.X[s], self.V[s])
            self.plan.update(coef, xf)
            idx, E, _ = self.plan.eval(self.D[s], out=(self.idx[s], self.E[s], None), second=False)
            if self.gather_fn is not None:
                idx, E = self.gather_fn(idx, E)
            self.comp_done[s].record(self.compute)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.comp_done[s])
            for t in (idx, E):  # (a gloo gather hands back host tensors)
                if t.is_cuda:
                    t.record_stream(self.d2h)
            idx_h.copy_(idx.reshape(idx_h.shape), non_blocking=True)
            E_h.copy_(E.reshape(E_h.shape), non_blocking=True)
            self.out_done[s].record(self.d2h)
        return self.out_done[s]

    def close(self):
        self.torch.cuda.synchronize(self.dev)
        self.plan.close()
