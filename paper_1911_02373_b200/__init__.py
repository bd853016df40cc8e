"""B200 (sm_100a) hot path of the rational-program method of arXiv 1911.02373 (KLARAPTOR).

Thin Python binding over ``librp.so`` (C ABI in ``include/rp.h``): argument marshalling only.
Every step of the method -- transform, design rows, Gram, solve, occupancy, masks, metric
evaluation, the MWP-CWP estimate and the argmin -- runs in the library's CUDA kernels.  There is
no CPU fallback: if ``librp.so`` is missing, importing this package raises, and on a machine
without a GPU every compute call raises ``RPError`` (RP_ERR_CUDA).

Arrays may be torch tensors (CUDA or CPU) or numpy arrays; CUDA tensors are used in place on
the current torch stream, host arrays are staged by the library itself (see rp.h).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RP_LIBRP overrides the in-tree library (developer knob for A/B builds of the same sources)
LIB_PATH = os.environ.get("RP_LIBRP") or os.path.join(_HERE, "librp.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

RP_MAX_VARS = 8
RP_MAX_METRICS = 3
STATUS = {0: "RP_OK", 1: "RP_ERR_INVALID_ARG", 2: "RP_ERR_CUDA", 3: "RP_ERR_DEGENERATE",
          4: "RP_ERR_NO_FEASIBLE", 5: "RP_ERR_UNSUPPORTED"}
TEMPLATES = {"mwpcwp": 0, "g1": 1}


class RPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class rp_basis(C.Structure):
    _fields_ = [("n_vars", C.c_int32), ("n_num", C.c_int32), ("n_den", C.c_int32),
                ("num_exp", C.c_void_p), ("den_exp", C.c_void_p)]


class rp_xform(C.Structure):
    _fields_ = [("c", C.c_double * RP_MAX_VARS), ("e", C.c_int32 * RP_MAX_VARS)]


class rp_hw(C.Structure):
    _fields_ = [("n_sm", C.c_int32), ("w_max", C.c_int32), ("b_max", C.c_int32), ("t_max", C.c_int32),
                ("r_max", C.c_int64), ("z_max", C.c_int64)] + \
               [(k, C.c_double) for k in ("freq_hz", "mem_bw", "load_bytes_per_warp", "mem_ld", "dd_coal",
                                          "dd_unc", "uncoal_per_mw", "issue_cycles")]


class rp_program(C.Structure):
    _fields_ = [("d", C.c_int32), ("p", C.c_int32), ("n_metrics", C.c_int32), ("e_template", C.c_int32),
                ("basis", rp_basis * RP_MAX_METRICS), ("coef", C.c_void_p * RP_MAX_METRICS),
                ("xform", rp_xform), ("hw", rp_hw), ("regs_per_thread", C.c_int32),
                ("grid_map", C.c_int32 * 3), ("smem_words_base", C.c_int64),
                ("smem_words_per_thread", C.c_int64)]


class rp_decision(C.Structure):
    _fields_ = [("idx", C.c_int32), ("from_history", C.c_int32), ("E", C.c_double),
                ("launch", C.c_int32 * 6), ("pad", C.c_int32 * 2)]


DECISION_DTYPE = np.dtype([("idx", np.int32), ("from_history", np.int32), ("E", np.float64),
                           ("launch", np.int32, (6,)), ("pad", np.int32, (2,))])
assert DECISION_DTYPE.itemsize == C.sizeof(rp_decision) == 48


class rp_fit_info(C.Structure):
    _fields_ = [("rank", C.c_int32), ("status", C.c_int32), ("resid2", C.c_double),
                ("min_pivot", C.c_double), ("cond_est", C.c_double), ("iters", C.c_int32), ("reserved", C.c_int32)]


_vp, _i32, _i64 = C.c_void_p, C.c_int32, C.c_int64
_lib.rp_abi_version.restype = _i32
_lib.rp_last_error.restype = C.c_char_p
_lib.rp_device_count.restype = _i32
_SIGS = {
    "rp_xform_from_box": [_i32, _vp, _vp, C.POINTER(rp_xform)],
    "rp_minmax": [_vp, _i64, _i32, _vp, _vp, _vp],
    "rp_gram_accumulate": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), C.POINTER(rp_xform), _vp, _vp],
    "rp_solve_normal": [_vp, _i32, C.POINTER(rp_basis), _vp, _vp, _vp],
    "rp_fit": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), _vp, C.POINTER(rp_xform), _vp, _vp],
    "rp_gram_accumulate_weighted": [_vp, _vp, _vp, _i64, _i32, C.POINTER(rp_basis), C.POINTER(rp_xform), _vp, _vp],
    "rp_fit_sk": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), _i32, _vp, C.POINTER(rp_xform), _vp, _vp],
    "rp_minmax_dev": [_vp, _i64, _i32, _vp, _vp],
    "rp_xform_dev": [_vp, _i32, _vp, _vp],
    "rp_gram_accumulate_dev": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), _vp, _vp, _vp],
    "rp_solve_normal_dev": [_vp, _i32, C.POINTER(rp_basis), _vp, _vp, _vp],
    "rp_fit_dev": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), _vp, _vp, _vp, _vp],
    "rp_plan_update_program": [_vp, _i32, _vp, _i32, _vp, _vp],
    "rp_fit_svd": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), _vp, _vp, C.POINTER(rp_xform), _vp, _vp],
    "rp_tsqr_accumulate": [_vp, _vp, _i64, _i32, C.POINTER(rp_basis), C.POINTER(rp_xform), _vp, _vp],
    "rp_svd_rows": [_vp, _i64, _i32, C.POINTER(rp_basis), _vp, _vp, _vp, _vp],
    "rp_codegen": [C.POINTER(rp_program), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
    "rp_jit_create": [C.POINTER(rp_program), C.POINTER(_vp)],
    "rp_jit_eval_argmin": [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp],
    "rp_jit_destroy": [_vp],
    "rp_eval_metrics": [C.POINTER(rp_program), _vp, _i64, _vp, _vp],
    "rp_eval_argmin": [C.POINTER(rp_program), _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp],
    "rp_eval_argmin_batched": [_vp, _i32, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp],
    "rp_plan_create": [_vp, _i32, _vp, _i32, C.POINTER(_vp), _vp],
    "rp_plan_eval_argmin": [_vp, _vp, _i64, _vp, _vp, _vp, _vp],
    "rp_plan_static_feasible": [_vp, _i32, C.POINTER(_i32)],
    "rp_plan_destroy": [_vp],
    "rp_plan_decide": [_vp, _i32, _vp, _i64, C.c_double, _vp, _vp],
    "rp_plan_history_enable": [_vp, _i32, _i32, C.c_double],
    "rp_decider_create": [_vp, _i32, C.c_double, _vp],
    "rp_decider_decide": [_vp, _vp, _vp],
    "rp_decider_destroy": [_vp],
    "rp_plan_history_stats": [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)],
    "rp_plan_history_clear": [_vp, _vp],
    "rp_plan_enable_timing": [_vp, _i32],
    "rp_plan_last_timing": [_vp, _vp],
    "rp_pipeline_create": [_vp, _i32, C.POINTER(rp_basis), _i32, _i64, _i32, _i64, _i32, C.POINTER(_vp)],
    "rp_pipeline_submit": [_vp, _vp, _vp, _vp, _vp, _vp],
    "rp_pipeline_sync": [_vp],
    "rp_pipeline_timer_start": [_vp],
    "rp_pipeline_timer_stop": [_vp, _vp],
    "rp_pipeline_destroy": [_vp],
    "rp_gram_sum_ordered": [_vp, _i32, _i64, _vp, _vp],
    "rp_program_save": [C.POINTER(rp_program), _vp, _i64, C.POINTER(_i64)],
    "rp_program_load": [_vp, _i64, C.POINTER(_vp)],
    "rp_program_blob_free": [_vp],
    "rp_plan_history_save": [_vp, _vp, _i64, C.POINTER(_i64)],
    "rp_plan_history_load": [_vp, _vp, _i64],
}
for _name, _args in _SIGS.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = C.c_int

_lib.rp_program_blob_program.argtypes = [_vp]
_lib.rp_program_blob_program.restype = C.POINTER(rp_program)
EXPORTED = ["rp_abi_version", "rp_last_error", "rp_device_count", "rp_program_blob_program"] + list(_SIGS)


def lib():
    return _lib


def _check(status: int):
    if status != 0:
        raise RPError(status, _lib.rp_last_error().decode(errors="replace"))


def abi_version() -> int:
    return int(_lib.rp_abi_version())


def device_count() -> int:
    return int(_lib.rp_device_count())


# --------------------------------------------------------------------------------------------
# array marshalling
# --------------------------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _ptr(a) -> int:
    """Raw data pointer of a contiguous torch tensor or numpy array."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream_of(*arrays):
    torch = _torch()
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
    return C.c_void_p(0)


def _contig(a, dtype):
    """Contiguous array of `dtype` (torch stays torch, on its device; else numpy)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int16: torch.int16}[dtype]
        return a.to(dtype=tdt).contiguous()
    return np.ascontiguousarray(a, dtype=dtype)


def _empty_like_family(ref, shape, dtype):
    torch = _torch()
    if isinstance(ref, torch.Tensor):
        tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        return torch.empty(shape, dtype=tdt, device=ref.device)
    return np.empty(shape, dtype=dtype)


# --------------------------------------------------------------------------------------------
# transform, basis
# --------------------------------------------------------------------------------------------

def xform_from_box(lo, hi):
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    out = rp_xform()
    _check(_lib.rp_xform_from_box(len(lo), _ptr(lo), _ptr(hi), C.byref(out)))
    n = len(lo)
    return np.array(out.c[:n]), np.array(out.e[:n], dtype=np.int32)


def _xform_struct(c, e) -> rp_xform:
    x = rp_xform()
    for k in range(len(c)):
        x.c[k] = float(c[k])
        x.e[k] = int(e[k])
    return x


class Basis:
    """Numerator / denominator exponent lists (held alive for the C struct)."""

    def __init__(self, num_exp, den_exp):
        self.num = np.ascontiguousarray(num_exp, dtype=np.int16)
        self.den = np.ascontiguousarray(den_exp, dtype=np.int16)
        assert self.num.ndim == 2 and self.den.ndim == 2 and self.num.shape[1] == self.den.shape[1]
        self.c = rp_basis(self.num.shape[1], len(self.num), len(self.den), _ptr(self.num), _ptr(self.den))

    @property
    def n_c(self) -> int:
        return len(self.num) + len(self.den)


# --------------------------------------------------------------------------------------------
# programs
# --------------------------------------------------------------------------------------------

class Program:
    """An ``rp_program`` built from a program description with the attributes of
    ``synth.ProgramSpec`` (d, p, num_exp, den_exp, coef, hw, R, Z0, Z1, grid_map, template and
    either box_lo/box_hi -- transform derived by the library -- or xform_c/xform_e)."""

    def __init__(self, spec):
        self.spec = spec
        self._keep = []
        pr = rp_program()
        pr.d, pr.p = spec.d, spec.p
        pr.n_metrics = len(spec.coef)
        pr.e_template = TEMPLATES[spec.template]
        for i in range(pr.n_metrics):
            b = Basis(spec.num_exp[i], spec.den_exp[i])
            cf = np.ascontiguousarray(spec.coef[i], dtype=np.float64)
            assert cf.size == b.n_c
            self._keep += [b, cf]
            pr.basis[i] = b.c
            pr.coef[i] = _ptr(cf)
        if getattr(spec, "xform_c", None) is not None:
            c, e = spec.xform_c, spec.xform_e
        else:
            c, e = xform_from_box(spec.box_lo, spec.box_hi)
        pr.xform = _xform_struct(c, e)
        self.xform = (np.asarray(c, dtype=np.float64), np.asarray(e, dtype=np.int32))
        hw = spec.hw
        pr.hw = rp_hw(**{k: hw[k] for k, _ in rp_hw._fields_})
        pr.regs_per_thread = int(spec.R)
        for k in range(3):
            pr.grid_map[k] = int(spec.grid_map[k]) if k < len(spec.grid_map) else -1
        pr.smem_words_base = int(spec.Z0)
        pr.smem_words_per_thread = int(spec.Z1)
        self.c = pr

    @property
    def d(self):
        return self.c.d

    @property
    def p(self):
        return self.c.p

    @property
    def n_metrics(self):
        return self.c.n_metrics


class LoadedProgram:
    """A program read back by :func:`load_program`, with the attributes :class:`Program`
    accepts (copies of the blob's arrays; the transform is explicit)."""

    def __init__(self, pr):
        inv = {v: k for k, v in TEMPLATES.items()}
        self.d, self.p = pr.d, pr.p
        self.template = inv[pr.e_template]
        n = pr.d + pr.p
        self.num_exp, self.den_exp, self.coef = [], [], []
        for i in range(pr.n_metrics):
            b = pr.basis[i]
            num = np.ctypeslib.as_array(C.cast(b.num_exp, C.POINTER(C.c_int16)), (b.n_num * b.n_vars,))
            den = np.ctypeslib.as_array(C.cast(b.den_exp, C.POINTER(C.c_int16)), (b.n_den * b.n_vars,))
            cf = np.ctypeslib.as_array(C.cast(pr.coef[i], C.POINTER(C.c_double)), (b.n_num + b.n_den,))
            self.num_exp.append(num.reshape(b.n_num, b.n_vars).copy())
            self.den_exp.append(den.reshape(b.n_den, b.n_vars).copy())
            self.coef.append(cf.copy())
        self.hw = {k: getattr(pr.hw, k) for k, _ in rp_hw._fields_}
        self.R = pr.regs_per_thread
        self.Z0, self.Z1 = pr.smem_words_base, pr.smem_words_per_thread
        self.grid_map = tuple(pr.grid_map[k] for k in range(3))
        self.xform_c = [pr.xform.c[k] for k in range(n)]
        self.xform_e = [pr.xform.e[k] for k in range(n)]
        self.box_lo = self.box_hi = None


def save_program(prog) -> bytes:
    """rp_program_save: the rational program as bytes (exact coefficients)."""
    prog = prog if isinstance(prog, Program) else Program(prog)
    n = _i64()
    _check(_lib.rp_program_save(C.byref(prog.c), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(_lib.rp_program_save(C.byref(prog.c), buf, n.value, C.byref(n)))
    return buf.raw[:n.value]


def load_program(blob: bytes) -> LoadedProgram:
    """rp_program_load: a program saved by :func:`save_program`."""
    h = _vp()
    _check(_lib.rp_program_load(blob, len(blob), C.byref(h)))
    try:
        return LoadedProgram(_lib.rp_program_blob_program(h).contents)
    finally:
        _lib.rp_program_blob_free(h)


def _programs(progs):
    progs = [p if isinstance(p, Program) else Program(p) for p in progs]
    arr = (rp_program * len(progs))(*[p.c for p in progs])
    return progs, arr


# --------------------------------------------------------------------------------------------
# sweep
# --------------------------------------------------------------------------------------------

def eval_argmin_batched(progs, D, F, second: bool = True, out=None):
    """Per-D argmin of E over F for each program: (idx int32 [n_prog][nD], E float64
    [n_prog][nD], second float64 [n_prog][nD] or None)."""
    progs, arr = _programs(progs)
    d, p = progs[0].d, progs[0].p
    D = _contig(D, np.int32)
    F = _contig(F, np.int32)
    nD = D.shape[0] if D.ndim > 1 else len(D) // d
    nF = F.shape[0] if F.ndim > 1 else len(F) // p
    shape = (len(progs), nD)
    if out is None:
        out = (_empty_like_family(D, shape, np.int32), _empty_like_family(D, shape, np.float64),
               _empty_like_family(D, shape, np.float64) if second else None)
    idx, E, S = out
    s = _stream_of(D, F, idx)
    _check(_lib.rp_eval_argmin_batched(C.cast(arr, _vp), len(progs), _ptr(D), nD, _ptr(F), nF, _ptr(idx),
                                       _ptr(E), _ptr(S) if S is not None else None, s))
    return idx, E, S


def eval_argmin(prog, D, F, second: bool = True):
    idx, E, S = eval_argmin_batched([prog], D, F, second)
    return idx[0], E[0], (S[0] if S is not None else None)


def codegen(prog) -> str:
    """rp_codegen (NEXT row f3): the CUDA C source of the rational program, constants as
    immediates (step 3)."""
    pr = prog if isinstance(prog, Program) else Program(prog)
    n = C.c_size_t(0)
    _check(_lib.rp_codegen(C.byref(pr.c), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(_lib.rp_codegen(C.byref(pr.c), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class Jit:
    """rp_jit_create / rp_jit_eval_argmin: the generated program compiled by NVRTC for sm_100a
    and searched exhaustively, one warp per data tuple."""

    def __init__(self, prog):
        self.prog = prog if isinstance(prog, Program) else Program(prog)
        self.d, self.p = self.prog.d, self.prog.p
        h = _vp()
        _check(_lib.rp_jit_create(C.byref(self.prog.c), C.byref(h)))
        self.h = h

    def eval(self, D, F, second: bool = True, out=None):
        D = _contig(D, np.int32)
        F = _contig(F, np.int32)
        nD = D.shape[0] if D.ndim > 1 else len(D) // self.d
        nF = F.shape[0] if F.ndim > 1 else len(F) // self.p
        if out is None:
            out = (_empty_like_family(D, (nD,), np.int32), _empty_like_family(D, (nD,), np.float64),
                   _empty_like_family(D, (nD,), np.float64) if second else None)
        idx, E, S = out
        _check(_lib.rp_jit_eval_argmin(self.h, _ptr(D), nD, _ptr(F), nF, _ptr(idx), _ptr(E),
                                       _ptr(S) if S is not None else None, _stream_of(D, F, idx)))
        return idx, E, S

    def close(self):
        if getattr(self, "h", None):
            _lib.rp_jit_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """a1 once per (programs, F) -- static mask, occupancy, P-monomials, compaction on the
    device -- then many sweeps over D batches."""

    def __init__(self, progs, F, device=None):
        self.progs, arr = _programs(progs)
        self.d, self.p = self.progs[0].d, self.progs[0].p
        F = _contig(F, np.int32)
        self.nF = F.shape[0] if F.ndim > 1 else len(F) // self.p
        self.handle = C.c_void_p()
        self.generation = 0  # bumped by update(): host-side caches of decisions key on it
        self._history = None  # (prog, log2_capacity, margin) of the enabled runtime history
        s = _stream_of(F)
        _check(_lib.rp_plan_create(C.cast(arr, _vp), len(self.progs), _ptr(F), self.nF, C.byref(self.handle), s))

    def update(self, coef, xf=None, prog: int = 0):
        """rp_plan_update_program: new coefficients [n_metrics][n_c] (and transform [n][2]) of
        program `prog` from device tensors: the staging matrix and the configurations' monomials are
        refreshed on the device in one launch (stream-ordered)."""
        coef = coef.contiguous()
        _check(_lib.rp_plan_update_program(self.handle, prog, _ptr(coef), coef.shape[-1],
                                           _ptr(xf.contiguous()) if xf is not None else None, _stream_of(coef)))
        self.generation += 1

    def static_feasible(self, prog: int = 0) -> int:
        v = C.c_int32()
        _check(_lib.rp_plan_static_feasible(self.handle, prog, C.byref(v)))
        return int(v.value)

    def eval(self, D, out=None, second: bool = True):
        D = _contig(D, np.int32)
        nD = D.shape[0] if D.ndim > 1 else len(D) // self.d
        shape = (len(self.progs), nD)
        if out is None:
            out = (_empty_like_family(D, shape, np.int32), _empty_like_family(D, shape, np.float64),
                   _empty_like_family(D, shape, np.float64) if second else None)
        idx, E, S = out
        s = _stream_of(D, idx)
        _check(_lib.rp_plan_eval_argmin(self.handle, _ptr(D), nD, _ptr(idx), _ptr(E),
                                        _ptr(S) if S is not None else None, s))
        return idx, E, S

    # ---- f2: runtime decisions -------------------------------------------------------------
    def decide(self, D, prog: int = 0, margin: float = 0.0, out=None):
        """One decision per data tuple (rp_plan_decide): a numpy structured array of
        DECISION_DTYPE (idx, from_history, E, launch = (gx, gy, gz, bx, by, bz)) for host D,
        or a uint8 device tensor [n][48] for device D / out."""
        D = _contig(D, np.int32)
        n = D.shape[0] if D.ndim > 1 else len(D) // self.d
        if out is None:
            torch = _torch()
            if isinstance(D, torch.Tensor) and D.is_cuda:
                out = torch.empty((n, 48), dtype=torch.uint8, device=D.device)
            else:
                out = np.zeros(n, dtype=DECISION_DTYPE)
        _check(_lib.rp_plan_decide(self.handle, prog, _ptr(D), n, float(margin), _ptr(out), _stream_of(D, out)))
        return out

    def enable_history(self, prog: int = 0, log2_capacity: int = 16, margin: float = 0.0):
        _check(_lib.rp_plan_history_enable(self.handle, prog, log2_capacity, float(margin)))
        self._history = (prog, log2_capacity, float(margin))

    def history_stats(self) -> dict:
        h, m, e = _i64(), _i64(), _i64()
        _check(_lib.rp_plan_history_stats(self.handle, C.byref(h), C.byref(m), C.byref(e)))
        return {"hits": h.value, "misses": m.value, "entries": e.value}

    def clear_history(self):
        _check(_lib.rp_plan_history_clear(self.handle, C.c_void_p(0)))

    def save_history(self) -> bytes:
        """rp_plan_history_save: the runtime history as bytes (bound to the program and F)."""
        n = _i64()
        _check(_lib.rp_plan_history_save(self.handle, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(_lib.rp_plan_history_save(self.handle, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def load_history(self, blob: bytes):
        """rp_plan_history_load: insert a saved history into this plan's enabled history."""
        _check(_lib.rp_plan_history_load(self.handle, blob, len(blob)))

    def enable_timing(self, on: bool = True):
        """Per-phase CUDA events in every later eval (rp_plan_enable_timing)."""
        _check(_lib.rp_plan_enable_timing(self.handle, 1 if on else 0))

    def last_timing(self) -> dict:
        """ms of the last eval's phases: D1 grouping, sweep kernel, winner refinement."""
        ms = (C.c_float * 3)()
        _check(_lib.rp_plan_last_timing(self.handle, ms))
        return {"group_ms": ms[0], "sweep_ms": ms[1], "refine_ms": ms[2]}

    def close(self):
        if self.handle:
            _lib.rp_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eval_metrics(prog, X):
    """g_i at the rows of X: float64 [n_metrics][K]."""
    prog = prog if isinstance(prog, Program) else Program(prog)
    X = _contig(X, np.float64)
    K = X.shape[0]
    out = _empty_like_family(X, (prog.n_metrics, K), np.float64)
    _check(_lib.rp_eval_metrics(C.byref(prog.c), _ptr(X), K, _ptr(out), _stream_of(X, out)))
    return out


# --------------------------------------------------------------------------------------------
# fit
# --------------------------------------------------------------------------------------------

def minmax(X):
    X = _contig(X, np.float64)
    K, n = X.shape
    lo = np.zeros(n)
    hi = np.zeros(n)
    _check(_lib.rp_minmax(_ptr(X), K, n, _ptr(lo), _ptr(hi), _stream_of(X)))
    return lo, hi


def gram(X, V, num_exp, den_exp, c, e, out=None):
    """G [n_v][n_c][n_c] of the linearised system for n_v metrics V [n_v][K] sharing X."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    xf = _xform_struct(c, e)
    G = out if out is not None else _empty_like_family(X, (n_v, b.n_c, b.n_c), np.float64)
    _check(_lib.rp_gram_accumulate(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), C.byref(xf), _ptr(G), _stream_of(X, V, G)))
    return G


def gram_weighted(X, V, S, num_exp, den_exp, c, e, out=None):
    """rp_gram_accumulate_weighted: every design row of metric m scaled by S[m][r]."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    S = _contig(S, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    xf = _xform_struct(c, e)
    G = out if out is not None else _empty_like_family(X, (n_v, b.n_c, b.n_c), np.float64)
    _check(_lib.rp_gram_accumulate_weighted(_ptr(X), _ptr(V), _ptr(S), K, n_v, C.byref(b.c), C.byref(xf), _ptr(G),
                                            _stream_of(X, V, G)))
    return G


def fit_sk(X, V, num_exp, den_exp, iters: int = 3, raise_on_degenerate: bool = True):
    """rp_fit_sk: Sanathanan-Koerner refit (NEXT row f4); returns like fit()."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    coef = np.zeros((n_v, b.n_c))
    xf = rp_xform()
    infos = (rp_fit_info * n_v)()
    st = _lib.rp_fit_sk(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), iters, _ptr(coef), C.byref(xf), C.cast(infos, _vp),
                        _stream_of(X, V))
    if st != 0 and (st != 3 or raise_on_degenerate):
        _check(st)
    n = b.num.shape[1]
    return coef, (np.array(xf.c[:n]), np.array(xf.e[:n], dtype=np.int32)), _infos(infos)


def _infos(infos):
    return [dict(rank=i.rank, status=i.status, resid2=i.resid2, min_pivot=i.min_pivot, cond_est=i.cond_est,
                 iters=i.iters)
            for i in infos]


def solve_normal(G, num_exp, den_exp, raise_on_degenerate: bool = True):
    b = Basis(num_exp, den_exp)
    G = _contig(G, np.float64)
    n_v = G.shape[0] if G.ndim == 3 else 1
    coef = np.zeros((n_v, b.n_c))
    infos = (rp_fit_info * n_v)()
    st = _lib.rp_solve_normal(_ptr(G), n_v, C.byref(b.c), _ptr(coef), C.cast(infos, _vp), _stream_of(G))
    if st != 0 and (st != 3 or raise_on_degenerate):
        _check(st)
    return coef, _infos(infos)


def fit(X, V, num_exp, den_exp, raise_on_degenerate: bool = True):
    """rp_fit: transform from the sample box, Gram, beta_0 = 1 solve, for n_v metrics sharing
    X.  Returns (coef float64 [n_v][n_c] in the u-basis, (c, e), infos)."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    coef = np.zeros((n_v, b.n_c))
    xf = rp_xform()
    infos = (rp_fit_info * n_v)()
    st = _lib.rp_fit(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), _ptr(coef), C.byref(xf), C.cast(infos, _vp),
                     _stream_of(X, V))
    if st != 0 and (st != 3 or raise_on_degenerate):
        _check(st)
    n = b.num.shape[1]
    return coef, (np.array(xf.c[:n]), np.array(xf.e[:n], dtype=np.int32)), _infos(infos)


# ---- device-resident (stream-ordered) forms: torch CUDA tensors in and out, no host sync ----

def _dev_empty(ref, shape):
    return _torch().empty(shape, dtype=_torch().float64, device=ref.device)


def gram_sum_ordered(parts, out=None):
    """rp_gram_sum_ordered: the rank-ordered sum of stacked partial Grams [n_parts][...] (device)."""
    parts = parts.contiguous()
    out = out if out is not None else _dev_empty(parts, tuple(parts.shape[1:]))
    _check(_lib.rp_gram_sum_ordered(_ptr(parts), parts.shape[0], parts[0].numel(), _ptr(out), _stream_of(parts)))
    return out


def minmax_dev(X, out=None):
    """lohi [n][2] (min, max per column) on the device."""
    X = _contig(X, np.float64)
    K, n = X.shape
    lohi = out if out is not None else _dev_empty(X, (n, 2))
    _check(_lib.rp_minmax_dev(_ptr(X), K, n, _ptr(lohi), _stream_of(X)))
    return lohi


def xform_dev(lohi, out=None):
    """xf [n][2] = (c_k, e_k) from lohi [n][2] on the device (reading R14)."""
    n = lohi.shape[0]
    xf = out if out is not None else _dev_empty(lohi, (n, 2))
    _check(_lib.rp_xform_dev(_ptr(lohi), n, _ptr(xf), _stream_of(lohi)))
    return xf


def gram_dev(X, V, num_exp, den_exp, xf, out=None):
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    n_v = V.shape[0] if V.ndim == 2 else 1
    G = out if out is not None else _dev_empty(X, (n_v, b.n_c, b.n_c))
    _check(_lib.rp_gram_accumulate_dev(_ptr(X), _ptr(V), X.shape[0], n_v, C.byref(b.c), _ptr(xf), _ptr(G),
                                       _stream_of(X, V, G)))
    return G


def solve_dev(G, num_exp, den_exp, coef=None, info=None):
    """coef [n_v][n_c] and info [n_v][5] (status, rank, resid2, min_pivot, cond_est) on the device."""
    b = Basis(num_exp, den_exp)
    n_v = G.shape[0]
    coef = coef if coef is not None else _dev_empty(G, (n_v, b.n_c))
    info = info if info is not None else _dev_empty(G, (n_v, 5))
    _check(_lib.rp_solve_normal_dev(_ptr(G), n_v, C.byref(b.c), _ptr(coef), _ptr(info), _stream_of(G)))
    return coef, info


def fit_dev(X, V, num_exp, den_exp, coef=None, xf=None, info=None):
    """rp_fit_dev: the fit entirely on the device, no host round trip.  Returns device tensors
    (coef [n_v][n_c], xf [n][2], info [n_v][5])."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K, n = X.shape
    n_v = V.shape[0] if V.ndim == 2 else 1
    coef = coef if coef is not None else _dev_empty(X, (n_v, b.n_c))
    xf = xf if xf is not None else _dev_empty(X, (n, 2))
    info = info if info is not None else _dev_empty(X, (n_v, 5))
    _check(_lib.rp_fit_dev(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), _ptr(coef), _ptr(xf), _ptr(info), _stream_of(X, V)))
    return coef, xf, info


def fit_svd(X, V, num_exp, den_exp, raise_on_degenerate: bool = True):
    """rp_fit_svd (NEXT row f1): the homogeneous system by SVD -- TSQR of the design rows, then
    Jacobi SVD of R.  Returns (coef [n_v][n_c], sigma [n_v][n_c] ascending, (c, e), infos)."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    coef = np.zeros((n_v, b.n_c))
    sigma = np.zeros((n_v, b.n_c))
    xf = rp_xform()
    infos = (rp_fit_info * n_v)()
    st = _lib.rp_fit_svd(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), _ptr(coef), _ptr(sigma), C.byref(xf),
                         C.cast(infos, _vp), _stream_of(X, V))
    if st != 0 and (st != 3 or raise_on_degenerate):
        _check(st)
    n = b.num.shape[1]
    return coef, sigma, (np.array(xf.c[:n]), np.array(xf.e[:n], dtype=np.int32)), _infos(infos)


def tsqr(X, V, num_exp, den_exp, c, e, out=None):
    """rp_tsqr_accumulate: R [n_v][n_c][n_c] (upper triangular, A^T A = R^T R) of this shard's
    design rows under the agreed transform (c, e)."""
    b = Basis(num_exp, den_exp)
    X = _contig(X, np.float64)
    V = _contig(V, np.float64)
    K = X.shape[0]
    n_v = V.shape[0] if V.ndim == 2 else 1
    xf = _xform_struct(c, e)
    R = out if out is not None else _empty_like_family(X, (n_v, b.n_c, b.n_c), np.float64)
    _check(_lib.rp_tsqr_accumulate(_ptr(X), _ptr(V), K, n_v, C.byref(b.c), C.byref(xf), _ptr(R), _stream_of(X, V, R)))
    return R


def svd_rows(rows, num_exp, den_exp, raise_on_degenerate: bool = True):
    """rp_svd_rows: TSQR + SVD of dense rows [n_v][n_rows][n_c] (e.g. stacked per-rank R factors).
    Returns (coef, sigma, infos)."""
    b = Basis(num_exp, den_exp)
    rows = _contig(rows, np.float64)
    n_v, n_rows = rows.shape[0], rows.shape[1]
    coef = np.zeros((n_v, b.n_c))
    sigma = np.zeros((n_v, b.n_c))
    infos = (rp_fit_info * n_v)()
    st = _lib.rp_svd_rows(_ptr(rows), n_rows, n_v, C.byref(b.c), _ptr(coef), _ptr(sigma), C.cast(infos, _vp),
                          _stream_of(rows))
    if st != 0 and (st != 3 or raise_on_degenerate):
        _check(st)
    return coef, sigma, _infos(infos)


def decisions_from_device(out) -> np.ndarray:
    """A uint8 [n][48] device tensor of rp_decision records as a DECISION_DTYPE array."""
    return np.frombuffer(out.cpu().numpy().tobytes(), dtype=DECISION_DTYPE)


class Decider:
    """rp_decider: one data tuple in, one decision out, through host-mapped pinned memory and a
    CUDA graph of the decide kernel captured once (no copy nodes, no per-call allocation).
    Enable the plan's history (Plan.enable_history) before creating one if it is to be used."""

    def __init__(self, plan: "Plan", prog: int = 0, margin: float = 0.0):
        self.plan = plan
        self.handle = C.c_void_p()
        _check(_lib.rp_decider_create(plan.handle, prog, float(margin), C.byref(self.handle)))
        self._D = (C.c_int32 * max(plan.d, 1))()
        self._out = np.zeros(1, dtype=DECISION_DTYPE)

    def __call__(self, D) -> np.void:
        for k, v in enumerate(np.asarray(D).ravel()[: self.plan.d]):
            self._D[k] = int(v)
        _check(_lib.rp_decider_decide(self.handle, C.cast(self._D, _vp), _ptr(self._out)))
        return self._out[0].copy()

    def close(self):
        if self.handle:
            _lib.rp_decider_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DecisionService:
    """The single-launch latency path of NEXT row f2, for a user's launch site: a host memo in
    front of a Decider (rp_decider: mapped memory, the decide kernel as a captured CUDA graph),
    which itself probes the plan's device history (the rational program runs
    "immediately preceding the launch of a kernel"; 2120-2122: the runtime history)."""

    def __init__(self, plan: "Plan", prog: int = 0, margin: float = 0.0, history_log2: int | None = 16,
                 host_memo: int = 1 << 16):
        self.plan, self.prog, self.margin = plan, prog, margin
        self.memo = {} if host_memo else None
        self.memo_cap = host_memo
        self._gen = plan.generation
        # the history may already serve another service of the same (program, margin): enabling
        # it again would only clear it (rp.h), so it is left as it is
        if history_log2 and plan._history != (prog, history_log2, float(margin)):
            plan.enable_history(prog, history_log2, margin)
        self.decider = Decider(plan, prog, margin)

    def __call__(self, D) -> np.void:
        if self.plan.generation != self._gen:  # Plan.update: every memoised decision is stale
            self._gen = self.plan.generation
            if self.memo is not None:
                self.memo.clear()
        key = tuple(int(v) for v in np.asarray(D).ravel()[: self.plan.d])
        hit = self.memo.get(key) if self.memo is not None else None
        if hit is not None:  # host memo in front of the device history: no GPU round trip
            return hit
        r = self.decider(key)
        if self.memo is not None and len(self.memo) < self.memo_cap:
            self.memo[key] = r
        return r
