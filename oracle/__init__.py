"""CPU oracle of the rational-program hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package.  The product (``paper_1911_02373_b200``) never does,
and this package never imports the product: the two share only the seeded generators in
``synth/``.

A thin ctypes wrapper over ``oracle/liboracle.so`` (plain C, x87 ``long double``), built from
``rp_oracle.c`` with ``make -C oracle`` on first use.  Every arithmetic step lives in the C file,
which cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LOCK = threading.Lock()

MAXV = 8
MAXM = 3
LD = np.longdouble


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    srcs = [os.path.join(_HERE, f) for f in ("rp_oracle.c", "rp_oracle_q.c", "rp_oracle_pair.inc", "rp_oracle.h")]
    if not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(f) for f in srcs):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return path


class _RatFunc(C.Structure):
    _fields_ = [("n_vars", C.c_int), ("n_num", C.c_int), ("n_den", C.c_int),
                ("num_exp", C.c_void_p), ("den_exp", C.c_void_p), ("coef", C.c_void_p)]


class _HW(C.Structure):
    _fields_ = [(k, C.c_longlong) for k in ("n_sm", "w_max", "b_max", "t_max", "r_max", "z_max")] + \
               [(k, C.c_double) for k in ("freq_hz", "mem_bw", "load_bytes_per_warp", "mem_ld", "dd_coal",
                                          "dd_unc", "uncoal_per_mw", "issue_cycles")]


class _Program(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("n_metrics", C.c_int), ("e_template", C.c_int),
                ("g", _RatFunc * MAXM), ("xc", C.c_double * MAXV), ("xe", C.c_int * MAXV),
                ("hw", _HW), ("R", C.c_longlong), ("Z0", C.c_longlong), ("Z1", C.c_longlong),
                ("grid_map", C.c_int * 3)]


class _Trace(C.Structure):
    _fields_ = [("feasible", C.c_int), ("mask", C.c_int), ("branch", C.c_int), ("mwp_case", C.c_int),
                ("T", C.c_longlong), ("B_active", C.c_longlong), ("W_active", C.c_longlong),
                ("blocks", C.c_longlong), ("sm_active", C.c_longlong),
                ("g", C.c_longdouble * MAXM), ("kappa", C.c_longdouble), ("MWP", C.c_longdouble),
                ("CWP", C.c_longdouble), ("E", C.c_longdouble), ("case_margin", C.c_longdouble)]


def lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            L = C.CDLL(build())
            vp, i, ll, d = C.c_void_p, C.c_int, C.c_longlong, C.c_double
            L.orc_xform_from_box.argtypes = [i, vp, vp, vp, vp]
            L.orc_minmax.argtypes = [vp, ll, i, vp, vp]
            L.orc_active_blocks.argtypes = [C.POINTER(_HW), ll, ll, ll, C.POINTER(C.c_int)]
            L.orc_active_blocks.restype = ll
            L.orc_active_warps.argtypes = [C.POINTER(_HW), ll, ll, ll]
            L.orc_active_warps.restype = ll
            L.orc_eval_ratfunc.argtypes = [C.POINTER(_RatFunc), vp, vp, vp, ll, vp, vp]
            for q in ("", "_q"):
                getattr(L, "orc_eval_pair" + q).argtypes = [C.POINTER(_Program), vp, vp, C.POINTER(_Trace)]
                getattr(L, "orc_eval_pair" + q).restype = i
                getattr(L, "orc_sweep" + q).argtypes = [C.POINTER(_Program), vp, ll, vp, i, vp, vp, vp, vp, vp, vp, i,
                                                        vp, vp]
            L.orc_decide.argtypes = [C.POINTER(_Program), vp, vp, i, d, vp, vp, vp]
            L.orc_decide.restype = i
            L.orc_design_row.argtypes = [i, i, i, vp, vp, vp, vp, vp, d, vp]
            L.orc_gram.argtypes = [vp, vp, ll, i, i, i, vp, vp, vp, vp, vp, i]
            L.orc_solve.argtypes = [vp, i, i, vp, vp, vp]
            L.orc_solve.restype = i
            L.orc_fit_sk.argtypes = [vp, vp, ll, i, i, i, vp, vp, i, vp, vp, vp, i]
            L.orc_fit_sk.restype = i
            L.orc_fit_svd.argtypes = [vp, vp, ll, i, i, i, vp, vp, vp, vp, vp, vp]
            L.orc_fit_svd.restype = i
            L.orc_svd_rows.argtypes = [vp, ll, i, i, vp, vp]
            L.orc_svd_rows.restype = i
            _LIB = L
        return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _hw(hw: dict) -> _HW:
    return _HW(**{k: hw[k] for k, _ in _HW._fields_})


# --------------------------------------------------------------------------------------------
# a10 transform
# --------------------------------------------------------------------------------------------


def xform_from_box(lo, hi):
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    c = np.zeros(len(lo))
    e = np.zeros(len(lo), dtype=np.int32)
    lib().orc_xform_from_box(len(lo), _p(lo), _p(hi), _p(c), _p(e))
    return c, e


def minmax(X):
    X = np.ascontiguousarray(X, dtype=np.float64)
    K, n = X.shape
    lo = np.zeros(n)
    hi = np.zeros(n)
    lib().orc_minmax(_p(X), K, n, _p(lo), _p(hi))
    return lo, hi


# --------------------------------------------------------------------------------------------
# a5 occupancy
# --------------------------------------------------------------------------------------------


def active_blocks(hw: dict, R: int, Z: int, T: int):
    b = C.c_int(0)
    h = _hw(hw)
    B = lib().orc_active_blocks(C.byref(h), R, Z, T, C.byref(b))
    return int(B), int(b.value)


def active_warps(hw: dict, R: int, Z: int, T: int) -> int:
    h = _hw(hw)
    return int(lib().orc_active_warps(C.byref(h), R, Z, T))


# --------------------------------------------------------------------------------------------
# programs
# --------------------------------------------------------------------------------------------

TEMPLATES = {"mwpcwp": 0, "g1": 1}


def program_xform(spec):
    if spec.xform_c is not None:
        return np.asarray(spec.xform_c, dtype=np.float64), np.asarray(spec.xform_e, dtype=np.int32)
    return xform_from_box(spec.box_lo, spec.box_hi)


class _ProgramHolder:
    """orc_program plus the numpy arrays it points into (kept alive)."""

    def __init__(self, spec):
        self.keep = []
        pr = _Program()
        pr.d, pr.p, pr.n_metrics = spec.d, spec.p, spec.n_metrics
        pr.e_template = TEMPLATES[spec.template]
        n = spec.d + spec.p
        for i in range(spec.n_metrics):
            ne = np.ascontiguousarray(spec.num_exp[i], dtype=np.int16)
            de = np.ascontiguousarray(spec.den_exp[i], dtype=np.int16)
            cf = np.ascontiguousarray(spec.coef[i], dtype=np.float64)
            assert ne.shape[1] == n and de.shape[1] == n and cf.size == len(ne) + len(de)
            self.keep += [ne, de, cf]
            pr.g[i] = _RatFunc(n, len(ne), len(de), _p(ne).value, _p(de).value, _p(cf).value)
        c, e = program_xform(spec)
        for k in range(n):
            pr.xc[k] = float(c[k])
            pr.xe[k] = int(e[k])
        pr.hw = _hw(spec.hw)
        pr.R, pr.Z0, pr.Z1 = spec.R, spec.Z0, spec.Z1
        for k in range(3):
            pr.grid_map[k] = spec.grid_map[k] if k < len(spec.grid_map) else -1
        self.pr = pr


def eval_pair(spec, D, P, quad: bool = False) -> dict:
    """Trace of one (D, P) pair; quad=True evaluates in IEEE binary128 (orc_eval_pair_q)."""
    h = _ProgramHolder(spec)
    Da = np.ascontiguousarray(D, dtype=np.int32)
    Pa = np.ascontiguousarray(P, dtype=np.int32)
    tr = _Trace()
    (lib().orc_eval_pair_q if quad else lib().orc_eval_pair)(C.byref(h.pr), _p(Da), _p(Pa), C.byref(tr))
    out = {k: getattr(tr, k) for k, _ in _Trace._fields_ if k != "g"}
    out["g"] = [LD(tr.g[i]) for i in range(spec.n_metrics)]
    for k in ("kappa", "MWP", "CWP", "E", "case_margin"):
        out[k] = LD(out[k])
    return out


COUNTER_NAMES = ["branch1", "branch2", "branch3", "branch4", "branch5", "case1", "case2", "case3",
                 "feasible", "pairs", "masked_static", "masked_D", "masked_B0", "masked_E"]


def sweep(spec, D, F, nthreads: int = 0, quad: bool = False) -> dict:
    """Per-D argmin of E over F (lowest index on exact ties): idx (-1 if none), best, second
    (+inf if none), idx2 (the runner-up's index), kappa / kappa2 at the winner / runner-up, the
    case margin, and coverage counters.  quad=True: the binary128 instance (orc_sweep_q)."""
    h = _ProgramHolder(spec)
    D = np.ascontiguousarray(D, dtype=np.int32).reshape(-1, spec.d)
    F = np.ascontiguousarray(F, dtype=np.int32).reshape(-1, spec.p)
    nD = len(D)
    idx = np.zeros(nD, dtype=np.int32)
    idx2 = np.zeros(nD, dtype=np.int32)
    best = np.zeros(nD)
    second = np.zeros(nD)
    kappa = np.zeros(nD)
    kappa2 = np.zeros(nD)
    margin = np.zeros(nD)
    cnt = np.zeros(16, dtype=np.int64)
    (lib().orc_sweep_q if quad else lib().orc_sweep)(C.byref(h.pr), _p(D), nD, _p(F), len(F), _p(idx), _p(best),
                                                     _p(second), _p(kappa), _p(margin), _p(cnt), nthreads, _p(idx2),
                                                     _p(kappa2))
    return dict(idx=idx, best=best, second=second, kappa=kappa, margin=margin, idx2=idx2, kappa2=kappa2,
                counters={k: int(cnt[i]) for i, k in enumerate(COUNTER_NAMES)})


def decide(spec, D, F, margin: float = 0.0) -> dict:
    """One runtime decision for the data tuple D: chosen index (-1 if none), its E, the six
    launch integers (gx, gy, gz, bx, by, bz) and the margin-boundary gap (diagnostic)."""
    h = _ProgramHolder(spec)
    Da = np.ascontiguousarray(D, dtype=np.int32).ravel()
    Fa = np.ascontiguousarray(F, dtype=np.int32).reshape(-1, spec.p)
    E = np.zeros(1)
    six = np.zeros(6, dtype=np.int32)
    gap = np.zeros(1)
    j = lib().orc_decide(C.byref(h.pr), _p(Da), _p(Fa), len(Fa), float(margin), _p(E), _p(six), _p(gap))
    return dict(idx=int(j), E=float(E[0]), launch=tuple(int(v) for v in six), boundary=float(gap[0]))


def eval_ratfunc(num_exp, den_exp, coef, c, e, X):
    """g(x) = p(u)/q(u) at the rows of X (x-space); returns (values, kappa) as long double."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    K, n = X.shape
    ne = np.ascontiguousarray(num_exp, dtype=np.int16)
    de = np.ascontiguousarray(den_exp, dtype=np.int16)
    cf = np.ascontiguousarray(coef, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.int32)
    f = _RatFunc(n, len(ne), len(de), _p(ne).value, _p(de).value, _p(cf).value)
    out = np.zeros(K, dtype=LD)
    kap = np.zeros(K, dtype=LD)
    lib().orc_eval_ratfunc(C.byref(f), _p(c), _p(e), _p(X), K, _p(out), _p(kap))
    return out, kap


def program_metrics(spec, X):
    """The program's l metrics g_i at the rows of X: long double [l][K]."""
    c, e = program_xform(spec)
    return np.stack([eval_ratfunc(spec.num_exp[i], spec.den_exp[i], spec.coef[i], c, e, X)[0]
                     for i in range(spec.n_metrics)])


# --------------------------------------------------------------------------------------------
# fit
# --------------------------------------------------------------------------------------------


def design_row(num_exp, den_exp, c, e, x, v):
    ne = np.ascontiguousarray(num_exp, dtype=np.int16)
    de = np.ascontiguousarray(den_exp, dtype=np.int16)
    n = ne.shape[1]
    c = np.ascontiguousarray(c, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    row = np.zeros(len(ne) + len(de), dtype=LD)
    lib().orc_design_row(n, len(ne), len(de), _p(ne), _p(de), _p(c), _p(e), _p(x), float(v), _p(row))
    return row


def gram(X, V, num_exp, den_exp, c, e, nthreads: int = 1):
    X = np.ascontiguousarray(X, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    K, n = X.shape
    ne = np.ascontiguousarray(num_exp, dtype=np.int16)
    de = np.ascontiguousarray(den_exp, dtype=np.int16)
    c = np.ascontiguousarray(c, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.int32)
    nc = len(ne) + len(de)
    G = np.zeros((nc, nc), dtype=LD)
    lib().orc_gram(_p(X), _p(V), K, n, len(ne), len(de), _p(ne), _p(de), _p(c), _p(e), _p(G), nthreads)
    return G


def solve(G, n_num: int):
    G = np.ascontiguousarray(G, dtype=LD)
    nc = G.shape[0]
    coef = np.zeros(nc, dtype=LD)
    r2 = np.zeros(1, dtype=LD)
    mp = np.zeros(1, dtype=LD)
    st = lib().orc_solve(_p(G), nc, n_num, _p(coef), _p(r2), _p(mp))
    return dict(coef=coef, status=int(st), resid2=r2[0], min_pivot=mp[0])


def fit(X, V, num_exp, den_exp, nthreads: int = 1, xform=None):
    """Oracle-fit: transform from the sample box, Gram, beta_0 = 1, solve."""
    if xform is None:
        lo, hi = minmax(X)
        c, e = xform_from_box(lo, hi)
    else:
        c, e = xform
    G = gram(X, V, num_exp, den_exp, c, e, nthreads)
    s = solve(G, len(num_exp))
    s.update(c=c, e=e, G=G)
    return s


def fit_sk(X, V, num_exp, den_exp, iters: int = 3, nthreads: int = 1):
    """Sanathanan-Koerner refit (NEXT row f4): `iters` weighted solves, weights 1/q_prev(x)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    K, n = X.shape
    ne = np.ascontiguousarray(num_exp, dtype=np.int16)
    de = np.ascontiguousarray(den_exp, dtype=np.int16)
    coef = np.zeros(len(ne) + len(de), dtype=LD)
    c = np.zeros(n)
    e = np.zeros(n, dtype=np.int32)
    st = lib().orc_fit_sk(_p(X), _p(V), K, n, len(ne), len(de), _p(ne), _p(de), iters, _p(coef), _p(c), _p(e),
                          nthreads)
    return dict(coef=coef, c=c, e=e, status=int(st))


def fit_svd(X, V, num_exp, den_exp):
    """Homogeneous least squares by one-sided Jacobi SVD (NEXT row f1): the right singular vector
    of the smallest singular value, beta_0 = 1.  Returns coef, ascending sigma, (c, e)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    K, n = X.shape
    ne = np.ascontiguousarray(num_exp, dtype=np.int16)
    de = np.ascontiguousarray(den_exp, dtype=np.int16)
    nc = len(ne) + len(de)
    coef = np.zeros(nc, dtype=LD)
    sigma = np.zeros(nc, dtype=LD)
    c = np.zeros(n)
    e = np.zeros(n, dtype=np.int32)
    st = lib().orc_fit_svd(_p(X), _p(V), K, n, len(ne), len(de), _p(ne), _p(de), _p(coef), _p(sigma), _p(c), _p(e))
    return dict(coef=coef, sigma=sigma, c=c, e=e, status=int(st))


def svd_rows(rows, n_num: int):
    """The oracle's Jacobi SVD of an explicit matrix rows [K][n_c] (e.g. stacked design rows of
    several shards): coef with beta_0 = 1 and ascending sigma (NEXT row f1)."""
    rows = np.ascontiguousarray(rows, dtype=LD)
    K, nc = rows.shape
    coef = np.zeros(nc, dtype=LD)
    sigma = np.zeros(nc, dtype=LD)
    st = lib().orc_svd_rows(_p(rows), K, nc, n_num, _p(coef), _p(sigma))
    return dict(coef=coef, sigma=sigma, status=int(st))
