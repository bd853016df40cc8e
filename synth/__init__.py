"""Seeded synthetic inputs for the rational-program hot path.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the CUDA path
(``paper_1911_02373_b200/``).  It draws random numbers and enumerates index sets; it holds none
of the method's arithmetic: no occupancy, no masks, no variable transform, no rational-function
evaluation, no MWP-CWP program, no design rows, no Gram, no solve.  Noise-free metric values V
for a fit are NOT made here (that is rational-function evaluation): tests obtain them from the
oracle's evaluator, ``bench.py`` from the product's ``rp_eval_metrics``.

Recipe:
  * one global seed 1911023730 and a per-(config, stream) sub-seed from ``zlib.crc32`` (never the
    salted ``hash()``), numpy ``PCG64(SeedSequence([global, crc(config), crc(stream)]))``;
  * the five BASELINE configs ``tiny``, ``polybench``, ``large``, ``fitheavy``, ``multikernel``
    with the shapes of PAPER.md's workloads: data sizes N (or (D1, D2)) log-uniform integers,
    thread-block shapes from the CUDA rules of PAPER.md:2172-2177, 2284, profiled sample sets K
    in a box design (class F) or the paper's small-N launch design (class L,
    PAPER.md:2119-2120);
  * "class-F" program coefficients: generic, full-degree, pole-free on the transform box
    (SURVEY §8(d) "Program generators").  They are expressed in the centred variables u of the
    program's box; each side derives the transform from the box with its own code.
"""
from __future__ import annotations

import itertools
import math
import zlib
from dataclasses import dataclass, field

import numpy as np

GLOBAL_SEED = 1911023730

# --------------------------------------------------------------------------------------------
# seeding
# --------------------------------------------------------------------------------------------


def rng(config: str, stream: str = "") -> np.random.Generator:
    """Deterministic generator for (config, stream); independent of process and platform."""
    ss = np.random.SeedSequence([GLOBAL_SEED, zlib.crc32(config.encode()), zlib.crc32(stream.encode())])
    return np.random.Generator(np.random.PCG64(ss))


# --------------------------------------------------------------------------------------------
# monomial bases (explicit exponent lists; SURVEY §8(c) readings #10, #11)
# --------------------------------------------------------------------------------------------


def basis_total_degree(n_vars: int, degree: int) -> np.ndarray:
    """All exponent vectors e in N^n with |e| <= degree, graded by |e| then ascending
    lexicographic (first variable major).  The zero vector comes first (beta_0 slot)."""
    out = []
    for deg in range(degree + 1):
        level = [e for e in itertools.product(range(deg + 1), repeat=n_vars) if sum(e) == deg]
        out.extend(sorted(level))
    return np.asarray(out, dtype=np.int16).reshape(-1, n_vars)


def basis_box(bounds) -> np.ndarray:
    """All e with 0 <= e_k <= bounds[k] (the per-variable degree-bound display of
    PAPER.md:2567-2576), graded then ascending lexicographic."""
    ranges = [range(b + 1) for b in bounds]
    es = sorted(itertools.product(*ranges), key=lambda e: (sum(e), e))
    return np.asarray(es, dtype=np.int16).reshape(-1, len(bounds))


# --------------------------------------------------------------------------------------------
# configuration sets F; tuple order = index order
# --------------------------------------------------------------------------------------------

POW2 = [1 << k for k in range(11)]  # 1 .. 1024


def F_pow2_2d(t_lo: int = 32, t_hi: int = 1024) -> np.ndarray:
    """2-D power-of-two blocks (bx, by), t_lo <= bx*by <= t_hi, lexicographic."""
    F = [(bx, by) for bx in POW2 for by in POW2 if t_lo <= bx * by <= t_hi]
    return np.asarray(F, dtype=np.int32)


def F_pow2_3d(bz_max: int = 64, t_hi: int = 1024) -> np.ndarray:
    """3-D power-of-two blocks with bz <= bz_max and bx*by*bz <= t_hi (no warp rule: the
    method's mask removes T mod 32 != 0), lexicographic."""
    F = [(bx, by, bz) for bx in POW2 for by in POW2 for bz in POW2
         if bz <= bz_max and bx * by * bz <= t_hi]
    return np.asarray(F, dtype=np.int32)


def F_large() -> np.ndarray:
    """All integer (bx, by) in [1,1024]^2 with bx*by a multiple of 32 and <= 2048 (1,021
    tuples, lexicographic), then (1,1), (2,1), (4,1) appended: 1,024 configs.  Exercises the
    T <= T_max rule (T up to 2048) and the warp rule (the 3 appended tuples)."""
    F = [(bx, by) for bx in range(1, 1025) for by in range(1, 1025)
         if (bx * by) % 32 == 0 and bx * by <= 2048]
    F += [(1, 1), (2, 1), (4, 1)]
    return np.asarray(F, dtype=np.int32)


# --------------------------------------------------------------------------------------------
# data batches D
# --------------------------------------------------------------------------------------------


def tiny_sizes() -> np.ndarray:
    """N in {2^k, 1.5*2^k : k = 3..10}: 8, 12, 16, 24, ..., 1024, 1536 (16 sizes)."""
    out = []
    for k in range(3, 11):
        out += [1 << k, 3 << (k - 1)]
    return np.asarray(out, dtype=np.int32).reshape(-1, 1)


def log_uniform_ints(g: np.random.Generator, lo: int, hi: int, size) -> np.ndarray:
    """Integers log-uniform on [lo, hi] (floor of exp(U(log lo, log(hi+1))), clipped)."""
    x = np.exp(g.uniform(math.log(lo), math.log(hi + 1), size=size))
    return np.clip(np.floor(x), lo, hi).astype(np.int32)


# --------------------------------------------------------------------------------------------
# hardware fixtures H (any fixed values work for parity)
# --------------------------------------------------------------------------------------------

HW_GTX1080TI = dict(n_sm=28, w_max=64, b_max=32, t_max=1024, r_max=65536, z_max=24576,
                    freq_hz=1.582e9, mem_bw=484e9, load_bytes_per_warp=128.0, mem_ld=450.0,
                    dd_coal=4.0, dd_unc=40.0, uncoal_per_mw=32.0, issue_cycles=4.0)
HW_B200 = dict(n_sm=148, w_max=64, b_max=32, t_max=1024, r_max=65536, z_max=58368,
               freq_hz=1.965e9, mem_bw=8e12, load_bytes_per_warp=128.0, mem_ld=600.0,
               dd_coal=4.0, dd_unc=40.0, uncoal_per_mw=32.0, issue_cycles=4.0)
# SPEC.md:224-246 occupancy fixture (unit vectors only)
HW_SPEC_OCC = dict(HW_GTX1080TI, w_max=64, b_max=32, r_max=65536, z_max=12288, t_max=1024)

# metric scales (s_comp, s_coal, s_uncoal): chosen by a scan so that all three MWP-CWP cases
# occur in `tiny` and in the `large` sweep (tests/test_oracle_sweep.py::test_case_coverage)
METRIC_SCALES = (130.0, 100.0, 0.05)

# --------------------------------------------------------------------------------------------
# class-F coefficients (generic, full degree, pole-free on the box)
# --------------------------------------------------------------------------------------------


def classf_coefficients(g: np.random.Generator, basis: np.ndarray, scale: float) -> np.ndarray:
    """[alpha | beta] over ``basis`` for numerator and denominator, in the centred variables u
    of the program's box (|m_e(u)| <= 1 there):
      alpha_e, beta_e ~ U(-1,1) * 0.5^|e| for e != 0;  sum_{e!=0} |beta_e| rescaled to 0.5,
      beta_0 = 1 (so q in [0.5, 1.5]);  alpha_0 = 1 + sum |alpha_e| (so p >= 1); alpha *= scale.
    All coefficients nonzero (generic), hence a 1-D null space of the linearised system."""
    deg = basis.sum(axis=1).astype(np.float64)
    w = 0.5 ** deg
    a = g.uniform(-1.0, 1.0, size=len(basis)) * w
    b = g.uniform(-1.0, 1.0, size=len(basis)) * w
    b[1:] *= 0.5 / np.abs(b[1:]).sum()
    b[0] = 1.0
    a[0] = 1.0 + np.abs(a[1:]).sum()
    a *= scale
    return np.concatenate([a, b])


# --------------------------------------------------------------------------------------------
# program specs (the shared input description of a rational program R)
# --------------------------------------------------------------------------------------------


@dataclass
class ProgramSpec:
    """Rational program R = template E + l fitted g_i + H + kernel resources.

    ``coef[i]`` is [alpha (n_num) | beta (n_den)] in the u-variables of ``box`` (or of an
    explicit ``xform`` = (c, e) when the program comes from a fit)."""

    d: int
    p: int
    num_exp: list  # l arrays int16 [n_num][n]
    den_exp: list  # l arrays int16 [n_den][n]
    coef: list  # l arrays float64 [n_num + n_den]
    hw: dict
    R: int
    Z0: int
    Z1: int
    grid_map: tuple  # which D_j each P_k tiles (-1: grid dim 1)
    template: str = "mwpcwp"  # "mwpcwp" (Appendix A) or "g1" (E := g_1)
    box_lo: list | None = None
    box_hi: list | None = None
    xform_c: list | None = None
    xform_e: list | None = None

    @property
    def n_vars(self) -> int:
        return self.d + self.p

    @property
    def n_metrics(self) -> int:
        return len(self.coef)


def classf_program(config: str, d: int, p: int, degree: int, box_lo, box_hi, hw: dict, R: int,
                   Z0: int, Z1: int, grid_map, scales=METRIC_SCALES, stream: str = "prog",
                   template: str = "mwpcwp") -> ProgramSpec:
    g = rng(config, stream)
    basis = basis_total_degree(d + p, degree)
    coefs = [classf_coefficients(g, basis, s) for s in scales]
    return ProgramSpec(d=d, p=p, num_exp=[basis] * len(scales), den_exp=[basis] * len(scales),
                       coef=coefs, hw=dict(hw), R=R, Z0=Z0, Z1=Z1, grid_map=tuple(grid_map),
                       template=template, box_lo=list(box_lo), box_hi=list(box_hi))


# --------------------------------------------------------------------------------------------
# profiled sample sets K (box design: class F; launch design: class L)
# --------------------------------------------------------------------------------------------


def box_grid_design(lo, hi, per_dim: int) -> np.ndarray:
    """Full grid of round(linspace(lo_k, hi_k, per_dim)) per variable (contains both corners)."""
    axes = [np.round(np.linspace(l, h, per_dim)) for l, h in zip(lo, hi)]
    return np.asarray(list(itertools.product(*axes)), dtype=np.float64)


def box_random_design(g: np.random.Generator, lo, hi, K: int) -> np.ndarray:
    """K integer points uniform on the box; rows 0 and 1 are the all-lo and all-hi corners so
    the sample's per-variable min/max equal the box (the fit's transform then equals the
    truth's)."""
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    X = np.empty((K, len(lo)), dtype=np.float64)
    for k in range(len(lo)):
        X[:, k] = g.integers(lo[k], hi[k] + 1, size=K)
    if K >= 2:
        X[0] = lo
        X[1] = hi
    return X


def noise_multipliers(g: np.random.Generator, K: int, sigma: float) -> np.ndarray:
    """(1 + sigma * N(0,1)) per sample (SPEC.md simulate_profile)."""
    return 1.0 + sigma * g.standard_normal(K)


# --------------------------------------------------------------------------------------------
# the five BASELINE configs
# --------------------------------------------------------------------------------------------

TINY_BOX = ([8, 1, 1], [1536, 1024, 1024])
POLY_BOX = ([8, 1, 1, 1], [16384, 1024, 1024, 64])
LARGE_BOX = ([8, 8, 1, 1], [16384, 16384, 1024, 1024])
MK_R = (16, 24, 32, 40, 48, 64, 72, 80, 96, 128, 168, 255)
MK_Z0 = (0, 1024, 4096, 8192)
MK_Z1 = (0, 1, 2)


@dataclass
class SweepCase:
    name: str
    programs: list  # list[ProgramSpec]
    D: np.ndarray  # int32 [nD][d]
    F: np.ndarray  # int32 [nF][p]
    meta: dict = field(default_factory=dict)


def tiny_sweep(hw=HW_GTX1080TI) -> SweepCase:
    prog = classf_program("tiny", 1, 2, 2, *TINY_BOX, hw=hw, R=32, Z0=0, Z1=0, grid_map=(0, 0, -1))
    return SweepCase("tiny", [prog], tiny_sizes(), F_pow2_2d())


def polybench_sweep(hw=HW_GTX1080TI, nD: int = 10_000) -> SweepCase:
    """gemm, 2mm K1, 2mm K2, jacobi-2d: 4 class-F programs over (N, bx, by, bz)."""
    progs = []
    for i, (name, R) in enumerate([("gemm", 32), ("2mm_k1", 32), ("2mm_k2", 32), ("jacobi2d", 24)]):
        progs.append(classf_program("polybench", 1, 3, 3, *POLY_BOX, hw=hw, R=R, Z0=0, Z1=0,
                                    grid_map=(0, 0, -1), stream=f"prog/{name}"))
    D = log_uniform_ints(rng("polybench", "D"), 8, 16384, nD).reshape(-1, 1)
    return SweepCase("polybench", progs, D, F_pow2_3d(), meta={"kernels": ["gemm", "2mm_k1", "2mm_k2", "jacobi2d"]})


def large_program(hw=HW_GTX1080TI) -> ProgramSpec:
    """The 3 class-F truths that ``fitheavy`` samples, over (D1, D2, bx, by), degree <= 4."""
    return classf_program("large", 2, 2, 4, *LARGE_BOX, hw=hw, R=40, Z0=0, Z1=0, grid_map=(1, 0, -1))


def large_D(nD: int = 1_000_000) -> np.ndarray:
    g = rng("large", "D")
    return log_uniform_ints(g, 8, 16384, (nD, 2))


def large_sweep(hw=HW_GTX1080TI, nD: int = 1_000_000) -> SweepCase:
    return SweepCase("large", [large_program(hw)], large_D(nD), F_large())


def large_subsample_index(nD: int = 1_000_000, every: int = 100, edge: int = 100) -> np.ndarray:
    """Every ``every``-th D plus the first and last ``edge`` (SURVEY §8(d) oracle scope)."""
    idx = set(range(0, nD, every)) | set(range(min(edge, nD))) | set(range(max(0, nD - edge), nD))
    return np.asarray(sorted(idx), dtype=np.int64)


def multikernel_sweep(hw=HW_GTX1080TI, n_kernels: int = 20, nD: int = 10_000) -> SweepCase:
    progs = []
    for k in range(n_kernels):
        progs.append(classf_program("multikernel", 1, 3, 3, *POLY_BOX, hw=hw, R=MK_R[k % len(MK_R)],
                                    Z0=MK_Z0[k % len(MK_Z0)], Z1=MK_Z1[(k // len(MK_Z0)) % len(MK_Z1)],
                                    grid_map=(0, 0, -1), stream=f"prog/{k}"))
    D = log_uniform_ints(rng("multikernel", "D"), 8, 16384, nD).reshape(-1, 1)
    return SweepCase("multikernel", progs, D, F_pow2_3d())


@dataclass
class FitCase:
    name: str
    X: np.ndarray  # float64 [K][n]
    num_exp: np.ndarray
    den_exp: np.ndarray
    truths: list  # ProgramSpec holding the truths (coef in u of box)
    noise: np.ndarray | None  # [l][K] multipliers (1 + sigma*eps) or None
    meta: dict = field(default_factory=dict)


def tiny_fit_box(sigma: float = 0.0) -> FitCase:
    prog = tiny_sweep().programs[0]
    X = box_grid_design(*TINY_BOX, per_dim=4)
    noise = None
    if sigma:
        g = rng("tiny", "fitnoise")
        noise = np.stack([noise_multipliers(g, len(X), sigma) for _ in range(prog.n_metrics)])
    return FitCase("tiny-box", X, prog.num_exp[0], prog.den_exp[0], [prog], noise)


def polybench_fit_box(sigma: float = 0.0, K: int = 2000) -> FitCase:
    prog = polybench_sweep(nD=1).programs[0]
    X = box_random_design(rng("polybench", "K"), *POLY_BOX, K)
    noise = None
    if sigma:
        g = rng("polybench", "fitnoise")
        noise = np.stack([noise_multipliers(g, K, sigma) for _ in range(prog.n_metrics)])
    return FitCase("polybench-box", X, prog.num_exp[0], prog.den_exp[0], [prog], noise)


def fitheavy(sigma: float = 0.0, K: int = 1_000_000) -> FitCase:
    """K box-sampled points (D1, D2, bx, by) of the ``large`` truths, total degree <= 4
    (n_num = n_den = 70, n_c = 140)."""
    prog = large_program()
    X = box_random_design(rng("fitheavy", "K"), *LARGE_BOX, K)
    noise = None
    if sigma:
        g = rng("fitheavy", f"fitnoise/{sigma}")
        noise = np.stack([noise_multipliers(g, K, sigma) for _ in range(prog.n_metrics)])
    return FitCase("fitheavy", X, prog.num_exp[0], prog.den_exp[0], [prog], noise)


def random_D_edge_cases(d: int) -> np.ndarray:
    """Degenerate data tuples: smallest sizes (D1 < 32 fires P1*P2 <= D1^2), D1 = 1."""
    rows = [[1] * d, [4] * d, [5] * d, [31] * d, [32] * d, [33] * d]
    return np.asarray(rows, dtype=np.int32)


# --------------------------------------------------------------------------------------------
# class L (SURVEY 8(c) "parity classes", 8(d) "Program generators"): the paper's own regime --
# samples profiled at small data sizes and launch shapes and
# kernel-flavoured truths of lower degree than the fit's bounds (non-unique fits, PAPER.md:
# 2609-2615).  Diagnostics, not gated fits.
# --------------------------------------------------------------------------------------------


def launch_design_tiny() -> np.ndarray:
    """64 points: N in {32, 64, 128, 256} x 16 seeded configurations of the 2-D pow2 set."""
    g = rng("tiny", "launch")
    F = F_pow2_2d()
    rows = []
    for N in (32, 64, 128, 256):
        for j in g.choice(len(F), size=16, replace=False):
            rows.append([N, F[j][0], F[j][1]])
    return np.asarray(rows, dtype=np.float64)


def launch_design_poly(config: str = "polybench", K: int = 2000) -> np.ndarray:
    """K points: N log-uniform in [32, 512], P uniform over the 231 warp-valid 3-D pow2 shapes."""
    g = rng(config, "launch")
    F = F_pow2_3d()
    F = F[(F.prod(axis=1) % 32) == 0]
    N = log_uniform_ints(g, 32, 512, K)
    P = F[g.integers(0, len(F), size=K)]
    return np.concatenate([N.reshape(-1, 1), P], axis=1).astype(np.float64)


def _rat(terms_num, terms_den, n=4):
    """(exponent list, coefficient list) pairs of one rational function in raw x (identity transform)."""
    ne = np.zeros((len(terms_num), n), dtype=np.int16)
    de = np.zeros((len(terms_den), n), dtype=np.int16)
    cn, cd = [], []
    for i, (c, e) in enumerate(terms_num):
        ne[i, :len(e)] = e
        cn.append(c)
    for i, (c, e) in enumerate(terms_den):
        de[i, :len(e)] = e
        cd.append(c)
    return ne, de, np.asarray(cn + cd, dtype=np.float64)


# kernel-flavoured truths over x = (N, bx, by, bz): (comp, coal, uncoal) per thread
KERNEL_FAMILIES = {
    "gemm": (  # also 2mm K1
        ([(10.0, ()), (8.0, (1,))], [(1.0, ())]),
        ([(2.0, (1, 1)), (1.0, (0, 1))], [(8.0, ()), (1.0, (0, 1))]),
        ([(16.0, ()), (16.0, (1,)), (2.0, (0, 1))], [(8.0, ()), (1.0, (0, 1))]),
    ),
    "2mm_k2": (
        ([(12.0, ()), (9.0, (1,))], [(1.0, ())]),
        ([(2.0, (1, 1)), (1.0, (0, 1))], [(8.0, ()), (1.0, (0, 1))]),
        ([(16.0, ()), (16.0, (1,)), (2.0, (0, 1))], [(8.0, ()), (1.0, (0, 1))]),
    ),
    "jacobi2d": (
        ([(14.0, ())], [(1.0, ())]),
        ([(6.0, (0, 1))], [(2.0, ()), (1.0, (0, 1))]),
        ([(12.0, ())], [(2.0, ()), (1.0, (0, 1))]),
    ),
}


def kernel_truth(family: str, hw=HW_GTX1080TI, R: int = 32, Z0: int = 0, Z1: int = 0, scale=None) -> ProgramSpec:
    """A kernel-flavoured truth as a program in the raw variables (identity transform); `scale`
    optionally multiplies each metric's numerator constants (the multikernel perturbations)."""
    num, den, coef = [], [], []
    for i, (tn, td) in enumerate(KERNEL_FAMILIES[family]):
        ne, de, c = _rat(tn, td)
        if scale is not None:
            c = c.copy()
            c[:len(ne)] *= scale[i]
        num.append(ne)
        den.append(de)
        coef.append(c)
    return ProgramSpec(d=1, p=3, num_exp=num, den_exp=den, coef=coef, hw=dict(hw), R=R, Z0=Z0, Z1=Z1,
                       grid_map=(0, 0, -1), xform_c=[0.0] * 4, xform_e=[0] * 4)


@dataclass
class ClassLCase:
    name: str
    X: np.ndarray            # launch-design samples [K][n]
    truths: list             # ProgramSpec per program (the data generators)
    basis: np.ndarray        # the fit's basis (numerator = denominator)
    noise: list              # per program [l][K] multipliers
    sweep: SweepCase         # the D x F grid the fitted programs are swept over
    fit_programs: list       # ProgramSpec per program: H, resources, grid rule of the swept kernel


def classL_case(name: str, sigma: float = 0.01, n_kernels: int = 20) -> ClassLCase:
    """tiny: the class-F truth on the launch design (degree <= 2); polybench: gemm, 2mm K1/K2,
    jacobi-2d kernel-flavoured truths; multikernel: seeded constant-perturbations of the three
    families with the multikernel resources (degree <= 3 in (N, bx, by, bz))."""
    if name == "tiny":
        sw = tiny_sweep()
        X = launch_design_tiny()
        truths = sw.programs
        basis = sw.programs[0].num_exp[0]
        fit_programs = sw.programs
    elif name == "polybench":
        sw = polybench_sweep()
        X = launch_design_poly("polybench")
        fams = ["gemm", "gemm", "2mm_k2", "jacobi2d"]
        truths = [kernel_truth(f, R=p.R) for f, p in zip(fams, sw.programs)]
        basis = sw.programs[0].num_exp[0]
        fit_programs = sw.programs
    elif name == "multikernel":
        sw = multikernel_sweep(n_kernels=n_kernels)
        X = launch_design_poly("multikernel")
        g = rng("multikernel", "perturb")
        fams = ["gemm", "2mm_k2", "jacobi2d"]
        truths = [kernel_truth(fams[k % 3], R=p.R, Z0=p.Z0, Z1=p.Z1, scale=g.uniform(0.8, 1.2, size=3))
                  for k, p in enumerate(sw.programs)]
        basis = sw.programs[0].num_exp[0]
        fit_programs = sw.programs
    else:
        raise ValueError(name)
    g = rng(name, "launch-noise")
    noise = [np.stack([noise_multipliers(g, len(X), sigma) for _ in range(3)]) for _ in truths]
    return ClassLCase(name, X, truths, basis, noise, sw, fit_programs)

