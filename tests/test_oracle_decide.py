"""Pins for the oracle's runtime decision (NEXT row f2): "several configurations which, up to
some margin, optimize E ... a secondary performance metric or some heuristic ... may be used to
refine the choice", returning "(gx, gx, gz, bx, by, bz)" (PAPER.md:2490-2491,
typo for gy).  Pinned by SPEC.md's worked selection / CLI example, the grid-formula example,
margin 0 == the argmin, and brute force over tiny grids."""
import numpy as np

import oracle
import synth
from helpers import golden, ratfunc_program


def test_spec_selection_example():
    ex, grid_ex = golden("spec_worked.json")["decision"]
    F = synth.F_pow2_2d()
    spec = ratfunc_program(synth.HW_GTX1080TI, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2, R=16)
    r = oracle.decide(spec, [ex["N"]], F, margin=1e-9)
    assert tuple(F[r["idx"]]) == tuple(ex["block"])
    assert r["launch"] == tuple(ex["launch"])
    assert r["E"] == 4.0
    # margin 0: the plain argmin (lowest index among the exact ties)
    r0 = oracle.decide(spec, [ex["N"]], F, margin=0.0)
    assert r0["idx"] == oracle.sweep(spec, np.array([[ex["N"]]]), F)["idx"][0]
    # grid formula example: single configuration (32, 8)
    r = oracle.decide(spec, [grid_ex["N"]], np.array([grid_ex["block"]], dtype=np.int32))
    assert r["launch"][:3] == tuple(grid_ex["grid"])


def test_margin_zero_is_argmin():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    ref = oracle.sweep(spec, case.D, case.F)
    for i, d in enumerate(case.D):
        r = oracle.decide(spec, d, case.F, margin=0.0)
        assert r["idx"] == ref["idx"][i]
        assert (r["idx"] < 0) or r["E"] == ref["best"][i]


def test_brute_force_tie_break():
    """margin > 0: the candidate set {E <= best (1 + margin)} and the secondary order
    (W_active desc, bx desc, by asc, bz asc, index asc), checked by brute force."""
    case = synth.polybench_sweep(nD=30)
    spec = case.programs[1]
    for margin in (0.05, 0.5, 1e300):
        for d in case.D[:12]:
            tr = [oracle.eval_pair(spec, d, P) for P in case.F]
            cand = [j for j, t in enumerate(tr) if t["feasible"]]
            r = oracle.decide(spec, d, case.F, margin=margin)
            if not cand:
                assert r["idx"] == -1 and r["launch"] == (0,) * 6
                continue
            best = min(tr[j]["E"] for j in cand)
            ties = [j for j in cand if tr[j]["E"] <= best * (1 + np.longdouble(margin))]
            key = lambda j: (-tr[j]["W_active"], -case.F[j][0], case.F[j][1], case.F[j][2], j)
            assert r["idx"] == min(ties, key=key)
            P = case.F[r["idx"]]
            N = int(d[0])
            assert r["launch"] == ((N + P[0] - 1) // P[0], (N + P[1] - 1) // P[1], 1, P[0], P[1], P[2])
