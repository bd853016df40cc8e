"""Pins for the oracle's sweep + argmin (a1-a8): exhaustive search over F
with lowest-index tie-breaking (reading R15).

Pinned by: brute force over tiny grids; special cases (every P masked -> idx -1; duplicated
configs; SPEC.md:492's all-tie example); argmin invariance when all metrics are scaled by 7
(SPEC.md:514, 604); coverage of all MWP-CWP cases and occupancy branches 1-4.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import golden, ratfunc_program


def _brute(spec, D, F):
    out = []
    for d in D:
        Es = []
        for j, P in enumerate(F):
            tr = oracle.eval_pair(spec, d, P)
            if tr["feasible"]:
                Es.append((tr["E"], j))
        if not Es:
            out.append((-1, np.inf, np.inf))
            continue
        Es.sort()  # (E, index): lowest E, then lowest index
        best = Es[0]
        second = Es[1][0] if len(Es) > 1 else np.inf
        out.append((best[1], float(best[0]), float(second)))
    return out


def test_brute_force_tiny():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    res = oracle.sweep(spec, case.D, case.F)
    bf = _brute(spec, case.D, case.F)
    for i, (j, b, s) in enumerate(bf):
        assert res["idx"][i] == j
        assert res["best"][i] == b
        assert res["second"][i] == s


def test_brute_force_edge_D_polybench():
    case = synth.polybench_sweep(nD=4)
    spec = case.programs[3]
    D = np.concatenate([synth.random_D_edge_cases(1), case.D])
    res = oracle.sweep(spec, D, case.F)
    bf = _brute(spec, D, case.F)
    assert [r[0] for r in bf] == res["idx"].tolist()
    assert np.array_equal(np.array([r[1] for r in bf]), res["best"])


def test_all_masked_gives_minus_one():
    """D1 = 4: every P has P1 P2 >= 32 > 16 = D1^2, so nothing is meaningful."""
    case = synth.tiny_sweep()
    res = oracle.sweep(case.programs[0], np.array([[4], [1]], dtype=np.int32), case.F)
    assert res["idx"].tolist() == [-1, -1]
    assert np.all(np.isinf(res["best"])) and np.all(np.isinf(res["second"]))


def test_duplicate_config_earlier_index_wins():
    case = synth.tiny_sweep()
    spec = case.programs[0]
    res = oracle.sweep(spec, case.D, case.F)
    w = int(res["idx"][10])
    F2 = np.concatenate([case.F[:3], case.F[w:w + 1], case.F[3:]])  # copy of the winner at index 3
    res2 = oracle.sweep(spec, case.D[10:11], F2)
    assert res2["idx"][0] == 3 and res2["best"][0] == res["best"][10]
    assert res2["second"][0] == res2["best"][0]  # an exact tie makes second == best
    F3 = np.concatenate([case.F, case.F[w:w + 1]])  # copy at the end: the original wins
    assert oracle.sweep(spec, case.D[10:11], F3)["idx"][0] == w


def test_spec_all_tie_example():
    """E = N^2/(bx*by) at N = 64 ties every T = 1024 block; lowest index wins."""
    ex = golden("spec_worked.json")["selection"][0]
    F = synth.F_pow2_2d()
    spec = ratfunc_program(synth.HW_GTX1080TI, [[2, 0, 0]], [[0, 1, 1]], [1.0, 1.0], d=1, p=2, R=16)
    res = oracle.sweep(spec, np.array([[ex["N"]]], dtype=np.int32), F)
    ties = [j for j, P in enumerate(F) if P[0] * P[1] == ex["tie_product"]]
    assert res["idx"][0] == ties[0]
    assert res["best"][0] == res["second"][0] == 4.0


def test_argmin_invariant_to_scaling_metric_by_7():
    """scaling the predicted metric by 7 changes no choice (template E := g1)."""
    case = synth.tiny_sweep()
    spec = case.programs[0]
    import copy
    s1 = copy.deepcopy(spec)
    s1.template = "g1"
    s7 = copy.deepcopy(s1)
    s7.coef = [c.copy() for c in s1.coef]
    s7.coef[0][: len(s1.num_exp[0])] *= 7.0
    a = oracle.sweep(s1, case.D, case.F)
    b = oracle.sweep(s7, case.D, case.F)
    assert np.array_equal(a["idx"], b["idx"])
    np.testing.assert_allclose(b["best"], 7 * a["best"], rtol=1e-15)


def test_case_coverage():
    """All three MWP-CWP cases occur in `tiny` and in a `large` subsample."""
    tiny = synth.tiny_sweep()
    c = oracle.sweep(tiny.programs[0], tiny.D, tiny.F)["counters"]
    assert c["case1"] > 0 and c["case2"] > 0 and c["case3"] > 0
    large = synth.large_sweep(nD=1)
    D = synth.large_D()[::2500]
    c = oracle.sweep(large.programs[0], D, large.F)["counters"]
    assert c["case1"] > 0 and c["case2"] > 0 and c["case3"] > 0
    assert c["masked_static"] == len(D) * (1024 - 464)


def test_multikernel_branch_coverage():
    """The multikernel R/Z sets reach occupancy branches 1-4 and the B_active = 0 mask."""
    mk = synth.multikernel_sweep(nD=1)
    tot = {}
    for spec in mk.programs:
        c = oracle.sweep(spec, np.array([[16384]], dtype=np.int32), mk.F)["counters"]
        for k, v in c.items():
            tot[k] = tot.get(k, 0) + v
    for b in ("branch1", "branch2", "branch3", "branch4"):
        assert tot[b] > 0, tot
    assert tot["masked_B0"] > 0 and tot["branch5"] == 0


def test_thread_count_does_not_change_result():
    case = synth.polybench_sweep(nD=300)
    a = oracle.sweep(case.programs[0], case.D, case.F, nthreads=1)
    b = oracle.sweep(case.programs[0], case.D, case.F, nthreads=4)
    for k in ("idx", "best", "second"):
        assert np.array_equal(a[k], b[k])


def test_nonpositive_data_and_huge_blocks_are_masked():
    """Reading R32: data parameters are sizes (D_k >= 1) and block dimensions are >= 1; the
    product T = P1 P2 P3 stops at T_max instead of wrapping around in 64 bits."""
    case = synth.tiny_sweep()
    spec = case.programs[0]
    res = oracle.sweep(spec, np.array([[0], [-64], [-2147483647], [64]], dtype=np.int32), case.F)
    assert res["idx"][:3].tolist() == [-1, -1, -1] and res["idx"][3] >= 0
    for d in ([0], [-5]):
        tr = oracle.eval_pair(spec, np.array(d, dtype=np.int32), case.F[0])
        assert not tr["feasible"] and tr["mask"] == 6
    # (2^30, 2^30): the product 2^60 fits, but with a third factor of 16 it would wrap to 0 mod 2^64
    spec3 = synth.polybench_sweep(nD=1).programs[0]
    for P in ([1 << 30, 1 << 30, 16], [0, 32, 1], [-32, -1, 1], [2147483647, 2147483647, 2147483647]):
        tr = oracle.eval_pair(spec3, np.array([1000], dtype=np.int32), np.array(P, dtype=np.int32))
        assert not tr["feasible"] and tr["mask"] in (1, 2), P
