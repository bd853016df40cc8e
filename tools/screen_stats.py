"""Design statistics for a tensor-core (split-tf32) screened sweep, on the bench workload (CPU).

For a sample of `large` data tuples against all of F_large, with the `large` truth program (what
the bench's fit recovers to ~1e-11):
  * rho = sum_j |t_j| / |sum_j t_j| of each of the 2l polynomials (t_j its monomial terms in the
    u-variables): the cancellation factor that scales an FP32/tensor-core contraction's relative
    error (an upper bound on the staged contraction's own factor, by the triangle inequality);
  * per tuple, how many feasible configurations have E within eta (relative) of the minimum: the
    candidates a screen with relative error bound eta must re-evaluate in FP64.
Analysis only (calls oracle.eval_pair for E); not part of the product path.

  python tools/screen_stats.py [n_tuples]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def poly_terms(exps, coef, U):
    """terms [n_pairs][n_terms] of sum_j coef_j prod_k U[:, k]^exps[j, k]"""
    T = np.ones((U.shape[0], len(exps)))
    for j, e in enumerate(exps):
        for k, ek in enumerate(e):
            if ek:
                T[:, j] *= U[:, k] ** int(ek)
    return T * coef[None, :]


def main():
    nT = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    spec = synth.large_program()
    F = synth.F_large()
    D = synth.large_D(1_000_000)[:: 1_000_000 // nT][:nT]
    c, e = oracle.program_xform(spec)
    n = spec.d + spec.p
    X = np.concatenate([np.repeat(D, len(F), 0), np.tile(F, (len(D), 1))], 1).astype(np.float64)
    U = (X - c[None, :n]) * np.ldexp(1.0, -e[None, :n].astype(np.int64))
    rho, rho_st, rho_cs = [], [], []
    for i in range(spec.n_metrics):
        nn = len(spec.num_exp[i])
        for exps, cf in ((spec.num_exp[i], spec.coef[i][:nn]), (spec.den_exp[i], spec.coef[i][nn:])):
            exps = np.asarray(exps)
            T = poly_terms(exps, np.asarray(cf), U)
            p = T.sum(1)
            rho.append(np.abs(T).sum(1) / np.abs(p))
            # the staged form p = sum_pe C_pe(D) m_pe(P): group the terms by their P-exponents
            pes = sorted({tuple(e[spec.d:]) for e in exps})
            Cm = np.zeros((len(X), len(pes)))
            for j, e in enumerate(exps):
                Cm[:, pes.index(tuple(e[spec.d:]))] += T[:, j]
            mP = np.stack([np.prod(U[:, spec.d:] ** np.array(pe)[None, :], 1) for pe in pes], 1)
            C = Cm / np.where(mP == 0, 1, mP)
            rho_st.append(np.abs(Cm).sum(1) / np.abs(p))
            rho_cs.append(np.linalg.norm(C, axis=1) * np.linalg.norm(mP, axis=1) / np.abs(p))
    rho = np.max(np.stack(rho), 0)
    rho_st = np.max(np.stack(rho_st), 0)
    rho_cs = np.max(np.stack(rho_cs), 0)
    E = np.full(len(X), np.inf)
    for r in range(len(X)):
        t = oracle.eval_pair(spec, X[r, :spec.d].astype(np.int32), X[r, spec.d:].astype(np.int32))
        if t["feasible"]:
            E[r] = float(t["E"])
    feas = np.isfinite(E)
    out = {"tuples": nT, "configs": len(F), "feasible_pairs": int(feas.sum())}
    for R in (1.5, 2, 4, 8, 16, 64):
        out[f"frac_rho_gt_{R}"] = float(np.mean(rho[feas] > R))
    for name, r in (("full", rho), ("staged", rho_st), ("cauchy_schwarz", rho_cs)):
        out[f"rho_{name}_p50_p99_p999_max"] = [float(np.percentile(r[feas], q)) for q in (50, 99, 99.9)] + [float(r[feas].max())]
    E = E.reshape(nT, len(F))
    for eta in (1e-5, 1e-4, 3e-4, 1e-3):
        cnt = []
        for t in range(nT):
            m = E[t].min()
            if np.isfinite(m):
                cnt.append(int(np.sum(E[t] <= m * (1 + 2 * eta))))
        cnt = np.array(cnt)
        out[f"candidates_eta_{eta:g}"] = {"mean": float(cnt.mean()), "p99": float(np.percentile(cnt, 99)),
                                          "max": int(cnt.max())}
    import json
    print(json.dumps(out))


if __name__ == "__main__":
    main()
