/* rp_oracle.c -- CPU oracle of the rational-program hot path (arXiv 1911.02373).
 *
 * TEST INFRASTRUCTURE ONLY (see rp_oracle.h).  Never linked into, or called by, the product.
 *
 * Conventions.  "PAPER.md:L" is a line of /root/reference/PAPER.md (flattened ICPP chunk,
 * lines 1245-2998) with the section / equation / figure it falls in.  "R<k>" is reading k of
 * DESIGN.md "Readings" (the paper is silent, ambiguous or garbled there).  The MWP-CWP program
 * "E" is DESIGN.md Appendix A (reading R1: Hong & Kim ISCA'09 Eqs. 1-18, the model cited at
 * PAPER.md:1913), transcribed line by line below.
 *
 * parity pins: see tests/test_oracle_*.py (worked examples SPEC.md:224-246, 303, 57; the paper's
 * counts PAPER.md:1973-1977; closed forms; brute force; exact recovery PAPER.md:2227-2230).
 */
#include "rp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;

/* ------------------------------------------------------------------------------------------
 * a10 -- variable transform (reading R14; motivated by PAPER.md:2601-2611 "essentially a
 * Vandermonde matrix ... very ill-conditioned").  c = (lo+hi)/2, e = the least integer with
 * 2^e >= max((hi-lo)/2, 1).  u = (x - c) * 2^-e lies in [-1, 1] on the box and is exact for
 * integer data below 2^52.
 * ---------------------------------------------------------------------------------------- */
void orc_xform_from_box(int n, const double *lo, const double *hi, double *c, int *e) {
  for (int k = 0; k < n; ++k) {
    c[k] = (lo[k] + hi[k]) / 2.0;
    double h = (hi[k] - lo[k]) / 2.0;
    if (h < 1.0) h = 1.0;
    int ek = 0;
    while (ldexp(1.0, ek) < h) ++ek;
    e[k] = ek;
  }
}

void orc_minmax(const double *X, long long K, int n, double *lo, double *hi) {
  for (int k = 0; k < n; ++k) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (long long r = 0; r < K; ++r)
    for (int k = 0; k < n; ++k) {
      double x = X[r * n + k];
      if (x < lo[k]) lo[k] = x;
      if (x > hi[k]) hi[k] = x;
    }
}

static ld to_u(double x, double c, int e) { return ldexpl((ld)x - (ld)c, -e); }

/* Pi_k u_k^{e_k} by repeated multiplication (X_1^{u_1} ... X_n^{u_n}) */
static ld monomial(const short *exps, int n, const ld *u) {
  ld m = 1.0L;
  for (int k = 0; k < n; ++k)
    for (int t = 0; t < exps[k]; ++t) m *= u[k];
  return m;
}

/* ------------------------------------------------------------------------------------------
 * a5 -- occupancy.  Fig. occupancysimpleflowchart: four decision
 * diamonds tried top to bottom, first "Yes" wins, else "Failure to Launch" (B_active = 0).
 * All products in 64-bit integers (reading R9: integer parts are exact).
 * ---------------------------------------------------------------------------------------- */
long long orc_active_blocks(const orc_hw *hw, long long R, long long Z, long long T, int *branch) {
  const long long Bmax = hw->b_max, Wmax = hw->w_max, Rmax = hw->r_max, Zmax = hw->z_max;
  /* PAPER.md:1789 "T B_max <= 32 W_max and R T B_max <= R_max and Z B_max <= Z_max?" */
  if (T * Bmax <= 32 * Wmax && R * T * Bmax <= Rmax && Z * Bmax <= Zmax) {
    if (branch) *branch = 1;
    return Bmax; /* PAPER.md:1797 B_active = B_max */
  }
  /* PAPER.md:1791 "32 W_max <= T B_max, and 32 W_max R <= R_max and 32 W_max Z <= Z_max T?" */
  if (32 * Wmax <= T * Bmax && 32 * Wmax * R <= Rmax && 32 * Wmax * Z <= Zmax * T) {
    if (branch) *branch = 2;
    return (32 * Wmax) / T; /* PAPER.md:1798 floor(32 W_max / T) */
  }
  /* PAPER.md:1793 "R_max <= R T B_max and R_max <= R 32 W_max and R_max Z <= R T Z_max?" */
  if (Rmax <= R * T * Bmax && Rmax <= R * 32 * Wmax && Rmax * Z <= R * T * Zmax) {
    if (branch) *branch = 3;
    return Rmax / (R * T); /* PAPER.md:1799 floor(R_max / (R T)) */
  }
  /* PAPER.md:1795 "Z_max <= B_max Z and Z_max T <= 32 W_max Z and Z_max R T <= Z R_max?" */
  if (Zmax <= Bmax * Z && Zmax * T <= 32 * Wmax * Z && Zmax * R * T <= Z * Rmax) {
    if (branch) *branch = 4;
    return Zmax / Z; /* PAPER.md:1800 floor(Z_max / Z) */
  }
  if (branch) *branch = 5; /* PAPER.md:1802 "B_active = 0 (Failure to Launch)" */
  return 0;
}

/* Eq. (1): W_active = min(floor(B_active T / 32), W_max) */
long long orc_active_warps(const orc_hw *hw, long long R, long long Z, long long T) {
  long long B = orc_active_blocks(hw, R, Z, T, NULL);
  long long w = (B * T) / 32;
  return w < hw->w_max ? w : hw->w_max;
}

/* ------------------------------------------------------------------------------------------
 * a4 -- g(x) = p(u)/q(u), direct monomial sums in basis order.
 * ---------------------------------------------------------------------------------------- */
static ld eval_pq(const orc_ratfunc *f, const ld *u, ld *kappa) {
  ld p = 0, q = 0, pa = 0, qa = 0;
  for (int j = 0; j < f->n_num; ++j) {
    ld t = (ld)f->coef[j] * monomial(f->num_exp + (long)j * f->n_vars, f->n_vars, u);
    p += t;
    pa += fabsl(t);
  }
  for (int j = 0; j < f->n_den; ++j) {
    ld t = (ld)f->coef[f->n_num + j] * monomial(f->den_exp + (long)j * f->n_vars, f->n_vars, u);
    q += t;
    qa += fabsl(t);
  }
  if (kappa) {
    ld kp = pa / fabsl(p), kq = qa / fabsl(q);
    *kappa = kp > kq ? kp : kq;
  }
  return p / q;
}

void orc_eval_ratfunc(const orc_ratfunc *f, const double *xc, const int *xe, const double *X,
                      long long K, long double *out, long double *kappa) {
  ld u[ORC_MAX_VARS];
  for (long long r = 0; r < K; ++r) {
    for (int k = 0; k < f->n_vars; ++k) u[k] = to_u(X[r * f->n_vars + k], xc[k], xe[k]);
    out[r] = eval_pq(f, u, kappa ? &kappa[r] : NULL);
  }
}

static ld rel_gap(ld a, ld b) {
  ld m = fabsl(a) > fabsl(b) ? fabsl(a) : fabsl(b);
  return m > 0 ? fabsl(a - b) / m : 0.0L;
}

/* ------------------------------------------------------------------------------------------
 * a1..a7 -- one (D, P) pair: masks, occupancy, grid, g_i, then E (DESIGN.md Appendix A).
 * ---------------------------------------------------------------------------------------- */
int orc_eval_pair(const orc_program *pr, const int *D, const int *P, orc_trace *tr) {
  orc_trace t;
  memset(&t, 0, sizeof t);
  t.E = INFINITY;
  t.case_margin = INFINITY;
  const orc_hw *hw = &pr->hw;

  /* Appendix A line 1 -- "multiple of the warp size (32)" and "bounded over by the maximum
   * number of threads per block" (reading R5: <= T_max), and the footnote
   * "P1 P2 <= D1^2 is meaningful" (reading R6: non-strict). */
  /* reading R32: data parameters are sizes, D_k >= 1; a block dimension is >= 1 */
  for (int k = 0; k < pr->d; ++k)
    if (D[k] < 1) { t.mask = 6; goto done; }
  long long T = 1;
  for (int k = 0; k < pr->p; ++k) {
    if (P[k] < 1) { t.mask = 1; goto done; }
    T *= P[k];
    if (T > hw->t_max) { t.T = T; t.mask = 2; goto done; } /* stop before the product can wrap */
  }
  t.T = T;
  if (T % 32 != 0) { t.mask = 1; goto done; }
  if (T > hw->t_max) { t.mask = 2; goto done; }
  {
    long long pp = P[0];
    if (pr->p >= 2) pp *= P[1];
    if (pp > (long long)D[0] * D[0]) { t.mask = 3; goto done; }
  }

  /* line 2 -- B_active by the flowchart; B_active = 0 cannot launch */
  long long Z = pr->Z0 + pr->Z1 * T;
  t.B_active = orc_active_blocks(hw, pr->R, Z, T, &t.branch);
  if (t.B_active == 0) { t.mask = 4; goto done; }
  /* line 3 -- Eq. (1) */
  t.W_active = (t.B_active * T) / 32;
  if (t.W_active > hw->w_max) t.W_active = hw->w_max;
  /* line 4 -- grid "gx = ceil[N/bx]", one factor per tiled dimension */
  long long blocks = 1;
  for (int k = 0; k < pr->p && k < 3; ++k) {
    int j = pr->grid_map[k];
    if (j >= 0) blocks *= ((long long)D[j] + P[k] - 1) / P[k];
  }
  t.blocks = blocks;
  t.sm_active = blocks < hw->n_sm ? blocks : hw->n_sm;

  /* a4 -- fitted low-level metrics g_i(D, P) */
  {
    ld u[ORC_MAX_VARS];
    int n = pr->d + pr->p;
    for (int k = 0; k < pr->d; ++k) u[k] = to_u((double)D[k], pr->xc[k], pr->xe[k]);
    for (int k = 0; k < pr->p; ++k) u[pr->d + k] = to_u((double)P[k], pr->xc[pr->d + k], pr->xe[pr->d + k]);
    (void)n;
    t.kappa = 0;
    for (int i = 0; i < pr->n_metrics; ++i) {
      ld kap;
      t.g[i] = eval_pq(&pr->g[i], u, &kap);
      if (kap > t.kappa) t.kappa = kap;
    }
  }

  ld E;
  if (pr->e_template == ORC_TEMPLATE_G1) {
    E = t.g[0]; /* E := g_1 (used for SPEC.md:492-style pins) */
  } else {
    /* Appendix A lines 5-18 (Hong & Kim ISCA'09 Eqs. 1-18; reading R1, R2) */
    const ld g1 = t.g[0], g2 = t.g[1], g3 = t.g[2];
    const ld U = hw->uncoal_per_mw;
    const ld Wact = (ld)t.W_active, Bact = (ld)t.B_active, SMact = (ld)t.sm_active;
    ld Mem = g2 + g3;                                     /* 5 */
    ld Tot = g1 + g2 + g3;                                /* 5 */
    ld W_unc = g3 / Mem;                                  /* 6 [HK Eq.4] */
    ld W_coal = g2 / Mem;                                 /* 6 [HK Eq.5] */
    ld L_unc = (ld)hw->mem_ld + (U - 1) * (ld)hw->dd_unc; /* 7 [HK Eq.1] */
    ld L_coal = (ld)hw->mem_ld;                           /* 7 [HK Eq.2] */
    ld Mem_L = L_unc * W_unc + L_coal * W_coal;           /* 8 [HK Eq.3] */
    ld Dep = (ld)hw->dd_unc * U * W_unc + (ld)hw->dd_coal * W_coal; /* 9 [HK Eq.6] */
    ld MWP_nb = Mem_L / Dep;                              /* 10 [HK Eq.7] */
    ld BWpw = (ld)hw->freq_hz * (ld)hw->load_bytes_per_warp / Mem_L; /* 11 [HK Eq.8] */
    ld MWP_bw = (ld)hw->mem_bw / (BWpw * SMact);          /* 11 [HK Eq.9] */
    ld MWP = MWP_nb;                                      /* 12 [HK Eq.10] */
    if (MWP_bw < MWP) MWP = MWP_bw;
    if (Wact < MWP) MWP = Wact;
    ld Comp_c = (ld)hw->issue_cycles * Tot;               /* 13 [HK Eq.11] */
    ld Mem_c = L_unc * g3 + L_coal * g2;                  /* 13 [HK Eq.12] */
    ld CWP_full = (Mem_c + Comp_c) / Comp_c;              /* 14 [HK Eq.13] */
    ld CWP = CWP_full < Wact ? CWP_full : Wact;           /* 14 [HK Eq.14] */
    ld Rep = (ld)t.blocks / (Bact * SMact);               /* 15 [HK Eq.15], not ceiled (R18) */
    ld mwp_free = MWP_nb < MWP_bw ? MWP_nb : MWP_bw;
    ld margin = rel_gap(mwp_free, Wact);
    ld m2 = rel_gap(CWP_full, Wact);
    if (m2 < margin) margin = m2;
    if (MWP == Wact && CWP == Wact) {                     /* 16 [HK Eq.16] */
      t.mwp_case = 1;
      E = (Mem_c + Comp_c + Comp_c / Mem * (MWP - 1)) * Rep;
    } else {
      ld m3 = rel_gap(CWP, MWP);
      if (m3 < margin) margin = m3;
      if (CWP >= MWP || (Comp_c > Mem_c)) {               /* 17 [HK Eq.17] */
        if (!(CWP >= MWP)) {
          ld m4 = rel_gap(Comp_c, Mem_c);
          if (m4 < margin) margin = m4;
        }
        t.mwp_case = 2;
        E = (Mem_c * Wact / MWP + Comp_c / Mem * (MWP - 1)) * Rep;
      } else {                                            /* 18 [HK Eq.18] */
        ld m4 = rel_gap(Comp_c, Mem_c);
        if (m4 < margin) margin = m4;
        t.mwp_case = 3;
        E = (Mem_L + Comp_c * Wact) * Rep;
      }
    }
    t.MWP = MWP;
    t.CWP = CWP;
    t.case_margin = margin;
  }
  /* line 19 -- reading R17: a non-finite or non-positive estimate is not a candidate */
  if (!(isfinite(E) && E > 0)) { t.mask = 5; t.E = E; goto done; }
  t.E = E;
  t.feasible = 1;
done:
  if (tr) *tr = t;
  return t.feasible;
}

/* ------------------------------------------------------------------------------------------
 * a8 -- "an exhaustive search is feasible": for each D, the lowest index
 * j minimising E over the candidates, by a strict-< scan in index order (reading R15: exact
 * ties go to the lowest index).  OpenMP over D: disjoint outputs, so the result does not
 * depend on the thread count.
 * ---------------------------------------------------------------------------------------- */
void orc_sweep(const orc_program *pr, const int *D, long long nD, const int *F, int nF, int *idx,
               double *best, double *second, double *kappa, double *margin, long long *counters,
               int nthreads) {
  long long cnt[16];
  memset(cnt, 0, sizeof cnt);
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#endif
#pragma omp parallel num_threads(nthreads)
  {
    long long lc[16];
    memset(lc, 0, sizeof lc);
#pragma omp for schedule(static)
    for (long long i = 0; i < nD; ++i) {
      const int *Di = D + i * pr->d;
      ld b = INFINITY, s = INFINITY, kb = 0, mb = INFINITY, ms = INFINITY;
      int bi = -1;
      for (int j = 0; j < nF; ++j) {
        orc_trace tr;
        int ok = orc_eval_pair(pr, Di, F + (long)j * pr->p, &tr);
        lc[9]++;
        if (tr.branch >= 1 && tr.branch <= 5) lc[tr.branch - 1]++;
        if (tr.mask == 1 || tr.mask == 2) lc[10]++;
        if (tr.mask == 3) lc[11]++;
        if (tr.mask == 4) lc[12]++;
        if (tr.mask == 5) lc[13]++;
        if (!ok) continue;
        lc[8]++;
        if (tr.mwp_case >= 1) lc[4 + tr.mwp_case]++;
        if (tr.E < b) {
          s = b;
          ms = mb;
          b = tr.E;
          bi = j;
          kb = tr.kappa;
          mb = tr.case_margin;
        } else if (tr.E < s) {
          s = tr.E;
          ms = tr.case_margin;
        }
      }
      idx[i] = bi;
      best[i] = (double)b;
      second[i] = (double)s;
      if (kappa) kappa[i] = (double)kb;
      if (margin) margin[i] = (double)(mb < ms ? mb : ms);
    }
#pragma omp critical
    for (int k = 0; k < 16; ++k) cnt[k] += lc[k];
  }
  if (counters)
    for (int k = 0; k < 16; ++k) counters[k] = cnt[k];
}

/* ------------------------------------------------------------------------------------------
 * f2 -- one runtime decision: "there may be several configurations which, up to some margin,
 * optimize E.  Then, a secondary performance metric or some heuristic ... may be used to
 * refine the choice"; returns the six launch integers of the IO function
 * "(gx, gy, gz, bx, by, bz)".  Secondary metric: occupancy W_active /
 * W_max, then larger bx, smaller by, smaller bz (reading R28).
 * ---------------------------------------------------------------------------------------- */
int orc_decide(const orc_program *pr, const int *D, const int *F, int nF, double margin,
               double *E_out, int *out6, double *boundary) {
  ld best = INFINITY;
  int bi = -1;
  orc_trace *tr = (orc_trace *)malloc(sizeof(orc_trace) * (nF > 0 ? nF : 1));
  for (int j = 0; j < nF; ++j) {
    orc_eval_pair(pr, D, F + (long)j * pr->p, &tr[j]);
    if (tr[j].feasible && tr[j].E < best) {
      best = tr[j].E;
      bi = j;
    }
  }
  int choice = bi;
  ld bgap = INFINITY;
  if (bi >= 0 && margin > 0) {
    const ld lim = best * (1.0L + (ld)margin);
    for (int j = 0; j < nF; ++j) {
      if (!tr[j].feasible) continue;
      ld gap = fabsl(tr[j].E - lim) / best;
      if (gap < bgap) bgap = gap;
      if (!(tr[j].E <= lim)) continue;
      const int *Pj = F + (long)j * pr->p, *Pc = F + (long)choice * pr->p;
      int Pj1 = pr->p >= 2 ? Pj[1] : 1, Pc1 = pr->p >= 2 ? Pc[1] : 1;
      int Pj2 = pr->p >= 3 ? Pj[2] : 1, Pc2 = pr->p >= 3 ? Pc[2] : 1;
      int better;
      if (tr[j].W_active != tr[choice].W_active) better = tr[j].W_active > tr[choice].W_active;
      else if (Pj[0] != Pc[0]) better = Pj[0] > Pc[0];
      else if (Pj1 != Pc1) better = Pj1 < Pc1;
      else if (Pj2 != Pc2) better = Pj2 < Pc2;
      else better = j < choice;
      if (better) choice = j;
    }
  }
  for (int k = 0; k < 6; ++k) out6[k] = 0;
  if (choice >= 0) {
    const int *Pc = F + (long)choice * pr->p;
    for (int k = 0; k < 3; ++k) {
      const int Pk = k < pr->p ? Pc[k] : 1;
      const int j = k < pr->p ? pr->grid_map[k] : -1;
      out6[k] = j >= 0 ? (int)(((long long)D[j] + Pk - 1) / Pk) : 1; /* gx = ceil[N/bx] */
      out6[3 + k] = Pk;
    }
    *E_out = (double)tr[choice].E;
  } else {
    *E_out = INFINITY;
  }
  if (boundary) *boundary = (double)bgap;
  free(tr);
  return choice;
}

/* ------------------------------------------------------------------------------------------
 * a11 -- one row of the linearised system p(x) - V q(x) = 0: a = [M(u) | -V N(u)]
 * ("over-determined system of linear equations"; draft PAPER.md:2590-2598
 * "the sample matrix for the denominator polynomial appended to the sample matrix for the
 * numerator polynomial"; SPEC.md:303 worked example [1, 2, -3, -6]).
 * ---------------------------------------------------------------------------------------- */
void orc_design_row(int n, int n_num, int n_den, const short *num_exp, const short *den_exp,
                    const double *xc, const int *xe, const double *x, double v, long double *row) {
  ld u[ORC_MAX_VARS];
  for (int k = 0; k < n; ++k) u[k] = to_u(x[k], xc[k], xe[k]);
  for (int j = 0; j < n_num; ++j) row[j] = monomial(num_exp + (long)j * n, n, u);
  for (int j = 0; j < n_den; ++j) row[n_num + j] = -(ld)v * monomial(den_exp + (long)j * n, n, u);
}

/* a12 -- G = A^T A = sum_r a_r a_r^T ("linear least squares"; the normal
 * equations are the north star's reading R13 of "solved ... by the method of linear least
 * squares"). */
void orc_gram(const double *X, const double *V, long long K, int n, int n_num, int n_den,
              const short *num_exp, const short *den_exp, const double *xc, const int *xe,
              long double *G, int nthreads) {
  const int nc = n_num + n_den;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  nthreads = 1;
#endif
  if (nthreads < 1) nthreads = 1;
  ld *part = (ld *)calloc((size_t)nthreads * nc * nc, sizeof(ld));
#pragma omp parallel num_threads(nthreads)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    long long r0 = K * tid / nthreads, r1 = K * (tid + 1) / nthreads;
    ld *Gt = part + (size_t)tid * nc * nc;
    ld *row = (ld *)malloc(sizeof(ld) * nc);
    for (long long r = r0; r < r1; ++r) {
      orc_design_row(n, n_num, n_den, num_exp, den_exp, xc, xe, X + r * n, V[r], row);
      for (int i = 0; i < nc; ++i) {
        ld ai = row[i];
        ld *Gi = Gt + (size_t)i * nc;
        for (int j = i; j < nc; ++j) Gi[j] += ai * row[j];
      }
    }
    free(row);
  }
  for (int i = 0; i < nc; ++i)
    for (int j = i; j < nc; ++j) {
      ld s = 0;
      for (int t = 0; t < nthreads; ++t) s += part[(size_t)t * nc * nc + (size_t)i * nc + j];
      G[(size_t)i * nc + j] = s;
      G[(size_t)j * nc + i] = s;
    }
  free(part);
}

/* ------------------------------------------------------------------------------------------
 * a14 -- normalise beta_0 = 1 (reading R12; the homogeneous system of the draft footnote
 * PAPER.md:2595-2598) and solve the normal equations G_ff z = -G_{f,beta0} by Gaussian
 * elimination with partial pivoting.  Degenerate (rank-deficient) when a
 * pivot falls below 1e-30 * max|G_ff|.
 * ---------------------------------------------------------------------------------------- */
int orc_solve(const long double *G, int nc, int beta0, long double *coef, long double *resid2,
              long double *min_pivot) {
  const int m = nc - 1;
  ld *A = (ld *)malloc(sizeof(ld) * (size_t)m * (m + 1));
  int *col = (int *)malloc(sizeof(int) * m);
  for (int i = 0, k = 0; i < nc; ++i)
    if (i != beta0) col[k++] = i;
  ld amax = 0;
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < m; ++j) {
      A[(size_t)i * (m + 1) + j] = G[(size_t)col[i] * nc + col[j]];
      if (fabsl(A[(size_t)i * (m + 1) + j]) > amax) amax = fabsl(A[(size_t)i * (m + 1) + j]);
    }
    A[(size_t)i * (m + 1) + m] = -G[(size_t)col[i] * nc + beta0];
  }
  ld pmin = INFINITY;
  int status = 0;
  for (int k = 0; k < m; ++k) {
    int piv = k;
    for (int i = k + 1; i < m; ++i)
      if (fabsl(A[(size_t)i * (m + 1) + k]) > fabsl(A[(size_t)piv * (m + 1) + k])) piv = i;
    if (piv != k)
      for (int j = 0; j <= m; ++j) {
        ld tmp = A[(size_t)k * (m + 1) + j];
        A[(size_t)k * (m + 1) + j] = A[(size_t)piv * (m + 1) + j];
        A[(size_t)piv * (m + 1) + j] = tmp;
      }
    ld p = A[(size_t)k * (m + 1) + k];
    if (fabsl(p) < pmin) pmin = fabsl(p);
    if (!(fabsl(p) > 1e-30L * amax)) { status = 3; break; }
    for (int i = k + 1; i < m; ++i) {
      ld f = A[(size_t)i * (m + 1) + k] / p;
      if (f == 0) continue;
      for (int j = k; j <= m; ++j) A[(size_t)i * (m + 1) + j] -= f * A[(size_t)k * (m + 1) + j];
    }
  }
  if (status == 0) {
    ld *z = (ld *)malloc(sizeof(ld) * m);
    for (int i = m - 1; i >= 0; --i) {
      ld s = A[(size_t)i * (m + 1) + m];
      for (int j = i + 1; j < m; ++j) s -= A[(size_t)i * (m + 1) + j] * z[j];
      z[i] = s / A[(size_t)i * (m + 1) + i];
    }
    for (int i = 0; i < m; ++i) coef[col[i]] = z[i];
    coef[beta0] = 1.0L;
    free(z);
    if (resid2) {
      ld r = 0;
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) r += coef[i] * G[(size_t)i * nc + j] * coef[j];
      *resid2 = r;
    }
  }
  if (min_pivot) *min_pivot = pmin;
  free(A);
  free(col);
  return status;
}

/* ------------------------------------------------------------------------------------------
 * f4 -- Sanathanan-Koerner iteration (reading R29): the linearised residual p - V q of
 * PAPER.md:2578-2584 weighs each row by q(x_r); dividing by the previous q_{t-1}(x_r) makes the
 * minimised quantity approach sum_r (p/q - V)^2, the error of the fitted value itself.
 * ---------------------------------------------------------------------------------------- */
int orc_fit_sk(const double *X, const double *V, long long K, int n, int n_num, int n_den,
               const short *num_exp, const short *den_exp, int iters, long double *coef,
               double *c, int *e, int nthreads) {
  const int nc = n_num + n_den;
  double lo[ORC_MAX_VARS], hi[ORC_MAX_VARS];
  orc_minmax(X, K, n, lo, hi);
  orc_xform_from_box(n, lo, hi, c, e);
  ld *G = (ld *)calloc((size_t)nc * nc, sizeof(ld));
  ld *row = (ld *)malloc(sizeof(ld) * nc);
  ld *s = (ld *)malloc(sizeof(ld) * (K > 0 ? K : 1));
  int status = 0;
  for (int t = 0; t < iters; ++t) {
    if (t == 0) {
      orc_gram(X, V, K, n, n_num, n_den, num_exp, den_exp, c, e, G, nthreads);
    } else {
      /* s_r = 1 / q_{t-1}(x_r) with the previous coefficients (denominator block) */
      ld u[ORC_MAX_VARS];
      for (long long r = 0; r < K; ++r) {
        for (int k = 0; k < n; ++k) u[k] = to_u(X[r * n + k], c[k], e[k]);
        ld q = 0;
        for (int j = 0; j < n_den; ++j) q += coef[n_num + j] * monomial(den_exp + (long)j * n, n, u);
        s[r] = 1.0L / q;
      }
      memset(G, 0, sizeof(ld) * (size_t)nc * nc);
      for (long long r = 0; r < K; ++r) {
        orc_design_row(n, n_num, n_den, num_exp, den_exp, c, e, X + r * n, V[r], row);
        for (int i = 0; i < nc; ++i) row[i] *= s[r];
        for (int i = 0; i < nc; ++i)
          for (int j = i; j < nc; ++j) G[(size_t)i * nc + j] += row[i] * row[j];
      }
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < i; ++j) G[(size_t)i * nc + j] = G[(size_t)j * nc + i];
    }
    status = orc_solve(G, nc, n_num, coef, NULL, NULL);
    if (status != 0) break;
  }
  free(G);
  free(row);
  free(s);
  return status;
}

/* ------------------------------------------------------------------------------------------
 * f1 -- "we use the computationally more intensive yet more numerically stable method of
 * singular value decomposition" on "a system of homogeneous equations"
 * (draft): min ||A c|| over ||c|| = 1 is the right singular vector of the
 * smallest singular value.  One-sided Jacobi (Hestenes): rotate column pairs of A until they are
 * orthogonal; the rotations accumulate into V, the column norms are the singular values.
 * ---------------------------------------------------------------------------------------- */
/* one-sided Jacobi SVD of an explicit matrix A [K][nc] (row-major, long double copy made
 * here): coef = the right singular vector of the smallest singular value with beta_0 (column
 * n_num) = 1; sigma[nc] ascending.  Returns 0, or 3 if that vector's beta_0 is below 1e-300. */
int orc_svd_rows(const long double *rows, long long K, int nc, int n_num, long double *coef,
                 long double *sigma) {
  ld *A = (ld *)malloc(sizeof(ld) * (size_t)K * nc); /* column-major: A[j * K + r] */
  for (long long r = 0; r < K; ++r)
    for (int j = 0; j < nc; ++j) A[(size_t)j * K + r] = rows[(size_t)r * nc + j];
  ld *W = (ld *)calloc((size_t)nc * nc, sizeof(ld)); /* V of the SVD, column-major */
  for (int j = 0; j < nc; ++j) W[(size_t)j * nc + j] = 1.0L;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int i = 0; i < nc - 1; ++i)
      for (int j = i + 1; j < nc; ++j) {
        ld *ai = A + (size_t)i * K, *aj = A + (size_t)j * K;
        ld al = 0, be = 0, ga = 0;
        for (long long r = 0; r < K; ++r) {
          al += ai[r] * ai[r];
          be += aj[r] * aj[r];
          ga += ai[r] * aj[r];
        }
        if (ga == 0 || fabsl(ga) <= 1e-18L * sqrtl(al * be)) continue;
        rotated = 1;
        const ld zeta = (be - al) / (2 * ga);
        const ld t = (zeta >= 0 ? 1.0L : -1.0L) / (fabsl(zeta) + sqrtl(1 + zeta * zeta));
        const ld cs = 1 / sqrtl(1 + t * t), sn = cs * t;
        for (long long r = 0; r < K; ++r) {
          const ld x = ai[r], y = aj[r];
          ai[r] = cs * x - sn * y;
          aj[r] = sn * x + cs * y;
        }
        ld *wi = W + (size_t)i * nc, *wj = W + (size_t)j * nc;
        for (int r = 0; r < nc; ++r) {
          const ld x = wi[r], y = wj[r];
          wi[r] = cs * x - sn * y;
          wj[r] = sn * x + cs * y;
        }
      }
    if (!rotated) break;
  }
  /* singular values = column norms; pick the smallest */
  int jmin = 0;
  ld smin = INFINITY;
  for (int j = 0; j < nc; ++j) {
    ld s2 = 0;
    for (long long r = 0; r < K; ++r) s2 += A[(size_t)j * K + r] * A[(size_t)j * K + r];
    sigma[j] = sqrtl(s2);
    if (sigma[j] < smin) {
      smin = sigma[j];
      jmin = j;
    }
  }
  /* ascending order of sigma (insertion sort, nc <= a few hundred) */
  for (int a = 1; a < nc; ++a) {
    ld v = sigma[a];
    int b = a - 1;
    while (b >= 0 && sigma[b] > v) {
      sigma[b + 1] = sigma[b];
      --b;
    }
    sigma[b + 1] = v;
  }
  int status = 0;
  const ld b0 = W[(size_t)jmin * nc + n_num];
  if (!(fabsl(b0) > 1e-300L)) status = 3;
  for (int r = 0; r < nc; ++r) coef[r] = status ? NAN : W[(size_t)jmin * nc + r] / b0;
  free(A);
  free(W);
  return status;
}

int orc_fit_svd(const double *X, const double *V, long long K, int n, int n_num, int n_den,
                const short *num_exp, const short *den_exp, long double *coef, long double *sigma,
                double *c, int *e) {
  const int nc = n_num + n_den;
  double lo[ORC_MAX_VARS], hi[ORC_MAX_VARS];
  orc_minmax(X, K, n, lo, hi);
  orc_xform_from_box(n, lo, hi, c, e);
  ld *rows = (ld *)malloc(sizeof(ld) * (size_t)K * nc);
  for (long long r = 0; r < K; ++r)
    orc_design_row(n, n_num, n_den, num_exp, den_exp, c, e, X + r * n, V[r], rows + (size_t)r * nc);
  const int status = orc_svd_rows(rows, K, nc, n_num, coef, sigma);
  free(rows);
  return status;
}
