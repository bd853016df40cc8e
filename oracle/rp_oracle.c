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

#define REAL ld
#define RABS(x) fabsl(x)
#define RFINITE(x) isfinite(x)
#define ORC_PFX(name) name
#include "rp_oracle_pair.inc"

void orc_eval_ratfunc(const orc_ratfunc *f, const double *xc, const int *xe, const double *X,
                      long long K, long double *out, long double *kappa) {
  ld u[ORC_MAX_VARS];
  for (long long r = 0; r < K; ++r) {
    for (int k = 0; k < f->n_vars; ++k) u[k] = to_u(X[r * f->n_vars + k], xc[k], xe[k]);
    out[r] = eval_pq(f, u, kappa ? &kappa[r] : NULL);
  }
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
