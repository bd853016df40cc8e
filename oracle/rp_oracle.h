/* rp_oracle.h -- CPU oracle of the rational-program hot path (arXiv 1911.02373, KLARAPTOR).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA product (paper_1911_02373_b200/, include/rp.h).
 *
 * Plain, slow and obviously correct: x87 `long double` (64-bit mantissa) arithmetic, direct
 * monomial sums, a strict-< scan over F in index order, the Gram as a plain sum of outer
 * products in row order, Gaussian elimination with partial pivoting.  Every function cites the
 * PAPER.md passage (line, section/equation/figure) it follows; where the paper is silent the
 * reading is the numbered one in DESIGN.md "Readings".
 */
#ifndef RP_ORACLE_H
#define RP_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_VARS 8
#define ORC_MAX_METRICS 3

/* f = p/q with explicit exponent lists (display of f_b = p_b/q_b). */
typedef struct {
  int n_vars, n_num, n_den;
  const short *num_exp; /* [n_num][n_vars] */
  const short *den_exp; /* [n_den][n_vars] */
  const double *coef;   /* alpha[n_num] then beta[n_den], in the u-variables */
} orc_ratfunc;

/* hardware parameters H (PAPER.md:1870-1878 Ex. ex:cuda; 1915-1918 Ex. ex:mwpcwp) */
typedef struct {
  long long n_sm, w_max, b_max, t_max, r_max, z_max;
  double freq_hz, mem_bw, load_bytes_per_warp, mem_ld, dd_coal, dd_unc, uncoal_per_mw,
      issue_cycles;
} orc_hw;

enum { ORC_TEMPLATE_MWPCWP = 0, ORC_TEMPLATE_G1 = 1 };

typedef struct {
  int d, p, n_metrics, e_template;
  orc_ratfunc g[ORC_MAX_METRICS];
  double xc[ORC_MAX_VARS]; /* variable transform u = (x - c) * 2^-e   (reading R14) */
  int xe[ORC_MAX_VARS];
  orc_hw hw;
  long long R, Z0, Z1; /* regs/thread; shared words per block = Z0 + Z1*T */
  int grid_map[3];     /* P_k tiles D_{grid_map[k]}; -1: that grid dimension is 1 */
} orc_program;

/* per-pair trace for tests */
typedef struct {
  int feasible;   /* 1 if E is a candidate */
  int mask;       /* 0 ok, 1 warp rule / P_k < 1, 2 T > T_max, 3 P1*P2 > D1^2, 4 B_active = 0, 5 E invalid,
                     6 some D_k < 1 (reading R32) */
  int branch;     /* occupancy flowchart branch 1..5 (0 if not reached) */
  int mwp_case;   /* 1..3 (0 if not reached / template g1) */
  long long T, B_active, W_active, blocks, sm_active;
  long double g[ORC_MAX_METRICS];
  long double kappa; /* max over the 2*l polynomials of sum|c m| / |sum c m| */
  long double MWP, CWP, E;
  long double case_margin; /* min relative gap of the case decisions taken */
} orc_trace;

/* ---- a10: variable transform ---------------------------------------------------------- */
void orc_xform_from_box(int n, const double *lo, const double *hi, double *c, int *e);
void orc_minmax(const double *X, long long K, int n, double *lo, double *hi);

/* ---- a5: occupancy (Fig. occupancysimpleflowchart, Eq. (1)) --------------------------- */
long long orc_active_blocks(const orc_hw *hw, long long R, long long Z, long long T, int *branch);
long long orc_active_warps(const orc_hw *hw, long long R, long long Z, long long T);

/* ---- a4: rational functions ------------------------------------------------------------ */
/* g(x) at K points x (row-major [K][n], x-space); out[K] long double, kappa[K] nullable */
void orc_eval_ratfunc(const orc_ratfunc *f, const double *xc, const int *xe, const double *X,
                      long long K, long double *out, long double *kappa);

/* ---- a1..a7: one (D,P) pair ------------------------------------------------------------ */
int orc_eval_pair(const orc_program *prog, const int *D, const int *P, orc_trace *tr);

/* ---- a1..a8: sweep + argmin --------------------------------------------------------------
 * idx[nD] (-1 if none feasible), best[nD] (+inf), second[nD] (+inf), kappa[nD] (nullable:
 * kappa at the winner), margin[nD] (nullable: min case_margin over winner and runner-up),
 * counters[16] (nullable): [0..4] occupancy branches 1..5 over statically valid pairs,
 * [5..7] MWP-CWP cases 1..3 over feasible pairs, [8] feasible pairs, [9] total pairs,
 * [10] masked by warp/T_max, [11] masked by P1P2<=D1^2, [12] B_active=0, [13] E invalid.   */
void orc_sweep(const orc_program *prog, const int *D, long long nD, const int *F, int nF,
               int *idx, double *best, double *second, double *kappa, double *margin,
               long long *counters, int nthreads, int *idx2, double *kappa2);
/* idx2[nD] (nullable): the runner-up's index (-1 if none; on an exact tie with the winner, the
 * next lowest index); kappa2[nD] (nullable): kappa at the runner-up.                          */

/* The same two functions in IEEE binary128 (__float128, 113-bit mantissa): the identical
 * transcription (rp_oracle_pair.inc) with 49 more mantissa bits than x87 long double.  For
 * fitted programs whose polynomials cancel (kappa up to ~1e7) the long double evaluation is
 * accurate to ~1e-13 only; these are accurate to ~1e-28 there.  Trace values are rounded to long
 * double on output.  Soft-float: ~50x slower than orc_eval_pair.                              */
int orc_eval_pair_q(const orc_program *prog, const int *D, const int *P, orc_trace *tr);
void orc_sweep_q(const orc_program *prog, const int *D, long long nD, const int *F, int nF,
                 int *idx, double *best, double *second, double *kappa, double *margin,
                 long long *counters, int nthreads, int *idx2, double *kappa2);

/* ---- f2: runtime decision (PAPER.md:2292-2305 step 5, 2490-2491 the six launch integers) --
 * margin == 0: the argmin of orc_sweep.  margin > 0: among the candidates with
 * E <= best (1 + margin) pick the one with the larger W_active (occupancy), then larger P1,
 * smaller P2, smaller P3, lower index (SPEC.md:489's secondary metric; reading R28).
 * out6 = (gx, gy, gz, bx, by, bz) of the choice (grid rule), zeros if none;
 * boundary = min over candidates of |E - best (1 + margin)| / best (diagnostic).              */
int orc_decide(const orc_program *prog, const int *D, const int *F, int nF, double margin,
               double *E_out, int *out6, double *boundary);

/* ---- a11..a14: least-squares fit ------------------------------------------------------- */
void orc_design_row(int n, int n_num, int n_den, const short *num_exp, const short *den_exp,
                    const double *xc, const int *xe, const double *x, double v, long double *row);
/* G[n_c][n_c] = sum_r a_r a_r^T (rows in order; nthreads contiguous row blocks summed in
 * thread order) */
void orc_gram(const double *X, const double *V, long long K, int n, int n_num, int n_den,
              const short *num_exp, const short *den_exp, const double *xc, const int *xe,
              long double *G, int nthreads);
/* beta_0 := 1 (column n_num), solve G_ff z = -G_{f,beta0} by partial-pivoting elimination.
 * coef[n_c]; returns 0 or 3 (degenerate).  resid2 = coef^T G coef; min_pivot = min |pivot|. */
int orc_solve(const long double *G, int n_c, int beta0, long double *coef, long double *resid2,
              long double *min_pivot);

/* ---- f4: Sanathanan-Koerner reweighted refit ----------------------------------------------
 * iters >= 1 solves; solve 1 is orc_gram + orc_solve; solve t > 1 weights row r by
 * s_r = 1 / q_{t-1}(x_r) (q of the previous solve, long double), i.e. minimises
 * sum_r ((p(x_r) - V_r q(x_r)) / q_{t-1}(x_r))^2 (reading R29).  The transform comes from the
 * sample box.  Returns the status of the last solve; coef[n_c], c[n], e[n] out.             */
int orc_fit_sk(const double *X, const double *V, long long K, int n, int n_num, int n_den,
               const short *num_exp, const short *den_exp, int iters, long double *coef,
               double *c, int *e, int nthreads);

/* ---- f1: the homogeneous system by SVD (draft footnote 2595-2598) -----
 * A = rows a_r = [M(u_r) | -V_r N(u_r)] (transform from the sample box), formed explicitly in
 * long double; one-sided (Hestenes) Jacobi SVD of A; coef = the right singular vector of the
 * smallest singular value scaled so that beta_0 = 1 (SPEC.md:33 canonical form).  sigma[n_c]
 * ascending.  Returns 0, or 3 if |beta_0| of that vector is below 1e-300 (degenerate).       */
int orc_svd_rows(const long double *rows, long long K, int nc, int n_num, long double *coef,
                 long double *sigma);
int orc_fit_svd(const double *X, const double *V, long long K, int n, int n_num, int n_den,
                const short *num_exp, const short *den_exp, long double *coef, long double *sigma,
                double *c, int *e);

#ifdef __cplusplus
}
#endif
#endif
