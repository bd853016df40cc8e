/* rp.h -- C ABI of librp, the B200 (sm_100a) hot path of the rational-program method of
 * arXiv 1911.02373 (KLARAPTOR: "rational programs" that pick CUDA launch parameters).
 *
 * Two halves, following the paper's statement of the problem:
 *   - compile time, step 2 "Rational function estimation":
 *     given the profiled points K with measured values V, find g_i = p_i/q_i by linear least
 *     squares on the linearised system p(x) - V q(x) = 0  ->  rp_fit (and its split form
 *     rp_minmax / rp_xform_from_box / rp_gram_accumulate / rp_solve_normal for K-sharding);
 *   - run time, steps 4-5 "Rational program evaluation" and "Selection of optimal values of
 *     program parameters": for each data tuple D evaluate the rational
 *     program R over all practically meaningful configurations P in F and take the argmin
 *     ->  rp_eval_argmin / rp_eval_argmin_batched / rp_plan_*.
 *
 * The estimate E is the MWP-CWP program of DESIGN.md Appendix A (PAPER.md:1909-1933 names the
 * model; its equations are Hong & Kim ISCA'09 Eqs. 1-18, reading R1) fed by l = 3 fitted
 * metrics (comp, coal, uncoal instructions per thread; reading R2), the occupancy flowchart
 * (Fig. occupancysimpleflowchart; Eq. (1)) and the grid
 * rule gx = ceil[N/bx].
 *
 * Conventions (all functions):
 *   - Return an rp_status; on failure rp_last_error() returns a thread-local message.
 *     Argument checks happen before any launch.  Nothing is written on failure except where
 *     stated.  Per-D infeasibility is data (idx -1, E +inf), never an error.
 *   - "device-or-host" pointers may be either: the library inspects them with
 *     cudaPointerGetAttributes; host inputs are staged through internal device workspace and
 *     host outputs are copied back before return (the call then synchronises the stream).
 *     With device pointers everything is stream-ordered and asynchronous unless noted.
 *   - The caller owns every buffer it passes.  The library owns only internal workspace
 *     (cached per device, freed at unload) and rp_plan objects (freed by rp_plan_destroy).
 *   - rp_stream is a cudaStream_t (NULL = the legacy default stream).
 *   - Every arithmetic step runs in the library's CUDA kernels; there is no CPU fallback.  On a
 *     machine without a CUDA device every compute entry point returns RP_ERR_CUDA.
 */
#ifndef RP_H
#define RP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RP_ABI_VERSION 1
#define RP_MAX_VARS 8    /* n = d + p variables (data parameters first, then program ones) */
#define RP_MAX_METRICS 3 /* l fitted metrics per rational program */

typedef enum {
  RP_OK = 0,
  RP_ERR_INVALID_ARG = 1,
  RP_ERR_CUDA = 2,
  RP_ERR_DEGENERATE = 3,  /* rank-deficient / non-SPD normal equations */
  RP_ERR_NO_FEASIBLE = 4, /* reserved */
  RP_ERR_UNSUPPORTED = 5  /* size or layout outside the compiled limits */
} rp_status;

typedef void *rp_stream;

/* A monomial basis as an explicit exponent list (the display of
 * f_b = p_b/q_b; reading R10).  Row j of num_exp is the exponent vector of alpha_j's monomial.
 * For a fit, den_exp[0] must be the zero vector: its coefficient beta_0 is normalised to 1
 * (reading R12).  Host pointers, read during the call only.                                  */
typedef struct {
  int32_t n_vars, n_num, n_den;
  const int16_t *num_exp; /* host int16 [n_num][n_vars] */
  const int16_t *den_exp; /* host int16 [n_den][n_vars] */
} rp_basis;

/* Variable transform u_k = (x_k - c_k) * 2^-e_k (reading R14; PAPER.md:2601-2611 motivates
 * it: the monomial system is "essentially a Vandermonde matrix" and "very ill-conditioned").
 * Coefficients always live in the u-variables.                                             */
typedef struct {
  double c[RP_MAX_VARS];
  int32_t e[RP_MAX_VARS];
} rp_xform;

/* Hardware parameters H (Ex. ex:cuda PAPER.md:1870-1878; Ex. ex:mwpcwp PAPER.md:1915-1918),
 * fixed at compile time of the user program (Obs. obs:faisability).
 * r_max / z_max are per SM (reading R3); z in 4-byte words.                                */
typedef struct {
  int32_t n_sm, w_max, b_max, t_max;
  int64_t r_max, z_max;
  double freq_hz, mem_bw, load_bytes_per_warp, mem_ld, dd_coal, dd_unc, uncoal_per_mw,
      issue_cycles;
} rp_hw;

typedef enum {
  RP_TEMPLATE_MWPCWP = 0, /* E = DESIGN.md Appendix A, metrics (comp, coal, uncoal)        */
  RP_TEMPLATE_G1 = 1      /* E = g_1 (the fitted metric itself), same masks               */
} rp_template;

/* The rational program R (step 3: "the CFG for computing E" plus one
 * sub-routine per fitted g_i).  Host struct; all pointers host, read during the call.       */
typedef struct {
  int32_t d, p;        /* numbers of data / program parameters; n = d + p <= RP_MAX_VARS, p <= 3 */
  int32_t n_metrics;   /* l; 3 for RP_TEMPLATE_MWPCWP, >= 1 for RP_TEMPLATE_G1              */
  int32_t e_template;  /* rp_template                                                        */
  rp_basis basis[RP_MAX_METRICS];
  const double *coef[RP_MAX_METRICS]; /* host float64 [n_num + n_den]: alpha then beta      */
  rp_xform xform;
  rp_hw hw;
  int32_t regs_per_thread;  /* R: registers per thread of the tuned kernel                 */
  int32_t grid_map[3];      /* P_k tiles D_{grid_map[k]} (gx = ceil(D/P_k)); -1: dimension 1 */
  int64_t smem_words_base;  /* Z = smem_words_base + smem_words_per_thread * T (words/block) */
  int64_t smem_words_per_thread;
} rp_program;

typedef struct {
  int32_t rank;      /* n_c - 1 on success                                                  */
  int32_t status;    /* rp_status of the solve                                              */
  double resid2;     /* coef^T G coef = sum_r (p(x_r) - V_r q(x_r))^2                        */
  double min_pivot;  /* smallest pivot of the equilibrated Cholesky factor (squared diag)   */
  double cond_est;   /* (max pivot / min pivot) of the equilibrated factorisation          */
  int32_t iters;     /* solves (rp_fit: 1, rp_fit_sk: iters) or Jacobi sweeps (rp_fit_svd)  */
  int32_t reserved;
} rp_fit_info;

/* ---- library --------------------------------------------------------------------------- */
int32_t rp_abi_version(void);
const char *rp_last_error(void);
/* Number of CUDA devices visible (0 without a GPU).  Never fails.                          */
int32_t rp_device_count(void);

/* ---- a10: transform -----------------------------------------------------------------------
 * rp_xform_from_box: c_k = (lo_k + hi_k)/2; e_k = least integer with 2^e_k >=
 * max((hi_k - lo_k)/2, 1), computed by a one-thread kernel on the legacy default stream
 * (synchronises).  lo, hi host float64 [n]; out host.  INVALID_ARG if n not in
 * [1, RP_MAX_VARS] or hi < lo.  rp_fit computes the same transform on the device without a
 * host round trip of the box.                                                               */
rp_status rp_xform_from_box(int32_t n, const double *lo, const double *hi, rp_xform *out);

/* rp_minmax: per-column min and max of X (device-or-host float64 [K][n], row-major) into host
 * lo[n], hi[n].  Synchronises.  INVALID_ARG if K < 1 or n out of range.                     */
rp_status rp_minmax(const double *X, int64_t K, int32_t n, double *lo, double *hi,
                    rp_stream s);

/* ---- a11-a12: Gram of the linearised system ---------------------------
 * G[m][n_c][n_c] (device-or-host float64, overwritten) = A_m^T A_m with, for row r of X,
 * a_r = [ M(u_r) | -V_m[r] N(u_r) ], M / N the numerator / denominator monomials of `basis`
 * in basis order (n_c = n_num + n_den), u_r = (X_r - c) 2^-e.  X device-or-host float64
 * [K][n]; V device-or-host float64 [n_v][K] (n_v >= 1 metrics sharing X).  Rows are split
 * over CTAs and the per-CTA partial Grams are summed in a fixed order (deterministic).
 * K = 0 gives G = 0.  UNSUPPORTED if n_c > 176 (shared-memory tile of the DMMA kernel).                                             */
rp_status rp_gram_accumulate(const double *X, const double *V, int64_t K, int32_t n_v,
                             const rp_basis *basis, const rp_xform *xform, double *G,
                             rp_stream s);

/* ---- a14: normalise + solve --------------------------------------------
 * For each of n_v Grams G (device-or-host float64 [n_v][n_c][n_c]): fix beta_0 = 1 (column
 * n_num) and solve G_ff z = -G_{f,beta0} by Jacobi-equilibrated Cholesky with one step of
 * iterative refinement (residual in double-double) on one CTA.  coef_out host float64
 * [n_v][n_c] (u-basis, coef[n_num] == 1).  info host [n_v] (nullable).  Synchronises.
 * DEGENERATE if a pivot <= 1e-13 (equilibrated) -- coef of that metric is then NaN and the
 * others are still solved; UNSUPPORTED if n_c > 161.                                       */
rp_status rp_solve_normal(const double *G, int32_t n_v, const rp_basis *basis, double *coef_out,
                          rp_fit_info *info, rp_stream s);

/* ---- a10-a14 in one call -------------------------------------------------------------------
 * Fit n_v metrics sharing the sample points X: transform from the sample box (rp_minmax +
 * rp_xform_from_box), Gram, solve.  X [K][n], V [n_v][K] device-or-host; coef_out host
 * [n_v][n_c]; xform_out host; info host [n_v] nullable.  Synchronises.                      */
rp_status rp_fit(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                 double *coef_out, rp_xform *xform_out, rp_fit_info *info, rp_stream s);

/* ---- stream-ordered (device-resident) forms of a10-a14 --------------------------------------
 * No host synchronisation and no host round trip: every pointer is a device pointer (INVALID_ARG
 * otherwise), results stay on the device, and the calls only enqueue work on the stream (their
 * temporaries come from the stream-ordered pool).  The transform travels as xf [n][2] doubles
 * (c_k, e_k) -- the layout rp_plan_update_program takes.
 * rp_minmax_dev: lohi [n][2] = per-column (min, max) of X [K][n].
 * rp_xform_dev: xf [n][2] from lohi [n][2] (reading R14).
 * rp_gram_accumulate_dev: rp_gram_accumulate with the transform from xf; G [n_v][n_c][n_c].
 * rp_solve_normal_dev: rp_solve_normal into coef [n_v][n_c] and info [n_v][5] (status, rank,
 *   resid2, min_pivot, cond_est as doubles; nullable).  A degenerate system leaves NaN
 *   coefficients and status 3 in info (no error is returned: nothing is read back).
 * rp_fit_dev: the four above in order; xf_out [n][2] nullable.                               */
/* rp_gram_sum_ordered: a13 in its deterministic form -- out[e] = ((parts[0][e] + parts[1][e]) +
 * parts[2][e]) + ... for the n_parts partial Grams of the K shards, stacked in rank order (device
 * float64 [n_parts][elems], e.g. an all_gather's output); out device float64 [elems] (may not
 * alias parts).  Bit-reproducible, unlike an all_reduce whose summation order is NCCL's.
 * INVALID_ARG for n_parts < 1 or host pointers.  Stream-ordered.                           */
rp_status rp_gram_sum_ordered(const double *parts, int32_t n_parts, int64_t elems, double *out, rp_stream s);
rp_status rp_minmax_dev(const double *X, int64_t K, int32_t n, double *lohi, rp_stream s);
rp_status rp_xform_dev(const double *lohi, int32_t n, double *xf, rp_stream s);
rp_status rp_gram_accumulate_dev(const double *X, const double *V, int64_t K, int32_t n_v,
                                 const rp_basis *basis, const double *xf, double *G, rp_stream s);
rp_status rp_solve_normal_dev(const double *G, int32_t n_v, const rp_basis *basis, double *coef,
                              double *info, rp_stream s);
rp_status rp_fit_dev(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                     double *coef, double *xf_out, double *info, rp_stream s);

/* ---- f4: Sanathanan-Koerner reweighted refit ---------------------------------------------------
 * The linearised rows p(x) - V q(x) of PAPER.md:2578-2584 weigh each sample by q(x), which biases
 * noisy fits.  rp_gram_accumulate_weighted is rp_gram_accumulate with every
 * design row of metric m scaled by S[m][r] (device-or-host float64 [n_v][K]); rp_fit_sk runs
 * `iters` solves: the first is rp_fit, each later one refits with S[m][r] = 1 / q_m(x_r) of the
 * previous solution (reading R29), i.e. minimises sum_r ((p - V q) / q_prev)^2 -> sum (p/q - V)^2.
 * Same layouts, ownership and errors as rp_gram_accumulate / rp_fit.                          */
rp_status rp_gram_accumulate_weighted(const double *X, const double *V, const double *S, int64_t K,
                                      int32_t n_v, const rp_basis *basis, const rp_xform *xform,
                                      double *G, rp_stream s);
rp_status rp_fit_sk(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                    int32_t iters, double *coef_out, rp_xform *xform_out, rp_fit_info *info,
                    rp_stream s);

/* ---- f1: the homogeneous system by singular value decomposition ------------------------------
 * "we use the computationally more intensive yet more numerically stable method of singular
 * value decomposition" on the homogeneous system p(x) - V q(x) = 0 (draft
 * footnote PAPER.md:2595-2598): coef = the right singular vector of the smallest singular value
 * of A_m = [M(u_r) | -V_m[r] N(u_r)] (rows as in rp_gram_accumulate), scaled so that beta_0 = 1
 * (reading R12).  A is never formed in memory: its triangular factor R (A^T A = R^T R) comes from
 * design rows generated on chip -- for K >= 4 n_c (and a basis whose exponent-sum simplex fits
 * the moment kernel) as the Cholesky factor of A^T A formed from double-double moments and
 * factored in double-double (reading R34; RP_SVD_R=tsqr disables it), otherwise by a
 * Householder TSQR -- and an SVD of R (one CTA per metric) gives the right singular vectors.
 * Deterministic (fixed reduction orders, fixed merge tree).
 *
 * rp_fit_svd: transform from the sample box as rp_fit, then R + SVD.  X [K][n], V [n_v][K]
 *   device-or-host; coef_out host [n_v][n_c]; sigma_out host [n_v][n_c] ascending singular values
 *   (nullable); xform_out host (nullable); info host [n_v] (nullable) with rank = #{sigma >
 *   1e-13 sigma_max}, resid2 = ||A coef||^2, min_pivot = sigma_min, cond_est = sigma_max /
 *   sigma_min.  Synchronises.  DEGENERATE if beta_0 of that singular vector is 0 (coef NaN;
 *   other metrics still solved); UNSUPPORTED if n_c outside [2, 144].
 * rp_tsqr_accumulate: the split form for K-sharding -- R_m of this rank's rows under an agreed
 *   transform: R device-or-host float64 [n_v][n_c][n_c], row-major upper triangular (zeros
 *   below the diagonal; A_m^T A_m = R_m^T R_m).  K = 0 gives R = 0.
 * rp_svd_rows: TSQR + SVD of dense rows (device-or-host float64 [n_v][n_rows][n_c]), e.g. the
 *   ranks' stacked factors [R_0; R_1; ...]; outputs as rp_fit_svd.                          */
rp_status rp_fit_svd(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                     double *coef_out, double *sigma_out, rp_xform *xform_out, rp_fit_info *info,
                     rp_stream s);
rp_status rp_tsqr_accumulate(const double *X, const double *V, int64_t K, int32_t n_v,
                             const rp_basis *basis, const rp_xform *xform, double *R, rp_stream s);
rp_status rp_svd_rows(const double *rows, int64_t n_rows, int32_t n_v, const rp_basis *basis,
                      double *coef_out, double *sigma_out, rp_fit_info *info, rp_stream s);

/* ---- f3: step 3, "convert [the rational program] into code" ------------
 * rp_codegen: the CUDA C source of the rational program R of `prog` with every constant an
 *   immediate (fitted coefficients, transform, H, R, Z, grid rule; hexadecimal float literals,
 *   exact): the occupancy flowchart, the masks, g_i as direct monomial sums, the MWP-CWP CFG of
 *   DESIGN.md Appendix A line by line (or E = g_1), and `rp_jit_argmin`, the exhaustive per-D
 *   search of steps 4-5.  Host buffer out_src of cap bytes (nullable:
 *   query); *len = the source length without the NUL.  UNSUPPORTED if cap <= *len.
 * rp_jit_create: rp_codegen, then NVRTC (libnvrtc.so.12, loaded with dlopen) for sm_100a and
 *   cudaLibraryLoadData on the current device.  UNSUPPORTED without NVRTC; CUDA on a compile or
 *   load failure (the NVRTC log is in rp_last_error()).  Free with rp_jit_destroy.
 * rp_jit_eval_argmin: the generated search over D (device-or-host int32 [nD][d]) and F
 *   (device-or-host int32 [nF][p]); outputs as rp_eval_argmin (best_idx [nD], best_E [nD],
 *   second_E [nD] nullable), one warp per tuple.  Same masks and tie rule as rp_eval_argmin; E
 *   is evaluated in the literal order of Appendix A (IEEE divisions).                         */
typedef struct rp_jit_s *rp_jit;
rp_status rp_codegen(const rp_program *prog, char *out_src, size_t cap, size_t *len);
rp_status rp_jit_create(const rp_program *prog, rp_jit *out);
rp_status rp_jit_eval_argmin(rp_jit jit, const int32_t *D, int64_t nD, const int32_t *F, int32_t nF,
                             int32_t *best_idx, double *best_E, double *second_E, rp_stream s);
rp_status rp_jit_destroy(rp_jit jit);

/* ---- a4 alone: fitted metrics at points ----------------------------------------------------
 * out[i][r] = g_i(X_r) = p_i(u_r)/q_i(u_r) for i < prog->n_metrics (device-or-host float64
 * [n_metrics][K]); X device-or-host float64 [K][d+p].                                      */
rp_status rp_eval_metrics(const rp_program *prog, const double *X, int64_t K, double *out,
                          rp_stream s);

/* ---- a1-a8: sweep + per-D argmin ------------------------------------------------------------
 * For every D (device-or-host int32 [nD][d]) evaluate E over the configurations F
 * (device-or-host int32 [nF][p], tuple order = index order), masking P that are not
 * practically meaningful (T mod 32 != 0, T > t_max, P1 P2 > D1^2, B_active = 0, E not finite
 * or <= 0), and return the lowest index minimising E: best_idx int32 [nD] (-1 if no P is
 * feasible), best_E float64 [nD] (+inf if none), second_E float64 [nD] (nullable; the
 * second-smallest E over the other feasible P, == best_E on an exact tie).  Outputs
 * device-or-host.  nD = 0 is a no-op.  UNSUPPORTED if nF > 65536 or a basis exceeds the
 * compiled staging limits.                                   */
rp_status rp_eval_argmin(const rp_program *prog, const int32_t *D, int64_t nD, const int32_t *F,
                         int32_t nF, int32_t *best_idx, double *best_E, double *second_E,
                         rp_stream s);

/* Same for n_prog programs over one D batch and one F (all programs share d and p): outputs
 * [n_prog][nD].  One launch covers every program.                                           */
rp_status rp_eval_argmin_batched(const rp_program *progs, int32_t n_prog, const int32_t *D,
                                 int64_t nD, const int32_t *F, int32_t nF, int32_t *best_idx,
                                 double *best_E, double *second_E, rp_stream s);

/* ---- plans: a1 once per (programs, F), then many sweeps ------------------------------------
 * rp_plan_create stages the programs (coefficients, H, resources) to the device and
 * precomputes the per-configuration table (static mask, B_active, W_active, P-monomials)
 * and the compaction of statically feasible configurations, on the device.  F
 * device-or-host.  The plan is bound to the current device.  rp_plan_eval_argmin is
 * rp_eval_argmin_batched without the setup.  rp_plan_static_feasible returns the number of
 * configurations of program `prog` that survive the static mask (synchronises).  Plan memory
 * comes from the stream-ordered pool; rp_plan_destroy frees it in order on the stream of the
 * last rp_plan_eval_argmin (or of the creation): if the plan was used on several streams,
 * synchronise them before destroying it.  rp_plan_create synchronises its stream.            */
typedef struct rp_plan_s *rp_plan;
rp_status rp_plan_create(const rp_program *progs, int32_t n_prog, const int32_t *F, int32_t nF,
                         rp_plan *out, rp_stream s);
rp_status rp_plan_eval_argmin(rp_plan plan, const int32_t *D, int64_t nD, int32_t *best_idx,
                              double *best_E, double *second_E, rp_stream s);
rp_status rp_plan_static_feasible(rp_plan plan, int32_t prog, int32_t *n_static_feasible);
/* rp_plan_update_program: replace the coefficients (and, if xform is non-null, the transform) of
 * program `prog` from DEVICE memory -- coef [n_metrics][stride] in each metric's basis order
 * (stride >= its n_c; rp_fit_dev's output has stride n_c), xform [n][2] (c_k, e_k).  The
 * configuration table (a1 masks, a5 occupancy, its order) depends on F, the hardware and the
 * kernel's resources only, so one device launch refreshes what the new values change: the
 * staging matrix of the coefficients and the configurations' program-part monomials.
 * Stream-ordered, no host synchronisation: a fit and the sweep that uses it chain on the device.
 * The bases (hence the term layout) are those of the plan's creation.
 * Clears the plan's runtime history.                                                       */
rp_status rp_plan_update_program(rp_plan plan, int32_t prog, const double *coef, int32_t stride,
                                 const double *xform, rp_stream s);
rp_status rp_plan_destroy(rp_plan plan);

/* Per-phase device timing of rp_plan_eval_argmin (measurement support; off by default).
 * rp_plan_enable_timing(plan, 1) creates CUDA events that every later rp_plan_eval_argmin records
 * on its stream around its phases; rp_plan_last_timing waits for the last call's final event and
 * writes ms[0] = tuple grouping (the D1 buckets), ms[1] = the sweep kernel (a1-a8),
 * ms[2] = the winner refinement (k_refine; 0 when disabled by RP_SWEEP_REFINE=0).  ms host
 * float[3].  INVALID_ARG if timing was not enabled.  Events add ~2 us per call.               */
rp_status rp_plan_enable_timing(rp_plan plan, int32_t on);
rp_status rp_plan_last_timing(rp_plan plan, float *ms);

/* ---- f2: runtime decision service ----------------------------------------------------------
 * One decision per data tuple, as the paper's driver program makes before every kernel launch
 * (PAPER.md:2094-2099): evaluate R over F, take the optimum (step 5) and
 * return the six launch integers "(gx, gy, gz, bx, by, bz)" of the IO function
 * (the paper's text has a "gx, gx" typo).  "There may be several
 * configurations which, up to some margin, optimize E.  Then, a secondary performance metric
 * ... may be used to refine the choice": with margin > 0 every candidate with
 * E <= E_best (1 + margin) ties, and the tie goes to the larger W_active (occupancy, Eq. (1)),
 * then the larger P1, the smaller P2, the smaller P3, the lower index (reading
 * R28).  margin == 0 returns exactly the argmin of rp_plan_eval_argmin (lowest index on exact
 * ties).  One CTA per tuple; nFc <= 8192 statically feasible configurations.
 * D device-or-host int32 [n][d]; out device-or-host [n].                                      */
typedef struct {
  int32_t idx;          /* chosen configuration (index in F); -1 if none is feasible          */
  int32_t from_history; /* 1 if served by the runtime history                                  */
  double E;             /* its estimate (+inf if none)                                         */
  int32_t launch[6];    /* gx, gy, gz, bx, by, bz (grid rule gx = ceil(D/P), 1 for unmapped
                           dimensions); zeros if none                                          */
  int32_t pad[2];
} rp_decision;

rp_status rp_plan_decide(rp_plan plan, int32_t prog, const int32_t *D, int64_t n, double margin,
                         rp_decision *out, rp_stream s);

/* Runtime history ("maintaining a runtime history to instantly provide results for future kernel
 * launches"): a device-resident open-addressing hash table D -> decision,
 * owned by the plan, 2^log2_capacity slots (4..24), for one program of the plan and one
 * margin; rp_plan_decide then probes it first and inserts its fresh decisions (a full table
 * keeps serving hits and computes the rest).  Enabling again clears it: with the same capacity
 * in place (a live rp_decider of the same program and margin keeps working; another program or
 * margin is INVALID_ARG while deciders live), with another capacity by reallocation (refused,
 * INVALID_ARG, while any rp_decider of the plan lives: its graph holds the table).             */
rp_status rp_plan_history_enable(rp_plan plan, int32_t prog, int32_t log2_capacity, double margin);
rp_status rp_plan_history_stats(rp_plan plan, int64_t *hits, int64_t *misses, int64_t *entries);
rp_status rp_plan_history_clear(rp_plan plan, rp_stream s);

/* ---- persistence --------------------------------------------------------------------------
 * The paper keeps two artefacts across runs: the rational program built at compile time (step 3,
 * PAPER.md:2243-2258) and the runtime history that "instantly provide[s] results for future
 * kernel launches".  Both are saved as self-describing little-endian byte
 * blobs with a magic, a version and an FNV-1a 64 checksum; coefficients keep their IEEE bits
 * (a load reproduces the program exactly).  Writers: buf may be null to query *size; a non-null
 * buf shorter than the blob is INVALID_ARG (with *size set).  Readers: INVALID_ARG on a wrong
 * magic, a checksum mismatch, truncation or content that rp_plan_create would reject.
 *   rp_program_save     -- rp_program (host) -> bytes (validated like rp_plan_create).
 *   rp_program_load     -- bytes -> an owned rp_program_blob; rp_program_blob_program returns
 *                          the rp_program inside (valid until rp_program_blob_free).
 *   rp_plan_history_save -- the ready entries of the plan's runtime history (in slot order), its
 *                          program index and margin, and a fingerprint of the device program
 *                          (its coefficients and transform as they are now) and of F.
 *                          INVALID_ARG if the history is not enabled.  Synchronises.
 *   rp_plan_history_load -- inserts the saved entries into the plan's enabled history through the
 *                          decision kernel's own hashing (rp_plan_decide then serves them as
 *                          hits).  INVALID_ARG unless the data arity, program index, margin and
 *                          fingerprint match: a history never outlives the program and
 *                          configuration set that made it.  Synchronises.                      */
typedef struct rp_program_blob_s *rp_program_blob;
rp_status rp_program_save(const rp_program *prog, void *buf, int64_t cap, int64_t *size);
rp_status rp_program_load(const void *buf, int64_t size, rp_program_blob *out);
const rp_program *rp_program_blob_program(rp_program_blob blob);
rp_status rp_program_blob_free(rp_program_blob blob);
rp_status rp_plan_history_save(rp_plan plan, void *buf, int64_t cap, int64_t *size);
rp_status rp_plan_history_load(rp_plan plan, const void *buf, int64_t size);

/* Single-launch decider (the per-launch use of PAPER.md:2094-2099, "immediately preceding the
 * launch of a kernel", with the lowest host-visible latency the library offers): one data tuple
 * in, one rp_decision out, through host-mapped pinned memory (no copy nodes) and a CUDA graph of
 * the rp_plan_decide kernel captured once on a private stream.
 *   rp_decider_create  -- for program `prog` of `plan` and `margin`; if the plan's runtime history
 *                         is used, enable it BEFORE creating the decider (the graph captures the
 *                         table) and do not re-enable it while the decider lives.
 *   rp_decider_decide  -- D: host array of the plan's d data parameters; out: host rp_decision.
 *                         Synchronous (returns when `out` is written).  Not thread-safe.
 *   rp_decider_destroy -- frees the mapped buffers, the graph and the stream.
 * The plan must outlive the decider.  Errors: RP_ERR_INVALID_ARG, RP_ERR_UNSUPPORTED (nF beyond
 * the decide kernel's limit), RP_ERR_CUDA.                                                    */
typedef struct rp_decider_s *rp_decider;
rp_status rp_decider_create(rp_plan plan, int32_t prog, double margin, rp_decider *out);
rp_status rp_decider_decide(rp_decider dc, const int32_t *D, rp_decision *out);
rp_status rp_decider_destroy(rp_decider dc);

/* ---- host-fed steps, pipelined (the e2e use: batches arrive in host memory) -------------------
 * One step = the whole path for one batch: fit of n_v metrics on the samples X (host float64
 * [K][n]) with measured V (host float64 [n_v][K]) -> rp_plan_update_program of program 0 of
 * `plan` (a single-program plan created for the program's bases, F, H and resources) -> sweep of
 * the data tuples D (host int32 [nD][d]) -> per-D winners into best_idx (host int32 [nD]) and
 * best_E (host float64 [nD]).  rp_pipeline_submit enqueues a step and returns at once: the H2D
 * copies of the step's inputs run on a copy stream while the previous step computes, and its
 * winners come back on another copy stream while the next step computes (up to `depth` steps in
 * flight, depth in [1, 4]; device buffers allocated once per slot at creation).  Host buffers must
 * stay valid and unmodified until rp_pipeline_sync returns (pinned memory makes the copies truly
 * asynchronous; pageable memory is still correct but the copies then block the submitting thread).
 * PAPER.md:2094-2099 (evaluate before each launch), 2222-2235 (re-estimate from samples).
 * Errors: INVALID_ARG (shapes, a multi-program plan), CUDA.  Not thread-safe per pipeline. */
typedef struct rp_pipeline_s *rp_pipeline;
rp_status rp_pipeline_create(rp_plan plan, int32_t prog, const rp_basis *basis, int32_t n_v, int64_t K,
                             int32_t d, int64_t nD, int32_t depth, rp_pipeline *out);
rp_status rp_pipeline_submit(rp_pipeline p, const double *X, const double *V, const int32_t *D, int32_t *best_idx,
                             double *best_E);
rp_status rp_pipeline_sync(rp_pipeline p);
/* Device time of a run of steps: timer_start records an event on the copy-in stream ahead of the
 * next submitted step's H2D (call rp_pipeline_sync first so no earlier step overlaps); timer_stop
 * records one after the last submitted step's D2H, waits for it and writes the elapsed ms.      */
rp_status rp_pipeline_timer_start(rp_pipeline p);
rp_status rp_pipeline_timer_stop(rp_pipeline p, float *ms);
rp_status rp_pipeline_destroy(rp_pipeline p);

#ifdef __cplusplus
}
#endif
#endif /* RP_H */
