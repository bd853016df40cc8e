// rp_internal.cuh -- internal types shared by librp's translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rp.h"

namespace rp {

// ---- errors ---------------------------------------------------------------------------------
void set_error(const char *fmt, ...);
rp_status cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define RP_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return rp::cuda_fail(e_, #call, __FILE__, __LINE__);    \
  } while (0)
#define RP_REQUIRE(cond, status, ...)   \
  do {                                  \
    if (!(cond)) {                      \
      rp::set_error(__VA_ARGS__);       \
      return (status);                  \
    }                                   \
  } while (0)

// ---- compiled program (device layout) --------------------------------------------------------
// The l numerators / denominators ("polys", k = 2i for p_i, 2i+1 for q_i) are split into
// data and program parts of each monomial: m_e(u) = m_{eD}(u_D) * m_{eP}(u_P).  For every
// poly k and every distinct program-part exponent pe, the data polynomial
//   C_{k,pe}(D) = sum_{terms with eP = pe} coef * m_{eD}(u_D)
// is staged once per D (a2), so that p_k(D,P) = sum_pe C_{k,pe}(D) * m_pe(u_P) (a4).
constexpr int kMaxVars = RP_MAX_VARS;
constexpr int kMaxMetrics = RP_MAX_METRICS;
constexpr int kMaxPolys = 2 * RP_MAX_METRICS;
constexpr int kMaxPE = 36;     // distinct program-part exponents (degree 4 in 3 vars = 35)
constexpr int kMaxDE = 64;     // distinct data-part exponents
constexpr int kMaxTerms = 1536;
constexpr int kMaxRows = kMaxPolys * kMaxPE;

struct DevProg {
  int32_t d, p, nm, tmpl, npoly, nPE, nDE, nterm;
  int32_t grid_map[3];
  int32_t n_sm, w_max, b_max, t_max;
  int64_t r_max, z_max, R, Z0, Z1;
  double freq, mem_bw, lbpw, mem_ld, dd_coal, dd_unc, U, issue;
  double xc[kMaxVars];
  int32_t xe[kMaxVars];
  int8_t de_exp[kMaxDE][kMaxVars];  // data-part exponents (first d entries used)
  int8_t pe_exp[kMaxPE][3];         // program-part exponents
  int16_t row_start[kMaxRows + 1];  // terms of row (k * nPE + pe) are [row_start[r], row_start[r+1])
  int16_t term_de[kMaxTerms];
  double term_coef[kMaxTerms];
  int16_t term_src[kMaxTerms];  // metric * kMaxSrc + index of the term's coefficient in coef[metric]
};
constexpr int kMaxSrc = 4096;   // term_src stride per metric (n_num + n_den < kMaxSrc)

// Per-configuration table of a plan (SoA over the statically feasible, compacted configs in
// ascending original index; program g at offset g * nFp, nFp = nF rounded up to 8 so that
// config octets of the DMMA tiles never straddle programs).
struct CfgRec {      // one statically feasible configuration, 64 B (4 x 16-byte loads)
  int64_t P01;               // P_1 P_2 (P_1 if p = 1), for the D rule P_1 P_2 <= D_1^2
  int32_t orig, Pm1_0;       // original index in F; P_0 - 1
  int32_t Pm1_1, Pm1_2;      // P_k - 1 (0 for k >= p)
  uint32_t M0, M1, M2;       // ceil(n / P_k) = (n + P_k - 1) * M_k >> s_k  (exact, n < 2^31)
  uint32_t s012;             // s_k in bits 8k..8k+7
  double W, rB;              // W_active, 1/B_active
  float W32, rB32;           // the same in FP32 (the screened sweep's inputs)
};
static_assert(sizeof(CfgRec) == 64, "CfgRec layout");

// Factored contraction of the sweep (k_plan_groups).  A group is a
// set of feasible configurations that share every P_k except P_hv (the Horner variable).  With
// x = u_hv(P_hv) and i_pe the exponent of u_hv in m_pe, every polynomial factors as
//   p_k(D, P) = sum_i x^i w_{k,i}(D),   w_{k,i}(D) = sum_{pe: i_pe = i} C_{k,pe}(D) Y_pe,
// Y_pe = prod_{j != hv} u_j(P_j)^{e_pe,j} (one value per group), so a tile of 8 configurations of
// one group is two DMMA.8x8x4 per polynomial instead of ceil(nPE / 4): A = the shares of w_{k,0},
// B = 1 (w_{k,0} in every column), then A = w_{k,1..4} of 8 tuples (lane q of a quad holds
// w_{k,1+q}), B = x^{1..4} of the 8 configurations.
// Lane q of a quad evaluates w_{k,1+q} from kGS1 terms and its share of w_{k,0} (terms q, q + 4 of
// the i = 0 list) from kGW0 terms; a DMMA with B = 1 sums the four shares.
constexpr int kGS1 = 4, kGW0 = 2, kGS = kGS1 + kGW0;
constexpr int kMaxGroups = 128;      // groups per program
constexpr int kGroupMaxPlan = 2048;  // plans with more feasible configurations stay dense
struct GroupDesc {
  int32_t tile_begin, tile_end, hv, nmem;  // tiles [tile_begin, tile_end) of the schedule
  int32_t P[3], pad;                       // the members' P (P[hv] unused)
  int32_t off[4][kGS];                     // lane q, term s: pe (s < kGS1: of w_{1+q}; else of w_0's share)
  double y[4][kGS];                        // Y_pe of that term (0 for padding)
  double ype[kMaxPE];                      // Y_pe by pe (0 past nPE): the setup DMMA's B operand
  int8_t ipe[kMaxPE];                      // i_pe = exponent of u_hv in m_pe (-1 past nPE)
};

struct CfgTable {
  int32_t nFp;     // padded stride (multiple of 8)
  CfgRec *rec;     // [n_prog][nFp]  sorted by (P1 P2, original index)
  CfgRec *srec;    // [n_prog][nFp]  scratch: compacted in index order
  double *smP;     // [n_prog][npe_pad][nFp]  scratch
  double *mP;      // [n_prog][npe_pad][nFp]  program-part monomials (0 for pe >= nPE or pad)
  double *rSM;     // [n_prog][kRSMTab]  1/k for SM_act = k (k <= n_sm)
  double *Cmat;    // [n_prog][6 * npe_pad][nde_pad]  dense coefficient matrix of the staging:
                   // row k * npe_pad + pe, column de: coef of m_de(u_D) m_pe(u_P) in poly k
  int32_t nde_pad; // data-part monomials padded to a multiple of 4 (the DMMA K step)
  int32_t *nFc;    // [n_prog][2]: number of feasible configurations, sorted flag
  // winner refinement (k_refine): the union of the polynomials' (de, pe) terms
  int32_t *rterm;  // [n_prog][npe_pad * nde_pad]: de | pe << 16 of term j (j < nRT)
  double *rcoef;   // [n_prog][npe_pad * nde_pad][kMaxPolys]: coefficient of term j in poly k
  double *rinfo;   // [n_prog][8]: A_k = sum_j |rcoef[j][k]| (k < 6), max total degree, nRT
  int32_t *inv;    // [n_prog][nFp]: original index -> position in srec (-1: statically infeasible)
  int32_t nrt_max; // host bound on the union term count of any program (shared-memory sizing)
  // the sweep's tile schedule (k_plan_groups): factored tiles of the groups, then dense tiles of
  // the remaining configurations in (P1 P2, index) order; every tile is 8 slots
  int32_t nGp;        // slots per program (multiple of 8, >= nFp + 8)
  CfgRec *grec;       // [n_prog][nGp]: records of the slots (zero record, orig INT_MAX: padding)
  double *gmP;        // [n_prog][npe_pad][nGp]: B operands (factored: x^{1+q} in rows q < 4)
  int32_t *ghv;       // [n_prog][nGp]: slot's Horner variable, -1 dense, -2 padding
  GroupDesc *gdesc;   // [n_prog][kMaxGroups]
  int32_t *gcnt;      // [n_prog][4]: groups, factored tiles, tiles, -
  // (last: the sweep kernel's code generation is sensitive to the offsets of the fields above)
  double2 *mPdd;      // [n_prog][nFp][npe_pad]: m_pe(u_P) of srec position pos, double-double (k_refine)
};
constexpr int kRSMTab = 1024;  // n_sm <= 1023 uses the table

// Host-side marshalling of an rp_program into DevProg (layout only: splitting exponent vectors,
// sorting terms, copying coefficients; no arithmetic on values).
rp_status compile_program(const rp_program *prog, DevProg *out);

// ---- launchers (defined in the kernel TUs) ----------------------------------------------------
cudaError_t launch_plan_configs(const DevProg *d_progs, int n_prog, const int32_t *d_F, int nF,
                                int npe_pad, CfgTable tab, cudaStream_t s);
cudaError_t launch_sweep(const DevProg *d_progs, int n_prog, bool mwp, CfgTable tab, int npe_pad,
                         int nde_max, int n_sm_max, int d, const int32_t *d_D, int64_t nD,
                         int32_t *idx, double *bestE, double *secondE, const int32_t *perm,
                         int32_t *idx2, cudaEvent_t *ev /* nullable: [1] before the sweep kernel,
                         [2] before the refinement */, cudaStream_t s);
cudaError_t launch_bucket_perm(const int32_t *d_D, int64_t nD, int d, int kb, unsigned *d_hist,
                               int32_t *d_perm, cudaStream_t s);
cudaError_t launch_eval_metrics(const DevProg *d_prog, int nm, const double *X, int64_t K,
                                double *out, cudaStream_t s);
cudaError_t launch_minmax(const double *X, int64_t K, int n, double *d_part, int nblk,
                          double *d_out, cudaStream_t s);
int minmax_blocks(int64_t K);
cudaError_t launch_xform(const double *d_lohi, int n, double *d_out, cudaStream_t s);
struct GramBasis;
cudaError_t launch_xform_to_basis(const double *d_xf, int n, GramBasis *d_gb, cudaStream_t s);

struct GramBasis {  // exponents of the n_c design columns (numerator then denominator)
  int32_t n, n_num, n_den, nc, maxdeg;
  int8_t exp[256][kMaxVars];
  double xc[kMaxVars];
  int32_t xe[kMaxVars];
  // fused path (numerator basis == denominator basis): the m = n_num monomials with their
  // exponents packed 4 bits per variable
  int32_t fused;
  uint32_t pexp[256];
  // monomial tree of the m numerator columns (fused path): column j of degree >= 1 is
  // M_j = M_parent[j] * u_var[j]; levels lists the columns by degree (lv_start[d] .. lv_start[d+1])
  int32_t tree;       // every non-constant column has its parent in the basis, one constant column
  int32_t n_lv;       // number of levels (max degree + 1)
  int16_t parent[256];
  int8_t pvar[256];
  int16_t lv_cols[256];
  int16_t lv_start[18];
};
cudaError_t launch_gram(const GramBasis *d_basis, const GramBasis &h_basis, const double *X,
                        const double *V, const double *S, int64_t K, int n_v, double *G,
                        double *d_part, size_t part_elems, cudaStream_t s);
size_t gram_partial_elems(const GramBasis &h_basis, int n_v, int64_t K, int num_sms, bool weighted);
// a12 as a moment contraction (rp_moments.cu): the default where the exponent-sum simplex is small
bool mom_supported(const GramBasis &h_basis, int n_v, bool weighted);
size_t mom_partial_elems(const GramBasis &h_basis, int n_v, int64_t K, bool weighted);
// f1: R = chol(A^T A) with the Gram and the factorisation in double-double (rp_moments.cu)
bool gram_dd_supported(const GramBasis &h_basis, int n_v, int64_t K);
size_t gram_dd_workspace_bytes(const GramBasis &h_basis, int n_v, int64_t K);
cudaError_t launch_gram_dd_chol(const GramBasis *d_basis, const GramBasis &h_basis, const double *X, const double *V,
                                int64_t K, int n_v, void *ws, size_t ws_bytes, double *R, cudaStream_t s);
cudaError_t launch_gram_mom(const GramBasis *d_basis, const GramBasis &h_basis, const double *X, const double *V,
                            const double *S, int64_t K, int n_v, double *G, double *d_part, size_t part_elems,
                            cudaStream_t s);
cudaError_t launch_sum_ordered(const double *parts, int n_parts, int64_t elems, double *out, cudaStream_t s);
cudaError_t launch_den_weights(const GramBasis *d_basis, const double *X, int64_t K, int n_v,
                               const double *d_coef, double *S, cudaStream_t s);

cudaError_t launch_solve(const double *G, int n_v, int nc, int beta0, double *coef_out,
                         double *info_out, cudaStream_t s);

// f1 (rp_svd.cu): Householder TSQR of the design rows (X, V[, S] through d_basis) or of dense
// rows [n_v][K][nc], then the one-sided Jacobi SVD of R (one CTA per metric, V in L2).
int tsqr_leaves(int64_t K, int n_v);
size_t tsqr_workspace_bytes(int nc, int n_v, int leaves);
cudaError_t launch_tsqr(const GramBasis *d_basis, const double *X, const double *V, const double *S,
                        const double *rows, int64_t K, int n, int nc, int n_v, void *ws, size_t ws_bytes,
                        double *R_out, cudaStream_t s);
cudaError_t launch_svd_jacobi(const double *R, int nc, int n_num, int n_v, double *V_ws, double *coef,
                              double *sigma, double *info, cudaStream_t s);

}  // namespace rp
int rp_jit_dims(rp_jit jit, int which);  // d (0) or p (1) of the program a jit was made from
namespace rp {
// device-resident refit of a plan's program (rp_plan_update_program)
cudaError_t launch_plan_refresh(DevProg *d_prog, int g, const double *d_coef, int stride, const double *d_xf,
                                int npe_pad, CfgTable tab, cudaStream_t s);
// f3 (rp_codegen.cu)
cudaError_t launch_jit(rp_jit jit, const int32_t *D, int64_t nD, const int32_t *F, int32_t nF, int32_t *idx,
                       double *bestE, double *secondE, cudaStream_t s);

int num_sms();
int plan_num_programs(rp_plan plan);     // rp_pipeline: shape checks against the plan
int plan_num_data_params(rp_plan plan);
void plan_forget_stream(rp_plan plan, cudaStream_t s);

}  // namespace rp
