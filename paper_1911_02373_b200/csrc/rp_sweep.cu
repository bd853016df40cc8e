// rp_sweep.cu -- the runtime sweep of the rational program R over (D, P) with per-D argmin.
//
// PAPER.md:2259-2305 (steps 4 and 5): for the runtime data parameters D and "all practically
// meaningful values of P from the set F, we compute an estimate of E using R", then "an
// exhaustive search is feasible" picks the optimum.
//
// Kernels:
//   k_plan_configs -- a1 + a5, once per (program, F): per configuration T, the static mask
//                     (warp rule, T <= T_max, B_active > 0), B_active (occupancy flowchart),
//                     W_active (Eq. (1)), the program-part monomials m_pe(u_P) and a few
//                     reciprocals; compaction of the feasible configurations in index order.
//   k_sweep        -- a2 (stage the data polynomials C_{k,pe}(D) of a tile of 32 tuples in
//                     shared memory), a4 (the contraction p_k(D,P) = sum_pe C_{k,pe}(D) m_pe(P)
//                     on the FP64 tensor pipe: DMMA.8x8x4, A = C of 8 tuples, B = m of 8
//                     configurations, so each lane ends up with all 2l polynomials of 2 (D,P)
//                     pairs), a3 (P1 P2 <= D1^2), a6 (grid), a7 (E in common-denominator form,
//                     4-5 Newton reciprocals instead of ~11 divisions), a8 (argmin on the exact
//                     key (E, original index) + runner-up, lane -> quad -> warp -> CTA).
#include <cstdio>

#include "rp_device.cuh"

namespace rp {

constexpr int kSortMaxPlan = 8192;  // plans with more feasible configurations keep index order

// ---- a5: occupancy, Fig. occupancysimpleflowchart, 64-bit integers ----
__device__ __forceinline__ int64_t occupancy_blocks(int64_t T, int64_t R, int64_t Z,
                                                    const DevProg &pg) {
  const int64_t Bm = pg.b_max, W32 = 32 * (int64_t)pg.w_max, Rm = pg.r_max, Zm = pg.z_max;
  if (T * Bm <= W32 && R * T * Bm <= Rm && Z * Bm <= Zm) return Bm;                   // none
  if (W32 <= T * Bm && W32 * R <= Rm && W32 * Z <= Zm * T) return W32 / T;             // warps
  if (Rm <= R * T * Bm && Rm <= R * W32 && Rm * Z <= R * T * Zm) return Rm / (R * T);  // regs
  if (Zm <= Bm * Z && Zm * T <= W32 * Z && Zm * R * T <= Z * Rm) return Zm / Z;         // smem
  return 0;                                                                             // fail
}

// ---- a1 + a5 + P-monomials, compaction in index order --------------------------------------
__global__ void __launch_bounds__(1024) k_plan_configs(const DevProg *progs, const int32_t *F,
                                                       int nF, int npe_pad, CfgTable tab) {
  const int g = blockIdx.x;
  const DevProg &pg = progs[g];
  const int nFp = tab.nFp;
  __shared__ int warp_tot[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < nF; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    int ok = 0;
    int32_t Pk[3] = {1, 1, 1};
    int64_t T = 1, B = 0, W = 0;
    if (c < nF) {
      for (int k = 0; k < pg.p; ++k) Pk[k] = F[(int64_t)c * pg.p + k];
      bool pos = true;
      for (int k = 0; k < pg.p; ++k) {
        T *= Pk[k];
        pos = pos && Pk[k] >= 1;
      }
      // "a multiple of the warp size (32)" and "bounded over by the maximum number of threads
      // per block"
      ok = pos && (T % 32 == 0) && (T <= pg.t_max);
      if (ok) {
        const int64_t Z = pg.Z0 + pg.Z1 * T;
        B = occupancy_blocks(T, pg.R, Z, pg);
        ok = B > 0;        // B_active = 0: "Failure to Launch"
        W = (B * T) / 32;  // Eq. (1)
        if (W > pg.w_max) W = pg.w_max;
      }
    }
    const unsigned ball = __ballot_sync(0xffffffffu, ok);
    const int pre = __popc(ball & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[wid] = __popc(ball);
    __syncthreads();
    if (wid == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      warp_tot[lane] = incl - v;
    }
    __syncthreads();
    const int pos = base + warp_tot[wid] + pre;
    if (ok) {
      const int64_t off = (int64_t)g * nFp;
      CfgRec r;
      r.P01 = (int64_t)Pk[0] * (pg.p >= 2 ? Pk[1] : 1);
      r.orig = c;
      r.Pm1_0 = Pk[0] - 1;
      r.Pm1_1 = Pk[1] - 1;
      r.Pm1_2 = Pk[2] - 1;
      // division by the invariant P: M = ceil(2^s / P), s = 31 + ceil(log2 P) gives
      // floor(n / P) = (n * M) >> s exactly for 0 <= n < 2^31 (error (M P - 2^s) n / (P 2^s) < 1/P)
      uint32_t Ms[3], ss[3];
      for (int k = 0; k < 3; ++k) {
        const uint32_t P = (uint32_t)Pk[k];
        uint32_t l = 0;
        while ((1ull << l) < P) ++l;
        ss[k] = 31 + l;
        Ms[k] = (uint32_t)(((1ull << ss[k]) + P - 1) / P);
      }
      r.M0 = Ms[0];
      r.M1 = Ms[1];
      r.M2 = Ms[2];
      r.s012 = ss[0] | (ss[1] << 8) | (ss[2] << 16);
      r.W = (double)W;
      r.rB = 1.0 / (double)B;
      r.rW = 1.0 / (double)W;
      tab.srec[off + pos] = r;
      double u[3];
      for (int k = 0; k < pg.p; ++k)
        u[k] = ((double)Pk[k] - pg.xc[pg.d + k]) * ldexp(1.0, -pg.xe[pg.d + k]);
      for (int pe = 0; pe < npe_pad; ++pe) {
        double m = 0.0;
        if (pe < pg.nPE) {
          m = 1.0;
          for (int k = 0; k < pg.p; ++k)
            for (int t = 0; t < pg.pe_exp[pe][k]; ++t) m *= u[k];
        }
        tab.smP[(int64_t)g * npe_pad * nFp + (int64_t)pe * nFp + pos] = m;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base = pos + ok;
    __syncthreads();
  }
  __syncthreads();
  const int nFc = base;
  // order the feasible configurations by (P1 P2, original index) so a warp can stop at the
  // first octet whose smallest P1 P2 exceeds every D1^2 of its tuples (a3); rank sort, O(n^2)
  // per plan, skipped above kSortMax (then index order and no early exit)
  const bool sorted = nFc <= kSortMaxPlan;
  for (int i = threadIdx.x; i < nFc; i += blockDim.x) {
    const CfgRec ri = tab.srec[(int64_t)g * nFp + i];
    int rank = i;
    if (sorted) {
      rank = 0;
      for (int j = 0; j < nFc; ++j) {
        const int64_t pj = tab.srec[(int64_t)g * nFp + j].P01;
        rank += (pj < ri.P01) || (pj == ri.P01 && j < i);
      }
    }
    tab.rec[(int64_t)g * nFp + rank] = ri;
    for (int pe = 0; pe < npe_pad; ++pe)
      tab.mP[(int64_t)g * npe_pad * nFp + (int64_t)pe * nFp + rank] =
          tab.smP[(int64_t)g * npe_pad * nFp + (int64_t)pe * nFp + i];
  }
  if (threadIdx.x == 0) {
    tab.nFc[2 * g] = nFc;
    tab.nFc[2 * g + 1] = sorted ? 1 : 0;
  }
  // dense staging matrix: Cmat[k * npe_pad + pe][de] = coefficient of m_de(u_D) m_pe(u_P) in
  // polynomial k (zero elsewhere; the buffer is zeroed at plan creation)
  double *Cm = tab.Cmat + (int64_t)g * kMaxPolys * npe_pad * tab.nde_pad;
  for (int r = threadIdx.x; r < pg.npoly * pg.nPE; r += blockDim.x) {
    const int k = r / pg.nPE, pe = r % pg.nPE;
    for (int j = pg.row_start[r]; j < pg.row_start[r + 1]; ++j)
      Cm[(int64_t)(k * npe_pad + pe) * tab.nde_pad + pg.term_de[j]] = pg.term_coef[j];
  }
  // 1/k for SM_act = k (line 15 of Appendix A); correctly rounded, computed once per plan
  for (int k = threadIdx.x; k < kRSMTab; k += blockDim.x)
    tab.rSM[(int64_t)g * kRSMTab + k] = k > 0 ? 1.0 / (double)k : 0.0;
}

// rp_plan_update_program in one launch: the configuration table (a1 masks, a5 occupancy, the
// P1 P2 order) depends on F, the hardware and the kernel's resources only, so a refit changes
// just the coefficients (the dense staging matrix Cmat) and the transform (the program-part
// monomials mP of the sorted feasible configurations).
__global__ void __launch_bounds__(1024) k_plan_refresh(DevProg *pgp, int g, const double *coef, int stride,
                                                       const double *xf, int npe_pad, CfgTable tab) {
  DevProg &pg = *pgp;
  const int nterm = pg.nterm;
  for (int j = threadIdx.x; j < nterm; j += blockDim.x) {
    const int src = pg.term_src[j];
    pg.term_coef[j] = coef[(int64_t)(src / kMaxSrc) * stride + src % kMaxSrc];
  }
  if (xf && threadIdx.x < pg.d + pg.p) {
    pg.xc[threadIdx.x] = xf[2 * threadIdx.x];
    pg.xe[threadIdx.x] = (int32_t)xf[2 * threadIdx.x + 1];
  }
  __syncthreads();
  const int nFp = tab.nFp, nFc = tab.nFc[2 * g];
  const CfgRec *rec = tab.rec + (int64_t)g * nFp;
  double *mP = tab.mP + (int64_t)g * npe_pad * nFp;
  for (int t = threadIdx.x; t < nFc * npe_pad; t += blockDim.x) {
    const int pos = t / npe_pad, pe = t % npe_pad;
    double m = 0.0;
    if (pe < pg.nPE) {
      const CfgRec &r = rec[pos];
      const int32_t Pk[3] = {r.Pm1_0 + 1, r.Pm1_1 + 1, r.Pm1_2 + 1};
      m = 1.0;
      for (int k = 0; k < pg.p; ++k) {
        const double u = ((double)Pk[k] - pg.xc[pg.d + k]) * ldexp(1.0, -pg.xe[pg.d + k]);
        for (int e = 0; e < pg.pe_exp[pe][k]; ++e) m *= u;
      }
    }
    mP[(int64_t)pe * nFp + pos] = m;
  }
  double *Cm = tab.Cmat + (int64_t)g * kMaxPolys * npe_pad * tab.nde_pad;
  for (int r = threadIdx.x; r < pg.npoly * pg.nPE; r += blockDim.x) {
    const int k = r / pg.nPE, pe = r % pg.nPE;
    for (int j = pg.row_start[r]; j < pg.row_start[r + 1]; ++j)
      Cm[(int64_t)(k * npe_pad + pe) * tab.nde_pad + pg.term_de[j]] = pg.term_coef[j];
  }
}

cudaError_t launch_plan_refresh(DevProg *d_prog, int g, const double *d_coef, int stride, const double *d_xf,
                                int npe_pad, CfgTable tab, cudaStream_t s) {
  k_plan_refresh<<<1, 1024, 0, s>>>(d_prog, g, d_coef, stride, d_xf, npe_pad, tab);
  return cudaGetLastError();
}

cudaError_t launch_plan_configs(const DevProg *d_progs, int n_prog, const int32_t *d_F, int nF,
                                int npe_pad, CfgTable tab, cudaStream_t s) {
  k_plan_configs<<<n_prog, 1024, 0, s>>>(d_progs, d_F, nF, npe_pad, tab);
  return cudaGetLastError();
}

// ---- tuple grouping by D1 (a3 early exit) ------------------------------------------------------
// Only tuples with D1 < kb (kb^2 > the largest P1 P2 of the plan) can fail the D rule, so a
// counting sort on min(D1, kb) groups them by D1 in front; everything else keeps one bucket.
// Which tile computes a tuple does not change its result (rows of the DMMA tiles are
// independent), so outputs are bit-identical to the identity order.
constexpr int kBucketMax = 256;  // kb + 1 <= kBucketMax (t_max <= 65025)

__global__ void k_bucket_count(const int32_t *D, int64_t nD, int d, int kb, unsigned *hist) {
  __shared__ unsigned sh[kBucketMax];
  for (int b = threadIdx.x; b <= kb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nD; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d1 = D[i * d];
    atomicAdd(&sh[d1 < kb ? (d1 < 0 ? 0 : d1) : kb], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b <= kb; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}
__global__ void k_bucket_scan(unsigned *hist, int kb) {  // exclusive scan of kb+1 counters, 1 thread
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int b = 0; b <= kb; ++b) {
      const unsigned c = hist[b];
      hist[b] = run;
      run += c;
    }
  }
}
// each block claims one contiguous range per bucket for the tuples of its grid-stride pass
__global__ void k_bucket_scatter(const int32_t *D, int64_t nD, int d, int kb, unsigned *pos, int32_t *perm) {
  __shared__ unsigned sh[kBucketMax], base[kBucketMax];
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < nD; c0 += (int64_t)gridDim.x * blockDim.x) {
    for (int b = threadIdx.x; b <= kb; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const int64_t i = c0 + threadIdx.x;
    int bk = -1;
    unsigned local = 0;
    if (i < nD) {
      const int32_t d1 = D[i * d];
      bk = d1 < kb ? (d1 < 0 ? 0 : d1) : kb;
      local = atomicAdd(&sh[bk], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b <= kb; b += blockDim.x) base[b] = sh[b] ? atomicAdd(&pos[b], sh[b]) : 0;
    __syncthreads();
    if (bk >= 0) perm[base[bk] + local] = (int32_t)i;
    __syncthreads();
  }
}

cudaError_t launch_bucket_perm(const int32_t *d_D, int64_t nD, int d, int kb, unsigned *d_hist,
                               int32_t *d_perm, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_hist, 0, sizeof(unsigned) * (kb + 1), s);
  if (e != cudaSuccess) return e;
  int64_t b = (nD + 255) / 256;
  const int cap = 4 * num_sms();
  const int grid = (int)(b > cap ? cap : (b < 1 ? 1 : b));
  k_bucket_count<<<grid, 256, 0, s>>>(d_D, nD, d, kb, d_hist);
  k_bucket_scan<<<1, 32, 0, s>>>(d_hist, kb);
  k_bucket_scatter<<<grid, 256, 0, s>>>(d_D, nD, d, kb, d_hist, d_perm);
  return cudaGetLastError();
}

// ---- the sweep ------------------------------------------------------------------------------
struct SweepArgs {
  const DevProg *progs;
  CfgTable tab;
  int npe_pad;
  int d;
  int nde_stride;  // row stride of the data-monomial tile in shared memory (= 4 mod 16)
  const int32_t *D;
  int64_t nD;
  int32_t *idx;
  double *bestE;
  double *secondE;
  const int32_t *perm;  // tuple order of the tiles (grouped by D1), or null: identity
};

#ifndef RP_SWEEP_MINB
#define RP_SWEEP_MINB 4
#endif
constexpr int kSweepWarps = 4;
constexpr int kSweepThreads = 32 * kSweepWarps;
constexpr int kTD = 8 * kSweepWarps;  // tuples per CTA: one octet (the DMMA M side) per warp

template <int NPOLY, int NPE>
__host__ __device__ constexpr int c_stride() {  // per-tuple stride of sC in doubles, = 4 mod 16
  int s = NPOLY * NPE;
  while (s % 16 != 4) ++s;
  return s;
}

static int md_stride(int nde_pad) {  // = 4 mod 16: conflict-free B fragments
  int s = nde_pad;
  while (s % 16 != 4) ++s;
  return s;
}

template <int NPOLY, int NPE>
size_t sweep_smem_bytes(int nde_stride, int n_sm) {
  const int rsm = (n_sm + 2) & ~1;
  return sizeof(double) * ((size_t)kTD * c_stride<NPOLY, NPE>() + (size_t)kTD * nde_stride + rsm) +
         sizeof(int32_t) * kTD * kMaxVars;
}

template <int NPE, bool MWP, bool SECOND>
__global__ void __launch_bounds__(kSweepThreads, RP_SWEEP_MINB) k_sweep(SweepArgs a) {
  constexpr int NPOLY = MWP ? 6 : 2;
  constexpr int KS = NPE / 4;
  constexpr int CS = c_stride<NPOLY, NPE>();
  constexpr double kInf = __builtin_huge_val();
  const int g = blockIdx.y;
  const DevProg &pg = a.progs[g];
  const int d = a.d;
  const int64_t d0 = (int64_t)blockIdx.x * kTD;
  const int tmax = (int)((a.nD - d0) < kTD ? (a.nD - d0) : kTD);
  const int nde = a.nde_stride;
  const int n_sm = pg.n_sm;

  extern __shared__ __align__(16) double smem[];
  double *sC = smem;                   // [kTD][CS]
  double *sMD = sC + kTD * CS;         // [kTD][nde]
  double *sRSM = sMD + kTD * nde;      // [n_sm + 1]
  int32_t *sDv = reinterpret_cast<int32_t *>(sRSM + ((n_sm + 2) & ~1));  // [kTD][kMaxVars]

  // ---- a2: stage the tile (D values, data monomials, data polynomials) --------------------------
  const int nDE = pg.nDE, ndp = a.tab.nde_pad;
  for (int i = threadIdx.x; i < kTD * d; i += blockDim.x) {
    const int t = i / d, k = i % d;
    const int64_t src = (t < tmax) ? (a.perm ? (int64_t)a.perm[d0 + t] : d0 + t) : 0;
    sDv[t * kMaxVars + k] = (t < tmax) ? a.D[src * d + k] : 1;
  }
  const double *gRSM = a.tab.rSM + (int64_t)g * kRSMTab;
  const bool rsm_tab = n_sm < kRSMTab;
  if (rsm_tab)
    for (int i = threadIdx.x; i <= n_sm; i += blockDim.x) sRSM[i] = gRSM[i];
  __syncthreads();
  // data monomials m_de(u_D), u = (D - c) 2^-e, zero for the padding de >= nDE
  for (int i = threadIdx.x; i < kTD * ndp; i += blockDim.x) {
    const int t = i / ndp, de = i % ndp;
    double m = 0.0;
    if (de < nDE) {
      m = 1.0;
      for (int k = 0; k < d; ++k) {
        const double u = ((double)sDv[t * kMaxVars + k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
        for (int e = 0; e < pg.de_exp[de][k]; ++e) m *= u;
      }
    }
    sMD[t * nde + de] = m;
  }
  __syncthreads();
  // staged data polynomials C[t][k NPE + pe] = sum_de Cmat[k NPE + pe][de] m_de(t): a
  // (NPOLY NPE x ndp) x (ndp x 32) product on DMMA.8x8x4 (A from the plan's dense matrix,
  // B = the monomials of the tile); output tiles (8 rows x 8 tuples) spread over the warps
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double *Cm = a.tab.Cmat + (int64_t)g * kMaxPolys * NPE * ndp;
    constexpr int MT = NPOLY * NPE / 8;  // 8-row tiles of the staging matrix
    constexpr int NT = kTD / 8;          // 8-tuple tiles
    for (int tile = wid; tile < MT * NT; tile += kSweepWarps) {
      const int mt = tile / NT, nt = tile % NT;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < ndp / 4; ++ks) {
        const double av = __ldg(Cm + (int64_t)(mt * 8 + (lane >> 2)) * ndp + ks * 4 + (lane & 3));
        const double bv = sMD[(nt * 8 + (lane >> 2)) * nde + ks * 4 + (lane & 3)];
        dmma(c0, c1, av, bv);
      }
      const int row = mt * 8 + (lane >> 2), t = nt * 8 + 2 * (lane & 3);
      sC[t * CS + row] = c0;
      sC[(t + 1) * CS + row] = c1;
    }
  }
  __syncthreads();

  // ---- per-program constants of Appendix A, folded once ----------------------------------------
  const EConst kc = make_econst(pg);
  const int map0 = pg.grid_map[0], map1 = pg.p >= 2 ? pg.grid_map[1] : -1,
            map2 = pg.p >= 3 ? pg.grid_map[2] : -1;
  const double rNSM = 1.0 / (double)n_sm;

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nFc = a.tab.nFc[2 * g];
  const bool sorted = a.tab.nFc[2 * g + 1] != 0;
  const int nFp = a.tab.nFp;
  const CfgRec *rec = a.tab.rec + (int64_t)g * nFp;
  const double *mP = a.tab.mP + (int64_t)g * a.npe_pad * nFp;

  // this warp's octet of tuples: row lane/4 of the DMMA tiles
  const int t = wid * 8 + (lane >> 2);
  const bool tok = t < tmax;
  const int32_t *Dt = sDv + t * kMaxVars;
  const int64_t D1 = Dt[0];
  const int64_t D1sq = D1 * D1;
  const int32_t Da = map0 >= 0 ? Dt[map0] : 1, Db = map1 >= 0 ? Dt[map1] : 1,
                Dc = map2 >= 0 ? Dt[map2] : 1;
  const double *arow = sC + t * CS + (lane & 3);

  Best st;
  st.e = kInf;
  st.i = 0x7fffffff;
  st.s = kInf;

  // the largest D1^2 among the warp's tuples (a3 early exit over configurations sorted by P1 P2)
  int64_t maxD1sq = tok ? D1sq : 0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, maxD1sq, o);
    maxD1sq = x > maxD1sq ? x : maxD1sq;
  }
  const int nOctF = (nFc + 7) >> 3;
  // a4 for one octet of configurations: p_k(D_t, P_c) for the octet of tuples x the octet of
  // configurations (k-step major: the NPOLY accumulation chains are independent, so consecutive
  // DMMAs do not wait).  B fragments: m_pe(u_P), pe = 4 ks + lane % 4, configuration 8 oc + lane / 4
#define RP_AFR(k, ks) arow[(k) * NPE + (ks) * 4]
  auto mma_oct = [&](int oc, double (&acc)[NPOLY][2]) {
    double bfr[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bfr[ks] = __ldg(mP + (int64_t)(ks * 4 + (lane & 3)) * nFp + oc * 8 + (lane >> 2));
#pragma unroll
    for (int k = 0; k < NPOLY; ++k) acc[k][0] = acc[k][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int k = 0; k < NPOLY; ++k) dmma(acc[k][0], acc[k][1], RP_AFR(k, ks), bfr[ks]);
    }
  };
#undef RP_AFR
  // a3, a6, a7, a8 for the 2 pairs of this lane in one octet
  auto epi_oct = [&](int oc, const double (&acc)[NPOLY][2]) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      // output column 2 (lane % 4) + v; padded configurations (c >= nFc) have zero records
      // and zero monomials, so their E is NaN and they are masked below
      const CfgRec *cr = rec + oc * 8 + 2 * (lane & 3) + v;
      const longlong2 h0 = __ldg(reinterpret_cast<const longlong2 *>(cr));      // P01 | orig, Pm1_0
      const int4 h1 = __ldg(reinterpret_cast<const int4 *>(cr) + 1);             // Pm1_1, Pm1_2, M0, M1
      const int32_t orig = (int32_t)(h0.y & 0xffffffff);
      // a3: "P1 P2 <= D1^2 is meaningful"
      const bool ok = tok && h0.x <= D1sq;
      double E;
      if (MWP) {
        const int4 h2 = __ldg(reinterpret_cast<const int4 *>(cr) + 2);           // M2, s012, W
        const double2 h3 = __ldg(reinterpret_cast<const double2 *>(cr) + 3);     // rB, rW
        const int32_t Pm1_0 = (int32_t)(h0.y >> 32);
        const uint32_t s012 = (uint32_t)h2.y;
        const double W = __hiloint2double(h2.w, h2.z);
        // a6: #Blocks = prod ceil(D / P); SM_act = min(#Blocks, n_SM)
        int64_t blocks = 1;
        if (map0 >= 0) blocks *= ceil_div_magic(Da, Pm1_0, (uint32_t)h1.z, s012 & 255);
        if (map1 >= 0) blocks *= ceil_div_magic(Db, h1.x, (uint32_t)h1.w, (s012 >> 8) & 255);
        if (map2 >= 0) blocks *= ceil_div_magic(Dc, h1.y, (uint32_t)h2.x, (s012 >> 16) & 255);
        const int64_t smact = blocks < n_sm ? blocks : n_sm;
        const double rSM = smact == n_sm ? rNSM : (rsm_tab ? sRSM[smact] : 1.0 / (double)smact);
        const double Rep = (double)blocks * h3.x * rSM;  // line 15: #Blocks / (B_act SM_act)
        E = mwpcwp_E(acc[0][v], acc[1][v], acc[2][v], acc[3][v], acc[4][v], acc[5][v], W, Rep,
                     rSM, (double)smact, kc);
      } else {
        E = acc[0][v] * frcp(acc[1][v]);  // template g1: E = g_1
      }
      // line 19 / reading R17: only finite positive estimates of meaningful pairs compete
      E = (ok && pos_finite(E)) ? E : kInf;
      // a8: exact lexicographic key (E, original index): ties go to the lowest index (E and the
      // running best are positive or +inf, so their bit patterns compare as integers)
      const long long eb = __double_as_longlong(E), sb = __double_as_longlong(st.e);
      const bool better = eb < sb || (eb == sb && orig < st.i);
      if (SECOND) st.s = better ? st.e : fmin(st.s, E);
      st.i = better ? orig : st.i;
      st.e = better ? E : st.e;
    }
  };
  if (wid * 8 < tmax) {
    // a3 early exit: configurations are sorted by P1 P2, so every octet from the first one whose
    // smallest P1 P2 exceeds the largest D1^2 of the warp's tuples fails the D rule
    int nEff = nOctF;
    if (sorted)
      for (int b0 = 0; b0 < nOctF; b0 += 32) {
        const int oc = b0 + lane;
        const unsigned stop = __ballot_sync(0xffffffffu, oc < nOctF && __ldg(&rec[oc * 8].P01) > maxD1sq);
        if (stop) {
          nEff = b0 + __ffs(stop) - 1;
          break;
        }
      }
    for (int oc = 0; oc < nEff; ++oc) {
      double acc[NPOLY][2];
      mma_oct(oc, acc);
      epi_oct(oc, acc);
    }
  }
  // ---- a8: the 4 lanes of a quad hold the same tuple ------------------------------------------
  st = merge(st, shfl_xor(st, 1));
  st = merge(st, shfl_xor(st, 2));
  if ((lane & 3) == 0 && tok) {
    const int64_t o = (int64_t)g * a.nD + (a.perm ? (int64_t)a.perm[d0 + t] : d0 + t);
    a.idx[o] = (st.e < kInf) ? st.i : -1;
    a.bestE[o] = st.e;
    if (SECOND) a.secondE[o] = st.s;
  }
}

template <int NPE, bool MWP, bool SECOND>
static cudaError_t launch3(const SweepArgs &a, int n_prog, int n_sm_max, cudaStream_t s) {
  const size_t smem = sweep_smem_bytes<MWP ? 6 : 2, NPE>(a.nde_stride, n_sm_max);
  const int64_t tiles = (a.nD + kTD - 1) / kTD;
  if (tiles > 0x7fffffffll || n_prog > 65535) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_sweep<NPE, MWP, SECOND>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_sweep<NPE, MWP, SECOND><<<dim3((unsigned)tiles, (unsigned)n_prog), kSweepThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NPE>
static cudaError_t launch_npe(const SweepArgs &a, int n_prog, bool mwp, int n_sm_max, cudaStream_t s) {
  const bool second = a.secondE != nullptr;
  if (mwp)
    return second ? launch3<NPE, true, true>(a, n_prog, n_sm_max, s)
                  : launch3<NPE, true, false>(a, n_prog, n_sm_max, s);
  return second ? launch3<NPE, false, true>(a, n_prog, n_sm_max, s)
                : launch3<NPE, false, false>(a, n_prog, n_sm_max, s);
}

cudaError_t launch_sweep(const DevProg *d_progs, int n_prog, bool mwp, CfgTable tab, int npe_pad,
                         int nde_max, int n_sm_max, int d, const int32_t *d_D, int64_t nD,
                         int32_t *idx, double *bestE, double *secondE, const int32_t *perm,
                         cudaStream_t s) {
  if (nD == 0) return cudaSuccess;
  if (n_sm_max >= kRSMTab) n_sm_max = 0;  // no table: 1/SM_act computed directly
  (void)nde_max;
  SweepArgs a{d_progs, tab, npe_pad, d, md_stride(tab.nde_pad), d_D, nD, idx, bestE, secondE, perm};
  switch (npe_pad) {
    case 4: return launch_npe<4>(a, n_prog, mwp, n_sm_max, s);
    case 8: return launch_npe<8>(a, n_prog, mwp, n_sm_max, s);
    case 16: return launch_npe<16>(a, n_prog, mwp, n_sm_max, s);
    case 20: return launch_npe<20>(a, n_prog, mwp, n_sm_max, s);
    case 24: return launch_npe<24>(a, n_prog, mwp, n_sm_max, s);
    case 36: return launch_npe<36>(a, n_prog, mwp, n_sm_max, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rp
