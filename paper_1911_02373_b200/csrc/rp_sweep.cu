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
#include <cstdlib>
#include <cstring>

#include "rp_device.cuh"
#include "rp_umma.cuh"

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

// m = prod u_k^{e_k} as a double-double (hi exact product chain by FMA, lo the running error)
__device__ __forceinline__ double2 dd_monomial(const int8_t *e, int n, const double *u) {
  double h = 1.0, l = 0.0;
  for (int k = 0; k < n; ++k)
    for (int t = 0; t < e[k]; ++t) {
      const double nh = h * u[k];
      l = fma(l, u[k], fma(h, u[k], -nh));
      h = nh;
    }
  return make_double2(h, l);
}

__device__ void build_refine_terms(int g, const DevProg &pg, const CfgTable &tab, int npe_pad);
__device__ void schedule_slot_mp(const DevProg &pg, const CfgRec &r, int hv, int npe_pad, double *col, int nGp);
__device__ bool group_lists(const DevProg &pg, int hv, int32_t (*off)[kGS]);
__device__ void group_y(const DevProg &pg, GroupDesc &gd);

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
      // running product with an early bound: every P_k >= 1, so once T exceeds T_max it stays
      // above it (no int64 wrap-around for P_k up to 2^31 - 1)
      bool pos = true, big = false;
      for (int k = 0; k < pg.p; ++k) {
        pos = pos && Pk[k] >= 1;
        if (pos && !big) {
          T *= Pk[k];
          big = T > pg.t_max;
        }
      }
      // "a multiple of the warp size (32)" and "bounded over by the maximum number of threads
      // per block"
      ok = pos && !big && (T % 32 == 0) && (T <= pg.t_max);
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
    if (c < nF) tab.inv[(int64_t)g * nFp + c] = ok ? pos : -1;
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
      r.W32 = (float)W;
      r.rB32 = (float)r.rB;
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
        // the refinement's double-double copy, by srec position
        tab.mPdd[((int64_t)g * nFp + pos) * npe_pad + pe] =
            pe < pg.nPE ? dd_monomial(pg.pe_exp[pe], pg.p, u) : make_double2(0.0, 0.0);
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
  __syncthreads();
  build_refine_terms(g, pg, tab, npe_pad);
}

// rp_plan_update_program: the configuration table (a1 masks, a5 occupancy, the P1 P2 order, the
// tile schedule) depends on F, the hardware and the kernel's resources only, so a refit changes
// just the coefficients (the dense staging matrix Cmat and the refinement's term table) and the
// transform (the program-part monomials of the configurations, the factored tiles' powers and
// the groups' Y values).  Three launches: the new values into the program (one CTA), the tables
// that depend on them (grid-stride over every entry), the refinement terms (one CTA: a compaction).
__global__ void __launch_bounds__(1024) k_plan_refresh_prog(DevProg *pgp, const double *coef, int stride,
                                                            const double *xf) {
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
}

__global__ void __launch_bounds__(256) k_plan_refresh_tables(const DevProg *pgp, int g, int npe_pad, CfgTable tab) {
  const DevProg &pg = *pgp;
  const int nFp = tab.nFp, nFc = tab.nFc[2 * g];
  const int nGp = tab.nGp, nslot = tab.gcnt[4 * g + 2] * 8, ngr = tab.gcnt[4 * g + 0];
  const int nrow = pg.npoly * pg.nPE;
  const CfgRec *rec = tab.rec + (int64_t)g * nFp;
  double *mP = tab.mP + (int64_t)g * npe_pad * nFp;
  const CfgRec *grec = tab.grec + (int64_t)g * nGp;
  double *gmP = tab.gmP + (int64_t)g * npe_pad * nGp;
  const int32_t *ghv = tab.ghv + (int64_t)g * nGp;
  GroupDesc *gdesc = tab.gdesc + (int64_t)g * kMaxGroups;
  double *Cm = tab.Cmat + (int64_t)g * kMaxPolys * npe_pad * tab.nde_pad;
  // work items: [configuration monomials | schedule slots | staging rows | groups | the
  // refinement's double-double monomials by srec position]
  const int n0 = nFc * npe_pad, n1 = n0 + nslot, n2 = n1 + nrow, n3 = n2 + ngr, n4 = n3 + nFc * npe_pad;
  const CfgRec *srec = tab.srec + (int64_t)g * nFp;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += gridDim.x * blockDim.x) {
    if (t >= n3) {
      const int pos = (t - n3) / npe_pad, pe = (t - n3) % npe_pad;
      double2 m = make_double2(0.0, 0.0);
      if (pe < pg.nPE) {
        const CfgRec &r = srec[pos];
        const int32_t Pk[3] = {r.Pm1_0 + 1, r.Pm1_1 + 1, r.Pm1_2 + 1};
        double u[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < pg.p; ++k) u[k] = ((double)Pk[k] - pg.xc[pg.d + k]) * ldexp(1.0, -pg.xe[pg.d + k]);
        m = dd_monomial(pg.pe_exp[pe], pg.p, u);
      }
      tab.mPdd[((int64_t)g * nFp + pos) * npe_pad + pe] = m;
      continue;
    }
    if (t < n0) {
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
    } else if (t < n1) {
      const int sl = t - n0;
      schedule_slot_mp(pg, grec[sl], ghv[sl], npe_pad, gmP + sl, nGp);
    } else if (t < n2) {
      const int r = t - n1, k = r / pg.nPE, pe = r % pg.nPE;
      for (int j = pg.row_start[r]; j < pg.row_start[r + 1]; ++j)
        Cm[(int64_t)(k * npe_pad + pe) * tab.nde_pad + pg.term_de[j]] = pg.term_coef[j];
    } else {
      GroupDesc &gd = gdesc[t - n2];
      // off[][] holds 0 for padding terms now: rebuild the lists (Y = 0 marks them)
      int32_t off[4][kGS];
      group_lists(pg, gd.hv, off);
      for (int q = 0; q < 4; ++q)
        for (int s = 0; s < kGS; ++s) gd.off[q][s] = off[q][s];
      group_y(pg, gd);
    }
  }
}

__global__ void __launch_bounds__(1024) k_plan_refresh_terms(const DevProg *pgp, int g, int npe_pad, CfgTable tab) {
  build_refine_terms(g, *pgp, tab, npe_pad);
}

// ---- the sweep's tile schedule: factored tiles of configuration groups, then dense tiles ----------
// u_k of program variable k (the transform of k_plan_configs)
__device__ __forceinline__ double prog_u(const DevProg &pg, int k, int32_t P) {
  return ((double)P - pg.xc[pg.d + k]) * ldexp(1.0, -pg.xe[pg.d + k]);
}

// B operands of one schedule slot: a factored slot holds x^{1+q} (x = u_hv(P_hv)) in rows q < 4,
// a dense slot the program-part monomials m_pe(u_P) (as k_plan_configs computes them)
__device__ void schedule_slot_mp(const DevProg &pg, const CfgRec &r, int hv, int npe_pad, double *col, int nGp) {
  const int32_t Pk[3] = {r.Pm1_0 + 1, r.Pm1_1 + 1, r.Pm1_2 + 1};
  if (hv == -2) {  // padding
    for (int pe = 0; pe < npe_pad; ++pe) col[(int64_t)pe * nGp] = 0.0;
    return;
  }
  if (hv >= 0) {  // factored slots are hv-major (k_plan_groups): P_hv at position 0
    const double x = prog_u(pg, hv, Pk[0]);
    double m = 1.0;
    for (int q = 0; q < npe_pad; ++q) {
      m = q < 4 ? m * x : 0.0;
      col[(int64_t)q * nGp] = m;
    }
    return;
  }
  double u[3];
  for (int k = 0; k < pg.p; ++k) u[k] = prog_u(pg, k, Pk[k]);
  for (int pe = 0; pe < npe_pad; ++pe) {
    double m = 0.0;
    if (pe < pg.nPE) {
      m = 1.0;
      for (int k = 0; k < pg.p; ++k)
        for (int t = 0; t < pg.pe_exp[pe][k]; ++t) m *= u[k];
    }
    col[(int64_t)pe * nGp] = m;
  }
}

// the term lists of Horner variable hv: lane q sums w_{1+q} over off[q][0..kGS1) and its share of
// w_0 over off[q][kGS1..kGS) (entries q, q + 4 of the i = 0 list); false when the program's
// monomials do not fit them (then no groups on hv)
__device__ bool group_lists(const DevProg &pg, int hv, int32_t (*off)[kGS]) {
  int cnt[5] = {0, 0, 0, 0, 0};
  for (int q = 0; q < 4; ++q)
    for (int s = 0; s < kGS; ++s) off[q][s] = -1;  // padding terms (Y = 0)
  for (int pe = 0; pe < pg.nPE; ++pe) {
    const int i = pg.pe_exp[pe][hv];
    if (i > 4) return false;
    if (i == 0) {
      if (cnt[0] >= 4 * kGW0) return false;
      off[cnt[0] % 4][kGS1 + cnt[0] / 4] = pe;
    } else {
      if (cnt[i] >= kGS1) return false;
      off[i - 1][cnt[i]] = pe;
    }
    ++cnt[i];
  }
  return true;
}

// Y_pe of a group's terms (they depend on the transform: recomputed at every refit)
__device__ void group_y(const DevProg &pg, GroupDesc &gd) {
  double u[3] = {1.0, 1.0, 1.0};
  for (int k = 0; k < pg.p; ++k) u[k] = prog_u(pg, k, gd.P[k]);
  for (int q = 0; q < 4; ++q)
    for (int s = 0; s < kGS; ++s) {
      const int pe = gd.off[q][s];
      double y = 0.0;
      if (pe >= 0) {
        y = 1.0;
        for (int k = 0; k < pg.p; ++k)
          if (k != gd.hv)
            for (int t = 0; t < pg.pe_exp[pe][k]; ++t) y *= u[k];
      }
      gd.y[q][s] = y;
    }
  for (int q = 0; q < 4; ++q)  // padding terms read a valid column with Y = 0
    for (int s = 0; s < kGS; ++s) gd.off[q][s] = gd.off[q][s] < 0 ? 0 : gd.off[q][s];
  for (int pe = 0; pe < kMaxPE; ++pe) {  // the same values by pe, with the Horner exponent
    double y = 0.0;
    int8_t ip = -1;
    if (pe < pg.nPE) {
      y = 1.0;
      for (int k = 0; k < pg.p; ++k)
        if (k != gd.hv)
          for (int t = 0; t < pg.pe_exp[pe][k]; ++t) y *= u[k];
      ip = pg.pe_exp[pe][gd.hv];
    }
    gd.ype[pe] = y;
    gd.ipe[pe] = ip;
  }
}

// One CTA per program, after k_plan_configs.  Candidate groups: for every Horner variable whose
// term lists fit, the sets of feasible configurations with equal P_k (k != hv) and >= 8 members.
// Greedy, largest first (ties: lower hv, then lower position): a group takes the floor(n / 8) * 8
// lowest-P1P2 members nobody took yet (full tiles only).  The rest is dense, in (P1 P2, index) order.
// Which tile evaluates a pair changes only the rounding of p_k (the exact key (E, index) decides).
__global__ void __launch_bounds__(1024) k_plan_groups(const DevProg *progs, int npe_pad, CfgTable tab, int enable) {
  const int g = blockIdx.x;
  const DevProg &pg = progs[g];
  const int nFp = tab.nFp, nGp = tab.nGp;
  const int nFc = tab.nFc[2 * g];
  const bool sorted = tab.nFc[2 * g + 1] != 0;
  const CfgRec *rec = tab.rec + (int64_t)g * nFp;
  const double *mP = tab.mP + (int64_t)g * npe_pad * nFp;
  CfgRec *grec = tab.grec + (int64_t)g * nGp;
  double *gmP = tab.gmP + (int64_t)g * npe_pad * nGp;
  int32_t *ghv = tab.ghv + (int64_t)g * nGp;
  GroupDesc *gdesc = tab.gdesc + (int64_t)g * kMaxGroups;

  __shared__ int32_t s_slot[kGroupMaxPlan + 8];   // schedule slot -> position in rec (-1: padding)
  __shared__ int8_t s_hv[kGroupMaxPlan + 8];      // slot's Horner variable (-1 dense)
  __shared__ uint8_t s_taken[kGroupMaxPlan];
  __shared__ int32_t s_P[3][kGroupMaxPlan];       // P_k - 1 of the sorted configurations
  // candidates: a key has >= 8 members, so at most 3 nFc / 8 of them
  constexpr int kMaxCand = 3 * kGroupMaxPlan / 8;
  __shared__ int32_t s_cand[kMaxCand];   // hv << 16 | first member position
  __shared__ int32_t s_csize[kMaxCand];
  __shared__ int32_t s_corder[kMaxCand];
  __shared__ int32_t s_off[3][4][kGS];
  __shared__ int32_t s_wsum[32];
  __shared__ int s_hvok[3], s_ncand, s_ngroups, s_ntiles, s_ngt, s_ns, s_cnt;
  const bool grouping = enable && sorted && pg.p >= 2 && nFc <= kGroupMaxPlan;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int hv = 0; hv < 3; ++hv) s_hvok[hv] = grouping && hv < pg.p && group_lists(pg, hv, s_off[hv]);
    s_ncand = 0;
    s_ns = 0;
  }
  for (int i = threadIdx.x; i < kGroupMaxPlan; i += blockDim.x) {
    s_taken[i] = 0;
    if (grouping && i < nFc) {
      s_P[0][i] = rec[i].Pm1_0;
      s_P[1][i] = rec[i].Pm1_1;
      s_P[2][i] = rec[i].Pm1_2;
    }
  }
  __syncthreads();
  auto same_key = [&](int a, int b, int hv) {  // configurations a, b share every P_k, k != hv
    return (hv == 0 || s_P[0][a] == s_P[0][b]) && (hv == 1 || s_P[1][a] == s_P[1][b]) &&
           (hv == 2 || s_P[2][a] == s_P[2][b]);
  };
  // block-wide exclusive prefix of one count per thread (deterministic; all threads call it)
  auto block_scan = [&](int v, int &total) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int w = lane < nwarp ? s_wsum[lane] : 0;
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      s_wsum[lane] = wi - w;  // exclusive prefix of the warps
      if (lane == 31) s_cnt = wi;
    }
    __syncthreads();
    const int ex = s_wsum[wid] + incl - v;
    total = s_cnt;
    __syncthreads();
    return ex;
  };
  if (grouping) {
    for (int hv = 0; hv < 3; ++hv) {
      if (!s_hvok[hv]) continue;
      for (int c = threadIdx.x; c < nFc; c += blockDim.x) {
        int n = 0;
        bool first = true;
        for (int j = 0; j < nFc; ++j) {
          const bool m = same_key(j, c, hv);
          n += m;
          first = first && !(m && j < c);
        }
        if (first && n >= 8) {
          const int k = atomicAdd(&s_ncand, 1);
          s_cand[k] = hv << 16 | c;
          s_csize[k] = n;
        }
      }
      __syncthreads();
    }
    // order: size descending, then (hv, position) ascending -- a rank sort, deterministic
    const int nc = s_ncand;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      int rank = 0;
      for (int j = 0; j < nc; ++j)
        rank += s_csize[j] > s_csize[i] || (s_csize[j] == s_csize[i] && s_cand[j] < s_cand[i]);
      s_corder[rank] = i;
    }
    __syncthreads();
  }
  // greedy assignment, one candidate at a time; each thread owns the contiguous positions
  // [per t, per (t + 1)) so member ranks follow the position order
  const int per = (nFc + blockDim.x - 1) / blockDim.x;
  const int p0 = threadIdx.x * per, p1 = min(nFc, p0 + per);
  int ngroups = 0;
  const int ncand = grouping ? s_ncand : 0;
  for (int r = 0; r < ncand && ngroups < kMaxGroups; ++r) {
    const int cd = s_cand[s_corder[r]], hv = cd >> 16, c0 = cd & 0xffff;
    int mine = 0;
    for (int q = p0; q < p1; ++q) mine += q >= c0 && !s_taken[q] && same_key(q, c0, hv);
    int n;
    int rank = block_scan(mine, n);
    const int take = n / 8 * 8;
    if (take == 0) continue;  // (uniform)
    const int ns = s_ns;
    for (int q = p0; q < p1 && rank < take; ++q)
      if (q >= c0 && !s_taken[q] && same_key(q, c0, hv)) {
        s_taken[q] = 1;
        s_slot[ns + rank] = q;
        s_hv[ns + rank] = (int8_t)hv;
        ++rank;
      }
    if (threadIdx.x == 0) {
      GroupDesc &gd = gdesc[ngroups];
      gd.tile_begin = ns / 8;
      gd.tile_end = (ns + take) / 8;
      gd.hv = hv;
      gd.nmem = take;
      gd.P[0] = s_P[0][c0] + 1;
      gd.P[1] = s_P[1][c0] + 1;
      gd.P[2] = s_P[2][c0] + 1;
      gd.pad = 0;
      for (int q = 0; q < 4; ++q)
        for (int t = 0; t < kGS; ++t) gd.off[q][t] = s_off[hv][q][t];
      group_y(pg, gd);
      s_ns = ns + take;
    }
    ++ngroups;
    __syncthreads();
  }
  // the dense remainder in (P1 P2, index) order, then padding to a whole tile
  if (nFc <= kGroupMaxPlan) {
    int mine = 0;
    for (int q = p0; q < p1; ++q) mine += !s_taken[q];
    int tot;
    int rank = block_scan(mine, tot);
    const int ns = s_ns;
    if (threadIdx.x == 0) s_ngt = ns / 8;
    for (int q = p0; q < p1; ++q)
      if (!s_taken[q]) {
        s_slot[ns + rank] = q;
        s_hv[ns + rank] = -1;
        ++rank;
      }
    int end = ns + tot;
    for (int t = end + threadIdx.x; t < ((end + 7) & ~7); t += blockDim.x) {
      s_slot[t] = -1;
      s_hv[t] = -2;
    }
    if (threadIdx.x == 0) {
      s_ngroups = ngroups;
      s_ntiles = ((end + 7) & ~7) / 8;
    }
  }
  __syncthreads();
  const int nslots = s_ntiles * 8;
  // nFc > kGroupMaxPlan: the slots are the table itself, 1:1 (no shared list)
  const bool big = nFc > kGroupMaxPlan;
  const int nsl = big ? ((nFc + 7) & ~7) : nslots;
  for (int s = threadIdx.x; s < nGp; s += blockDim.x) {
    int pos = -1, hv = -2;
    if (s < nsl) {
      pos = big ? (s < nFc ? s : -1) : s_slot[s];
      hv = big ? (s < nFc ? -1 : -2) : s_hv[s];
    }
    CfgRec r;
    if (pos >= 0) {
      r = rec[pos];
      if (hv > 0) {  // factored slot, hv-major: P_hv's (P - 1, M, s) at position 0 for the sweep
        const int32_t Ph = hv == 1 ? r.Pm1_1 : r.Pm1_2;
        const uint32_t Mh = hv == 1 ? r.M1 : r.M2;
        const uint32_t sh = (r.s012 >> (8 * hv)) & 255u;
        if (hv == 1) {
          r.Pm1_1 = r.Pm1_0;
          r.M1 = r.M0;
        } else {
          r.Pm1_2 = r.Pm1_0;
          r.M2 = r.M0;
        }
        const uint32_t s0 = r.s012 & 255u;
        r.s012 = (r.s012 & ~(255u | (255u << (8 * hv)))) | sh | (s0 << (8 * hv));
        r.Pm1_0 = Ph;
        r.M0 = Mh;
      }
    } else {
      memset(&r, 0, sizeof(r));
      r.orig = 0x7fffffff;  // zero record: W = 0, 1/B_act = 0, so its E is never a candidate
    }
    grec[s] = r;
    ghv[s] = hv;
    if (hv == -1 && pos >= 0) {  // dense: the table's monomials, bit for bit
      for (int pe = 0; pe < npe_pad; ++pe) gmP[(int64_t)pe * nGp + s] = mP[(int64_t)pe * nFp + pos];
    } else {
      schedule_slot_mp(pg, r, hv, npe_pad, gmP + s, nGp);
    }
  }
  if (threadIdx.x == 0) {
    tab.gcnt[4 * g + 0] = big ? 0 : s_ngroups;
    tab.gcnt[4 * g + 1] = big ? 0 : s_ngt;
    tab.gcnt[4 * g + 2] = big ? nsl / 8 : s_ntiles;
    tab.gcnt[4 * g + 3] = 0;
  }
}

cudaError_t launch_plan_refresh(DevProg *d_prog, int g, const double *d_coef, int stride, const double *d_xf,
                                int npe_pad, CfgTable tab, cudaStream_t s) {
  k_plan_refresh_prog<<<1, 1024, 0, s>>>(d_prog, d_coef, stride, d_xf);
  k_plan_refresh_tables<<<4 * num_sms() < 64 ? 4 * num_sms() : 64, 256, 0, s>>>(d_prog, g, npe_pad, tab);
  k_plan_refresh_terms<<<1, 1024, 0, s>>>(d_prog, g, npe_pad, tab);
  return cudaGetLastError();
}

cudaError_t launch_plan_configs(const DevProg *d_progs, int n_prog, const int32_t *d_F, int nF,
                                int npe_pad, CfgTable tab, cudaStream_t s) {
  k_plan_configs<<<n_prog, 1024, 0, s>>>(d_progs, d_F, nF, npe_pad, tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const char *ge = getenv("RP_SWEEP_GROUPS");  // 0: dense tiles only (A/B measurements)
  k_plan_groups<<<n_prog, 1024, 0, s>>>(d_progs, npe_pad, tab, !(ge && ge[0] == '0'));
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
  int32_t *idx2 = nullptr;  // runner-up's original index [n_prog][nD] (SECOND; for the refinement)
  const unsigned char *tcpack = nullptr;  // k_sweep_tc: per-tile B operands, ||m||, records
  int tc_ntiles = 0;
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

// FAST (MWP-CWP programs whose winners k_refine re-evaluates): E only ranks here -- one-step
// reciprocals, Rep = 1/B_act when #Blocks < n_SM (SM_act = #Blocks cancels exactly) and, without a
// runner-up, a packed (E, index) key
template <int NPE, bool MWP, bool SECOND, bool FAST>
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
    constexpr int NT = kTD / 8;          // 8-tuple tiles (= kSweepWarps)
    // a warp takes whole row tiles: each A fragment (from the plan's matrix, L2) is loaded once
    // and used for the NT tuple tiles, and a row tile's k-step loads are issued together
    for (int mt = wid; mt < MT; mt += kSweepWarps) {
      const double *ca = Cm + (int64_t)(mt * 8 + (lane >> 2)) * ndp + (lane & 3);
      double c0[NT], c1[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) c0[nt] = c1[nt] = 0.0;
      for (int ks0 = 0; ks0 < ndp / 4; ks0 += 4) {
        double av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = ks0 + u < ndp / 4 ? __ldg(ca + (ks0 + u) * 4) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ks0 + u >= ndp / 4) break;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            dmma(c0[nt], c1[nt], av[u], sMD[(nt * 8 + (lane >> 2)) * nde + (ks0 + u) * 4 + (lane & 3)]);
        }
      }
      const int row = mt * 8 + (lane >> 2);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int t = nt * 8 + 2 * (lane & 3);
        sC[t * CS + row] = c0[nt];
        sC[(t + 1) * CS + row] = c1[nt];
      }
    }
  }
  __syncthreads();

  // ---- per-program constants of Appendix A, folded once ----------------------------------------
  const EConst kc = make_econst(pg);
  const int map0 = pg.grid_map[0], map1 = pg.p >= 2 ? pg.grid_map[1] : -1,
            map2 = pg.p >= 3 ? pg.grid_map[2] : -1;
  const double rNSM = 1.0 / (double)n_sm;
  const uint32_t sRSM_s = (uint32_t)__cvta_generic_to_shared(sRSM);

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool sorted = a.tab.nFc[2 * g + 1] != 0;
  // the tile schedule (k_plan_groups): factored tiles [0, ngt) in groups, dense tiles [ngt, ntile)
  const int nGp = a.tab.nGp;
  const int ngr = a.tab.gcnt[4 * g], ngt = a.tab.gcnt[4 * g + 1], ntile = a.tab.gcnt[4 * g + 2];
  const CfgRec *grec = a.tab.grec + (int64_t)g * nGp;
  const double *gmP = a.tab.gmP + (int64_t)g * a.npe_pad * nGp;
  const GroupDesc *gdesc = a.tab.gdesc + (int64_t)g * kMaxGroups;

  // this warp's octet of tuples: row lane/4 of the DMMA tiles
  const int t = wid * 8 + (lane >> 2);
  const int32_t *Dt = sDv + t * kMaxVars;
  // data parameters are sizes: a tuple with some D_k < 1 has no meaningful P (reading R32)
  bool dpos = true;
  for (int k = 0; k < d; ++k) dpos = dpos && Dt[k] >= 1;
  const bool tok = t < tmax && dpos;
  const int64_t D1 = Dt[0];
  const int64_t D1sq = D1 * D1;
  // the a3 test in 32 bits: P1 P2 of a compacted configuration is <= T_max < 2^31
  const int32_t D1sq32 = D1sq < 0x7fffffffll ? (int32_t)D1sq : 0x7fffffff;
  // (a tuple with some D_k < 1 is masked; its grid is computed from 1s so no index goes wild)
  const int32_t Da = map0 >= 0 && dpos ? Dt[map0] : 1, Db = map1 >= 0 && dpos ? Dt[map1] : 1,
                Dc = map2 >= 0 && dpos ? Dt[map2] : 1;
  const double *arow = sC + t * CS + (lane & 3);

  Best st;
  st.e = kInf;
  st.i = 0x7fffffff;
  st.s = kInf;
  st.j = 0x7fffffff;
  // FAST ranking without a runner-up: one 64-bit key per pair, E's bit pattern with its 13 low
  // mantissa bits replaced by the original index (< 8192: launch3 takes FAST only then) -- a
  // 2^-39 relative perturbation of a ranking value that is only ~1e-12 accurate anyway; the
  // refinement re-evaluates the winner exactly (4.282 -> 4.182 ms against the exact (E, index)
  // compare with its tie-break)
  unsigned long long pkey = ~0ull;

  // the largest D1^2 among the warp's tuples (a3 early exit over configurations sorted by P1 P2)
  int64_t maxD1sq = tok ? D1sq : 0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, maxD1sq, o);
    maxD1sq = x > maxD1sq ? x : maxD1sq;
  }
  // a4 for one dense tile of configurations: p_k(D_t, P_c) for the octet of tuples x the octet of
  // configurations (k-step major: the NPOLY accumulation chains are independent, so consecutive
  // DMMAs do not wait).  B fragments: m_pe(u_P), pe = 4 ks + lane % 4, configuration 8 oc + lane / 4
#define RP_AFR(k, ks) arow[(k) * NPE + (ks) * 4]
  // this lane's B-fragment column of the schedule's monomial table (4.160 -> 4.114 ms against
  // recomputing the 64-bit address of every load)
  const double *bbase = gmP + (int64_t)(lane & 3) * nGp + (lane >> 2);
  const int64_t bks = 4 * (int64_t)nGp;
  auto load_b = [&](int oc, double (&bfr)[KS]) {
    const double *bp = bbase + oc * 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bfr[ks] = __ldg(bp + ks * bks);
  };
  auto mma_oct = [&](double (&acc)[NPOLY][2], const double (&bfr)[KS]) {
#pragma unroll
    for (int k = 0; k < NPOLY; ++k) acc[k][0] = acc[k][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int k = 0; k < NPOLY; ++k) dmma(acc[k][0], acc[k][1], RP_AFR(k, ks), bfr[ks]);
    }
  };
#undef RP_AFR
  // a3, a6, a7, a8 for the 2 pairs of this lane in one tile
  // fact: a factored tile (grid factors other than P_hv's are the group's fcon; Dv = D_{map[hv]})
  auto epi_oct = [&](const CfgRec *trec, const double (&acc)[NPOLY][2], bool fact, uint64_t fcon, int32_t Dv) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      // output column 2 (lane % 4) + v; padding slots have zero records (W = 0, 1/B_act = 0),
      // so their E is 0 or NaN and they are masked below
      const CfgRec *cr = trec + 2 * (lane & 3) + v;
      const longlong2 h0 = __ldg(reinterpret_cast<const longlong2 *>(cr));      // P01 | orig, Pm1_0
      const int4 h1 = __ldg(reinterpret_cast<const int4 *>(cr) + 1);             // Pm1_1, Pm1_2, M0, M1
      const int32_t orig = (int32_t)(h0.y & 0xffffffff);
      // a3: "P1 P2 <= D1^2 is meaningful"
      const bool ok = tok && (int32_t)(h0.x & 0xffffffff) <= D1sq32;
      double E;
      if (MWP) {
        const int4 h2 = __ldg(reinterpret_cast<const int4 *>(cr) + 2);           // M2, s012, W
        const double2 h3 = __ldg(reinterpret_cast<const double2 *>(cr) + 3);     // rB, (W32, rB32)
        const int32_t Pm1_0 = (int32_t)(h0.y >> 32);
        const uint32_t s012 = (uint32_t)h2.y;
        const double W = __hiloint2double(h2.w, h2.z);
        // a6: #Blocks = prod ceil(D / P); SM_act = min(#Blocks, n_SM)
        // (each factor is < 2^32: 32-bit factors, 64-bit products only where needed)
        int64_t blocks;
        if (fact) {  // factored slot: position 0 holds P_hv; the other factors are the group's
          blocks = (int64_t)(fcon * ceil_div32(Dv, Pm1_0, (uint32_t)h1.z, s012 & 255));
        } else {
          const uint32_t f0 = map0 >= 0 ? ceil_div32(Da, Pm1_0, (uint32_t)h1.z, s012 & 255) : 1u;
          const uint32_t f1 = map1 >= 0 ? ceil_div32(Db, h1.x, (uint32_t)h1.w, (s012 >> 8) & 255) : 1u;
          blocks = (int64_t)((uint64_t)f0 * f1);
          if (map2 >= 0) blocks *= ceil_div32(Dc, h1.y, (uint32_t)h2.x, (s012 >> 16) & 255);
        }
        // (one 64-bit compare; SM_act itself fits 32 bits)
        const bool full = blocks >= n_sm;
        const int32_t smact = full ? n_sm : (int32_t)blocks;
        // (n_SM < kRSMTab for every program, compile_program: the 1/SM_act table exists; an
        // explicit shared-window load -- through the generic pointer the compiler rebuilt the
        // shared address from SR_CgaCtaId for every pair; with the 32-bit SM_act: 4.445 -> 4.374 ms)
        double rSM = rNSM;
        if (!full) asm("ld.shared.f64 %0, [%1];" : "=d"(rSM) : "r"(sRSM_s + 8u * (uint32_t)smact));
        // line 15: #Blocks / (B_act SM_act)
        const double Rep = FAST ? (full ? (double)blocks * h3.x * rNSM : h3.x) : (double)blocks * h3.x * rSM;
        E = mwpcwp_E<FAST>(acc[0][v], acc[1][v], acc[2][v], acc[3][v], acc[4][v], acc[5][v], W, Rep,
                           rSM, (double)smact, kc);
      } else {
        E = acc[0][v] * frcp(acc[1][v]);  // template g1: E = g_1
      }
      if constexpr (FAST && !SECOND) {
        // line 19 / reading R17 folded into the key: bits(E) - 1 as unsigned puts +0, negative
        // values and NaN above every positive finite E (and +inf at the top of that range, which
        // the "no winner" test below excludes); masked pairs get the largest key
        const unsigned long long eb1 = (unsigned long long)__double_as_longlong(E) - 1ull;
        const unsigned long long key = ok ? ((eb1 & ~0x1FFFull) | (unsigned long long)(uint32_t)orig) : ~0ull;
        pkey = key < pkey ? key : pkey;
        continue;
      }
      // line 19 / reading R17: only finite positive estimates of meaningful pairs compete
      E = (ok && pos_finite(E)) ? E : kInf;
      // a8: exact lexicographic key (E, original index): ties go to the lowest index (E and the
      // running best are positive or +inf, so their bit patterns compare as integers)
      const long long eb = __double_as_longlong(E), sb = __double_as_longlong(st.e);
      const bool better = eb < sb || (eb == sb && orig < st.i);
      if (SECOND) {  // runner-up on the same exact key
        const bool sec = !better && key_less(E, orig, st.s, st.j);
        st.s = better ? st.e : (sec ? E : st.s);
        st.j = better ? st.i : (sec ? orig : st.j);
      }
      st.i = better ? orig : st.i;
      st.e = better ? E : st.e;
    }
  };
#ifdef RP_SWEEP_PROBE
  const bool probe_on = false;  // timing probe: the prologue and outputs only
#else
  const bool probe_on = true;
#endif
  if (probe_on && wid * 8 < tmax) {
    // factored tiles (k_plan_groups): per group, the octet's Horner coefficients w_{k,i} are one
    // small DMMA product with the staged C (4.338 -> 4.282 ms against lane-wise FMA sums of
    // bank-conflicted shared-memory reads and quad shuffles); each tile of the group is then one
    // DMMA per polynomial: C = w_{k,0}, A = w_{k,1+q}, B = x^{1+q} of configuration lane / 4
    const int q = lane & 3;
#ifdef RP_SWEEP_PROBE_NOFACT  // timing probe: dense tiles only
    for (int gi = 0; gi < 0; ++gi) {
#else
    for (int gi = 0; gi < ngr; ++gi) {
#endif
      const GroupDesc *gd = gdesc + gi;
      const int tb = __ldg(&gd->tile_begin), te = __ldg(&gd->tile_end);
      if (sorted && __ldg(&grec[tb * 8].P01) > maxD1sq) continue;  // a3: every member fails
      double w1[NPOLY], a0[NPOLY];
      // on DMMA, A = the staged C of the octet (the dense tiles' fragments: conflict-free), B =
      // Y_pe routed to column 2q when i_pe = 1 + q and to column 2q + 1 when i_pe = 0, so lane q
      // receives w_{k,1+q} and w_{k,0} of its tuple directly (no quad sum)
      {
        const int col = lane >> 2, want = (col & 1) ? 0 : 1 + (col >> 1);
        double bfr[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int pe = ks * 4 + (lane & 3);
          bfr[ks] = __ldg(&gd->ipe[pe]) == want ? __ldg(&gd->ype[pe]) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NPOLY; ++k) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) dmma(c0, c1, arow[k * NPE + ks * 4], bfr[ks]);
          w1[k] = c0;
          a0[k] = c1;
        }
      }
      // a6 per group: every grid factor but P_hv's is the group's (exact, once per group)
      uint64_t fcon = 1;
      int32_t Dv = 1;
      {
        const int hv = __ldg(&gd->hv);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int mk = k == 0 ? map0 : (k == 1 ? map1 : map2);
          if (mk < 0) continue;
          const int32_t Dk = k == 0 ? Da : (k == 1 ? Db : Dc);
          if (k == hv) {
            Dv = Dk;
          } else {  // (32-bit unsigned division: D + P - 1 < 2^32; a 64-bit one costs ~70 instructions)
            const uint32_t Pk = (uint32_t)__ldg(&gd->P[k]);
            fcon *= (uint64_t)(((uint32_t)Dk + Pk - 1u) / Pk);
          }
        }
      }
      int tend = te;  // members in P1 P2 order: stop at the first tile that fails a3 everywhere
      if (sorted)  // (the group's tiles tested by the lanes at once)
        for (int t0 = tb + 1; t0 < te; t0 += 32) {
          const int tile = t0 + lane;
          const unsigned stop = __ballot_sync(0xffffffffu, tile < te && __ldg(&grec[tile * 8].P01) > maxD1sq);
          if (stop) {
            tend = t0 + __ffs(stop) - 1;
            break;
          }
        }
      int tile = tb;
      for (; tile < tend; ++tile) {
        const double b = __ldg(bbase + tile * 8);  // x^{1+q} of configuration lane / 4 (row q = lane & 3)
        double acc[NPOLY][2];
#pragma unroll
        for (int k = 0; k < NPOLY; ++k) {
          dmma_c(acc[k][0], acc[k][1], w1[k], b, a0[k], a0[k]);  // w_{k,0} + sum_i x^i w_{k,i}
        }
        epi_oct(grec + tile * 8, acc, true, fcon, Dv);
      }
    }
    // dense tiles; a3 early exit: they are sorted by P1 P2, so every tile from the first one whose
    // smallest P1 P2 exceeds the largest D1^2 of the warp's tuples fails the D rule
#ifdef RP_SWEEP_PROBE_NODENSE  // timing probe: factored tiles only
    const int nOctF = 0;
#else
    const int nOctF = ntile - ngt;
#endif
    const CfgRec *drec = grec + ngt * 8;
    int nEff = nOctF;
    if (sorted)
      for (int b0 = 0; b0 < nOctF; b0 += 32) {
        const int oc = b0 + lane;
        const unsigned stop = __ballot_sync(0xffffffffu, oc < nOctF && __ldg(&drec[oc * 8].P01) > maxD1sq);
        if (stop) {
          nEff = b0 + __ffs(stop) - 1;
          break;
        }
      }
    // two configuration octets per iteration: 4 independent pairs per lane in the epilogue
    int oc = ngt;
    nEff += ngt;
    for (; oc + 1 < nEff; oc += 2) {
      double acc[NPOLY][2], acc2[NPOLY][2], bfr[KS], bfr2[KS];
      load_b(oc, bfr);
      load_b(oc + 1, bfr2);
      mma_oct(acc, bfr);
      mma_oct(acc2, bfr2);
      epi_oct(grec + oc * 8, acc, false, 1ull, 1);
      epi_oct(grec + (oc + 1) * 8, acc2, false, 1ull, 1);
    }
    if (oc < nEff) {
      double acc[NPOLY][2], bfr[KS];
      load_b(oc, bfr);
      mma_oct(acc, bfr);
      epi_oct(grec + oc * 8, acc, false, 1ull, 1);
    }
  }
  // ---- a8: the 4 lanes of a quad hold the same tuple ------------------------------------------
  if constexpr (FAST && !SECOND) {
    if (pkey < (0x7FEFFFFFFFFFFFFFull & ~0x1FFFull)) {  // a positive finite E won
      st.e = __longlong_as_double((long long)((pkey & ~0x1FFFull) + 1ull));
      st.i = (int32_t)(pkey & 0x1FFFull);
    }
  }
  st = merge(st, shfl_xor(st, 1));
  st = merge(st, shfl_xor(st, 2));
  if ((lane & 3) == 0 && t < tmax) {  // every tuple of the tile is written (-1 / +inf if none)
    const int64_t o = (int64_t)g * a.nD + (a.perm ? (int64_t)a.perm[d0 + t] : d0 + t);
    a.idx[o] = (st.e < kInf) ? st.i : -1;
    a.bestE[o] = st.e;
    if (SECOND) {
      a.secondE[o] = st.s;
      if (a.idx2) a.idx2[o] = st.s < kInf ? st.j : -1;
    }
  }
}

// ============================================================================================
// Tensor-core screened sweep (RP_SWEEP_KERNEL=tc; MWP-CWP programs with nPE <= 16, no runner-up).
//
// The contraction p_k(D, P) = sum_pe C_{k,pe}(D) m_pe(P) runs on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM) as a 3-term split product
//   C m ~ C_hi m_hi + C_hi m_lo + C_lo m_hi      (x_hi = tf32(x), x_lo = tf32(x - x_hi)),
// asynchronously to the warps that screen E in FP32 (mwpcwp_E32 with a per-pair bound), so the
// FP64 datapath carries only the exact re-evaluation of the few candidates.  One CTA = 128 data
// tuples (the MMA M side, one TMEM lane each) x all configurations in tiles of 32 (N):
//   warp 16:     builds the B operands of tile i (m splits, K-major no-swizzle layout) into ring
//                slot i % 2, issues 36 MMAs (6 polynomials x 2 K-steps x 3 split terms) into TMEM
//                buffer i % 2, commits to full[i % 2];
//   warps 0-15:  warpgroups 2b, 2b+1 screen the tiles of buffer b (16 configurations each), keep
//                per thread the kKC smallest lower bounds E32 (1 - eta), then re-evaluate them
//                exactly in FP64; a tuple whose dropped lower bounds could reach its winner is
//                re-swept in FP64 by one warp (rare).
// Error model: |p32 - p| <= 64 u S, S = sum |C m| <=
// ||C_k||_2 ||m||_2 (Cauchy-Schwarz; u = 2^-24; measured <= 9.8 u S, tools/microbench/umma_tf32.cu),
// so with rho = max_k ||C_k|| ||m|| / |p32_k| <= 64 each input carries eps = 64 u rho relative error;
// E is a product / quotient / positive-sum expression in which each input enters at most 18 times
// (6 for every compared quantity), hence |E32 - E| <= 1.1 (18 eps + 80 u) E + 1e-6 E.
// ============================================================================================
constexpr int kTcM = 128;           // tuples per CTA (TMEM lanes)
constexpr int kTcN = 32;            // configurations per MMA tile (8 per screening warpgroup)
constexpr int kTcNB = 2;            // TMEM buffers = B operand ring slots
constexpr int kTcNR = 4;            // ring slots of the tile's records and ||m||
constexpr int kTcColStride = 256;   // TMEM columns per buffer (6 kTcN used)
constexpr int kTcNPE = 16;          // MMA K (program-part monomials, padded)
#ifndef RP_TC_KC
#define RP_TC_KC 4
#endif
constexpr int kTcKC = RP_TC_KC;     // kept candidates per screening thread
#ifndef RP_TC_EPI
#define RP_TC_EPI 512
#endif
constexpr int kTcEpi = RP_TC_EPI;   // screening threads (512: 4 warpgroups at 96 registers; 256: 2 at 168)
constexpr int kTcWG = kTcEpi / 128;             // screening warpgroups
constexpr int kTcCfgWG = kTcN / kTcWG;          // configurations of a tile per warpgroup
constexpr int kTcProd = kTcEpi / 32;            // the producer warp's index
constexpr int kTcThreads = kTcEpi + 32;
constexpr uint32_t kTcLBO = 128, kTcSBO = 512;        // K-major no-swizzle core-matrix strides
constexpr uint32_t kTcAbytes = kTcM / 8 * kTcSBO;     // one [128 x 16] tf32 operand: 8 KB
constexpr uint32_t kTcBbytes = kTcN / 8 * kTcSBO;     // one [32 x 16] tf32 operand: 2 KB
constexpr int kTcMaxNdp = 32;
// shared-memory map (bytes)
constexpr uint32_t kTcOffA = 0;                                   // [2 splits][6 polys] A operands; later FP64 C [128][96]
constexpr uint32_t kTcOffB = kTcOffA + 12 * kTcAbytes;            // [2 slots][2 splits] B operands
constexpr uint32_t kTcOffMn = kTcOffB + 2 * kTcNB * kTcBbytes;    // [slots][kTcN] ||m(P)||
constexpr uint32_t kTcOffMD = kTcOffMn + kTcNR * kTcN * 4;           // [128][ndp <= 32] data monomials (FP64)
constexpr uint32_t kTcOffRSM = kTcOffMD + kTcM * kTcMaxNdp * 8;   // [kRSMTab] 1/SM_act (FP32)
constexpr uint32_t kTcOffDv = kTcOffRSM + kRSMTab * 4;            // [128][kMaxVars] D values
constexpr uint32_t kTcOffCn = kTcOffDv + kTcM * kMaxVars * 4;     // [128][6] ||C_k(D)||
constexpr uint32_t kTcOffPart = kTcOffCn + kTcM * 6 * 4;          // [4][128] {e, i, tnl, ovf}
constexpr uint32_t kTcOffFb = kTcOffPart + 4 * kTcM * 24;         // [128] fallback tuples + count
constexpr uint32_t kTcOffBar = (kTcOffFb + (kTcM + 2) * 4 + 7) & ~7u;  // full[2], empty[2], tmem base, maxD1sq
constexpr uint32_t kTcOffRec = (kTcOffBar + 128 + 15) & ~15u;                // [slots][kTcN] CfgRec of the tile
constexpr uint32_t kTcSmem = kTcOffRec + kTcNR * kTcN * 64;
// per-tile pack built once per launch by k_tc_pack (the tile's B operands in their shared-memory
// layout, ||m(P)|| and records), moved by three bulk copies per tile
constexpr uint32_t kTcPackB = 2 * kTcBbytes, kTcPackMn = kTcN * 4, kTcPackRec = kTcN * 64;
constexpr uint32_t kTcPack = kTcPackB + kTcPackMn + kTcPackRec;  // 6272 B
static_assert(kTcOffB % 1024 == 0 && kTcSmem <= 227 * 1024, "tc sweep shared memory");
static_assert(12 * kTcAbytes >= kTcM * 96 * 8, "FP64 C fits the A operands' space");
// the per-SM scratch slot of g_tc_C has one owner at a time only if two CTAs cannot share an SM
static_assert(2 * kTcSmem > 228 * 1024, "k_sweep_tc must hold its SM alone");

__device__ unsigned long long g_tc_stats[2];
#ifdef RP_TC_TRACE  // timeline of CTA 0: [tile][0..3] = producer empty-wait done, copy landed, committed; screen start (warp 0)
__device__ long long g_tc_trace[64][6];
#endif  // [0] tuples re-swept in FP64, [1] tuples
// FP64 staged C of the CTA's tuples for the exact re-evaluation, one slot per SM (the kernel's
// shared memory admits one CTA per SM, so a slot has one owner at a time; 14.7 MB, L2-resident)
constexpr int kTcMaxSM = 160;
__device__ double g_tc_C[kTcMaxSM][kTcM * 96];

__global__ void __launch_bounds__(kTcThreads, 1) k_sweep_tc(SweepArgs a) {
  constexpr int NPOLY = 6, NPE = kTcNPE;
  constexpr double kInf = __builtin_huge_val();
  const int g = blockIdx.y;
  const DevProg &pg = a.progs[g];
  const int d = a.d;
  const int64_t d0 = (int64_t)blockIdx.x * kTcM;
  const int tmax = (int)((a.nD - d0) < kTcM ? (a.nD - d0) : kTcM);
  const int n_sm = pg.n_sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char *sA = sm + kTcOffA, *sB = sm + kTcOffB;
  float *sMn = reinterpret_cast<float *>(sm + kTcOffMn);
  double *sMD = reinterpret_cast<double *>(sm + kTcOffMD);
  float *sRSM32 = reinterpret_cast<float *>(sm + kTcOffRSM);
  int32_t *sDv = reinterpret_cast<int32_t *>(sm + kTcOffDv);
  float *sCn = reinterpret_cast<float *>(sm + kTcOffCn);
  unsigned char *sPart = sm + kTcOffPart;
  int32_t *sFb = reinterpret_cast<int32_t *>(sm + kTcOffFb);  // [0]: count, [1..]: tuples
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + kTcOffBar);  // full[kTcNB], empty[kTcNB]
  uint32_t *sTmem = reinterpret_cast<uint32_t *>(bars + 3 * kTcNB);  // (bars + 2 kTcNB: bulk-copy barriers)
  unsigned long long *sMaxD1 = reinterpret_cast<unsigned long long *>(bars + 3 * kTcNB + 1);
  int4 *sRec = reinterpret_cast<int4 *>(sm + kTcOffRec);  // [slots][kTcN][4]
  uint32_t smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  double *gCd = g_tc_C[smid % kTcMaxSM];  // FP64 C [128][96] of this CTA's tuples
  const double *gRSM = a.tab.rSM + (int64_t)g * kRSMTab;
  const int nDE = pg.nDE, ndp = a.tab.nde_pad;
  const double *Cm = a.tab.Cmat + (int64_t)g * kMaxPolys * NPE * ndp;

  if (tid == 0) {
    for (int i = 0; i < kTcNB; ++i) {
      mbar_init(smem_u32(bars + i), 1);                  // full: the MMA commit
      mbar_init(smem_u32(bars + kTcNB + i), kTcEpi / 32);  // empty: every screening warp copied it out
      mbar_init(smem_u32(bars + 2 * kTcNB + i), 1);        // the tile pack's bulk copies landed
    }
    sFb[0] = 0;
    *sMaxD1 = 0ull;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (wid == kTcProd) tmem_alloc(smem_u32(sTmem), 512);
  for (int i = tid; i < kTcM * d; i += kTcThreads) {
    const int t = i / d, k = i % d;
    const int64_t src = (t < tmax) ? (a.perm ? (int64_t)a.perm[d0 + t] : d0 + t) : 0;
    sDv[t * kMaxVars + k] = (t < tmax) ? a.D[src * d + k] : 1;
  }
  for (int i = tid; i <= n_sm; i += kTcThreads) sRSM32[i] = (float)gRSM[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // data monomials m_de(u_D) (FP64), and the largest D1^2 of the tile (a3 early exit)
  for (int i = tid; i < kTcM * ndp; i += kTcThreads) {
    const int t = i / ndp, de = i % ndp;
    double m = 0.0;
    if (de < nDE) {
      m = 1.0;
      for (int k = 0; k < d; ++k) {
        const double u = ((double)sDv[t * kMaxVars + k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
        for (int e = 0; e < pg.de_exp[de][k]; ++e) m *= u;
      }
    }
    sMD[t * ndp + de] = m;
  }
  if (tid < kTcM) {  // warps 0-3: a shuffle max, then one shared atomic per warp
    const long long D1 = tid < tmax ? sDv[tid * kMaxVars] : 0;
    unsigned long long m = (unsigned long long)(D1 * D1);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
      m = x > m ? x : m;
    }
    if (lane == 0) atomicMax(sMaxD1, m);
  }
  __syncthreads();
  // staged data polynomials C_{k,pe}(D) in FP64 (a2): the (96 x ndp) x (ndp x 128) product of the
  // plan's coefficient matrix and the tile's data monomials on DMMA.8x8x4 (8x8 output tiles spread
  // over the warps, as in k_sweep).  to_ops: stored as tf32 splits in the A operands, with
  // ||C_k(D)||_2^2 summed into sNrm (shared FP64 atomics: two addends onto 0, order-independent);
  // the FP64 rows also go to gCd[t][96] for the exact re-evaluation.
  double *sNrm = reinterpret_cast<double *>(sPart);  // [128][6][2] half sums, before the merge needs sPart
  auto stage_C = [&](bool to_ops, int nwarps) {
    constexpr int MT = NPOLY * NPE / 8, NT = kTcM / 8;
    for (int tile = wid; tile < MT * NT; tile += nwarps) {
      const int mt = tile / NT, nt = tile % NT;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < ndp / 4; ++ks) {
        const double av = __ldg(Cm + (int64_t)(mt * 8 + (lane >> 2)) * ndp + ks * 4 + (lane & 3));
        const double bv = sMD[(nt * 8 + (lane >> 2)) * ndp + ks * 4 + (lane & 3)];
        dmma(c0, c1, av, bv);
      }
      const int row = mt * 8 + (lane >> 2), t = nt * 8 + 2 * (lane & 3);
      const int k = row / NPE, pe = row % NPE;
      gCd[t * 96 + row] = c0;
      gCd[(t + 1) * 96 + row] = c1;
      if (to_ops) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double c = j ? c1 : c0;
          const float hi = to_tf32((float)c), lo = to_tf32((float)(c - (double)hi));
          const uint32_t o = umma_off(t + j, pe, kTcLBO, kTcSBO);
          *reinterpret_cast<float *>(sA + k * kTcAbytes + o) = hi;
          *reinterpret_cast<float *>(sA + (NPOLY + k) * kTcAbytes + o) = lo;
        }
        double q0 = c0 * c0, q1 = c1 * c1;
#pragma unroll
        for (int m = 4; m <= 16; m <<= 1) {
          q0 += __shfl_xor_sync(0xffffffffu, q0, m);
          q1 += __shfl_xor_sync(0xffffffffu, q1, m);
        }
        if (lane < 4) {  // each (tuple, polynomial, row-tile half) written by one lane: no atomics
          sNrm[(t * 6 + k) * 2 + (mt & 1)] = q0;
          sNrm[((t + 1) * 6 + k) * 2 + (mt & 1)] = q1;
        }
      }
    }
  };
  stage_C(true, kTcThreads / 32);
  __syncthreads();
  for (int i = tid; i < kTcM * 6; i += kTcThreads) sCn[i] = (float)(sqrt(sNrm[2 * i] + sNrm[2 * i + 1]) * (1.0 + 1e-6));
  fence_async_smem();
  __syncthreads();

  const int nFc = a.tab.nFc[2 * g];
  const bool sorted = a.tab.nFc[2 * g + 1] != 0;
  const int nFp = a.tab.nFp;
  const CfgRec *rec = a.tab.rec + (int64_t)g * nFp;
  const double *mP = a.tab.mP + (int64_t)g * a.npe_pad * nFp;
  const int nTiles = (nFc + kTcN - 1) / kTcN;
  int nEff = tmax > 0 ? nTiles : 0;
  if (sorted && nEff > 0) {  // configurations sorted by P1 P2: stop at the first tile past max D1^2
    const long long mx = (long long)*sMaxD1;
    for (int b0 = 0; b0 < nTiles; b0 += 32) {
      const int j = b0 + lane;
      const unsigned stop = __ballot_sync(0xffffffffu, j < nTiles && __ldg(&rec[j * kTcN].P01) > mx);
      if (stop) {
        nEff = b0 + __ffs(stop) - 1;
        break;
      }
    }
  }
  const uint32_t tm = *sTmem;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kTcNB);

  if (wid == kTcProd) {
    // ---- producer / MMA warp ------------------------------------------------------------------
    const uint32_t idesc = umma_idesc_tf32(kTcM, kTcN);
    const uint32_t bfull0 = smem_u32(bars + 2 * kTcNB);
    const unsigned char *pack = a.tcpack + (int64_t)g * a.tc_ntiles * kTcPack;
    for (int i = 0; i < nEff; ++i) {
      const int s = i % kTcNB, use = i / kTcNB, r = i % kTcNR;
      // TMEM buffer s and B slot s free (every warp copied tile i - 2 out); record slot r was last
      // read for tile i - 4, finished by every warp before its empty arrival for tile i - 2
      if (use > 0) mbar_wait(empty0 + 8 * s, (use - 1) & 1);
#ifdef RP_TC_TRACE
      if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][0] = clock64();
#endif
      if (lane == 0) {
        const unsigned char *src = pack + (int64_t)i * kTcPack;
        const uint32_t bar = bfull0 + 8 * s;
        mbar_expect_tx(bar, kTcPack);
        bulk_g2s(smem_u32(sB + 2 * s * kTcBbytes), src, kTcPackB, bar);
        bulk_g2s(smem_u32(sMn + r * kTcN), src + kTcPackB, kTcPackMn, bar);
        bulk_g2s(smem_u32(sRec + r * kTcN * 4), src + kTcPackB + kTcPackMn, kTcPackRec, bar);
        mbar_wait(bar, use & 1);
#ifdef RP_TC_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][1] = clock64();
#endif
        tc_fence_after();
        // (opaque base: keeps the loop-invariant A descriptors from being hoisted out of the tile
        // loop as live registers)
        uint32_t a_hi;
        asm volatile("mov.u32 %0, %1;" : "=r"(a_hi) : "r"(smem_u32(sA)));
        const uint32_t a_lo = a_hi + NPOLY * kTcAbytes;
        const uint32_t b_hi = smem_u32(sB + 2 * s * kTcBbytes), b_lo = b_hi + kTcBbytes;
#pragma unroll
        for (int k = 0; k < NPOLY; ++k) {
          const uint32_t dcol = tm + s * kTcColStride + k * kTcN;
#pragma unroll
          for (int kk = 0; kk < NPE / 8; ++kk) {
            const uint32_t ko = kk * 2 * kTcLBO;
            const uint32_t ah = a_hi + k * kTcAbytes + ko, al = a_lo + k * kTcAbytes + ko;
            umma_tf32(dcol, umma_sdesc(ah, kTcLBO, kTcSBO), umma_sdesc(b_hi + ko, kTcLBO, kTcSBO), idesc, kk > 0);
            umma_tf32(dcol, umma_sdesc(ah, kTcLBO, kTcSBO), umma_sdesc(b_lo + ko, kTcLBO, kTcSBO), idesc, 1);
            umma_tf32(dcol, umma_sdesc(al, kTcLBO, kTcSBO), umma_sdesc(b_hi + ko, kTcLBO, kTcSBO), idesc, 1);
          }
        }
        umma_commit(full0 + 8 * s);
#ifdef RP_TC_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][2] = clock64();
#endif
      }
      __syncwarp();
    }
  } else {
    // ---- screening warps ----------------------------------------------------------------------
    const int wg = wid >> 2;  // configurations 8 wg .. 8 wg + 7 of every tile
    const int t = (wid & 3) * 32 + lane;  // TMEM lane = tuple
    const bool tok = t < tmax;
    const int32_t *Dt = sDv + t * kMaxVars;
    bool dpos = true;  // reading R32: data parameters are sizes >= 1
    for (int k = 0; k < d; ++k) dpos = dpos && Dt[k] >= 1;
    // a tuple with some D_k < 1 has no candidate: its D1^2 is taken as 0 (no P1 P2 <= 0)
    const int64_t D1sq = dpos ? (int64_t)Dt[0] * Dt[0] : -1;
    const int map0 = pg.grid_map[0], map1 = pg.p >= 2 ? pg.grid_map[1] : -1, map2 = pg.p >= 3 ? pg.grid_map[2] : -1;
    const int32_t Da = map0 >= 0 && dpos ? Dt[map0] : 1, Db = map1 >= 0 && dpos ? Dt[map1] : 1,
                  Dc = map2 >= 0 && dpos ? Dt[map2] : 1;
    const EConst32 kc32 = to_econst32(make_econst(pg));
    const float rNSM32 = sRSM32[n_sm];
    float rcn[NPOLY];  // 1 / ||C_k(D)||: rho = ||m|| / min_k (|p_k| / ||C_k||), one reciprocal per pair
#pragma unroll
    for (int k = 0; k < NPOLY; ++k) rcn[k] = 1.0f / sCn[t * 6 + k];
    float ck[kTcKC];
    int cp[kTcKC];
#pragma unroll
    for (int i = 0; i < kTcKC; ++i) {
      ck[i] = __int_as_float(0x7f800000);
      cp[i] = 0x7fffffff;
    }
    float tnl = __int_as_float(0x7f800000);  // smallest lower bound not kept
    float ub = __int_as_float(0x7f800000);   // smallest upper bound E32 (1 + eta) of a trusted pair
    bool ovf = false;                        // an untrusted pair fell off the list
    const uint32_t tl = tm + ((uint32_t)((wid & 3) * 32) << 16);
    constexpr float u = 5.9604645e-8f;  // 2^-24
    for (int i = 0; i < nEff; ++i) {
      const int b = i % kTcNB, r = i % kTcNR;
#ifdef RP_TC_TRACE
      if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][3] = clock64();
      if (tid == 480 && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][5] = clock64();
#endif
      mbar_wait(full0 + 8 * b, (i / kTcNB) & 1);
#ifdef RP_TC_TRACE
      if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) g_tc_trace[i][4] = clock64();
#endif
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < kTcCfgWG / 4; ++h) {  // groups of 4 configurations: 24 live TMEM values
        const int col = wg * kTcCfgWG + 4 * h;
        float pv[NPOLY][4];
#pragma unroll
        for (int k = 0; k < NPOLY; ++k) tmem_ld4(tl + b * kTcColStride + k * kTcN + col, pv[k]);
        tmem_ld_wait();
        if (h == kTcCfgWG / 4 - 1) {  // the buffer is free for the MMAs of tile i + 2 once every warp holds its values
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(empty0 + 8 * b);
        }
#ifdef RP_TC_SKEL  // timing experiment: the pipeline without the screen
        {
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int k = 0; k < NPOLY; ++k) acc += pv[k][v];
          tnl = fminf(tnl, acc > 1e30f ? acc : __int_as_float(0x7f800000));
          continue;
        }
#endif
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int pos = i * kTcN + col + v;
          const int4 *cr = sRec + (r * kTcN + col + v) * 4;
          const int4 r0 = cr[0];
          const longlong2 h0 = make_longlong2(((long long)(uint32_t)r0.y << 32) | (uint32_t)r0.x,
                                              ((long long)(uint32_t)r0.w << 32) | (uint32_t)r0.z);
          const int4 h1 = cr[1];
          const int4 h2 = cr[2];
          const int4 r3 = cr[3];
          const int2 h3 = make_int2(r3.z, r3.w);  // W32, rB32
          const bool ok = tok && pos < nFc && h0.x <= D1sq;               // a3
          if (!ok) continue;  // masked: never a candidate (mostly warp-uniform: tuples sorted by D1)
          const uint32_t s012 = (uint32_t)h2.y;
          // a6 (as k_sweep): 32-bit factors, the 64-bit product only where needed
          const uint32_t f0 = map0 >= 0 ? ceil_div32(Da, (int32_t)(h0.y >> 32), (uint32_t)h1.z, s012 & 255) : 1u;
          const uint32_t f1 = map1 >= 0 ? ceil_div32(Db, h1.x, (uint32_t)h1.w, (s012 >> 8) & 255) : 1u;
          int64_t blocks = (int64_t)((uint64_t)f0 * f1);
          if (map2 >= 0) blocks *= ceil_div32(Dc, h1.y, (uint32_t)h2.x, (s012 >> 16) & 255);
          const int smact = (int)(blocks < n_sm ? blocks : n_sm);
          float rSMf = rNSM32;  // SM_act = n_SM for most pairs: the table read only otherwise
          if (smact < n_sm) rSMf = sRSM32[smact];
          const float Rep = (float)blocks * __int_as_float(h3.y) * rSMf;
          const float mn = sMn[r * kTcN + col + v];
          float qmin = fabsf(pv[0][v]) * rcn[0];
#pragma unroll
          for (int k = 1; k < NPOLY; ++k) qmin = fminf(qmin, fabsf(pv[k][v]) * rcn[k]);
          const float rho = mn * rcp32(qmin);  // = max_k ||C_k|| ||m|| / |p32_k| (to a few ulp)
          const float eps = 64.f * u * 1.001f * rho;
          const float tol = 2.2f * (6.f * eps + 25.f * u) + 1e-6f;
          bool unc;
          const float E32 = mwpcwp_E32(pv[0][v], pv[1][v], pv[2][v], pv[3][v], pv[4][v], pv[5][v],
                                       __int_as_float(h3.x), Rep, rSMf, (float)smact, kc32, unc, tol);
          const float eta = 1.1f * (18.f * eps + 80.f * u) + 1e-6f;
          unc = unc | !(rho <= 64.f);
          ub = unc ? ub : fminf(ub, E32 * (1.0f + eta));
          float key = unc ? -1.0f : E32 * (1.0f - eta);
          int q = pos;
          if (key < ck[kTcKC - 1]) {  // (mostly warp-uniform false once the list holds small keys)
#pragma unroll
            for (int j = 0; j < kTcKC; ++j) {  // positions grow along the stream: ties keep the earlier
              const bool lt = key < ck[j];
              const float tk = ck[j];
              const int tq = cp[j];
              ck[j] = lt ? key : tk;
              cp[j] = lt ? q : tq;
              key = lt ? tk : key;
              q = lt ? tq : q;
            }
          }
          ovf = ovf | (key < 0.f);
          tnl = fminf(tnl, key);
        }
      }
    }
    // ---- exact re-evaluation of the kept candidates --------------------------------------------
    *reinterpret_cast<float *>(sPart + (wg * kTcM + t) * 24 + 20) = ub;
    asm volatile("bar.sync 1, %0;" ::"r"(kTcEpi) : "memory");  // every MMA consumed: A space free
    asm volatile("bar.sync 1, %0;" ::"r"(kTcEpi) : "memory");
    // only candidates whose lower bound reaches the tuple's smallest upper bound can win
    float ubt = ub;
#pragma unroll
    for (int w2 = 0; w2 < kTcWG; ++w2) ubt = fminf(ubt, *reinterpret_cast<const float *>(sPart + (w2 * kTcM + t) * 24 + 20));
    const EConst kc = make_econst(pg);
    auto pair_E64 = [&](int tt, int pos, const double *pk, int32_t &orig) -> double {
      const int32_t *Dq = sDv + tt * kMaxVars;
      bool dq = true;  // reading R32
      for (int k = 0; k < d; ++k) dq = dq && Dq[k] >= 1;
      const int64_t D1q = dq ? (int64_t)Dq[0] * Dq[0] : -1;
      const int32_t qa = map0 >= 0 && dq ? Dq[map0] : 1, qb = map1 >= 0 && dq ? Dq[map1] : 1,
                    qc = map2 >= 0 && dq ? Dq[map2] : 1;
      const CfgRec *cr = rec + pos;
      const longlong2 h0 = __ldg(reinterpret_cast<const longlong2 *>(cr));
      const int4 h1 = __ldg(reinterpret_cast<const int4 *>(cr) + 1);
      const int4 h2 = __ldg(reinterpret_cast<const int4 *>(cr) + 2);
      const double2 h3 = __ldg(reinterpret_cast<const double2 *>(cr) + 3);
      orig = (int32_t)(h0.y & 0xffffffff);
      const bool ok = tt < tmax && pos < nFc && h0.x <= D1q;  // a3
      const uint32_t s012 = (uint32_t)h2.y;
      const int64_t blocks = ceil_div_magic(qa, (int32_t)(h0.y >> 32), (uint32_t)h1.z, s012 & 255) *
                             ceil_div_magic(qb, h1.x, (uint32_t)h1.w, (s012 >> 8) & 255) *
                             ceil_div_magic(qc, h1.y, (uint32_t)h2.x, (s012 >> 16) & 255);
      const int64_t smact = blocks < n_sm ? blocks : n_sm;
      const double rSM = __ldg(gRSM + smact);
      const double Rep = (double)blocks * h3.x * rSM;  // line 15
      const double E = mwpcwp_E(pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], __hiloint2double(h2.w, h2.z), Rep, rSM,
                                (double)smact, kc);
      return (ok && pos_finite(E)) ? E : kInf;  // line 19, R17
    };
    auto exact_pk = [&](int tt, int pos, double (&pk)[NPOLY]) {
      double mvv[NPE];
#pragma unroll
      for (int pe = 0; pe < NPE; ++pe) mvv[pe] = __ldg(mP + (int64_t)pe * nFp + pos);
      const double *crow = gCd + tt * 96;
#pragma unroll
      for (int k = 0; k < NPOLY; ++k) {
        double sacc = 0.0;
#pragma unroll
        for (int pe = 0; pe < NPE; ++pe) sacc = fma(crow[k * NPE + pe], mvv[pe], sacc);
        pk[k] = sacc;
      }
    };
    auto take = [](Best &bb, double E, int32_t orig) {  // a8: exact key (E, original index)
      const long long eb = __double_as_longlong(E), sb = __double_as_longlong(bb.e);
      const bool better = eb < sb || (eb == sb && orig < bb.i);
      bb.i = better ? orig : bb.i;
      bb.e = better ? E : bb.e;
    };
    Best st;
    st.e = kInf;
    st.i = 0x7fffffff;
    st.s = kInf;
    st.j = 0x7fffffff;
#pragma unroll 1
    for (int j = 0; j < kTcKC; ++j) {
      if (cp[j] != 0x7fffffff && !(ck[j] > ubt)) {
        double pk[NPOLY];
        exact_pk(t, cp[j], pk);
        int32_t orig;
        const double E = pair_E64(t, cp[j], pk, orig);
        take(st, E, orig);
      }
    }
    unsigned char *pp = sPart + (wg * kTcM + t) * 24;
    *reinterpret_cast<double *>(pp) = st.e;
    *reinterpret_cast<int32_t *>(pp + 8) = st.i;
    *reinterpret_cast<float *>(pp + 12) = tnl;
    *reinterpret_cast<int32_t *>(pp + 16) = ovf ? 1 : 0;
    asm volatile("bar.sync 1, %0;" ::"r"(kTcEpi) : "memory");
    if (wg == 0 && tok) {
      for (int w2 = 1; w2 < kTcWG; ++w2) {
        const unsigned char *qq = sPart + (w2 * kTcM + t) * 24;
        take(st, *reinterpret_cast<const double *>(qq), *reinterpret_cast<const int32_t *>(qq + 8));
        tnl = fminf(tnl, *reinterpret_cast<const float *>(qq + 12));
        ovf = ovf || *reinterpret_cast<const int32_t *>(qq + 16) != 0;
      }
      // exact unless a dropped pair's lower bound reaches the winner (E > lower bound > winner)
      const bool fb = ovf || (tnl < __int_as_float(0x7f800000) && !((double)tnl > st.e));
      if (fb) {
        sFb[1 + atomicAdd(&sFb[0], 1)] = t;
      } else {
        const int64_t o = (int64_t)g * a.nD + (a.perm ? (int64_t)a.perm[d0 + t] : d0 + t);
        a.idx[o] = (st.e < kInf) ? st.i : -1;
        a.bestE[o] = st.e;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kTcEpi) : "memory");
    // ---- rare: a flagged tuple re-swept exactly in FP64 by one warp (lanes over configurations)
    const int nfb = sFb[0];
    if (tid == 0 && nfb > 0) atomicAdd(&g_tc_stats[0], (unsigned long long)nfb);
    if (tid == 0) atomicAdd(&g_tc_stats[1], (unsigned long long)tmax);
    for (int f = wid; f < nfb; f += kTcEpi / 32) {
      const int tt = sFb[1 + f];
      Best sf;
      sf.e = kInf;
      sf.i = 0x7fffffff;
      sf.s = kInf;
      sf.j = 0x7fffffff;
      for (int pos = lane; pos < nEff * kTcN && pos < nFc; pos += 32) {
        double pk[NPOLY];
        exact_pk(tt, pos, pk);
        int32_t orig;
        const double E = pair_E64(tt, pos, pk, orig);
        take(sf, E, orig);
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) sf = merge(sf, shfl_xor(sf, m));
      if (lane == 0) {
        const int64_t o = (int64_t)g * a.nD + (a.perm ? (int64_t)a.perm[d0 + tt] : d0 + tt);
        a.idx[o] = (sf.e < kInf) ? sf.i : -1;
        a.bestE[o] = sf.e;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == kTcProd) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

// one warp per (configuration tile, program): the tile's B operands (tf32 splits of m(P) in the
// K-major no-swizzle layout), ||m(P)||_2 and its records, as k_sweep_tc's producer copies them
__global__ void k_tc_pack(SweepArgs a, unsigned char *pack) {
  const int g = blockIdx.y, j = blockIdx.x, lane = threadIdx.x;
  const int nFp = a.tab.nFp;
  const CfgRec *rec = a.tab.rec + (int64_t)g * nFp;
  const double *mP = a.tab.mP + (int64_t)g * a.npe_pad * nFp;
  unsigned char *dst = pack + ((int64_t)g * a.tc_ntiles + j) * kTcPack;
  const int pos = j * kTcN + lane;
  double mn2 = 0.0;
  for (int pe = 0; pe < kTcNPE; ++pe) {
    const double m = pos < nFp ? mP[(int64_t)pe * nFp + pos] : 0.0;
    const float hi = to_tf32((float)m), lo = to_tf32((float)(m - (double)hi));
    const uint32_t o = umma_off(lane, pe, kTcLBO, kTcSBO);
    *reinterpret_cast<float *>(dst + o) = hi;
    *reinterpret_cast<float *>(dst + kTcBbytes + o) = lo;
    mn2 = fma(m, m, mn2);
  }
  reinterpret_cast<float *>(dst + kTcPackB)[lane] = (float)(sqrt(mn2) * (1.0 + 1e-6));
  const int4 *src = reinterpret_cast<const int4 *>(rec + (pos < nFp ? pos : nFp - 1));
  int4 *rd = reinterpret_cast<int4 *>(dst + kTcPackB + kTcPackMn) + lane * 4;
  for (int q = 0; q < 4; ++q) rd[q] = src[q];
}

static cudaError_t launch_tc(SweepArgs a, int n_prog, cudaStream_t s) {
  const int64_t tiles = (a.nD + kTcM - 1) / kTcM;
  if (tiles > 0x7fffffffll || n_prog > 65535) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_sweep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
  if (e != cudaSuccess) return e;
  a.tc_ntiles = (a.tab.nFp + kTcN - 1) / kTcN;
  unsigned char *pack = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void **>(&pack), (size_t)n_prog * a.tc_ntiles * kTcPack, s);
  if (e != cudaSuccess) return e;
  k_tc_pack<<<dim3((unsigned)a.tc_ntiles, (unsigned)n_prog), 32, 0, s>>>(a, pack);
  a.tcpack = pack;
  k_sweep_tc<<<dim3((unsigned)tiles, (unsigned)n_prog), kTcThreads, kTcSmem, s>>>(a);
  e = cudaGetLastError();
  cudaFreeAsync(pack, s);
  if (e == cudaSuccess && getenv("RP_SWEEP_TC_STATS")) {
    unsigned long long st[2];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(st, g_tc_stats, sizeof(st));
    fprintf(stderr, "[k_sweep_tc] tuples re-swept in FP64: %llu of %llu\n", st[0], st[1]);
    const unsigned long long z[2] = {0ull, 0ull};
    cudaMemcpyToSymbol(g_tc_stats, z, sizeof(z));
  }
#ifdef RP_TC_TRACE
  {
    long long tr[64][6];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(tr, g_tc_trace, sizeof(tr));
    for (int i = 0; i < 40; ++i)
      fprintf(stderr, "tile %2d: empty_ok %8lld copy %8lld commit %8lld | w0 start %8lld full_ok %8lld | w15 start %8lld\n", i,
              tr[i][0] - tr[0][0], tr[i][1] - tr[0][0], tr[i][2] - tr[0][0], tr[i][3] - tr[0][0], tr[i][4] - tr[0][0],
              tr[i][5] - tr[0][0]);
  }
#endif
  return e;
}

template <int NPE, bool MWP, bool SECOND, bool FAST>
static cudaError_t launch4(const SweepArgs &a, int n_prog, int n_sm_max, cudaStream_t s) {
  const size_t smem = sweep_smem_bytes<MWP ? 6 : 2, NPE>(a.nde_stride, n_sm_max);
  const int64_t tiles = (a.nD + kTD - 1) / kTD;
  if (tiles > 0x7fffffffll || n_prog > 65535) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_sweep<NPE, MWP, SECOND, FAST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_sweep<NPE, MWP, SECOND, FAST><<<dim3((unsigned)tiles, (unsigned)n_prog), kSweepThreads, smem, s>>>(a);
  return cudaGetLastError();
}
static bool refine_enabled();
template <int NPE, bool MWP, bool SECOND>
static cudaError_t launch3(const SweepArgs &a, int n_prog, int n_sm_max, cudaStream_t s) {
  if constexpr (MWP) {  // (FAST packs the original index into 13 bits of its ranking key)
    if (refine_enabled() && a.tab.nFp <= 8192) return launch4<NPE, MWP, SECOND, true>(a, n_prog, n_sm_max, s);
  }
  return launch4<NPE, MWP, SECOND, false>(a, n_prog, n_sm_max, s);
}

template <int NPE>
static cudaError_t launch_npe(const SweepArgs &a, int n_prog, bool mwp, int n_sm_max, cudaStream_t s) {
  const bool second = a.secondE != nullptr;
  // RP_SWEEP_KERNEL=tc: the tensor-core screened sweep (MWP-CWP programs with nPE <= 16 and no
  // runner-up); default: k_sweep
  const char *kern = getenv("RP_SWEEP_KERNEL");
  if (NPE == kTcNPE && mwp && !second && kern && strcmp(kern, "tc") == 0 && a.tab.nde_pad <= kTcMaxNdp &&
      num_sms() <= kTcMaxSM)
    return launch_tc(a, n_prog, s);
  if (mwp)
    return second ? launch3<NPE, true, true>(a, n_prog, n_sm_max, s)
                  : launch3<NPE, true, false>(a, n_prog, n_sm_max, s);
  return second ? launch3<NPE, false, true>(a, n_prog, n_sm_max, s)
                : launch3<NPE, false, false>(a, n_prog, n_sm_max, s);
}

// ============================================================================================
// Winner refinement (default on; RP_SWEEP_REFINE=0 disables it).  A program fitted to noisy
// samples has polynomials whose terms cancel (kappa = sum |c m| / |p| up to ~1e7 on the bench's
// program, reading R31), so the FP64 sweep's E can be ~1e-9 off the exact value of
// the chosen pair.  k_refine re-evaluates, per tuple, the sweep's winner (and with a runner-up
// output also the runner-up, re-ranking the two) with every p_k accurate to ~u + n^2 u^2 kappa:
//   * monomials m = m_de(u_D) m_pe(u_P) in double-double (error-free products by FMA);
//   * each p_k = sum c m accumulated by error-free extraction against a power of two
//     sigma_k >= 4 sum |c m| (a bound from the plan: A_k = sum |c|, times max(1, |u|)^maxdeg):
//     x = fma(c, m_hi, sigma) rounds c m_hi to a multiple of ulp(sigma)/2, t = x - sigma is exact
//     (Sterbenz), the t are summed exactly in hi (multiples of ulp(sigma)/2 below sigma), and
//     the remainders fma(c, m_hi, -t) (one rounding of a value below ulp(sigma)) and c m_lo
//     go to lo -- 6 FP64 operations per term and polynomial instead of the ~11 of a TwoSum
//     chain;
//   * then a6 and Appendix A exactly as the sweep evaluates them.
// The plan keeps the union of the polynomials' (de, pe) terms with one coefficient per
// polynomial (zero where a polynomial lacks the term), so the monomial product is shared by the
// 2l polynomials.  One thread per tuple; the tuple's data monomials and the chosen configurations'
// program monomials sit in shared memory (thread-private columns, no barrier).
// ============================================================================================
constexpr int kRefThreads = 128;

// the union term list of program g's polynomials (rterm, rcoef) and its bounds (rinfo), from the
// staging matrix Cmat; called by every thread of a plan kernel after Cmat is written
__device__ void build_refine_terms(int g, const DevProg &pg, const CfgTable &tab, int npe_pad) {
  __shared__ int rt_warp[32];
  __shared__ int rt_base;
  const int ndp = tab.nde_pad, ncell = npe_pad * ndp;
  const double *Cm = tab.Cmat + (int64_t)g * kMaxPolys * npe_pad * ndp;
  double *rc = tab.rcoef + (int64_t)g * ncell * kMaxPolys;
  int32_t *rt = tab.rterm + (int64_t)g * ncell;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) rt_base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < ncell; c0 += blockDim.x) {
    const int cell = c0 + threadIdx.x, pe = cell / ndp, de = cell % ndp;
    bool nz = false;
    if (cell < ncell && pe < pg.nPE && de < pg.nDE)
      for (int k = 0; k < pg.npoly; ++k) nz = nz || Cm[(int64_t)(k * npe_pad + pe) * ndp + de] != 0.0;
    const unsigned ball = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) rt_warp[wid] = __popc(ball);
    __syncthreads();
    if (wid == 0) {
      const int v = lane < (int)(blockDim.x >> 5) ? rt_warp[lane] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      rt_warp[lane] = incl - v;
    }
    __syncthreads();
    const int pos = rt_base + rt_warp[wid] + __popc(ball & ((1u << lane) - 1u));
    if (nz) {
      rt[pos] = de | (pe << 16);
      for (int k = 0; k < kMaxPolys; ++k)
        rc[(int64_t)pos * kMaxPolys + k] = k < pg.npoly ? Cm[(int64_t)(k * npe_pad + pe) * ndp + de] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) rt_base = pos + nz;
    __syncthreads();
  }
  const int nrt = rt_base;
  double *ri = tab.rinfo + (int64_t)g * 8;
  // A_k = sum |c| over the terms of polynomial k (warp k: lane-strided partial sums, then a fixed
  // butterfly: deterministic); warp kMaxPolys: the largest total degree and the term count
  if (wid < kMaxPolys) {
    double A = 0.0;
    for (int j = lane; j < nrt; j += 32) A += fabs(rc[(int64_t)j * kMaxPolys + wid]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) A += __shfl_xor_sync(0xffffffffu, A, o);
    if (lane == 0) ri[wid] = A;
  } else if (wid == kMaxPolys) {
    int md = 0;
    for (int j = lane; j < nrt; j += 32) {
      const int de = rt[j] & 0xffff, pe = rt[j] >> 16;
      int dg = 0;
      for (int k = 0; k < pg.d; ++k) dg += pg.de_exp[de][k];
      for (int k = 0; k < pg.p; ++k) dg += pg.pe_exp[pe][k];
      md = dg > md ? dg : md;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const int x = __shfl_xor_sync(0xffffffffu, md, o);
      md = x > md ? x : md;
    }
    if (lane == 0) {
      ri[6] = (double)md;
      ri[7] = (double)nrt;
    }
  }
}

// the smallest power of two > 4 B (B >= 0 finite); 1 for B = 0; 0 if it would overflow
__device__ __forceinline__ double extract_sigma(double B) {
  if (!(B > 0.0)) return B == 0.0 ? 1.0 : 0.0;
  const long long ex = ((__double_as_longlong(B) >> 52) & 0x7ff) - 1023;  // B in [2^ex, 2^(ex+1))
  if (ex + 3 > 1023) return 0.0;
  return __longlong_as_double((ex + 3 + 1023) << 52);
}

// a6 + Appendix A for one pair from its polynomial values (as k_sweep evaluates them)
// ---- double-double arithmetic for the refined E (the literal order of Appendix A) ----------------
// When the metrics have mixed signs (a fitted g_i < 0 somewhere) the sums of Appendix A cancel and
// an FP64 evaluation of E from exact inputs can be off by 1e4 ulp; in double-double (~2^-104) the
// estimate of the refined pair is accurate to the rounding of its final value.
struct ddv {
  double h, l;
};
__device__ __forceinline__ ddv dd_qts(double a, double b) {  // |a| >= |b|
  const double s = a + b;
  return ddv{s, b - (s - a)};
}
__device__ __forceinline__ ddv dd_ts(double a, double b) {
  const double s = a + b, bb = s - a;
  return ddv{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ ddv dd_add(ddv x, ddv y) {
  ddv s = dd_ts(x.h, y.h), t = dd_ts(x.l, y.l);
  s.l += t.h;
  s = dd_qts(s.h, s.l);
  s.l += t.l;
  return dd_qts(s.h, s.l);
}
__device__ __forceinline__ ddv dd_neg(ddv x) { return ddv{-x.h, -x.l}; }
__device__ __forceinline__ ddv dd_sub(ddv x, ddv y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ ddv dd_mul(ddv x, ddv y) {
  const double p = x.h * y.h;
  double e = fma(x.h, y.h, -p);
  e = fma(x.h, y.l, fma(x.l, y.h, e));
  return dd_qts(p, e);
}
__device__ __forceinline__ ddv dd_muld(ddv x, double b) {
  const double p = x.h * b;
  return dd_qts(p, fma(x.l, b, fma(x.h, b, -p)));
}
// x / y: three quotient digits from one ~1-ulp reciprocal of y.h; each remainder step removes
// the previous digit's error (QD's accurate division with the IEEE divisions replaced)
__device__ __forceinline__ ddv dd_div(ddv x, ddv y) {
  const double ry = frcp(y.h);
  const double q1 = x.h * ry;
  ddv r = dd_sub(x, dd_muld(y, q1));
  const double q2 = r.h * ry;
  r = dd_sub(r, dd_muld(y, q2));
  const double q3 = r.h * ry;
  return dd_add(dd_qts(q1, q2), ddv{q3, 0.0});
}
__device__ __forceinline__ bool dd_lt(ddv x, ddv y) { return x.h < y.h || (x.h == y.h && x.l < y.l); }
__device__ __forceinline__ bool dd_eq(ddv x, ddv y) { return x.h == y.h && x.l == y.l; }
__device__ __forceinline__ ddv dd_min(ddv x, ddv y) { return dd_lt(y, x) ? y : x; }
__device__ __forceinline__ ddv dd_d(double a) { return ddv{a, 0.0}; }

// Appendix A lines 5-18 in double-double, in the oracle's literal order (DESIGN.md Appendix A)
__device__ double mwpcwp_E_dd(const ddv *pk, double W, int64_t blocks, double B, int64_t smact,
                              const DevProg &pg) {
  const ddv g1 = dd_div(pk[0], pk[1]), g2 = dd_div(pk[2], pk[3]), g3 = dd_div(pk[4], pk[5]);
  const ddv Wact = dd_d(W), SMact = dd_d((double)smact);
  const ddv Mem = dd_add(g2, g3), Tot = dd_add(dd_add(g1, g2), g3);             // 5
  const ddv W_unc = dd_div(g3, Mem), W_coal = dd_div(g2, Mem);                   // 6
  const ddv L_unc = dd_add(dd_d(pg.mem_ld), dd_muld(dd_d(pg.U - 1.0), pg.dd_unc));  // 7
  const ddv L_coal = dd_d(pg.mem_ld);
  const ddv Mem_L = dd_add(dd_mul(L_unc, W_unc), dd_mul(L_coal, W_coal));        // 8
  const ddv Dep = dd_add(dd_mul(dd_muld(dd_d(pg.dd_unc), pg.U), W_unc), dd_muld(W_coal, pg.dd_coal));  // 9
  const ddv MWP_nb = dd_div(Mem_L, Dep);                                         // 10
  const ddv BWpw = dd_div(dd_muld(dd_d(pg.freq), pg.lbpw), Mem_L);               // 11
  const ddv MWP_bw = dd_div(dd_d(pg.mem_bw), dd_mul(BWpw, SMact));
  ddv MWP = MWP_nb;                                                              // 12
  if (dd_lt(MWP_bw, MWP)) MWP = MWP_bw;
  if (dd_lt(Wact, MWP)) MWP = Wact;
  const ddv Comp_c = dd_muld(Tot, pg.issue);                                     // 13
  const ddv Mem_c = dd_add(dd_mul(L_unc, g3), dd_mul(L_coal, g2));
  const ddv CWP_full = dd_div(dd_add(Mem_c, Comp_c), Comp_c);                    // 14
  const ddv CWP = dd_lt(CWP_full, Wact) ? CWP_full : Wact;
  const ddv Rep = dd_div(dd_d((double)blocks), dd_muld(SMact, B));               // 15
  const ddv tail = dd_mul(dd_div(Comp_c, Mem), dd_sub(MWP, dd_d(1.0)));
  ddv E;
  if (dd_eq(MWP, Wact) && dd_eq(CWP, Wact))                                      // 16
    E = dd_mul(dd_add(dd_add(Mem_c, Comp_c), tail), Rep);
  else if (!dd_lt(CWP, MWP) || dd_lt(Mem_c, Comp_c))                             // 17
    E = dd_mul(dd_add(dd_div(dd_mul(Mem_c, Wact), MWP), tail), Rep);
  else                                                                           // 18
    E = dd_mul(dd_add(Mem_L, dd_mul(Comp_c, Wact)), Rep);
  return E.h + E.l;
}

// the same E in double-double in the sweep's common-denominator arrangement (g_i = a_i / Q;
// rp_device.cuh mwpcwp_E): 4 divisions instead of the literal order's 12, identical to it up to
// double-double rounding; the case tests compare the same quantities as Appendix A
__device__ double mwpcwp_E_dd2(const ddv *pk, double W, int64_t blocks, double B, int64_t smact,
                               const DevProg &pg) {
  const EConst k = make_econst(pg);
  const ddv q23 = dd_mul(pk[3], pk[5]), q13 = dd_mul(pk[1], pk[5]), q12 = dd_mul(pk[1], pk[3]);
  const ddv Q = dd_mul(pk[1], q23);
  const ddv a1 = dd_mul(pk[0], q23), a2 = dd_mul(pk[2], q13), a3 = dd_mul(pk[4], q12);
  const ddv s23 = dd_add(a2, a3), s = dd_add(a1, s23);                           // Mem Q, Tot Q
  const ddv mc = dd_add(dd_muld(a3, k.Lunc), dd_muld(a2, k.Lcoal));              // Mem_c Q
  const ddv dn = dd_add(dd_muld(a3, k.DdU), dd_muld(a2, k.ddc));                 // Dep Mem Q
  const ddv cc = dd_muld(s, k.issue);                                            // Comp_c Q
  const ddv SM = dd_d((double)smact), Wd = dd_d(W), one = dd_d(1.0);
  const ddv Mem_c = dd_div(mc, Q), Comp_c = dd_div(cc, Q);
  const ddv MWP_nb = dd_div(mc, dn);                                             // 10
  const ddv MWP_bw = dd_div(dd_muld(mc, k.Kbw), dd_mul(s23, SM));               // 11
  const ddv CWPf = dd_add(one, dd_div(mc, cc));                                  // 14
  const bool bw = dd_lt(MWP_bw, MWP_nb);
  const ddv mwp0 = bw ? MWP_bw : MWP_nb;
  const bool mwpW = !dd_lt(mwp0, Wd);                                            // 12: MWP = W_act
  const ddv mwp = mwpW ? Wd : mwp0;
  const bool cwpf = dd_lt(CWPf, Wd);
  const ddv cwp = cwpf ? CWPf : Wd;
  const ddv cpm = dd_div(cc, s23);                                               // Comp_c / Mem
  const ddv tail = dd_mul(cpm, dd_sub(mwp, one));
  ddv X;
  if (mwpW && !cwpf)                                                             // 16
    X = dd_add(dd_add(Mem_c, Comp_c), tail);
  else if (!dd_lt(cwp, mwp) || dd_lt(Mem_c, Comp_c))                             // 17
    X = dd_add(mwpW ? Mem_c : dd_div(dd_mul(Mem_c, Wd), mwp0), tail);
  else                                                                           // 18
    X = dd_add(dd_div(mc, s23), dd_mul(Comp_c, Wd));
  const ddv E = dd_div(dd_mul(X, dd_d((double)blocks)), dd_muld(SM, B));         // 15: x #Blocks / (B SM)
  return E.h + E.l;
}

// pk: the refined polynomial values; (ph, pl): their unevaluated high / low sums
template <int NPOLY>
__device__ __forceinline__ double pair_E(const DevProg &pg, const CfgTable &tab, int g, const int32_t *Dt,
                                         const CfgRec &r, const double *pk, const double *ph, const double *pl) {
  if (NPOLY != 6) {  // template g1: E = p_0 / q_0
    const ddv p0 = dd_ts(ph[0], pl[0]), q0 = dd_ts(ph[1], pl[1]);
    const ddv E = dd_div(p0, q0);
    return E.h + E.l;
  }
  const int P[3] = {r.Pm1_0 + 1, r.Pm1_1 + 1, r.Pm1_2 + 1};
  int64_t blocks = 1;
  for (int k = 0; k < pg.p && k < 3; ++k)
    if (pg.grid_map[k] >= 0) blocks *= ((int64_t)Dt[pg.grid_map[k]] + P[k] - 1) / P[k];
  const int64_t smact = blocks < pg.n_sm ? blocks : pg.n_sm;
  // all six values positive: every sum of Appendix A adds positive terms and FP64 is accurate to
  // ~20 ulp; otherwise (a metric <= 0 somewhere, sums that cancel) the double-double form
  bool pos = true;
#pragma unroll
  for (int k = 0; k < 6; ++k) pos = pos && pk[k] > 0.0;
#ifdef RP_REFINE_PROBE_NODD  // timing probe: never the double-double Appendix A
  pos = true;
#endif
  if (!pos) {
    ddv pd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) pd[k] = dd_ts(ph[k], pl[k]);
#ifdef RP_REFINE_LITERAL_DD
    return mwpcwp_E_dd(pd, r.W, blocks, rint(1.0 / r.rB), smact, pg);  // B_active: a small integer
#else
    return mwpcwp_E_dd2(pd, r.W, blocks, rint(1.0 / r.rB), smact, pg);
#endif
  }
  const double rSM = tab.rSM[(int64_t)g * kRSMTab + smact];
  const double Rep = (double)blocks * r.rB * rSM;
  return mwpcwp_E(pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], r.W, Rep, rSM, (double)smact, make_econst(pg));
}

// shared memory of k_refine: the term list (int32, padded to 16 B), its coefficients
// [nrt][kMaxPolys] and the tuples' data monomials [nDE][T] (double-double)
__host__ __device__ inline size_t refine_smem_bytes(int nrt, int nDE, int T) {
  return (size_t)((nrt + 3) & ~3) * 4 + (size_t)nrt * kMaxPolys * 8 + (size_t)nDE * T * 16;
}

template <int NPOLY, bool SECOND>
__global__ void __launch_bounds__(kRefThreads) k_refine(SweepArgs a) {
  const int g = blockIdx.y;
  const int T = blockDim.x, tid = threadIdx.x;
  const DevProg &pg = a.progs[g];
  const double *ri = a.tab.rinfo + (int64_t)g * 8;
  const int maxdeg = (int)ri[6], nrt = (int)ri[7];
  const int d = a.d, nDE = pg.nDE;
  // stage the term list and its coefficients (read by every thread in the same order: broadcast)
  extern __shared__ __align__(16) unsigned char rsh[];
  int32_t *sT = reinterpret_cast<int32_t *>(rsh);
  double2 *sCf = reinterpret_cast<double2 *>(rsh + (size_t)((nrt + 3) & ~3) * 4);  // [nrt][kMaxPolys / 2]
  double2 *sMD = sCf + (size_t)nrt * (kMaxPolys / 2);                              // [nDE][T]
  {
    const int32_t *rt = a.tab.rterm + (int64_t)g * a.npe_pad * a.tab.nde_pad;
    const double2 *rc = reinterpret_cast<const double2 *>(a.tab.rcoef + (int64_t)g * a.npe_pad * a.tab.nde_pad * kMaxPolys);
    for (int i = tid; i < nrt; i += T) sT[i] = rt[i];
    for (int i = tid; i < nrt * (kMaxPolys / 2); i += T) sCf[i] = rc[i];
  }
  __shared__ int8_t sDE[kMaxDE][kMaxVars];  // the data-part exponents (broadcast reads)
  for (int i = tid; i < nDE * kMaxVars; i += T) sDE[i / kMaxVars][i % kMaxVars] = pg.de_exp[i / kMaxVars][i % kMaxVars];
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * T + tid;
  if (t >= a.nD) return;
  const int64_t o = (int64_t)g * a.nD + t;
  const int32_t win = a.idx[o];
  if (win < 0) return;
  const CfgRec *sr = a.tab.srec + (int64_t)g * a.tab.nFp;
  const int32_t *inv = a.tab.inv + (int64_t)g * a.tab.nFp;
  const int p1 = __ldg(inv + win);
  if (p1 < 0) return;
  const CfgRec *r1 = sr + p1;
  const int32_t run = SECOND ? a.idx2[o] : -1;
  const int p2 = (SECOND && run >= 0) ? __ldg(inv + run) : -1;
  const CfgRec *r2 = p2 >= 0 ? sr + p2 : nullptr;
  const bool two = SECOND && r2 != nullptr;
  const int32_t *Dt = a.D + t * d;

  double u[kMaxVars];
  double R = 1.0;  // max(1, |u_k|) over the variables of both pairs
  for (int k = 0; k < d; ++k) {
    u[k] = ((double)Dt[k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
    R = fmax(R, fabs(u[k]));
  }
  for (int de = 0; de < nDE; ++de) sMD[(size_t)de * T + tid] = dd_monomial(sDE[de], d, u);
  double uP[3] = {0.0, 0.0, 0.0}, uP2[3] = {0.0, 0.0, 0.0};
  {
    const int P1[3] = {r1->Pm1_0 + 1, r1->Pm1_1 + 1, r1->Pm1_2 + 1};
    for (int k = 0; k < pg.p; ++k) {
      uP[k] = ((double)P1[k] - pg.xc[d + k]) * ldexp(1.0, -pg.xe[d + k]);
      R = fmax(R, fabs(uP[k]));
    }
  }
  if (two) {
    const int P2[3] = {r2->Pm1_0 + 1, r2->Pm1_1 + 1, r2->Pm1_2 + 1};
    for (int k = 0; k < pg.p; ++k) {
      uP2[k] = ((double)P2[k] - pg.xc[d + k]) * ldexp(1.0, -pg.xe[d + k]);
      R = fmax(R, fabs(uP2[k]));
    }
  }
  double Rp = 1.0;
  for (int i = 0; i < maxdeg; ++i) Rp *= R;
  double sg[NPOLY];
  bool okb = true;
#pragma unroll
  for (int k = 0; k < NPOLY; ++k) {
    sg[k] = extract_sigma(ri[k] * Rp * 1.0000000001);  // |c m| <= |c| R^maxdeg (+ rounding)
    okb = okb && sg[k] > 0.0;
  }
  if (!okb) return;  // bounds overflow: keep the sweep's values
  double h1[NPOLY], l1[NPOLY], h2[NPOLY], l2[NPOLY];
#pragma unroll
  for (int k = 0; k < NPOLY; ++k) h1[k] = l1[k] = h2[k] = l2[k] = 0.0;
  // terms in (pe, de) order: the program monomial m_pe(u_P) changes ~nPE times per tuple and is
  // recomputed then (uniform across the warp), the data monomial comes from shared memory
  int cur_pe = -1;
  double2 mp1 = make_double2(0.0, 0.0), mp2 = make_double2(0.0, 0.0);
  const double2 *mpd1 = a.tab.mPdd + ((int64_t)g * a.tab.nFp + p1) * a.npe_pad;
  const double2 *mpd2 = a.tab.mPdd + ((int64_t)g * a.tab.nFp + (p2 >= 0 ? p2 : p1)) * a.npe_pad;
  for (int j = 0; j < nrt; ++j) {
    const int32_t tt = sT[j];
    const int pe = tt >> 16;
    if (pe != cur_pe) {
      cur_pe = pe;
      // (the plan's double-double program monomials: computing them here was 30% of the kernel)
      mp1 = __ldg(mpd1 + pe);
      if (two) mp2 = __ldg(mpd2 + pe);
    }
    const double2 md = sMD[(size_t)(tt & 0xffff) * T + tid];
    double c[NPOLY];
#pragma unroll
    for (int k = 0; k < NPOLY; k += 2) {
      const double2 cc = sCf[(size_t)j * (kMaxPolys / 2) + k / 2];
      c[k] = cc.x;
      c[k + 1] = cc.y;
    }
    {
      const double mh = md.x * mp1.x;
      const double ml = fma(md.x, mp1.y, fma(md.y, mp1.x, fma(md.x, mp1.x, -mh)));
#pragma unroll
      for (int k = 0; k < NPOLY; ++k) {
        const double tq = fma(c[k], mh, sg[k]) - sg[k];
        h1[k] += tq;
        l1[k] = fma(c[k], ml, l1[k] + fma(c[k], mh, -tq));
      }
    }
    if (two) {
      const double mh = md.x * mp2.x;
      const double ml = fma(md.x, mp2.y, fma(md.y, mp2.x, fma(md.x, mp2.x, -mh)));
#pragma unroll
      for (int k = 0; k < NPOLY; ++k) {
        const double tq = fma(c[k], mh, sg[k]) - sg[k];
        h2[k] += tq;
        l2[k] = fma(c[k], ml, l2[k] + fma(c[k], mh, -tq));
      }
    }
  }
  double pk[NPOLY];
#pragma unroll
  for (int k = 0; k < NPOLY; ++k) pk[k] = h1[k] + l1[k];
  double E1 = pair_E<NPOLY>(pg, a.tab, g, Dt, *r1, pk, h1, l1);
  if (!pos_finite(E1)) E1 = a.bestE[o];  // exact evaluation masks the pair: keep the sweep's value
  if (!SECOND) {
    a.bestE[o] = E1;
    return;
  }
  double E2 = a.secondE[o];
  if (two) {
#pragma unroll
    for (int k = 0; k < NPOLY; ++k) pk[k] = h2[k] + l2[k];
    const double e2 = pair_E<NPOLY>(pg, a.tab, g, Dt, *r2, pk, h2, l2);
    if (pos_finite(e2)) E2 = e2;
  }
  // re-rank the two on the exact key (E, original index)
  if (two && key_less(E2, run, E1, win)) {
    a.idx[o] = run;
    a.bestE[o] = E2;
    a.secondE[o] = E1;
    a.idx2[o] = win;
  } else {
    a.bestE[o] = E1;
    a.secondE[o] = E2;
  }
}

static bool refine_enabled() {
  const char *v = getenv("RP_SWEEP_REFINE");
  return !(v && v[0] == '0');
}

template <int NPOLY, bool SECOND>
static cudaError_t launch_refine_t(const SweepArgs &a, int n_prog, int nDE, int nPE, cudaStream_t s) {
  (void)nPE;
  // union terms <= npe_pad * nde_pad (the plan's bound; the kernel reads the actual count)
  const int nrt_max = a.tab.nrt_max;
  int T = kRefThreads;
  auto bytes = [&](int th) { return refine_smem_bytes(nrt_max, nDE, th); };
  while (T > 32 && bytes(T) > 200 * 1024) T >>= 1;
  const size_t smem = bytes(T);
  cudaError_t e = cudaFuncSetAttribute(k_refine<NPOLY, SECOND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (a.nD + T - 1) / T;
  if (blocks > 0x7fffffffll) return cudaErrorInvalidValue;
  k_refine<NPOLY, SECOND><<<dim3((unsigned)blocks, (unsigned)n_prog), T, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const DevProg *d_progs, int n_prog, bool mwp, CfgTable tab, int npe_pad,
                         int nde_max, int n_sm_max, int d, const int32_t *d_D, int64_t nD,
                         int32_t *idx, double *bestE, double *secondE, const int32_t *perm,
                         int32_t *idx2, cudaEvent_t *ev, cudaStream_t s) {
  if (nD == 0) return cudaSuccess;
  if (ev) cudaEventRecord(ev[1], s);
  // n_sm < kRSMTab for every program (compile_program): the 1/SM_act tables always exist
  SweepArgs a{d_progs, tab, npe_pad, d, md_stride(tab.nde_pad), d_D, nD, idx, bestE, secondE, perm};
  a.idx2 = refine_enabled() ? idx2 : nullptr;
  cudaError_t e;
  switch (npe_pad) {
    case 4: e = launch_npe<4>(a, n_prog, mwp, n_sm_max, s); break;
    case 8: e = launch_npe<8>(a, n_prog, mwp, n_sm_max, s); break;
    case 16: e = launch_npe<16>(a, n_prog, mwp, n_sm_max, s); break;
    case 20: e = launch_npe<20>(a, n_prog, mwp, n_sm_max, s); break;
    case 24: e = launch_npe<24>(a, n_prog, mwp, n_sm_max, s); break;
    case 36: e = launch_npe<36>(a, n_prog, mwp, n_sm_max, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[2], s);
  if (e == cudaSuccess && refine_enabled()) {  // the winners' E (and runner-ups') accurate
    const bool second = secondE != nullptr && a.idx2 != nullptr;
    if (mwp)
      e = second ? launch_refine_t<6, true>(a, n_prog, nde_max, npe_pad, s)
                 : launch_refine_t<6, false>(a, n_prog, nde_max, npe_pad, s);
    else
      e = second ? launch_refine_t<2, true>(a, n_prog, nde_max, npe_pad, s)
                 : launch_refine_t<2, false>(a, n_prog, nde_max, npe_pad, s);
  }
  return e;
}

}  // namespace rp
