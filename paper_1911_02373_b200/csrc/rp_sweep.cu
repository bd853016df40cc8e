// rp_sweep.cu -- the runtime sweep of the rational program R over (D, P) with per-D argmin.
//
// PAPER.md:2259-2305 (steps 4 and 5): for the runtime data parameters D and "all practically
// meaningful values of P from the set F, we compute an estimate of E using R", then an
// exhaustive search picks the optimum.  Here one CTA owns a tile of TD data tuples and sweeps
// every statically feasible configuration of F for them; one thread owns one configuration at
// a time (its program-part monomials live in registers) and walks the TD tuples, whose staged
// data polynomials C_{k,pe}(D) are broadcast from shared memory.  The argmin key is the exact
// lexicographic (E, original config index), so exact ties go to the lowest index (reading R15).
//
// Kernels:
//   k_plan_configs -- a1 + a5: per configuration T, the static mask (warp rule, T <= T_max,
//                     B_active > 0), B_active (occupancy flowchart), W_active (Eq. (1)) and the
//                     program-part monomials; compaction of the feasible ones in index order.
//   k_sweep        -- a2 (stage C(D)), a3 (P1 P2 <= D1^2), a4 (g_i), a6 (grid), a7 (E),
//                     a8 (argmin + second best), for a tile of D x all feasible configs.
#include <cstdio>

#include "rp_internal.cuh"

namespace rp {

// ---- a5: occupancy, Fig. occupancysimpleflowchart, 64-bit integers ----
__device__ __forceinline__ int64_t occupancy_blocks(int64_t T, int64_t R, int64_t Z,
                                                    const DevProg &pg) {
  const int64_t Bm = pg.b_max, W32 = 32 * (int64_t)pg.w_max, Rm = pg.r_max, Zm = pg.z_max;
  if (T * Bm <= W32 && R * T * Bm <= Rm && Z * Bm <= Zm) return Bm;             // no limit
  if (W32 <= T * Bm && W32 * R <= Rm && W32 * Z <= Zm * T) return W32 / T;       // warps
  if (Rm <= R * T * Bm && Rm <= R * W32 && Rm * Z <= R * T * Zm) return Rm / (R * T);  // regs
  if (Zm <= Bm * Z && Zm * T <= W32 * Z && Zm * R * T <= Z * Rm) return Zm / Z;   // smem
  return 0;                                                                       // failure
}

// ---- a1 + a5 + P-monomials, compaction in index order --------------------------------------
__global__ void __launch_bounds__(1024) k_plan_configs(const DevProg *progs, const int32_t *F,
                                                       int nF, int npe_pad, CfgTable tab) {
  const int g = blockIdx.x;
  const DevProg &pg = progs[g];
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
      for (int k = 0; k < pg.p; ++k) T *= Pk[k];
      ok = (T % 32 == 0) && (T <= pg.t_max) && (T > 0);
      if (ok) {
        const int64_t Z = pg.Z0 + pg.Z1 * T;
        B = occupancy_blocks(T, pg.R, Z, pg);
        ok = B > 0;
        W = (B * T) / 32;  // Eq. (1)
        if (W > pg.w_max) W = pg.w_max;
      }
    }
    // block-wide exclusive scan of ok (index order preserved)
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
      const int64_t off = (int64_t)g * nF;
      tab.orig[off + pos] = c;
      for (int k = 0; k < 3; ++k) tab.P[(int64_t)g * 3 * nF + (int64_t)k * nF + pos] = Pk[k];
      tab.B[off + pos] = (int32_t)B;
      tab.W[off + pos] = (int32_t)W;
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
        tab.mP[(int64_t)g * npe_pad * nF + (int64_t)pe * nF + pos] = m;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base = pos + ok;
    __syncthreads();
  }
  if (threadIdx.x == 0) tab.nFc[g] = base;
}

cudaError_t launch_plan_configs(const DevProg *d_progs, int n_prog, const int32_t *d_F, int nF,
                                int npe_pad, CfgTable tab, cudaStream_t s) {
  k_plan_configs<<<n_prog, 1024, 0, s>>>(d_progs, d_F, nF, npe_pad, tab);
  return cudaGetLastError();
}

// ---- argmin state: exact lexicographic (E, index) with the runner-up E ----------------------
struct Best {
  double e;    // best E (+inf: none)
  int32_t i;   // its original config index (INT_MAX: none)
  double s;    // second-smallest E among the others
};
__device__ __forceinline__ bool key_less(double e1, int32_t i1, double e2, int32_t i2) {
  return e1 < e2 || (e1 == e2 && i1 < i2);
}
__device__ __forceinline__ Best merge(const Best &a, const Best &b) {
  Best r;
  if (key_less(a.e, a.i, b.e, b.i)) {
    r.e = a.e; r.i = a.i; r.s = fmin(a.s, b.e);
  } else {
    r.e = b.e; r.i = b.i; r.s = fmin(b.s, a.e);
  }
  return r;
}
__device__ __forceinline__ Best shfl_xor(const Best &a, int m) {
  Best r;
  r.e = __shfl_xor_sync(0xffffffffu, a.e, m);
  r.i = __shfl_xor_sync(0xffffffffu, a.i, m);
  r.s = __shfl_xor_sync(0xffffffffu, a.s, m);
  return r;
}

// ---- a7: the MWP-CWP estimate (DESIGN.md Appendix A = Hong & Kim ISCA'09 Eqs. 1-18) --------
__device__ __forceinline__ double mwpcwp_E(double g1, double g2, double g3, double Wact,
                                           double Bact, double SMact, double blocks,
                                           const DevProg &pg) {
  const double Mem = g2 + g3;
  const double Tot = g1 + g2 + g3;
  const double W_unc = g3 / Mem;
  const double W_coal = g2 / Mem;
  const double L_unc = pg.mem_ld + (pg.U - 1.0) * pg.dd_unc;
  const double L_coal = pg.mem_ld;
  const double Mem_L = L_unc * W_unc + L_coal * W_coal;
  const double Dep = pg.dd_unc * pg.U * W_unc + pg.dd_coal * W_coal;
  const double MWP_nb = Mem_L / Dep;
  const double BWpw = pg.freq * pg.lbpw / Mem_L;
  const double MWP_bw = pg.mem_bw / (BWpw * SMact);
  double MWP = MWP_nb;
  if (MWP_bw < MWP) MWP = MWP_bw;
  if (Wact < MWP) MWP = Wact;
  const double Comp_c = pg.issue * Tot;
  const double Mem_c = L_unc * g3 + L_coal * g2;
  const double CWP_full = (Mem_c + Comp_c) / Comp_c;
  const double CWP = CWP_full < Wact ? CWP_full : Wact;
  const double Rep = blocks / (Bact * SMact);
  double E;
  if (MWP == Wact && CWP == Wact)
    E = (Mem_c + Comp_c + Comp_c / Mem * (MWP - 1.0)) * Rep;
  else if (CWP >= MWP || Comp_c > Mem_c)
    E = (Mem_c * Wact / MWP + Comp_c / Mem * (MWP - 1.0)) * Rep;
  else
    E = (Mem_L + Comp_c * Wact) * Rep;
  return E;
}

// ---- the sweep ------------------------------------------------------------------------------
struct SweepArgs {
  const DevProg *progs;
  CfgTable tab;
  int nF;
  int d;
  const int32_t *D;
  int64_t nD;
  int32_t *idx;
  double *bestE;
  double *secondE;
};

constexpr int kSweepThreads = 256;

template <int NPE, int TD>
__global__ void __launch_bounds__(kSweepThreads, 2) k_sweep(SweepArgs a) {
  const int g = blockIdx.y;
  const DevProg &pg = a.progs[g];
  const int d = a.d;
  const int nPE = pg.nPE, nDE = pg.nDE, npoly = pg.npoly, nm = pg.nm;
  const int64_t d0 = (int64_t)blockIdx.x * TD;

  // dynamic shared memory (sweep_smem_bytes<NPE, TD>())
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto sC = reinterpret_cast<double(*)[kMaxPolys][NPE]>(smem_raw);
  auto sMD = reinterpret_cast<double(*)[kMaxDE]>(smem_raw + sizeof(double) * TD * kMaxPolys * NPE);
  auto sBe = reinterpret_cast<double(*)[kSweepThreads]>(&sMD[TD][0]);
  auto sBs = reinterpret_cast<double(*)[kSweepThreads]>(&sBe[TD][0]);
  auto sRed = reinterpret_cast<Best(*)[kSweepThreads / 32]>(&sBs[TD][0]);
  auto sBi = reinterpret_cast<int32_t(*)[kSweepThreads]>(&sRed[TD][0]);
  auto sD = reinterpret_cast<int32_t(*)[kMaxVars]>(&sBi[TD][0]);

  // a2: load the D tile (tuples past nD are replaced by D = 1, and their results dropped)
  for (int i = threadIdx.x; i < TD * d; i += blockDim.x) {
    const int t = i / d, k = i % d;
    sD[t][k] = (d0 + t < a.nD) ? a.D[(d0 + t) * d + k] : 1;
  }
  __syncthreads();
  // a2: data-part monomials m_de(u_D), u = (D - c) 2^-e
  for (int i = threadIdx.x; i < TD * nDE; i += blockDim.x) {
    const int t = i / nDE, de = i % nDE;
    double m = 1.0;
    for (int k = 0; k < d; ++k) {
      const double u = ((double)sD[t][k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
      for (int e = 0; e < pg.de_exp[de][k]; ++e) m *= u;
    }
    sMD[t][de] = m;
  }
  __syncthreads();
  // a2: staged data polynomials C_{k,pe}(D) (zero padding for k >= npoly or pe >= nPE)
  for (int i = threadIdx.x; i < TD * kMaxPolys * NPE; i += blockDim.x) {
    const int t = i / (kMaxPolys * NPE), r = i % (kMaxPolys * NPE);
    const int k = r / NPE, pe = r % NPE;
    double acc = 0.0;
    if (k < npoly && pe < nPE) {
      const int row = k * nPE + pe;
      for (int j = pg.row_start[row]; j < pg.row_start[row + 1]; ++j)
        acc = fma(pg.term_coef[j], sMD[t][pg.term_de[j]], acc);
    }
    sC[t][k][pe] = acc;
  }
  __syncthreads();

  // running argmin state of (tuple t, thread): shared memory, updated in place
  for (int t = 0; t < TD; ++t) {
    sBe[t][threadIdx.x] = __longlong_as_double(0x7ff0000000000000ll);
    sBs[t][threadIdx.x] = __longlong_as_double(0x7ff0000000000000ll);
    sBi[t][threadIdx.x] = 0x7fffffff;
  }
  const int nFc = a.tab.nFc[g];
  const int64_t off = (int64_t)g * a.nF;
  const int dmap0 = pg.grid_map[0], dmap1 = pg.grid_map[1], dmap2 = pg.grid_map[2];
  const int p = pg.p;
  const double n_sm = (double)pg.n_sm;
  const int tmax = (int)((a.nD - d0) < TD ? (a.nD - d0) : TD);

  for (int c = threadIdx.x; c < nFc; c += blockDim.x) {
    const int32_t orig = a.tab.orig[off + c];
    const int32_t P0 = a.tab.P[off * 3 + c];
    const int32_t P1 = a.tab.P[off * 3 + a.nF + c];
    const int32_t P2 = a.tab.P[off * 3 + 2 * a.nF + c];
    const double Bact = (double)a.tab.B[off + c];
    const double Wact = (double)a.tab.W[off + c];
    double mP[NPE];
#pragma unroll
    for (int pe = 0; pe < NPE; ++pe) mP[pe] = a.tab.mP[off * NPE + (int64_t)pe * a.nF + c];
    const int64_t P01 = (int64_t)P0 * (p >= 2 ? P1 : 1);

#pragma unroll 1
    for (int t = 0; t < tmax; ++t) {
      // a3: "P1 P2 <= D1^2 is meaningful"
      const int64_t D1 = sD[t][0];
      if (P01 > D1 * D1) continue;
      // a6: grid gx = ceil(D/bx), ...; SM_act = min(#blocks, n_SM)
      int64_t blocks = 1;
      if (dmap0 >= 0) blocks *= (sD[t][dmap0] + P0 - 1) / P0;
      if (p >= 2 && dmap1 >= 0) blocks *= (sD[t][dmap1] + P1 - 1) / P1;
      if (p >= 3 && dmap2 >= 0) blocks *= (sD[t][dmap2] + P2 - 1) / P2;
      const double dblocks = (double)blocks;
      const double SMact = fmin(dblocks, n_sm);
      // a4: g_i = p_i / q_i with p_k = sum_pe C_{k,pe}(D) m_pe(P)
      double gv[kMaxMetrics];
#pragma unroll
      for (int i = 0; i < kMaxMetrics; ++i) {
        double pn = 0.0, qd = 0.0;
        if (i < nm) {
#pragma unroll
          for (int pe = 0; pe < NPE; ++pe) {
            pn = fma(sC[t][2 * i][pe], mP[pe], pn);
            qd = fma(sC[t][2 * i + 1][pe], mP[pe], qd);
          }
        }
        gv[i] = pn / qd;
      }
      // a7
      double E;
      if (pg.tmpl == RP_TEMPLATE_G1)
        E = gv[0];
      else
        E = mwpcwp_E(gv[0], gv[1], gv[2], Wact, Bact, SMact, dblocks, pg);
      if (!(E > 0.0 && E < __longlong_as_double(0x7ff0000000000000ll))) continue;  // R17
      // a8: running argmin (exact key (E, original index); configs arrive in index order)
      const double be = sBe[t][threadIdx.x];
      if (E < be) {
        sBs[t][threadIdx.x] = be;
        sBe[t][threadIdx.x] = E;
        sBi[t][threadIdx.x] = orig;
      } else if (E < sBs[t][threadIdx.x]) {
        sBs[t][threadIdx.x] = E;
      }
    }
  }

  // a8: warp then block reduction of the TD states
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = 0; t < TD; ++t) {
    Best b;
    b.e = sBe[t][threadIdx.x];
    b.i = sBi[t][threadIdx.x];
    b.s = sBs[t][threadIdx.x];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) b = merge(b, shfl_xor(b, m));
    if (lane == 0) sRed[t][wid] = b;
  }
  __syncthreads();
  if (threadIdx.x < TD) {
    const int t = threadIdx.x;
    const int64_t di = d0 + t;
    if (di < a.nD) {
      Best b = sRed[t][0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = merge(b, sRed[t][w]);
      const int64_t o = (int64_t)g * a.nD + di;
      const bool none = !(b.e < __longlong_as_double(0x7ff0000000000000ll));
      a.idx[o] = none ? -1 : b.i;
      a.bestE[o] = b.e;
      if (a.secondE) a.secondE[o] = b.s;
    }
  }
}

template <int NPE, int TD>
constexpr size_t sweep_smem_bytes() {
  return sizeof(double) * TD * kMaxPolys * NPE + sizeof(double) * TD * kMaxDE +
         2 * sizeof(double) * TD * kSweepThreads + sizeof(Best) * TD * (kSweepThreads / 32) +
         sizeof(int32_t) * TD * kSweepThreads + sizeof(int32_t) * TD * kMaxVars;
}

template <int NPE>
static cudaError_t launch_npe(const SweepArgs &a, int n_prog, cudaStream_t s) {
  constexpr int TD = 8;
  constexpr size_t smem = sweep_smem_bytes<NPE, TD>();
  const int64_t tiles = (a.nD + TD - 1) / TD;
  if (tiles > 0x7fffffffll) return cudaErrorInvalidValue;
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep<NPE, TD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((unsigned)tiles, (unsigned)n_prog);
  k_sweep<NPE, TD><<<grid, kSweepThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const DevProg *d_progs, int n_prog, CfgTable tab, int nF, int npe_pad,
                         int d, const int32_t *d_D, int64_t nD, int32_t *idx, double *bestE,
                         double *secondE, cudaStream_t s) {
  if (nD == 0) return cudaSuccess;
  SweepArgs a{d_progs, tab, nF, d, d_D, nD, idx, bestE, secondE};
  switch (npe_pad) {
    case 4: return launch_npe<4>(a, n_prog, s);
    case 8: return launch_npe<8>(a, n_prog, s);
    case 16: return launch_npe<16>(a, n_prog, s);
    case 20: return launch_npe<20>(a, n_prog, s);
    case 24: return launch_npe<24>(a, n_prog, s);
    case 36: return launch_npe<36>(a, n_prog, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rp
