// rp_moments.cu -- a12 (the Gram A^T A of the linearised least-squares system) as a contraction
// of MOMENTS instead of an outer product of design rows.
//
// PAPER.md:2578-2584 / 2601-2603: row r of the linearised system is a_r = [M(u_r) | -V_r N(u_r)]
// with M, N monomial columns ("essentially a Vandermonde matrix").  Every entry of
// G = sum_r s_r^2 a_r a_r^T is then a weighted moment of ONE monomial:
//   G[num i][num j] =  sum_r s_r^2       u_r^(e_i + e_j)
//   G[num i][den j] = -sum_r s_r^2 V_r   u_r^(e_i + f_j)
//   G[den i][den j] =  sum_r s_r^2 V_r^2 u_r^(f_i + f_j)
// (s_r = 1 unless the rows are weighted, f4).  So the Gram of the n_v metrics needs only the
// moments m_w(e) = sum_r w_r(r) u_r^e for the exponents e of total degree <= D = 2 max|e_i|
// (the simplex: 495 of them for 4 variables and degree-4 bases) and the weights
// w in {1, V_v, V_v^2} (unweighted: 1 + 2 n_v of them) or {s_v^2, s_v^2 V_v, s_v^2 V_v^2}:
// 2 x 8 x 496 = 7.9k flop per row instead of the 34.8k of the 7 symmetric 70 x 70 blocks that
// k_gram_ws accumulates.  The contraction over rows is the same dense FP64
// product, moments[w][e] += W^T[w][rows] Mon[rows][e], on DMMA.8x8x4 (A = 8 weights x 4 rows,
// B = 4 rows x 8 exponents).
//
// k_gram_mom: one CTA per SM (16 warps) owns a contiguous slab of 32-row stages.  Per stage:
//   inputs  -- X rows, V_v (and S_v) land in a 3-stage ring by cp.async.bulk (TMA engine) issued
//              3 stages ahead; one warp turns them into u = (x - c) 2^-e and the row weights;
//   monomials (a11) -- lane = row; warp w generates a contiguous slot range of the simplex in
//              lexicographic order, unit by unit (a unit fixes e_0 .. e_{n-2}; its entries run
//              over e_{n-1}, each one DMUL from the previous), into sM[slot][row] (conflict-free:
//              a warp stores 32 consecutive rows);
//   moments (a12) -- warp w owns a contiguous range of 8-slot tiles and accumulates them for the
//              8 (or 16) weights over the stage's 8 k-steps.
// Register accumulators are added into the CTA's partial every 1,024 rows (two-level
// summation, as k_gram_ws); k_mom_sum adds the partials in a fixed order (deterministic) and
// k_mom_assemble scatters the moments into G_v (the slot of e_i + e_j by its lexicographic rank).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "rp_internal.cuh"
#include "rp_umma.cuh"

namespace rp {

#ifndef RP_MOM_WARPS
#define RP_MOM_WARPS 16
#endif
constexpr int kMomWarps = RP_MOM_WARPS;            // consumers: monomials + moments of their own tiles
constexpr int kMomThreads = 32 * (kMomWarps + 1);  // + one producer warp: TMA issue, row weights
constexpr int kMomRT = 32;          // rows per stage (lane = row in the monomial step)
constexpr int kMomRTP = 36;         // row stride of sM in doubles (= 4 mod 16: conflict-free fragments)
constexpr int kMomMaxSlots = 640;   // simplex size limit (shared memory)
constexpr int kMomMaxUnits = 256;
#ifndef RP_MOM_IS
#define RP_MOM_IS 5
#endif
#ifndef RP_MOM_LEAD
#define RP_MOM_LEAD 3
#endif
constexpr int kMomIS = RP_MOM_IS;      // ring slots: raw inputs (+ X transposed, ones row) of a stage
constexpr int kMomLead = RP_MOM_LEAD;  // bulk copies are issued this many stages ahead
constexpr int kMomFlush = 32;       // stages between flushes of the register accumulators (1024 rows)

struct MomArgs {
  const GramBasis *basis;  // device: the transform (xc, xe) and the column exponents (assembly)
  const double *X;         // [K][n]
  const double *V;         // [nv][K]
  const double *S;         // [nv][K] row scales or null
  int64_t K;
  double *part;            // [gridDim.x][nT][WT][64]
  int n, D, nslot, nT, nv, nw, tma;
  int16_t wtile[kMomWarps + 1];  // tiles of consumer warp w: [wtile[w], wtile[w + 1])
  int16_t wunit[kMomWarps];      // the first unit overlapping its slots
  int16_t wuslot[kMomWarps];     // that unit's first slot
  uint32_t uexp[kMomMaxUnits];   // unit: e_0 .. e_{n-2}, 4 bits each
  uint8_t ulen[kMomMaxUnits];    // its entries: e_{n-1} = 0 .. ulen - 1
};

__device__ __forceinline__ void mom_dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// one ring slot: X [RT][n] | V_v rows | S_v rows (bulk copies) | a row of ones the producer
// writes (0 past the slab).  The per-row vectors are kMomVS apart (= 8 banks: the quads of a warp
// read up to four of them at the same row without conflicts); every vector starts 16-byte aligned
// (bulk-copy targets).  (The consumers square V_v and s_v themselves: scalar FP64 work in the
// producer waits behind its sub-partition's DMMAs and starves the ring -- measured 0.474 vs
// 0.431 ms.)
constexpr int kMomVS = kMomRT + 4;
__host__ __device__ inline int mom_vec_off(int n) { return (kMomRT * n + 1) & ~1; }
__host__ __device__ inline int mom_in_doubles(int n, int nv, bool weighted) {
  return mom_vec_off(n) + kMomVS * (nv + (weighted ? nv : 0) + 1);
}

static size_t mom_smem(int nT, int n, int nv, bool weighted, bool generic = true) {
  return sizeof(double) * ((size_t)nT * 8 * kMomRTP + (generic ? kMomWarps * kMaxVars * kMomRT : 0) +
                           kMomIS * kMaxVars * kMomRT +
                           (size_t)kMomIS * mom_in_doubles(n, nv, weighted)) +
         sizeof(uint64_t) * 3 * kMomIS;
}

// ---- the simplex's units and the warps' shares (one algorithm for the host plan and the
// compile-time specialisations) ------------------------------------------------------------------
struct MomTab {
  int nu, ns;
  int8_t ex[kMomMaxUnits][kMaxVars];  // e_0 .. e_{N-2} of unit u (e_{N-1} runs over 0 .. len - 1)
  int len[kMomMaxUnits], slot[kMomMaxUnits];
  int nT;                            // 8-slot tiles
  int tb[kMomWarps + 1];              // tiles of warp w: [tb[w], tb[w + 1]) (moments and monomials)
  int wu[kMomWarps], wue[kMomWarps];  // units overlapping warp w's slots [8 tb[w], min(8 tb[w + 1], ns))
};
// units in lexicographic order (e_0 slowest, e_{N-2} fastest); nu = 0 when the simplex is too large
__host__ __device__ constexpr MomTab mom_tab(int N, int D) {
  MomTab t{};
  int e[kMaxVars] = {};
  const int np = N - 1;
  int slot = 0;
  for (;;) {
    if (t.nu >= kMomMaxUnits) {
      t.nu = 0;
      return t;
    }
    int sum = 0;
    for (int k = 0; k < np; ++k) sum += e[k], t.ex[t.nu][k] = (int8_t)e[k];
    t.len[t.nu] = D - sum + 1;
    t.slot[t.nu] = slot;
    slot += D - sum + 1;
    ++t.nu;
    int k = np - 1;
    while (k >= 0) {
      ++e[k];
      int s2 = 0;
      for (int i = 0; i < np; ++i) s2 += e[i];
      if (s2 <= D) break;
      e[k] = 0;
      --k;
    }
    if (k < 0) break;
  }
  t.ns = slot;
  // every warp accumulates a contiguous range of tiles (the remainder to the first warps: the
  // last ones stay lighter) and generates the monomials of exactly those slots
  t.nT = (t.ns + 7) / 8;
  const int base = t.nT / kMomWarps, rem = t.nT % kMomWarps;
  t.tb[0] = 0;
  for (int w = 0; w < kMomWarps; ++w) t.tb[w + 1] = t.tb[w] + base + (w < rem ? 1 : 0);
  for (int w = 0; w < kMomWarps; ++w) {
    const int s0 = 8 * t.tb[w], s1 = 8 * t.tb[w + 1] < t.ns ? 8 * t.tb[w + 1] : t.ns;
    int u = 0;
    while (u < t.nu && t.slot[u] + t.len[u] <= s0) ++u;
    t.wu[w] = u;
    while (u < t.nu && t.slot[u] < s1) ++u;
    t.wue[w] = s1 > s0 ? u : t.wu[w];
  }
  return t;
}
template <int N, int D>
struct MomC {
  static constexpr MomTab t = mom_tab(N, D);
};

// a11 for the units [UI, UE) of one warp, every index and exponent a compile-time constant:
// the unit's prefix from the power table (or, for the next e_{N-2} of the same prefix, one DMUL
// from the previous unit's), then e_{N-1} = 0 .. len - 1 one DMUL each; lane = row
struct MomUnit {
  int len, slot;
  bool cont;               // the previous unit has the same prefix with e_{N-2} one less
  int8_t ex[kMaxVars];
};
template <int N, int D>
__host__ __device__ constexpr MomUnit mom_unit(int u) {
  const MomTab &T = MomC<N, D>::t;
  MomUnit x{};
  x.len = T.len[u];
  x.slot = T.slot[u];
  for (int k = 0; k < kMaxVars; ++k) x.ex[k] = T.ex[u][k];
  x.cont = u > 0 && N >= 2;
  for (int k = 0; k + 2 < N && x.cont; ++k) x.cont = T.ex[u][k] == T.ex[u - 1][k];
  if (x.cont) x.cont = T.ex[u][N - 2] == T.ex[u - 1][N - 2] + 1;
  return x;
}
template <int N, int D>
__host__ __device__ constexpr int mom_wu(int w, int which) {  // 0: first unit, 1: end unit, 2/3: slot window
  const MomTab &T = MomC<N, D>::t;
  if (which == 0) return T.wu[w];
  if (which == 1) return T.wue[w];
  if (which == 2) return 8 * T.tb[w];
  return 8 * T.tb[w + 1] < T.ns ? 8 * T.tb[w + 1] : T.ns;
}

// a11 for the units [UI, UE) overlapping the warp's slots [S0, S1), every index and exponent a
// compile-time constant: the unit's prefix from the power table (or, for the next e_{N-2} of the
// same prefix, one DMUL from the previous unit's), then its entries in the window, one DMUL each
// (lane = row)
template <int N, int D, int UB, int UI, int UE, int S0, int S1>
__device__ __forceinline__ void mom_gen_units(const double (&pw)[kMaxVars][16], double *dst, double am_prev) {
  if constexpr (UI < UE) {
    constexpr MomUnit U = mom_unit<N, D>(UI);
    double am;
    if constexpr (U.cont && UI > UB) {  // (the warp's first unit always starts from the table)
      am = am_prev * pw[N - 2][1];
    } else {
      am = 1.0;
      bool one = true;
#pragma unroll
      for (int k = 0; k + 1 < N; ++k)
        if (U.ex[k] > 0) {
          am = one ? pw[k][U.ex[k]] : am * pw[k][U.ex[k]];
          one = false;
        }
    }
    constexpr int jb = S0 > U.slot ? S0 - U.slot : 0;
    constexpr int je = S1 - U.slot < U.len ? S1 - U.slot : U.len;
    double m = jb == 0 ? am : am * pw[N - 1][jb];
#pragma unroll
    for (int j = jb; j < je; ++j) {
      dst[(U.slot + j) * kMomRTP] = m;
      if (j + 1 < je) m *= pw[N - 1][1];
    }
    mom_gen_units<N, D, UB, UI + 1, UE, S0, S1>(pw, dst, am);
  }
}

template <int N, int D, int W>
__device__ __forceinline__ void mom_gen_warp(const double (&u)[kMaxVars], double *dst) {
  // power table u_k^j (j <= D; only the entries this warp's units use survive)
  double pw[kMaxVars][16];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    pw[k][0] = 1.0;
    pw[k][1] = u[k];
#pragma unroll
    for (int j = 2; j <= D; ++j) pw[k][j] = pw[k][j - 1] * pw[k][1];
  }
  constexpr int ub = mom_wu<N, D>(W, 0), ue = mom_wu<N, D>(W, 1), s0 = mom_wu<N, D>(W, 2), s1 = mom_wu<N, D>(W, 3);
  mom_gen_units<N, D, ub, ub, ue, s0, s1>(pw, dst, 1.0);
}

// N, D > 0: the monomial step specialised for that simplex (mom_gen_warp); N = 0: generic
template <int WT, int TPW, int N, int D>
__global__ void __launch_bounds__(kMomThreads, 1) k_gram_mom(const __grid_constant__ MomArgs a) {
  extern __shared__ __align__(16) double msm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = a.n, nv = a.nv;
  const bool wtd = a.S != nullptr;
  const int nslotp = a.nT * 8;
  double *sM = msm;                                   // [nslotp][RTP]  monomials (each warp its own slots)
  double *sUg = sM + (size_t)nslotp * kMomRTP;        // [warps][kMaxVars][RT]  u (generic monomial step)
  double *sXt = sUg + (N > 0 ? 0 : kMomWarps * kMaxVars * kMomRT);  // [IS][kMaxVars][RT]  X transposed
  double *sIn = sXt + kMomIS * kMaxVars * kMomRT;     // [IS][INB]  raw inputs X | V | S
  const int INB = mom_in_doubles(n, nv, wtd);
  uint64_t *rfull = reinterpret_cast<uint64_t *>(sIn + kMomIS * INB);  // [IS] raw inputs landed
  uint64_t *wfull = rfull + kMomIS;                                     // [IS] X transposed, ones row written
  uint64_t *sempty = wfull + kMomIS;                                    // [IS] every consumer warp done
  __shared__ double sXc[kMaxVars], sXs[kMaxVars];  // the transform: c_k, 2^-e_k

  // slab: whole 32-row stages, so bulk-copy sources stay 16-byte aligned
  const int64_t nst_all = (a.K + kMomRT - 1) / kMomRT;
  const int64_t t0 = nst_all * blockIdx.x / gridDim.x, t1 = nst_all * (blockIdx.x + 1) / gridDim.x;
  const int64_t r_begin = kMomRT * t0;
  const int64_t r_end = (kMomRT * t1) < a.K ? kMomRT * t1 : a.K;
  const int ns = (int)(t1 - t0);
  auto full_stage = [&](int s) { return a.tma && r_begin + (int64_t)(s + 1) * kMomRT <= r_end; };

  // padding slots [nslot, nslotp) stay zero
  for (int i = threadIdx.x; i < (nslotp - a.nslot) * kMomRTP; i += blockDim.x) sM[(size_t)a.nslot * kMomRTP + i] = 0.0;
  if (threadIdx.x < kMaxVars) {
    sXc[threadIdx.x] = threadIdx.x < n ? a.basis->xc[threadIdx.x] : 0.0;
    sXs[threadIdx.x] = threadIdx.x < n ? ldexp(1.0, -a.basis->xe[threadIdx.x]) : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMomIS; ++i) {
      mbar_init(smem_u32(rfull + i), 1);
      mbar_init(smem_u32(wfull + i), 1);            // the producer (lane 0 after __syncwarp)
      mbar_init(smem_u32(sempty + i), kMomWarps);   // lane 0 of every consumer warp after __syncwarp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == kMomWarps) {
    // ---- producer: raw inputs of stage s into ring slot s % IS (TMA, or plain loads for a tail
    // or unaligned stage), then the row weights of the stage --------------------------------------
    auto issue = [&](int s) {  // lane 0
      const int st = s % kMomIS;
      double *dst = sIn + st * INB;
      const int64_t r0 = r_begin + (int64_t)s * kMomRT;
      const uint32_t bx = kMomRT * n * 8, bv = kMomRT * 8;
      const uint32_t bar = smem_u32(rfull + st);
      mbar_expect_tx(bar, bx + nv * bv * (wtd ? 2 : 1));
      bulk_g2s(smem_u32(dst), a.X + r0 * n, bx, bar);
      double *dv = dst + mom_vec_off(n);
      for (int v = 0; v < nv; ++v) bulk_g2s(smem_u32(dv + v * kMomVS), a.V + (int64_t)v * a.K + r0, bv, bar);
      if (wtd)
        for (int v = 0; v < nv; ++v) bulk_g2s(smem_u32(dv + (nv + v) * kMomVS), a.S + (int64_t)v * a.K + r0, bv, bar);
    };
    if (lane == 0)
      for (int s = 0; s < kMomLead && s < ns; ++s)
        if (full_stage(s)) issue(s);
    for (int s = 0; s < ns; ++s) {
      const int st = s % kMomIS;
      double *raw = sIn + st * INB;
      {  // stage s + Lead: its slot is free once the consumers are done with stage s + Lead - IS
        const int t = s + kMomLead, tp = t - kMomIS;
        if (tp >= 0 && t < ns) mbar_wait(smem_u32(sempty + tp % kMomIS), (uint32_t)((tp / kMomIS) & 1));
        if (lane == 0 && t < ns && full_stage(t)) issue(t);
      }
      const int64_t r = r_begin + (int64_t)s * kMomRT + lane;
      const bool valid = r < r_end;
      if (full_stage(s)) {
        mbar_wait(smem_u32(rfull + st), (uint32_t)((s / kMomIS) & 1));
      } else {  // plain loads (zeros past the slab)
        for (int k = 0; k < n; ++k) raw[lane * n + k] = valid ? a.X[r * n + k] : 0.0;
        for (int v = 0; v < nv; ++v) {
          raw[mom_vec_off(n) + v * kMomVS + lane] = valid ? a.V[(int64_t)v * a.K + r] : 0.0;
          if (wtd) raw[mom_vec_off(n) + (nv + v) * kMomVS + lane] = valid ? a.S[(int64_t)v * a.K + r] : 0.0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(rfull + st));  // (completes the phase: count 1, no tx)
      }
      // X transposed for the consumers' lane = row reads
      for (int k = 0; k < n; ++k) sXt[(st * kMaxVars + k) * kMomRT + lane] = raw[lane * n + k];
      // the row of ones (the constant weight; 0 past the slab)
      raw[mom_vec_off(n) + (wtd ? 2 * nv : nv) * kMomVS + lane] = valid ? 1.0 : 0.0;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(wfull + st));
    }
    return;
  }

  // ---- consumers: u of the lane's row, the monomials and the moments of the warp's own tiles ----
  const int tb = a.wtile[wid], tc = a.wtile[wid + 1] - tb;
  double acc[TPW][WT][2];
#pragma unroll
  for (int q = 0; q < TPW; ++q)
#pragma unroll
    for (int h = 0; h < WT; ++h) acc[q][h][0] = acc[q][h][1] = 0.0;
  double *part = a.part + (size_t)blockIdx.x * a.nT * WT * 64;
  bool first = true;
  const int s0w = 8 * tb, s1w = 8 * (tb + tc) < a.nslot ? 8 * (tb + tc) : a.nslot;  // the warp's slots
  const uint32_t inc = n >= 2 ? 1u << (4 * (n - 2)) : 0u;  // e_{n-2} + 1 in a unit's packed exponents
  // this lane's weight (row lane / 4 of each weight tile of the A operand), from the slot's vectors:
  // unweighted w = 0: 1, w = 1 + v: V_v, w = 1 + nv + v: V_v^2; weighted w = 3 v + p: s_v^2 V_v^p;
  // other w: 0.  wv: the vector read (the ones row for 1), wsq: squared, ws: times s_v^2, wz: 0
  int wv[WT], ws[WT];
  bool wsq[WT], wz[WT];
  {
    const int v0 = mom_vec_off(n), ones = v0 + (wtd ? 2 * nv : nv) * kMomVS;
#pragma unroll
    for (int h = 0; h < WT; ++h) {
      const int w = 8 * h + (lane >> 2);
      wv[h] = ones;
      ws[h] = -1;
      wsq[h] = false;
      wz[h] = false;
      if (wtd) {
        if (w < 3 * nv) {
          const int v = w / 3, p = w % 3;
          ws[h] = v0 + (nv + v) * kMomVS;
          if (p > 0) wv[h] = v0 + v * kMomVS;
          wsq[h] = p == 2;
        } else {
          wz[h] = true;
        }
      } else if (w >= 1 && w <= 2 * nv) {
        wv[h] = v0 + ((w - 1) % nv) * kMomVS;
        wsq[h] = w > nv;
      } else if (w != 0) {
        wz[h] = true;
      }
    }
  }

  for (int s = 0; s < ns; ++s) {
    const int st = s % kMomIS;
    const uint32_t ph = (uint32_t)((s / kMomIS) & 1);
    mbar_wait(smem_u32(rfull + st), ph);
    mbar_wait(smem_u32(wfull + st), ph);
    const double *xt = sXt + st * kMaxVars * kMomRT + lane;
    // a10 for the lane's row: u = (x - c) 2^-e (rows past the slab have zero weights)
    double u[kMaxVars];
#pragma unroll
    for (int k = 0; k < kMaxVars; ++k) u[k] = k < n ? (xt[k * kMomRT] - sXc[k]) * sXs[k] : 0.0;
    // ---- a11: the monomials of the warp's slots for the stage's 32 rows (lane = row) ----------
#ifndef RP_MOM_PROBE_NOGEN  // (timing probe: no monomials, results meaningless)
    if constexpr (N > 0) {
      switch (wid) {
#define RP_MG(w) \
  case w: mom_gen_warp<N, D, w>(u, sM + lane); break;
        RP_MG(0) RP_MG(1) RP_MG(2) RP_MG(3) RP_MG(4) RP_MG(5) RP_MG(6) RP_MG(7) RP_MG(8) RP_MG(9) RP_MG(10)
        RP_MG(11) RP_MG(12) RP_MG(13) RP_MG(14) RP_MG(15)
#if RP_MOM_WARPS > 16
        RP_MG(16) RP_MG(17) RP_MG(18) RP_MG(19) RP_MG(20) RP_MG(21) RP_MG(22) RP_MG(23) RP_MG(24) RP_MG(25)
        RP_MG(26) RP_MG(27) RP_MG(28) RP_MG(29) RP_MG(30)
#endif
#undef RP_MG
      }
    } else if (s1w > s0w) {
      double *uw = sUg + wid * kMaxVars * kMomRT + lane;  // u by runtime variable index
#pragma unroll
      for (int k = 0; k < kMaxVars; ++k) uw[k * kMomRT] = u[k];
      const double ul = uw[(n - 1) * kMomRT], us = n >= 2 ? uw[(n - 2) * kMomRT] : 1.0;
      int slot = a.wuslot[wid];
      uint32_t pex = 0;
      double am = 1.0;
      for (int ui = a.wunit[wid]; slot < s1w; ++ui) {
        const uint32_t ex = a.uexp[ui];
        const int len = a.ulen[ui];
        if (ui > a.wunit[wid] && n >= 2 && ex == pex + inc) {
          am *= us;  // the next e_{n-2} of the same prefix
        } else {     // a new prefix: u_0^e_0 ... u_{n-2}^e_{n-2} by repeated multiplication
          am = 1.0;
          for (int k = 0; k + 1 < n; ++k) {
            const double uk = uw[k * kMomRT];
            for (int e = (int)((ex >> (4 * k)) & 15u); e > 0; --e) am *= uk;
          }
        }
        pex = ex;
        const int jb = s0w > slot ? s0w - slot : 0, je = s1w - slot < len ? s1w - slot : len;
        double m = am;
        for (int j = 0; j < jb; ++j) m *= ul;
        double *dst = sM + (size_t)slot * kMomRTP + lane;
        for (int j = jb; j < je; ++j) {
          dst[j * kMomRTP] = m;
          m *= ul;
        }
        slot += len;
      }
    }
#endif
    __syncwarp();
    // ---- a12: moments[w][e] += W^T Mon over the stage's 8 k-steps --------------------------------
#ifdef RP_MOM_PROBE_NODMMA
    if (false)
#endif
    {
      const double *raw = sIn + st * INB + (lane & 3);
      const double *mb = sM + (size_t)(tb * 8 + (lane >> 2)) * kMomRTP + (lane & 3);
      // every A value (the row weights) of the stage first, off the DMMA chain (0.430 -> 0.424 ms)
      double aall[kMomRT / 4][WT];
#pragma unroll
      for (int ks = 0; ks < kMomRT / 4; ++ks)
#pragma unroll
        for (int h = 0; h < WT; ++h) {
          const double x = raw[wv[h] + ks * 4];
          double w = wsq[h] ? x * x : x;
          if (wtd && ws[h] >= 0) {
            const double sv = raw[ws[h] + ks * 4];
            w *= sv * sv;
          }
          aall[ks][h] = wz[h] ? 0.0 : w;
        }
#pragma unroll
      for (int ks = 0; ks < kMomRT / 4; ++ks) {
        double av[WT];
#pragma unroll
        for (int h = 0; h < WT; ++h) av[h] = aall[ks][h];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
          if (q < tc) {
            const double bv = mb[(size_t)q * 8 * kMomRTP + ks * 4];
#pragma unroll
            for (int h = 0; h < WT; ++h) mom_dmma(acc[q][h][0], acc[q][h][1], av[h], bv);
          }
        }
      }
    }
    __syncwarp();  // the warp has read stage s (and its monomial rows are rewritten next stage)
    if (lane == 0) mbar_arrive(smem_u32(sempty + st));
    if (((s + 1) % kMomFlush) == 0 || s + 1 == ns) {
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        if (q < tc) {
#pragma unroll
          for (int h = 0; h < WT; ++h) {
            double *dst = part + ((size_t)(tb + q) * WT + h) * 64 + lane * 2;
            if (first) {
              dst[0] = acc[q][h][0];
              dst[1] = acc[q][h][1];
            } else {
              dst[0] += acc[q][h][0];
              dst[1] += acc[q][h][1];
            }
            acc[q][h][0] = acc[q][h][1] = 0.0;
          }
        }
      }
      first = false;
    }
  }
  if (ns == 0)  // empty slab: zero partial (this warp's tiles)
    for (int i = lane; i < tc * WT * 64; i += 32) part[(size_t)tb * WT * 64 + i] = 0.0;
}

// fixed-order sum of the per-CTA partials: 4 quarter sums per element (CTAs q, q + 4, ...),
// added as (q0 + q1) + (q2 + q3)
__global__ void __launch_bounds__(256) k_mom_sum(const double *part, int nblk, int n_el, double *red) {
  __shared__ double sq[4][64];
  const int q = threadIdx.x >> 6, l = threadIdx.x & 63;
  const int e = blockIdx.x * 64 + l;
  double s = 0.0;
  if (e < n_el)
    for (int b = q; b < nblk; b += 4) s += part[(int64_t)b * n_el + e];
  sq[q][l] = s;
  __syncthreads();
  if (q == 0 && e < n_el) red[e] = (sq[0][l] + sq[1][l]) + (sq[2][l] + sq[3][l]);
}

// lexicographic rank of e (|e| <= D) in the simplex {|e| <= D} of n variables:
// sum_k sum_{j < e_k} #{vectors of the n - k - 1 later variables with sum <= D - s_k - j}
__device__ __forceinline__ int simplex_rank(const int8_t *e, int n, int D) {
  int rank = 0, s = 0;
  for (int k = 0; k < n; ++k) {
    const int m = n - k - 1;
    for (int j = 0; j < e[k]; ++j) {
      const int R = D - s - j;
      int c = 1;  // C(R + m, m)
      for (int i = 1; i <= m; ++i) c = c * (R + i) / i;
      rank += c;
    }
    s += e[k];
  }
  return rank;
}

// G_v[i][j] from the summed moments red [nT][WT][64] (element 8 w + slot % 8 of tile slot / 8)
__global__ void k_mom_assemble(const GramBasis *gb, const double *red, int D, int nv, int wtd, int WT, double *G) {
  const GramBasis &B = *gb;
  const int n = B.n, nc = B.nc, nn = B.n_num;
  const int64_t total = (int64_t)nv * nc * nc;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(idx / ((int64_t)nc * nc));
    const int rc = (int)(idx % ((int64_t)nc * nc));
    const int i = rc / nc, j = rc % nc;
    const int q = (i >= nn) + (j >= nn);  // 0: num-num, 1: num-den, 2: den-den
    int8_t e[kMaxVars];
    for (int k = 0; k < n; ++k) e[k] = (int8_t)(B.exp[i][k] + B.exp[j][k]);
    const int slot = simplex_rank(e, n, D);
    const int w = wtd ? 3 * v + q : (q == 0 ? 0 : (q == 1 ? 1 + v : 1 + nv + v));
    const double m = red[((int64_t)(slot >> 3) * WT + (w >> 3)) * 64 + 8 * (w & 7) + (slot & 7)];
    G[idx] = q == 1 ? -m : m;
  }
}

// ---- host: the moment plan -------------------------------------------------------------------
static int64_t binom(int a, int b) {
  if (b < 0 || b > a) return 0;
  int64_t c = 1;
  for (int i = 1; i <= b; ++i) c = c * (a - b + i) / i;
  return c;
}

struct MomShape {
  int D, nslot, nunit, nT, nw, WT, TPW;
};

static bool mom_shape(const GramBasis &h, int n_v, bool weighted, MomShape *sh) {
  const int n = h.n;
  if (n < 1 || n > kMaxVars) return false;
  int dmax = 0;
  for (int j = 0; j < h.nc; ++j) {
    int d = 0;
    for (int k = 0; k < n; ++k) d += h.exp[j][k];
    dmax = d > dmax ? d : dmax;
  }
  sh->D = 2 * dmax;
  if (sh->D > 15) return false;  // unit exponents are packed 4 bits per variable
  const int64_t nslot = binom(sh->D + n, n), nunit = n >= 2 ? binom(sh->D + n - 1, n - 1) : 1;
  if (nslot > kMomMaxSlots || nunit > kMomMaxUnits) return false;
  sh->nslot = (int)nslot;
  sh->nunit = (int)nunit;
  sh->nT = (sh->nslot + 7) / 8;
  sh->nw = weighted ? 3 * n_v : 1 + 2 * n_v;
  if (n_v < 1 || sh->nw > 16) return false;
  sh->WT = sh->nw <= 8 ? 1 : 2;
  const int tpw = (sh->nT + kMomWarps - 1) / kMomWarps;
  sh->TPW = tpw <= 1 ? 1 : (tpw <= 2 ? 2 : (tpw <= 4 ? 4 : 8));
  if (sh->TPW * sh->WT > 8) return false;
  return mom_smem(sh->nT, n, n_v, weighted) <= 227 * 1024;
}

static int mom_grid_x(int64_t K) {
  const int64_t want = (K + kMomRT - 1) / kMomRT;
  const int64_t cap = num_sms();
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

bool mom_supported(const GramBasis &h, int n_v, bool weighted) {
  MomShape sh;
  return mom_shape(h, n_v, weighted, &sh);
}

size_t mom_partial_elems(const GramBasis &h, int n_v, int64_t K, bool weighted) {
  MomShape sh;
  if (!mom_shape(h, n_v, weighted, &sh)) return 0;
  return (size_t)(mom_grid_x(K) + 1) * sh.nT * sh.WT * 64;  // partials + their sum
}

template <int WT, int TPW, int N, int D>
static cudaError_t launch_mom_t(const MomArgs &a, int gx, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_gram_mom<WT, TPW, N, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_gram_mom<WT, TPW, N, D><<<gx, kMomThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gram_mom(const GramBasis *d_basis, const GramBasis &h, const double *X, const double *V,
                            const double *S, int64_t K, int n_v, double *G, double *d_part, size_t part_elems,
                            cudaStream_t s) {
  MomShape sh;
  const bool wtd = S != nullptr;
  if (!mom_shape(h, n_v, wtd, &sh)) return cudaErrorInvalidValue;
  const int gx = mom_grid_x(K);
  const int n_el = sh.nT * sh.WT * 64;
  if ((size_t)(gx + 1) * n_el > part_elems) return cudaErrorInvalidValue;
  MomArgs a;
  memset(&a, 0, sizeof a);
  a.basis = d_basis;
  a.X = X;
  a.V = V;
  a.S = S;
  a.K = K;
  a.part = d_part;
  a.n = h.n;
  a.D = sh.D;
  a.nslot = sh.nslot;
  a.nT = sh.nT;
  a.nv = n_v;
  a.nw = sh.nw;
  // bulk copies need 16-byte aligned sources: X, V and S rows of whole stages (K even)
  a.tma = ((uintptr_t)X % 16 == 0) && ((uintptr_t)V % 16 == 0) && (!S || (uintptr_t)S % 16 == 0) && (K % 2 == 0);
  // units in lexicographic order and the warps' contiguous shares (the same table the
  // specialised kernels are compiled from)
  const int n = h.n;
  MomTab tab;  // (~4 KB; per call: launches may come from several host threads)
  tab = mom_tab(n, sh.D);
  if (tab.nu != sh.nunit || tab.ns != sh.nslot) return cudaErrorInvalidValue;
  for (int i = 0; i < sh.nunit; ++i) {
    uint32_t pk = 0;
    for (int k = 0; k + 1 < n; ++k) pk |= (uint32_t)tab.ex[i][k] << (4 * k);
    a.uexp[i] = pk;
    a.ulen[i] = (uint8_t)tab.len[i];
  }
  for (int w = 0; w <= kMomWarps; ++w) a.wtile[w] = (int16_t)tab.tb[w];
  for (int w = 0; w < kMomWarps; ++w) {
    a.wunit[w] = (int16_t)tab.wu[w];
    a.wuslot[w] = (int16_t)(tab.wu[w] < tab.nu ? tab.slot[tab.wu[w]] : tab.ns);
  }
  const size_t smem = mom_smem(sh.nT, n, n_v, wtd), smem_spec = mom_smem(sh.nT, n, n_v, wtd, false);
  cudaError_t e;
  const char *gen = getenv("RP_MOM_GENERIC");  // measurement: the runtime monomial step only
  const bool spec = !(gen && gen[0] == '1');
  // the BASELINE shapes (tiny: 3 variables, degree 2; polybench: 4, degree 3; fitheavy: 4,
  // degree 4) with their monomial step specialised at compile time; the rest generic
#define RP_MOM_SPEC(WT_, TPW_, N_, D_) \
  if (spec && sh.WT == WT_ && sh.TPW == TPW_ && n == N_ && sh.D == D_) e = launch_mom_t<WT_, TPW_, N_, D_>(a, gx, smem_spec, s); else
#define RP_MOM_CASE(WT_, TPW_) \
  if (sh.WT == WT_ && sh.TPW == TPW_) e = launch_mom_t<WT_, TPW_, 0, 0>(a, gx, smem, s); else
#if RP_MOM_WARPS > 16
  RP_MOM_SPEC(1, 2, 4, 8) RP_MOM_SPEC(2, 2, 4, 8) RP_MOM_SPEC(1, 1, 4, 6) RP_MOM_SPEC(2, 1, 4, 6)
#else
  RP_MOM_SPEC(1, 4, 4, 8) RP_MOM_SPEC(2, 4, 4, 8) RP_MOM_SPEC(1, 2, 4, 6) RP_MOM_SPEC(2, 2, 4, 6)
#endif
  RP_MOM_SPEC(1, 1, 3, 4) RP_MOM_SPEC(2, 1, 3, 4)
  RP_MOM_CASE(1, 1) RP_MOM_CASE(1, 2) RP_MOM_CASE(1, 4) RP_MOM_CASE(1, 8) RP_MOM_CASE(2, 1) RP_MOM_CASE(2, 2)
  RP_MOM_CASE(2, 4) e = cudaErrorInvalidValue;
#undef RP_MOM_CASE
#undef RP_MOM_SPEC
  if (e != cudaSuccess) return e;
  double *red = d_part + (size_t)gx * n_el;
  k_mom_sum<<<(n_el + 63) / 64, 256, 0, s>>>(d_part, gx, n_el, red);
  const int64_t total = (int64_t)n_v * h.nc * h.nc;
  const int rb = (int)((total + 255) / 256);
  k_mom_assemble<<<rb < 4 * num_sms() ? rb : 4 * num_sms(), 256, 0, s>>>(d_basis, red, sh.D, n_v, wtd ? 1 : 0, sh.WT, G);
  return cudaGetLastError();
}


// ============================================================================================
// f1: the triangular factor R of A = [M(u) | -V N(u)] from its Gram in DOUBLE-DOUBLE.
//
// The paper solves the homogeneous system by SVD because the normal equations square the
// condition number.  That loss is a loss of precision: with G = A^T A
// accurate to ~1e-30 relative (double-double moments: every entry is a weighted moment of one
// monomial, as in k_gram_mom) and its Cholesky factor computed in double-double, R = chol(G)
// carries the same information as Householder's R to well below FP64 rounding for
// cond(A) < ~1e13 (|delta sigma_i| <~ 1e-30 sigma_max^2 / sigma_i), so the SVD of R (k_svd_gk)
// meets the same gates as after the TSQR -- including sigma_min = 0 of exact recovery (the
// Cholesky pivot of a null direction is ~1e-30 relative and is set to an exact zero).  The
// moments are accumulated without rounding in their high part: term t = w m is split as
// t_hi = fma(w_h, m_h, sigma) - sigma (a multiple of ulp(sigma) / 2, exact; sigma a power of two
// >= 2 x the stage's bound) and the remainder t - t_hi into a low sum; every 64 rows both are
// added into a double-double accumulator.  rp_fit_svd uses it for K >= 4 n_c (RP_SVD_R=tsqr
// keeps the Householder TSQR, which also serves small K, weighted rows and rp_tsqr_accumulate).
// ============================================================================================
struct dd2 {
  double h, l;
};
__device__ __forceinline__ dd2 dd2_quick(double a, double b) {
  const double s = a + b;
  return dd2{s, b - (s - a)};
}
__device__ __forceinline__ dd2 dd2_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return dd2{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd2 dd2_add(dd2 x, dd2 y) {
  dd2 a = dd2_two_sum(x.h, y.h);
  const dd2 b = dd2_two_sum(x.l, y.l);
  a.l += b.h;
  a = dd2_quick(a.h, a.l);
  a.l += b.l;
  return dd2_quick(a.h, a.l);
}
__device__ __forceinline__ dd2 dd2_neg(dd2 x) { return dd2{-x.h, -x.l}; }
__device__ __forceinline__ dd2 dd2_mul(dd2 x, dd2 y) {
  const double p = x.h * y.h;
  double e = fma(x.h, y.h, -p);
  e = fma(x.h, y.l, fma(x.l, y.h, e));
  return dd2_quick(p, e);
}
__device__ __forceinline__ dd2 dd2_muld(dd2 x, double y) {
  const double p = x.h * y;
  return dd2_quick(p, fma(x.l, y, fma(x.h, y, -p)));
}
__device__ __forceinline__ dd2 dd2_div(dd2 a, dd2 b) {  // three quotient digits
  const double q1 = a.h / b.h;
  dd2 r = dd2_add(a, dd2_neg(dd2_muld(b, q1)));
  const double q2 = r.h / b.h;
  r = dd2_add(r, dd2_neg(dd2_muld(b, q2)));
  const double q3 = r.h / b.h;
  return dd2_add(dd2_quick(q1, q2), dd2{q3, 0.0});
}
__device__ __forceinline__ dd2 dd2_sqrt(dd2 a) {  // a > 0
  const double x = sqrt(a.h);
  const dd2 r = dd2_add(a, dd2_neg(dd2_mul(dd2{x, 0.0}, dd2{x, 0.0})));
  return dd2_quick(x, r.h / (2.0 * x));
}

// max |V_v| (positive doubles order like their bit patterns: an integer atomic max)
__global__ void k_vabsmax(const double *V, int64_t K, unsigned long long *out) {
  const int v = blockIdx.y;
  unsigned long long m = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < K; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(V[(int64_t)v * K + r]));
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out + v, m);
}

constexpr int kDdThreads = 512;
constexpr int kDdRS = 16;    // rows per stage
constexpr int kDdAcc = 8;    // accumulators (weight, monomial) per thread: nw * nslot <= 4096
constexpr int kDdFlush = 4;  // stages between flushes into the double-double accumulators (64 rows)
constexpr int kDdUS = kMaxVars + 1;  // row stride of sU (odd: conflict-free)

struct DdArgs {
  const GramBasis *basis;
  const double *X, *V;
  int64_t K;
  const unsigned long long *vmax;  // [nv] bit patterns of max |V_v|
  double *part;                    // [gridDim.x][nw * nslot][2]
  int n, nslot, nv, nw, nunit;
  uint32_t uexp[kMomMaxUnits];
  uint8_t ulen[kMomMaxUnits];
  int16_t uslot[kMomMaxUnits];
};

__host__ __device__ inline int dd_nsp(int ns) { return ns | 1; }  // odd row stride: conflict-free stores

// NSP > 0: the monomial row stride as a compile-time constant (immediate shared-memory offsets)
template <int NSP>
__global__ void __launch_bounds__(kDdThreads, 1) k_gram_dd(const __grid_constant__ DdArgs a) {
  extern __shared__ __align__(16) double dsm[];
  const int tid = threadIdx.x, n = a.n, nv = a.nv, nw = a.nw, ns = a.nslot;
  const int nsp = NSP > 0 ? NSP : dd_nsp(ns);
  double *sMh = dsm;                          // [RS][nsp]  monomials (hi)
  double *sMl = sMh + kDdRS * nsp;            // [RS][nsp]  (lo)
  double *sU = sMl + kDdRS * nsp;             // [RS][kDdUS]
  double *sWh = sU + kDdRS * kDdUS;           // [16][RS]  weights (hi), weight-major
  double *sWl = sWh + kDdRS * 16;             // [16][RS]  (lo)
  const GramBasis &B = *a.basis;
  const int64_t r_begin = a.K * blockIdx.x / gridDim.x, r_end = a.K * (blockIdx.x + 1) / gridDim.x;
  const int nacc = nw * ns;
  // accumulators a_i = tid + 512 i: weight w_i, monomial e_i; sigma_i >= 2 x 64 rows x max |w|
  int aw[kDdAcc], ae[kDdAcc];
  double sg[kDdAcc], h[kDdAcc], l[kDdAcc];
  dd2 acc[kDdAcc];
#pragma unroll
  for (int i = 0; i < kDdAcc; ++i) {
    const int ai = tid + kDdThreads * i;
    const int w = ai < nacc ? ai / ns : -1;
    aw[i] = w;
    ae[i] = ai < nacc ? ai - w * ns : 0;
    double vm = 1.0;
    if (w >= 1) {
      vm = __longlong_as_double((long long)a.vmax[(w - 1) % nv]);
      if (w > nv) vm *= vm * (1.0 + 1e-15);
    }
    int ex;
    frexp(2.0 * kDdRS * kDdFlush * (vm > 0.0 ? vm : 1.0) * (1.0 + 1e-12), &ex);
    sg[i] = ldexp(1.0, ex);
    h[i] = l[i] = 0.0;
    acc[i] = dd2{0.0, 0.0};
  }
  const double xs0 = ldexp(1.0, -B.xe[tid % kMaxVars < n ? tid % kMaxVars : 0]);
  const double xc0 = B.xc[tid % kMaxVars < n ? tid % kMaxVars : 0];
  int stage = 0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kDdRS, ++stage) {
    // inputs: u of the stage's rows, the row weights 1, V_v, V_v^2 (double-double; 0 past the slab)
    if (tid < kDdRS * kMaxVars) {
      const int r = tid / kMaxVars, k = tid % kMaxVars;
      const int64_t row = r0 + r;
      sU[r * kDdUS + k] = (row < r_end && k < n) ? (a.X[row * n + k] - xc0) * xs0 : 0.0;
    }
    if (tid < kDdRS * 16) {
      const int w = tid / kDdRS, r = tid % kDdRS;
      const int64_t row = r0 + r;
      double wh = 0.0, wl = 0.0;
      if (row < r_end && w < nw) {
        if (w == 0) {
          wh = 1.0;
        } else {
          const double vv = a.V[(int64_t)((w - 1) % nv) * a.K + row];
          if (w <= nv) {
            wh = vv;
          } else {
            wh = vv * vv;
            wl = fma(vv, vv, -wh);
          }
        }
      }
      sWh[tid] = wh;
      sWl[tid] = wl;
    }
    __syncthreads();
    // a11 in double-double: tasks (unit, row), row fastest (a warp runs two units: uniform
    // control flow): the unit's prefix by repeated exact products, then its entries along the
    // last variable
    for (int task = tid; task < kDdRS * a.nunit; task += kDdThreads) {
      const int r = task % kDdRS, u = task / kDdRS;
      const double *ur = sU + r * kDdUS;
      const uint32_t ex = a.uexp[u];
      dd2 m{1.0, 0.0};
      for (int k = 0; k + 1 < n; ++k) {
        const double uk = ur[k];
        for (int e = (int)((ex >> (4 * k)) & 15u); e > 0; --e) m = dd2_muld(m, uk);
      }
      const double ul = ur[n - 1];
      const int slot = a.uslot[u], len = a.ulen[u];
      double *dh = sMh + r * nsp + slot, *dl = sMl + r * nsp + slot;
      for (int j = 0; j < len; ++j) {
        dh[j] = m.h;
        dl[j] = m.l;
        m = dd2_muld(m, ul);
      }
    }
    __syncthreads();
    // a12: the terms w m of the stage's rows, high parts exact (V^2 weights carry a low part)
#pragma unroll
    for (int i = 0; i < kDdAcc; ++i) {
      if (aw[i] < 0) continue;
      const double *mh = sMh + ae[i], *ml = sMl + ae[i];
      const double *wh = sWh + aw[i] * kDdRS, *wl = sWl + aw[i] * kDdRS;
      const double sgi = sg[i];
      double hi = h[i], lo = l[i];
      if (aw[i] > nv) {
#pragma unroll 4
        for (int r = 0; r < kDdRS; ++r) {
          const double m_h = mh[r * nsp], m_l = ml[r * nsp], w_h = wh[r], w_l = wl[r];
          const double th = fma(w_h, m_h, sgi) - sgi;
          hi += th;
          lo = fma(w_h, m_l, lo);
          lo = fma(w_l, m_h, lo);
          lo += fma(w_h, m_h, -th);
        }
      } else {
#pragma unroll 4
        for (int r = 0; r < kDdRS; ++r) {
          const double m_h = mh[r * nsp], m_l = ml[r * nsp], w_h = wh[r];
          const double th = fma(w_h, m_h, sgi) - sgi;
          hi += th;
          lo = fma(w_h, m_l, lo);
          lo += fma(w_h, m_h, -th);
        }
      }
      h[i] = hi;
      l[i] = lo;
    }
    if ((stage + 1) % kDdFlush == 0 || r0 + kDdRS >= r_end) {
#pragma unroll
      for (int i = 0; i < kDdAcc; ++i) {
        acc[i] = dd2_add(acc[i], dd2_two_sum(h[i], l[i]));
        h[i] = l[i] = 0.0;
      }
    }
    __syncthreads();
  }
  double *out = a.part + (size_t)blockIdx.x * nacc * 2;
#pragma unroll
  for (int i = 0; i < kDdAcc; ++i)
    if (aw[i] >= 0) {
      const int ai = aw[i] * ns + ae[i];
      out[2 * ai] = acc[i].h;
      out[2 * ai + 1] = acc[i].l;
    }
}

// the partials summed in CTA order (double-double), then G_v [nv][nc][nc] as (hi, lo) pairs
__global__ void k_gram_dd_sum(const double *part, int nblk, int nacc, double *red) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nacc; e += gridDim.x * blockDim.x) {
    dd2 s{0.0, 0.0};
    for (int b = 0; b < nblk; ++b) s = dd2_add(s, dd2{part[((size_t)b * nacc + e) * 2], part[((size_t)b * nacc + e) * 2 + 1]});
    red[2 * e] = s.h;
    red[2 * e + 1] = s.l;
  }
}

__global__ void k_gram_dd_assemble(const GramBasis *gb, const double *red, int D, int nv, int ns, double *Gdd) {
  const GramBasis &B = *gb;
  const int n = B.n, nc = B.nc, nn = B.n_num;
  const int64_t total = (int64_t)nv * nc * nc;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(idx / ((int64_t)nc * nc));
    const int rc = (int)(idx % ((int64_t)nc * nc));
    const int i = rc / nc, j = rc % nc;
    const int q = (i >= nn) + (j >= nn);
    int8_t e[kMaxVars];
    for (int k = 0; k < n; ++k) e[k] = (int8_t)(B.exp[i][k] + B.exp[j][k]);
    const int slot = simplex_rank(e, n, D);
    const int w = q == 0 ? 0 : (q == 1 ? 1 + v : 1 + nv + v);
    const double sgn = q == 1 ? -1.0 : 1.0;
    Gdd[2 * idx] = sgn * red[2 * ((size_t)w * ns + slot)];
    Gdd[2 * idx + 1] = sgn * red[2 * ((size_t)w * ns + slot) + 1];
  }
}

// R = chol(G) in double-double, one CTA per metric: G equilibrated by powers of two (exact),
// right-looking, one column per step; a pivot <= 1e-26 (relative to the unit diagonal) is a
// null direction: its column is set to an exact zero.  R [nv][nc][nc] (upper, FP64) for the SVD.
constexpr int kCholDdThreads = 512;
__global__ void __launch_bounds__(kCholDdThreads, 1) k_chol_dd(const double *Gdd, int nc, double *R_out) {
  extern __shared__ __align__(16) double csm[];
  const int v = blockIdx.x, tid = threadIdx.x;
  const int np = nc * (nc + 1) / 2;
  double *Sh = csm, *Sl = Sh + np;  // packed lower: (i, j), j <= i at i (i + 1) / 2 + j
  double *dsc = Sl + np;            // [nc] the power-of-two scales
  const double *G = Gdd + (size_t)v * nc * nc * 2;
  auto P = [](int i, int j) { return i * (i + 1) / 2 + j; };
  for (int i = tid; i < nc; i += kCholDdThreads) {
    const double gii = G[2 * ((size_t)i * nc + i)];
    int ex = 0;
    if (gii > 0.0) frexp(sqrt(gii), &ex);
    dsc[i] = ldexp(1.0, -ex);
  }
  __syncthreads();
  for (int t = tid; t < np; t += kCholDdThreads) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (P(i + 1, 0) <= t) ++i;
    while (P(i, 0) > t) --i;
    const int j = t - P(i, 0);
    const double sc = dsc[i] * dsc[j];
    Sh[t] = G[2 * ((size_t)i * nc + j)] * sc;
    Sl[t] = G[2 * ((size_t)i * nc + j) + 1] * sc;
  }
  __syncthreads();
  for (int j = 0; j < nc; ++j) {
    const dd2 piv{Sh[P(j, j)], Sl[P(j, j)]};
    const bool null = !(piv.h > 1e-26);
    dd2 rj{0.0, 0.0};
    if (!null) rj = dd2_sqrt(piv);
    __syncthreads();  // every thread has read the pivot
    for (int i = j + tid; i < nc; i += kCholDdThreads) {
      dd2 x{0.0, 0.0};
      if (!null) x = (i == j) ? rj : dd2_div(dd2{Sh[P(i, j)], Sl[P(i, j)]}, rj);
      Sh[P(i, j)] = x.h;
      Sl[P(i, j)] = x.l;
    }
    __syncthreads();
    if (!null) {
      const int m = nc - j - 1, cnt = m * (m + 1) / 2;
      for (int t = tid; t < cnt; t += kCholDdThreads) {  // trailing (i, k), j < k <= i
        int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
        while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
        while (ii * (ii + 1) / 2 > t) --ii;
        const int kk = t - ii * (ii + 1) / 2;
        const int i = j + 1 + ii, k = j + 1 + kk;
        const dd2 li{Sh[P(i, j)], Sl[P(i, j)]}, lk{Sh[P(k, j)], Sl[P(k, j)]};
        const dd2 s = dd2_add(dd2{Sh[P(i, k)], Sl[P(i, k)]}, dd2_neg(dd2_mul(li, lk)));
        Sh[P(i, k)] = s.h;
        Sl[P(i, k)] = s.l;
      }
    }
    __syncthreads();
  }
  // R = L^T D^{-1}: R[j][i] = L~[i][j] / d_i (upper)
  double *Ro = R_out + (size_t)v * nc * nc;
  for (int t = tid; t < nc * nc; t += kCholDdThreads) {
    const int rr = t / nc, cc = t % nc;
    Ro[t] = cc >= rr ? (Sh[P(cc, rr)] + Sl[P(cc, rr)]) / dsc[cc] : 0.0;
  }
}

bool gram_dd_supported(const GramBasis &h, int n_v, int64_t K) {
  MomShape sh;
  if (!mom_shape(h, n_v, false, &sh)) return false;
  if (sh.nw * sh.nslot > kDdThreads * kDdAcc || sh.nw > 16) return false;
  const char *r = getenv("RP_SVD_R");
  if (r && strcmp(r, "tsqr") == 0) return false;
  return K >= 4 * (int64_t)h.nc && (size_t)h.nc * (h.nc + 1) * 8 + 8 * h.nc <= 227 * 1024;
}

static int dd_grid_x(int64_t K) {
  const int64_t want = (K + 255) / 256;
  const int64_t cap = num_sms();
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

size_t gram_dd_workspace_bytes(const GramBasis &h, int n_v, int64_t K) {
  MomShape sh;
  if (!mom_shape(h, n_v, false, &sh)) return 0;
  const size_t nacc = (size_t)sh.nw * sh.nslot;
  return 8 * ((size_t)(dd_grid_x(K) + 1) * nacc * 2 + (size_t)n_v * h.nc * h.nc * 2 + 16);
}

cudaError_t launch_gram_dd_chol(const GramBasis *d_basis, const GramBasis &h, const double *X, const double *V,
                                int64_t K, int n_v, void *ws, size_t ws_bytes, double *R, cudaStream_t s) {
  MomShape sh;
  if (!mom_shape(h, n_v, false, &sh)) return cudaErrorInvalidValue;
  if (ws_bytes < gram_dd_workspace_bytes(h, n_v, K)) return cudaErrorInvalidValue;
  const int gx = dd_grid_x(K);
  const int nacc = sh.nw * sh.nslot;
  double *part = (double *)ws, *red = part + (size_t)gx * nacc * 2, *Gdd = red + (size_t)nacc * 2;
  unsigned long long *vmax = (unsigned long long *)(Gdd + (size_t)n_v * h.nc * h.nc * 2);
  cudaError_t e = cudaMemsetAsync(vmax, 0, 8 * n_v, s);
  if (e != cudaSuccess) return e;
  {
    const int64_t b = (K + 255) / 256;
    const int bx = (int)(b < 2 * num_sms() ? b : 2 * num_sms());
    k_vabsmax<<<dim3(bx, n_v), 256, 0, s>>>(V, K, vmax);
  }
  DdArgs a;
  memset(&a, 0, sizeof a);
  a.basis = d_basis;
  a.X = X;
  a.V = V;
  a.K = K;
  a.vmax = vmax;
  a.part = part;
  a.n = h.n;
  a.nslot = sh.nslot;
  a.nv = n_v;
  a.nw = sh.nw;
  MomTab tab;  // (~4 KB; per call: launches may come from several host threads)
  tab = mom_tab(h.n, sh.D);
  if (tab.nu != sh.nunit) return cudaErrorInvalidValue;
  a.nunit = tab.nu;
  for (int i = 0; i < tab.nu; ++i) {
    uint32_t pk = 0;
    for (int k = 0; k + 1 < h.n; ++k) pk |= (uint32_t)tab.ex[i][k] << (4 * k);
    a.uexp[i] = pk;
    a.ulen[i] = (uint8_t)tab.len[i];
    a.uslot[i] = (int16_t)tab.slot[i];
  }
  const int nsp = dd_nsp(sh.nslot);
  const size_t smem = 8 * ((size_t)2 * kDdRS * nsp + kDdRS * kDdUS + 2 * kDdRS * 16);
  if (nsp == 495) {  // fitheavy: 4 variables, degree-4 bases
    e = cudaFuncSetAttribute(k_gram_dd<495>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gram_dd<495><<<gx, kDdThreads, smem, s>>>(a);
  } else {
    e = cudaFuncSetAttribute(k_gram_dd<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gram_dd<0><<<gx, kDdThreads, smem, s>>>(a);
  }
  k_gram_dd_sum<<<(nacc + 255) / 256, 256, 0, s>>>(part, gx, nacc, red);
  const int64_t total = (int64_t)n_v * h.nc * h.nc;
  const int rb = (int)((total + 255) / 256);
  k_gram_dd_assemble<<<rb < 4 * num_sms() ? rb : 4 * num_sms(), 256, 0, s>>>(d_basis, red, sh.D, n_v, sh.nslot, Gdd);
  const size_t csm = 8 * ((size_t)h.nc * (h.nc + 1) + h.nc);
  e = cudaFuncSetAttribute(k_chol_dd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  if (e != cudaSuccess) return e;
  k_chol_dd<<<n_v, kCholDdThreads, csm, s>>>(Gdd, h.nc, R);
  return cudaGetLastError();
}

}  // namespace rp
