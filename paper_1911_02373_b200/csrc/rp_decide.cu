// rp_decide.cu -- NEXT row f2: the runtime decision service.
//
// The paper's driver program evaluates the rational program before every kernel launch and
// returns the launch parameters, keeps "a runtime history to
// instantly provide results for future kernel launches", and may refine
// near-optimal choices "up to some margin" with "a secondary performance metric"
// (PAPER.md:2299-2305).  k_decide makes one decision per data tuple (one CTA each): probe the
// history, stage the data polynomials, evaluate E for every statically feasible configuration
// (same arithmetic as k_sweep: scalar dot products instead of DMMA tiles, the same E code),
// argmin on (E, index), tie-break within the margin by (W_active desc, P1 desc, P2 asc, P3 asc,
// index asc), compute the grid, insert into the history.
#include <cstdio>

#include "rp_device.cuh"
#include "rp_decide.cuh"

namespace rp {

__device__ __forceinline__ uint32_t hist_hash(const int32_t *key, int d) {
  uint32_t h = 2166136261u;  // FNV-1a over the bytes of the tuple
  for (int k = 0; k < d; ++k) {
    uint32_t v = (uint32_t)key[k];
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 255u;
      h *= 16777619u;
    }
  }
  return h;
}

__device__ bool hist_lookup(const HistTable &H, const int32_t *key, int d, rp_decision *out) {
  const uint32_t h = hist_hash(key, d);
  for (int probe = 0; probe < kHistProbes; ++probe) {
    HistSlot *sl = H.slots + ((h + probe) & H.mask);
    const uint32_t st = *((volatile uint32_t *)&sl->state);
    if (st == 0) return false;  // empty slot ends the probe sequence
    if (st != 2) continue;      // being written
    __threadfence();
    bool eq = true;
    for (int k = 0; k < d; ++k) eq = eq && (((volatile int32_t *)sl->key)[k] == key[k]);
    if (eq) {
      *out = sl->val;
      return true;
    }
  }
  return false;
}

__device__ void hist_insert(const HistTable &H, const int32_t *key, int d, const rp_decision &v) {
  const uint32_t h = hist_hash(key, d);
  for (int probe = 0; probe < kHistProbes; ++probe) {
    HistSlot *sl = H.slots + ((h + probe) & H.mask);
    uint32_t st = atomicCAS(&sl->state, 0u, 1u);
    while (st == 1) {  // another CTA is publishing this slot (it never waits): wait, then compare
      __nanosleep(32);
      st = *((volatile uint32_t *)&sl->state);
    }
    if (st == 0) {  // claimed: write, publish
      for (int k = 0; k < d; ++k) sl->key[k] = key[k];
      sl->val = v;
      __threadfence();
      atomicExch(&sl->state, 2u);
      atomicAdd(H.counters + 2, 1ull);
      return;
    }
    if (st == 2) {
      __threadfence();
      bool eq = true;
      for (int k = 0; k < d; ++k) eq = eq && (((volatile int32_t *)sl->key)[k] == key[k]);
      if (eq) return;  // already recorded (a concurrent decision for the same tuple)
    }
  }
}

// secondary order of the tie-break: larger W_active, larger P1, smaller P2, smaller P3, lower
// original index (reading R28)
__device__ __forceinline__ bool sec_better(const CfgRec &a, const CfgRec &b) {
  if (a.W != b.W) return a.W > b.W;
  if (a.Pm1_0 != b.Pm1_0) return a.Pm1_0 > b.Pm1_0;
  if (a.Pm1_1 != b.Pm1_1) return a.Pm1_1 < b.Pm1_1;
  if (a.Pm1_2 != b.Pm1_2) return a.Pm1_2 < b.Pm1_2;
  return a.orig < b.orig;
}

constexpr int kDecideThreads = 256;

template <int NPE, bool MWP>
__global__ void __launch_bounds__(kDecideThreads) k_decide(DecideArgs a) {
  constexpr int NPOLY = MWP ? 6 : 2;
  constexpr double kInf = __builtin_huge_val();
  const int g = a.prog;
  const DevProg &pg = a.progs[g];
  const int d = pg.d, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t ti = blockIdx.x;
  extern __shared__ __align__(16) double sE[];  // [nFc] estimates
  __shared__ int32_t sD[kMaxVars];
  __shared__ double sMD[kMaxDE];
  __shared__ double sC[NPOLY * NPE];
  __shared__ int s_hit;
  __shared__ double s_e[kDecideThreads / 32];
  __shared__ int s_c[kDecideThreads / 32];

  if (tid < d) sD[tid] = a.D[ti * d + tid];
  if (tid == 0) s_hit = 0;
  __syncthreads();
  if (a.hist.enabled && tid == 0) {
    rp_decision v;
    if (hist_lookup(a.hist, sD, d, &v)) {
      v.from_history = 1;
      a.out[ti] = v;
      s_hit = 1;
      atomicAdd(a.hist.counters + 0, 1ull);
    }
  }
  __syncthreads();
  if (s_hit) return;

  // a2: data monomials and staged data polynomials C[k NPE + pe] = sum_de Cmat m_de(u_D)
  const int nDE = pg.nDE, ndp = a.tab.nde_pad;
  for (int de = tid; de < ndp; de += blockDim.x) {
    double m = 0.0;
    if (de < nDE) {
      m = 1.0;
      for (int k = 0; k < d; ++k) {
        const double u = ((double)sD[k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
        for (int e = 0; e < pg.de_exp[de][k]; ++e) m *= u;
      }
    }
    sMD[de] = m;
  }
  __syncthreads();
  const double *Cm = a.tab.Cmat + (int64_t)g * kMaxPolys * NPE * ndp;
  for (int r = tid; r < NPOLY * NPE; r += blockDim.x) {
    double acc = 0.0;
    for (int de = 0; de < ndp; ++de) acc = fma(Cm[(int64_t)r * ndp + de], sMD[de], acc);
    sC[r] = acc;
  }
  __syncthreads();

  const int nFc = a.tab.nFc[2 * g];
  const int nFp = a.tab.nFp;
  const CfgRec *rec = a.tab.rec + (int64_t)g * nFp;
  const double *mP = a.tab.mP + (int64_t)g * a.npe_pad * nFp;
  const EConst kc = make_econst(pg);
  const int map0 = pg.grid_map[0], map1 = pg.p >= 2 ? pg.grid_map[1] : -1,
            map2 = pg.p >= 3 ? pg.grid_map[2] : -1;
  bool dpos = true;  // reading R32: data parameters are sizes >= 1
  for (int k = 0; k < d; ++k) dpos = dpos && sD[k] >= 1;
  // (a masked tuple's grid is computed from 1s so that no table index goes out of range)
  const int32_t Da = map0 >= 0 && dpos ? sD[map0] : 1, Db = map1 >= 0 && dpos ? sD[map1] : 1,
                Dc = map2 >= 0 && dpos ? sD[map2] : 1;
  const int64_t D1sq = (int64_t)sD[0] * sD[0];
  const int n_sm = pg.n_sm;
  const double *gRSM = a.tab.rSM + (int64_t)g * kRSMTab;

  // a4-a8 per configuration: E into shared memory, running argmin on (E, original index)
  double be = kInf;
  int bc = -1, bo = 0x7fffffff;
  for (int c = tid; c < nFc; c += blockDim.x) {
    const CfgRec cr = rec[c];
    double pk[NPOLY];
#pragma unroll
    for (int k = 0; k < NPOLY; ++k) {
      double acc = 0.0;
#pragma unroll 4
      for (int pe = 0; pe < NPE; ++pe) acc = fma(sC[k * NPE + pe], mP[(int64_t)pe * nFp + c], acc);
      pk[k] = acc;
    }
    double E;
    if constexpr (MWP) {
      const uint32_t s012 = cr.s012;
      int64_t blocks = 1;
      if (map0 >= 0) blocks *= ceil_div_magic(Da, cr.Pm1_0, cr.M0, s012 & 255);
      if (map1 >= 0) blocks *= ceil_div_magic(Db, cr.Pm1_1, cr.M1, (s012 >> 8) & 255);
      if (map2 >= 0) blocks *= ceil_div_magic(Dc, cr.Pm1_2, cr.M2, (s012 >> 16) & 255);
      const int64_t smact = blocks < n_sm ? blocks : n_sm;
      const double rSM = smact < kRSMTab ? gRSM[smact] : 1.0 / (double)smact;
      const double Rep = (double)blocks * cr.rB * rSM;
      E = mwpcwp_E(pk[0], pk[1], pk[2], pk[3], pk[4], pk[5], cr.W, Rep, rSM, (double)smact, kc);
    } else {
      E = pk[0] * frcp(pk[1]);
    }
    const bool ok = cr.P01 <= D1sq && dpos;
    E = (ok && E > 0.0 && E < kInf) ? E : kInf;
    sE[c] = E;
    if (E < kInf && (E < be || (E == be && cr.orig < bo))) {
      be = E;
      bc = c;
      bo = cr.orig;
    }
  }
  // block argmin
  for (int o = 16; o >= 1; o >>= 1) {
    const double e2 = __shfl_xor_sync(0xffffffffu, be, o);
    const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
    const int o2 = __shfl_xor_sync(0xffffffffu, bo, o);
    if (e2 < be || (e2 == be && o2 < bo)) {
      be = e2;
      bc = c2;
      bo = o2;
    }
  }
  if (lane == 0) {
    s_e[wid] = be;
    s_c[wid] = bc;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      const int c2 = s_c[w];
      if (c2 >= 0 && (s_e[w] < be || (s_e[w] == be && bc >= 0 && rec[c2].orig < rec[bc].orig))) {
        be = s_e[w];
        bc = c2;
      }
    }
    s_e[0] = be;
    s_c[0] = bc;
  }
  __syncthreads();
  be = s_e[0];
  int choice = s_c[0];
  // tie-break within the margin by the secondary order
  if (a.margin > 0.0 && choice >= 0) {
    const double lim = be * (1.0 + a.margin);
    int sc = -1;
    for (int c = tid; c < nFc; c += blockDim.x)
      if (sE[c] <= lim && (sc < 0 || sec_better(rec[c], rec[sc]))) sc = c;
    for (int o = 16; o >= 1; o >>= 1) {
      const int c2 = __shfl_xor_sync(0xffffffffu, sc, o);
      if (c2 >= 0 && (sc < 0 || sec_better(rec[c2], rec[sc]))) sc = c2;
    }
    __syncthreads();
    if (lane == 0) s_c[wid] = sc;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        const int c2 = s_c[w];
        if (c2 >= 0 && (sc < 0 || sec_better(rec[c2], rec[sc]))) sc = c2;
      }
      choice = sc;
    }
  }
  if (tid == 0) {
    rp_decision v;
    v.from_history = 0;
    v.pad[0] = v.pad[1] = 0;
    if (choice >= 0) {
      const CfgRec cr = rec[choice];
      v.idx = cr.orig;
      v.E = sE[choice];
      const uint32_t s012 = cr.s012;
      // grid rule gx = ceil[N / bx], 1 for an unmapped dimension
      v.launch[0] = map0 >= 0 ? (int32_t)ceil_div_magic(Da, cr.Pm1_0, cr.M0, s012 & 255) : 1;
      v.launch[1] = map1 >= 0 ? (int32_t)ceil_div_magic(Db, cr.Pm1_1, cr.M1, (s012 >> 8) & 255) : 1;
      v.launch[2] = map2 >= 0 ? (int32_t)ceil_div_magic(Dc, cr.Pm1_2, cr.M2, (s012 >> 16) & 255) : 1;
      v.launch[3] = cr.Pm1_0 + 1;
      v.launch[4] = cr.Pm1_1 + 1;
      v.launch[5] = cr.Pm1_2 + 1;
    } else {
      v.idx = -1;
      v.E = kInf;
      for (int k = 0; k < 6; ++k) v.launch[k] = 0;
    }
    a.out[ti] = v;
    if (a.hist.enabled) {
      atomicAdd(a.hist.counters + 1, 1ull);
      hist_insert(a.hist, sD, d, v);
    }
  }
}

template <int NPE>
static cudaError_t launch_decide_npe(const DecideArgs &a, bool mwp, int nFp, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)nFp;
  cudaError_t e;
  if (mwp) {
    e = cudaFuncSetAttribute(k_decide<NPE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_decide<NPE, true><<<(unsigned)a.n, kDecideThreads, smem, s>>>(a);
  } else {
    e = cudaFuncSetAttribute(k_decide<NPE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_decide<NPE, false><<<(unsigned)a.n, kDecideThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// ---- persistence of the runtime history (rp_plan_history_save / _load) ------------------------
// Export: the ready slots, compacted with their slot index (the host sorts by it: deterministic).
__global__ void k_hist_export(HistTable H, int d, int32_t *keys, rp_decision *vals, int32_t *slot_of,
                              unsigned *count) {
  const int64_t n = (int64_t)H.mask + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const HistSlot &sl = H.slots[i];
    if (sl.state != 2) continue;
    const unsigned j = atomicAdd(count, 1u);
    for (int k = 0; k < d; ++k) keys[(int64_t)j * d + k] = sl.key[k];
    vals[j] = sl.val;
    slot_of[j] = (int32_t)i;
  }
}

// Import: every entry goes through the decision kernel's own insertion (same hash, same probes),
// so rp_plan_decide finds it exactly where it would have put it
__global__ void k_hist_import(HistTable H, int d, const int32_t *keys, const rp_decision *vals, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    rp_decision v = vals[i];
    v.from_history = 0;
    hist_insert(H, keys + i * d, d, v);
  }
}

// FNV-1a 64 over device bytes, chained through *h (compile_program zeroes the device program
// first, and the refit kernel rewrites coefficients and transform in place): a saved history is
// bound to the program and the configuration set that made its decisions
__global__ void k_fnv64(const unsigned char *b, size_t n, unsigned long long *h) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long x = *h;
  for (size_t i = 0; i < n; ++i) {
    x ^= b[i];
    x *= 1099511628211ull;
  }
  *h = x;
}

cudaError_t launch_hist_export(const HistTable &H, int d, int32_t *keys, rp_decision *vals, int32_t *slot_of,
                               unsigned *count, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  const int64_t n = (int64_t)H.mask + 1;
  const int grid = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  k_hist_export<<<grid, 256, 0, s>>>(H, d, keys, vals, slot_of, count);
  return cudaGetLastError();
}

cudaError_t launch_hist_import(const HistTable &H, int d, const int32_t *keys, const rp_decision *vals, int64_t n,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)((n + 127) / 128 < 1024 ? (n + 127) / 128 : 1024);
  k_hist_import<<<grid, 128, 0, s>>>(H, d, keys, vals, n);
  return cudaGetLastError();
}

cudaError_t launch_fingerprint(const DevProg *pg, const int32_t *F, size_t f_bytes, unsigned long long *out,
                               cudaStream_t s) {
  const unsigned long long basis = 1469598103934665603ull;
  cudaError_t e = cudaMemcpyAsync(out, &basis, sizeof basis, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  k_fnv64<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned char *>(pg), sizeof(DevProg), out);
  k_fnv64<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned char *>(F), f_bytes, out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);  // (the pageable source of the async copy must outlive it)
}

cudaError_t launch_decide(const DecideArgs &a, bool mwp, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  if (a.n > 0x7fffffffll) return cudaErrorInvalidValue;
  const int nFp = a.tab.nFp;
  switch (a.npe_pad) {
    case 4: return launch_decide_npe<4>(a, mwp, nFp, s);
    case 8: return launch_decide_npe<8>(a, mwp, nFp, s);
    case 16: return launch_decide_npe<16>(a, mwp, nFp, s);
    case 20: return launch_decide_npe<20>(a, mwp, nFp, s);
    case 24: return launch_decide_npe<24>(a, mwp, nFp, s);
    case 36: return launch_decide_npe<36>(a, mwp, nFp, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rp
