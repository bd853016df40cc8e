// rp_gram.cu -- the compile-time least-squares fit's dense part, and small helpers.
//
// the coefficients alpha, beta of g = p/q are estimated by "linear least
// squares" on an "over-determined system of linear equations" whose rows are built "from the
// evaluation of monomial terms, resulting in essentially a Vandermonde matrix"
// (PAPER.md:2601-2603).  Row r of the linearised system p(x) - V q(x) = 0 is
// a_r = [M(u_r) | -V_r N(u_r)]; the normal equations need G = A^T A = sum_r a_r a_r^T.
//
// k_gram: one CTA per SM, 8 warps.  Each CTA owns a contiguous slab of rows, builds RT = 64
// design rows at a time in shared memory (never in HBM) and accumulates the upper-triangular
// 8x8 tiles of G with FP64 tensor-core mma.sync.m8n8k4 (SASS DMMA.8x8x4).  X / V tiles arrive
// in shared memory through the bulk-copy (TMA) engine: cp.async.bulk + mbarrier, double
// buffered, so the next slab streams in while the current one is multiplied.  Accuracy: the
// register accumulators are flushed into a shared-memory accumulator every kChunk rows
// (two-level summation), the per-CTA partials are summed in a fixed order by k_gram_reduce.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rp_internal.cuh"

namespace rp {

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ============================================================================================
// minmax (a10): per-column min / max of X [K][n]
// ============================================================================================
__global__ void k_minmax_part(const double *X, int64_t K, int n, double *part) {
  __shared__ double smin[32][kMaxVars], smax[32][kMaxVars];
  double lo[kMaxVars], hi[kMaxVars];
  for (int k = 0; k < kMaxVars; ++k) {
    lo[k] = __longlong_as_double(0x7ff0000000000000ll);
    hi[k] = -lo[k];
  }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < K;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < n; ++k) {
      const double x = X[r * n + k];
      lo[k] = fmin(lo[k], x);
      hi[k] = fmax(hi[k], x);
    }
  for (int k = 0; k < n; ++k)
    for (int o = 16; o >= 1; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
    for (int k = 0; k < n; ++k) {
      smin[wid][k] = lo[k];
      smax[wid][k] = hi[k];
    }
  __syncthreads();
  if (threadIdx.x < n) {
    const int k = threadIdx.x;
    double a = smin[0][k], b = smax[0][k];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      a = fmin(a, smin[w][k]);
      b = fmax(b, smax[w][k]);
    }
    part[((int64_t)blockIdx.x * n + k) * 2 + 0] = a;
    part[((int64_t)blockIdx.x * n + k) * 2 + 1] = b;
  }
}

// one CTA: every thread folds a strided subset of the partials (independent loads, not one
// dependent chain over nblk), then warp shuffles and a shared-memory pass
__global__ void k_minmax_final(const double *part, int nblk, int n, double *out) {
  __shared__ double smin[8][kMaxVars], smax[8][kMaxVars];
  double lo[kMaxVars], hi[kMaxVars];
  for (int k = 0; k < kMaxVars; ++k) {
    lo[k] = __longlong_as_double(0x7ff0000000000000ll);
    hi[k] = -lo[k];
  }
  for (int i = threadIdx.x; i < nblk; i += blockDim.x)
    for (int k = 0; k < n; ++k) {
      lo[k] = fmin(lo[k], part[((int64_t)i * n + k) * 2]);
      hi[k] = fmax(hi[k], part[((int64_t)i * n + k) * 2 + 1]);
    }
  for (int k = 0; k < n; ++k)
    for (int o = 16; o >= 1; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
    for (int k = 0; k < n; ++k) {
      smin[wid][k] = lo[k];
      smax[wid][k] = hi[k];
    }
  __syncthreads();
  if (threadIdx.x < n) {
    const int k = threadIdx.x;
    double a = smin[0][k], b = smax[0][k];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      a = fmin(a, smin[w][k]);
      b = fmax(b, smax[w][k]);
    }
    out[k * 2] = a;
    out[k * 2 + 1] = b;
  }
}

// a10: c_k = (lo_k + hi_k) / 2, e_k = least integer with 2^e_k >= max((hi_k - lo_k) / 2, 1)
// (reading R14).  lohi [n][2] -> out [n][2] = (c_k, (double)e_k).
__global__ void k_xform(const double *lohi, int n, double *out) {
  const int k = threadIdx.x;
  if (k >= n) return;
  const double lo = lohi[2 * k], hi = lohi[2 * k + 1];
  double h = (hi - lo) * 0.5;
  if (!(h >= 1.0)) h = 1.0;
  int e = 0;
  while (ldexp(1.0, e) < h) ++e;
  out[2 * k] = (lo + hi) * 0.5;
  out[2 * k + 1] = (double)e;
}

cudaError_t launch_xform(const double *d_lohi, int n, double *d_out, cudaStream_t s) {
  k_xform<<<1, 32, 0, s>>>(d_lohi, n, d_out);
  return cudaGetLastError();
}

// the transform of k_xform copied into the device-side GramBasis (c_k, e_k)
__global__ void k_xform_to_basis(const double *xf, int n, GramBasis *gb) {
  const int k = threadIdx.x;
  if (k >= n) return;
  gb->xc[k] = xf[2 * k];
  gb->xe[k] = (int32_t)xf[2 * k + 1];
}

cudaError_t launch_xform_to_basis(const double *d_xf, int n, GramBasis *d_gb, cudaStream_t s) {
  k_xform_to_basis<<<1, 32, 0, s>>>(d_xf, n, d_gb);
  return cudaGetLastError();
}

int minmax_blocks(int64_t K) {
  int64_t b = (K + 255) / 256;
  int64_t cap = 4LL * num_sms();
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

cudaError_t launch_minmax(const double *X, int64_t K, int n, double *d_part, int nblk,
                          double *d_out, cudaStream_t s) {
  k_minmax_part<<<nblk, 256, 0, s>>>(X, K, n, d_part);
  k_minmax_final<<<1, 256, 0, s>>>(d_part, nblk, n, d_out);
  return cudaGetLastError();
}

// ============================================================================================
// eval_metrics (a4 alone): out[i][r] = p_i(u_r) / q_i(u_r)
// ============================================================================================
__global__ void k_eval_metrics(const DevProg *pgp, int nm, const double *X, int64_t K,
                               double *out) {
  const DevProg &pg = *pgp;
  const int n = pg.d + pg.p;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < K;
       r += (int64_t)gridDim.x * blockDim.x) {
    double u[kMaxVars];
    for (int k = 0; k < n; ++k) u[k] = (X[r * n + k] - pg.xc[k]) * ldexp(1.0, -pg.xe[k]);
    double mD[kMaxDE];
    for (int de = 0; de < pg.nDE; ++de) {
      double m = 1.0;
      for (int k = 0; k < pg.d; ++k)
        for (int e = 0; e < pg.de_exp[de][k]; ++e) m *= u[k];
      mD[de] = m;
    }
    for (int i = 0; i < nm; ++i) {
      double pq[2];
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * i + h;
        double acc = 0.0;
        for (int pe = 0; pe < pg.nPE; ++pe) {
          const int row = k * pg.nPE + pe;
          double c = 0.0;
          for (int j = pg.row_start[row]; j < pg.row_start[row + 1]; ++j)
            c = fma(pg.term_coef[j], mD[pg.term_de[j]], c);
          double m = 1.0;
          for (int kk = 0; kk < pg.p; ++kk)
            for (int e = 0; e < pg.pe_exp[pe][kk]; ++e) m *= u[pg.d + kk];
          acc = fma(c, m, acc);
        }
        pq[h] = acc;
      }
      out[(int64_t)i * K + r] = pq[0] / pq[1];
    }
  }
}

cudaError_t launch_eval_metrics(const DevProg *d_prog, int nm, const double *X, int64_t K,
                                double *out, cudaStream_t s) {
  if (K == 0) return cudaSuccess;
  int64_t b = (K + 127) / 128;
  int cap = 8 * num_sms();
  k_eval_metrics<<<(int)(b > cap ? cap : b), 128, 0, s>>>(d_prog, nm, X, K, out);
  return cudaGetLastError();
}

// ============================================================================================
// Gram (a11 + a12)
// ============================================================================================
constexpr int kGramWarps = 8;
constexpr int kGramThreads = kGramWarps * 32;
constexpr int kRT = 64;             // design rows per smem tile (16 k-steps of 4)
constexpr int kMaxTilesPerWarp = 32;
constexpr int kTilesPerGroup = kGramWarps * kMaxTilesPerWarp;  // 256 upper tiles per CTA pass
constexpr int kChunkTiles = 8;      // flush register accumulators every 8 tiles (512 rows)

__host__ __device__ inline int gram_stride(int nb) {  // smem row stride (doubles), = 4 mod 16
  int s = nb * 8;
  while (s % 16 != 4) ++s;
  return s;
}

#ifdef RP_GRAM_DMMA_NV  // a pure function of its operands: the scheduler may move it
#define RP_GRAM_ASM asm
#else
#define RP_GRAM_ASM asm volatile
#endif
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  RP_GRAM_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine (SASS UBLKCP), completes on an mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct GramArgs {
  const GramBasis *basis;
  const double *X;
  const double *V;  // [n_v][K]
  const double *S;  // [n_v][K] row scales or null
  int64_t K;
  int n_v;
  int nb, ntiles, stride;
  double *part;     // [n_v][gridDim.y][gridDim.x][ntiles_in_group * 64] (tile-major)
};

// Shared memory layout (dynamic): sA [kRT][stride] | sAcc [kTilesPerGroup][64] |
// sX[2][kRT * 8] | sV[2][kRT] | sU[kRT * 8] | bars[2]
__global__ void __launch_bounds__(kGramThreads, 1) k_gram(GramArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const GramBasis &B = *a.basis;
  const int n = B.n, nc = B.nc, n_num = B.n_num;
  const int stride = a.stride;
  double *sA = (double *)smem_raw;
  double *sAcc = sA + kRT * stride;
  double *sX = sAcc + kTilesPerGroup * 64;
  double *sV = sX + 2 * kRT * kMaxVars;
  double *sU = sV + 2 * kRT;
  uint64_t *bars = (uint64_t *)(sU + kRT * kMaxVars);

  const int metric = blockIdx.z;
  const int group = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double *V = a.V + (int64_t)metric * a.K;

  // contiguous slab of rows for this CTA
  // (slab boundaries rounded to even rows so bulk copies of V stay 16-byte aligned)
  const int64_t r_begin = (a.K * blockIdx.x / gridDim.x) & ~1ll;
  const int64_t r_end =
      (blockIdx.x + 1 == gridDim.x) ? a.K : ((a.K * (blockIdx.x + 1) / gridDim.x) & ~1ll);

  // tiles of this warp: group tiles t_g = group * 256 + w + 8 * t, upper-triangular (bi <= bj)
  int toff[kMaxTilesPerWarp];  // (8*bi) | (8*bj) << 16, or -1
  {
    // enumerate upper tiles row-major: tile id -> (bi, bj)
#pragma unroll
    for (int t = 0; t < kMaxTilesPerWarp; ++t) {
      int id = group * kTilesPerGroup + wid + kGramWarps * t;
      toff[t] = -1;
      if (id < a.ntiles) {
        int bi = 0, rem = id;
        while (rem >= a.nb - bi) {
          rem -= a.nb - bi;
          ++bi;
        }
        const int bj = bi + rem;
        toff[t] = (8 * bi) | ((8 * bj) << 16);
      }
    }
  }
  for (int i = threadIdx.x; i < kTilesPerGroup * 64; i += blockDim.x) sAcc[i] = 0.0;
  // zero the pad columns of sA once (columns nc .. stride-1 stay zero)
  for (int i = threadIdx.x; i < kRT * stride; i += blockDim.x) sA[i] = 0.0;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nrows = r_end - r_begin;
  const int64_t ntile_rows = (nrows + kRT - 1) / kRT;
  // producer: one elected thread issues the bulk copies of X / V row tiles
  auto issue = [&](int64_t tr, int buf) {
    const int64_t r0 = r_begin + tr * kRT;
    const int64_t rows = (r_end - r0) < kRT ? (r_end - r0) : kRT;
    const unsigned bx = (unsigned)(rows * n * sizeof(double));
    const unsigned bv = (unsigned)(rows * sizeof(double));
    mbar_expect_tx(&bars[buf], bx + bv);
    bulk_g2s(sX + buf * kRT * kMaxVars, a.X + r0 * n, bx, &bars[buf]);
    bulk_g2s(sV + buf * kRT, V + r0, bv, &bars[buf]);
  };
  // bulk copies need 16-byte aligned sources and sizes: use them when the slab allows it
  const bool bulk_ok = ((((uintptr_t)(a.X + r_begin * n)) & 15) == 0) &&
                       ((((uintptr_t)(V + r_begin)) & 15) == 0) && ((kRT * n) % 2 == 0) &&
                       (nrows % 2 == 0);
  if (bulk_ok && threadIdx.x == 0 && ntile_rows > 0) issue(0, 0);

  double acc[kMaxTilesPerWarp][2];
#pragma unroll
  for (int t = 0; t < kMaxTilesPerWarp; ++t) acc[t][0] = acc[t][1] = 0.0;

  for (int64_t tr = 0; tr < ntile_rows; ++tr) {
    const int buf = (int)(tr & 1);
    const int64_t r0 = r_begin + tr * kRT;
    const int rows = (int)((r_end - r0) < kRT ? (r_end - r0) : kRT);
    const double *tX;
    const double *tV;
    if (bulk_ok) {
      if (threadIdx.x == 0 && tr + 1 < ntile_rows) issue(tr + 1, buf ^ 1);
      mbar_wait(&bars[buf], (unsigned)((tr >> 1) & 1));
      tX = sX + buf * kRT * kMaxVars;
      tV = sV + buf * kRT;
    } else {
      tX = a.X + r0 * n;  // generic path: plain loads
      tV = V + r0;
    }
    // a10: u = (x - c) 2^-e for the tile's rows
    for (int i = threadIdx.x; i < kRT * n; i += blockDim.x) {
      const int r = i / n, k = i % n;
      sU[i] = r < rows ? (tX[r * n + k] - B.xc[k]) * ldexp(1.0, -B.xe[k]) : 0.0;
    }
    __syncthreads();
    // a11: design rows [M(u) | -V N(u)] into sA (rows >= `rows` are zero: no contribution)
    for (int i = threadIdx.x; i < kRT * nc; i += blockDim.x) {
      const int r = i / nc, j = i % nc;
      double m = 0.0;
      if (r < rows) {
        m = 1.0;
        for (int k = 0; k < n; ++k) {
          const double u = sU[r * n + k];
          for (int e = 0; e < B.exp[j][k]; ++e) m *= u;
        }
        if (j >= n_num) m *= -tV[r];
        if (a.S) m *= a.S[(int64_t)metric * a.K + r0 + r];
      }
      sA[r * stride + j] = m;
    }
    __syncthreads();
    // a12: G_tile += A_bi^T A_bj over the 16 k-steps of this row tile
#pragma unroll 1
    for (int ks = 0; ks < kRT / 4; ++ks) {
      const double *row = sA + (ks * 4 + (lane & 3)) * stride + (lane >> 2);
#pragma unroll
      for (int t = 0; t < kMaxTilesPerWarp; ++t) {
        if (toff[t] >= 0) {
          const double av = row[toff[t] & 0xffff];
          const double bv = row[toff[t] >> 16];
          dmma_8x8x4(acc[t][0], acc[t][1], av, bv);
        }
      }
    }
    // two-level accumulation: flush registers every kChunkTiles row tiles
    if (((tr + 1) % kChunkTiles) == 0 || tr + 1 == ntile_rows) {
#pragma unroll
      for (int t = 0; t < kMaxTilesPerWarp; ++t) {
        if (toff[t] >= 0) {
          double *dst = sAcc + (wid + kGramWarps * t) * 64 + lane * 2;
          dst[0] += acc[t][0];
          dst[1] += acc[t][1];
          acc[t][0] = acc[t][1] = 0.0;
        }
      }
    }
    __syncthreads();
  }
  // write this CTA's partial tiles (tile-major, 64 doubles per tile in fragment order)
  const int64_t groups = gridDim.y;
  double *out = a.part + (((int64_t)metric * groups + group) * gridDim.x + blockIdx.x) *
                             (int64_t)kTilesPerGroup * 64;
  for (int i = threadIdx.x; i < kTilesPerGroup * 64; i += blockDim.x) out[i] = sAcc[i];
}

// Fixed-order sum of the per-CTA partials, scattered into the symmetric G.
__global__ void k_gram_reduce(const double *part, int nblk, int groups, int nb, int ntiles,
                              int nc, double *G) {
  const int metric = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)ntiles * 64;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(i / 64), e = (int)(i % 64);
    const int group = tile / kTilesPerGroup, tig = tile % kTilesPerGroup;
    // tig = wid + 8 * t within the group; element e = lane * 2 + v
    const int lane = e >> 1, v = e & 1;
    // tile id -> (bi, bj)
    int bi = 0, rem = tile;
    while (rem >= nb - bi) {
      rem -= nb - bi;
      ++bi;
    }
    const int bj = bi + rem;
    const int row = 8 * bi + (lane >> 2), col = 8 * bj + 2 * (lane & 3) + v;
    const double *src = part + ((int64_t)metric * groups + group) * nblk * (int64_t)kTilesPerGroup * 64 +
                         (int64_t)tig * 64 + e;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += src[(int64_t)b * kTilesPerGroup * 64];
    if (row < nc && col < nc) {
      double *Gm = G + (int64_t)metric * nc * nc;
      Gm[(int64_t)row * nc + col] = s;
      Gm[(int64_t)col * nc + row] = s;
    }
  }
}

// ============================================================================================
// Fused weighted Gram (numerator basis == denominator basis; every BASELINE config)
//
// With N = M the linearised rows a = [M | -V_i M] of the n_v metrics sharing X give
//   G_i = [[ M^T M , -M^T diag(V_i) M ], [ . , M^T diag(V_i^2) M ]],
// so 1 + 2 n_v symmetric m x m blocks replace n_v full (2m)^2 Grams.  With X_0 = M and
// X_{1+i} = V_i M (staged in shared memory), the blocks are X_0^T X_0, X_0^T X_{1+i} and
// X_{1+i}^T X_{1+i}; their upper-triangular 8x8 tiles are accumulated with DMMA.8x8x4.  Tiles
// are ordered by A-row group so the slots of one warp mostly share their A fragment.
// ============================================================================================
constexpr int kFW = 16;          // warps per CTA
constexpr int kFRT = 64;         // design rows per shared-memory tile (16 k-steps)
constexpr int kFlushTiles = 16;  // add register accumulators into the partial every 1024 rows

__host__ __device__ constexpr int fstride(int m8) {  // = 4 mod 16 (conflict-free fragments)
  int s = m8;
  while (s % 16 != 4) ++s;
  return s;
}

template <int NB, int NV>
struct FL {
  static constexpr int M8 = 8 * NB;
  static constexpr int T = NB * (NB + 1) / 2;  // upper tiles of one m x m block
  static constexpr int NP = 1 + 2 * NV;        // blocks: (0,0), (0,1+i), (1+i,1+i)
  static constexpr int NT = NP * T;
  static constexpr int SLOTS = (NT + kFW - 1) / kFW;
  static constexpr int NX = 1 + NV;
  static constexpr int S = fstride(M8);
};

// packed compile-time operand offsets (doubles) of a slot: A | B << 16, or kNoTile
constexpr uint32_t kNoTile = 0xffffffffu;

// tile id (A-row-group order) -> X arrays (pa, pb), block pair index and 8-blocks (bi <= bj)
template <int NB, int NV>
__host__ __device__ constexpr void fused_tile(int id, int &pa, int &pb, int &pair, int &bi, int &bj) {
  for (int a = 0; a <= NV; ++a)
    for (int i = 0; i < NB; ++i) {
      const int cnt = (a == 0 ? NV + 1 : 1) * (NB - i);
      if (id < cnt) {
        pa = a;
        bi = i;
        if (a == 0) {
          pb = id / (NB - i);
          bj = i + id % (NB - i);
          pair = pb;  // (0,0) -> 0, (0,1+v) -> 1+v
        } else {
          pb = a;
          bj = i + id;
          pair = 1 + NV + (a - 1);
        }
        return;
      }
      id -= cnt;
    }
  pa = pb = pair = bi = bj = -1;
}

__host__ __device__ constexpr int upper_index(int NB, int bi, int bj) {
  return bi * NB - bi * (bi - 1) / 2 + (bj - bi);
}

template <int NB, int NV, int NW = kFW>
__host__ __device__ constexpr uint32_t fused_slot_off(int wid, int j, int S, int RT) {
  const int NT = (1 + 2 * NV) * NB * (NB + 1) / 2;
  const int id = wid * ((NT + NW - 1) / NW) + j;
  if (id >= NT) return kNoTile;
  int pa = 0, pb = 0, pair = 0, bi = 0, bj = 0;
  fused_tile<NB, NV>(id, pa, pb, pair, bi, bj);
  return (uint32_t)(pa * RT * S + 8 * bi) | ((uint32_t)(pb * RT * S + 8 * bj) << 16);
}

// The MMA phase of one warp over the k-steps of a row tile: every operand offset is a
// compile-time constant (template on the warp id), so fragment loads are immediate-offset LDS
// and slots sharing an A fragment reuse the loaded value.
template <int NB, int NV, int WID, int SLOTS, int S, int RT, int NW = kFW>
__device__ __forceinline__ void fused_mma_warp(const double *sX, int lane, double (&acc)[SLOTS][2]) {
#pragma unroll 2
  for (int ks = 0; ks < RT / 4; ++ks) {
    const double *row = sX + (ks * 4 + (lane & 3)) * S + (lane >> 2);
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const uint32_t off = fused_slot_off<NB, NV, NW>(WID, j, S, RT);
      if (off != kNoTile) dmma_8x8x4(acc[j][0], acc[j][1], row[off & 0xffffu], row[off >> 16]);
    }
  }
}

struct FusedArgs {
  const GramBasis *basis;
  const double *X;
  const double *V;  // [NV][K]
  const double *S;  // [K] row scales (NV = 1, weighted refit) or null
  int64_t K;
  double *part;     // [gridDim.x][NT][64]  canonical (pair, upper tile) order
  int tma = 0;      // k_gram_ws: inputs of full tiles by bulk copy (16-byte aligned X, V rows, S)
};

template <int NB, int NV>
__global__ void __launch_bounds__(kFW * 32, 1) k_gram_fused(FusedArgs a) {
  using L = FL<NB, NV>;
  extern __shared__ __align__(16) double fsm[];
  const GramBasis &B = *a.basis;
  const int n = B.n, m = B.n_num, pw = B.maxdeg + 1;
  double *sX = fsm;                          // [NX][kFRT][S]
  double *sU = sX + L::NX * kFRT * L::S;     // [kFRT][n]
  double *sPow = sU + kFRT * kMaxVars;       // [kFRT][n][pw]
  double *sV = sPow + kFRT * n * pw;         // [NV][kFRT]
  double *sS = sV + NV * kFRT;                                     // [kFRT]
  uint32_t *sExp = reinterpret_cast<uint32_t *>(sS + kFRT);       // [M8]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  const int64_t r_begin = a.K * blockIdx.x / gridDim.x;
  const int64_t r_end = a.K * (blockIdx.x + 1) / gridDim.x;
  const int64_t ntr = (r_end - r_begin + kFRT - 1) / kFRT;

  for (int i = threadIdx.x; i < L::NX * kFRT * L::S; i += blockDim.x) sX[i] = 0.0;  // pads
  for (int j = threadIdx.x; j < m; j += blockDim.x) sExp[j] = B.pexp[j];

  double acc[L::SLOTS][2];
#pragma unroll
  for (int j = 0; j < L::SLOTS; ++j) acc[j][0] = acc[j][1] = 0.0;
  double *part = a.part + (int64_t)blockIdx.x * L::NT * 64;
  bool first = true;
  __syncthreads();

  for (int64_t tr = 0; tr < ntr; ++tr) {
    const int64_t r0 = r_begin + tr * kFRT;
    const int rows = (int)((r_end - r0) < kFRT ? (r_end - r0) : kFRT);
    // a10: u = (x - c) 2^-e; the metric values of the tile
    for (int i = threadIdx.x; i < kFRT * n; i += blockDim.x) {
      const int r = i / n, k = i % n;
      sU[r * kMaxVars + k] = r < rows ? (a.X[(r0 + r) * n + k] - B.xc[k]) * ldexp(1.0, -B.xe[k]) : 0.0;
    }
    for (int i = threadIdx.x; i < NV * kFRT; i += blockDim.x) {
      const int v = i / kFRT, r = i % kFRT;
      sV[i] = r < rows ? a.V[(int64_t)v * a.K + r0 + r] : 0.0;
    }
    if (a.S)  // weighted rows (f4): the power table of row r starts at s_r instead of 1
      for (int r = threadIdx.x; r < kFRT; r += blockDim.x) sS[r] = r < rows ? a.S[r0 + r] : 0.0;
    __syncthreads();
    // powers u^e, e <= maxdeg, by repeated multiplication
    for (int i = threadIdx.x; i < kFRT * n; i += blockDim.x) {
      const int r = i / n, k = i % n;
      const double u = sU[r * kMaxVars + k];
      double p = r < rows ? 1.0 : 0.0;  // rows past the slab: all-zero design row
      if (a.S && k == 0) p = sS[r];      // the row scale enters through variable 0's powers
      double *dst = sPow + (r * n + k) * pw;
      for (int e = 0; e < pw; ++e) {
        dst[e] = p;
        p *= u;
      }
    }
    __syncthreads();
    // a11: X_0 = M(u) and X_{1+v} = V_v M(u) (the design row is [X_0 | -X_{1+v}])
    for (int i = threadIdx.x; i < kFRT * m; i += blockDim.x) {
      const int r = i / m, j = i % m;
      const uint32_t w = sExp[j];
      const double *pr = sPow + r * n * pw;
      double prod = pr[w & 15];
      for (int k = 1; k < n; ++k) prod *= pr[k * pw + ((w >> (4 * k)) & 15)];
      sX[r * L::S + j] = prod;
#pragma unroll
      for (int v = 0; v < NV; ++v) sX[(1 + v) * kFRT * L::S + r * L::S + j] = sV[v * kFRT + r] * prod;
    }
    __syncthreads();
    // a12: the upper tiles of the 1 + 2 NV blocks (per-warp compile-time tile lists)
    switch (wid) {
#define RP_W(w) \
  case w: fused_mma_warp<NB, NV, w, L::SLOTS, L::S, kFRT>(sX, lane, acc); break;
      RP_W(0) RP_W(1) RP_W(2) RP_W(3) RP_W(4) RP_W(5) RP_W(6) RP_W(7)
      RP_W(8) RP_W(9) RP_W(10) RP_W(11) RP_W(12) RP_W(13) RP_W(14) RP_W(15)
#undef RP_W
    }
    __syncthreads();
    if (((tr + 1) % kFlushTiles) == 0 || tr + 1 == ntr) {
#pragma unroll
      for (int j = 0; j < L::SLOTS; ++j) {
        const int id = wid * L::SLOTS + j;
        if (id < L::NT) {
          int pa, pb, pair, bi, bj;
          fused_tile<NB, NV>(id, pa, pb, pair, bi, bj);
          double *dst = part + (int64_t)(pair * L::T + upper_index(NB, bi, bj)) * 64 + lane * 2;
          if (first) {
            dst[0] = acc[j][0];
            dst[1] = acc[j][1];
          } else {
            dst[0] += acc[j][0];
            dst[1] += acc[j][1];
          }
          acc[j][0] = acc[j][1] = 0.0;
        }
      }
      first = false;
    }
  }
  if (ntr == 0)  // empty slab: zero partial
    for (int i = threadIdx.x; i < L::NT * 64; i += blockDim.x) part[i] = 0.0;
}

// ============================================================================================
// Warp-specialised fused Gram (default).  In k_gram_fused every warp stages, then every warp
// multiplies, so the FP64 tensor pipe idles during staging (~30% of a tile, measured with
// -DRP_GRAM_TS).  Here the last warpgroup (kWsPW = 4 warps, one per SM sub-partition) only builds
// design rows and the first kWsMW warps (16: 20 accumulator slots each; 12: 27) only multiply.  A stage holds
// X_0 = M(u) of 32 rows and, per row, the scales V_v and V_v^2: since
//   X_0^T diag(V_v) X_0  and  X_0^T diag(V_v^2) X_0
// are the (0, 1+v) and (1+v, 1+v) blocks, the consumers scale their A fragment (one row per lane)
// instead of the producers writing X_{1+v} = V_v X_0 (4x less staging and shared memory).  Stages
// are handed over with named barriers (FULL[b]: producers arrive, consumers wait; EMPTY[b]:
// consumers arrive, producers wait); setmaxnreg gives the producers RP_WS_PREG registers and the
// consumers RP_WS_CREG (56 / 104 with 16 consumer warps).
// ============================================================================================
constexpr int kWsRT = 32;      // rows per tile
#ifndef RP_WS_MW
#define RP_WS_MW 16
#endif
constexpr int kWsMW = RP_WS_MW;  // MMA (consumer) warps: 16 (4 per sub-partition), 12 measured 1.5% slower
constexpr int kWsPW = 4;       // staging (producer) warps
#ifndef RP_WS_NS
#define RP_WS_NS 3
#endif
constexpr int kWsNS = RP_WS_NS;  // stages
#ifndef RP_WS_UNROLL
#define RP_WS_UNROLL 1
#endif
constexpr int kWsUnroll = RP_WS_UNROLL;  // k-steps per MMA loop body (code size: instruction cache)
constexpr int kWsFlush = 32;   // tiles between flushes of the register accumulators (1024 rows)
constexpr int kWsThreads = 32 * (kWsMW + kWsPW);
constexpr int kWsIS = 4;       // input stages (raw X / V / S of a tile, filled by the TMA engine)
// registers per thread after setmaxnreg: 12 x 32 x CREG + 4 x 32 x PREG <= 64K
#if RP_WS_MW > 12
#ifndef RP_WS_PREG
#define RP_WS_PREG 56
#endif
#ifndef RP_WS_CREG
#define RP_WS_CREG 104
#endif
#else
#ifndef RP_WS_PREG
#define RP_WS_PREG 72
#endif
#ifndef RP_WS_CREG
#define RP_WS_CREG 144
#endif
#endif
static_assert(kWsMW * 32 * RP_WS_CREG + kWsPW * 32 * RP_WS_PREG <= 65536, "register file");

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NB, int NV>
struct WsL {
  static constexpr int S = FL<NB, NV>::S;
  static constexpr int SCS = 2 * NV;                   // scales per row: V_v, V_v^2
  static constexpr int XB = kWsRT * S + kWsRT * SCS;   // doubles per stage: X_0 | scales
};

// doubles before the input ring: stages | producers' power tables | exponent / tree tables
template <int NB, int NV>
__host__ __device__ constexpr size_t ws_in_off(int n, int pw) {
  // rounded up to an even count: bulk-copy destinations are 16-byte aligned
  return ((size_t)kWsNS * WsL<NB, NV>::XB + (size_t)kWsPW * (8 * n * pw + 16) +
          ((size_t)kWsPW * 3 * FL<NB, NV>::M8 + 1) / 2 + 2) & ~(size_t)1;
}

// tile id of slot j of consumer warp WID: contiguous ranges of SLOTS tiles (measured faster than
// spreading them so that every sub-partition holds NT / 4: 1.464 vs 1.509 ms at K = 10^6)
template <int NT, int SLOTS>
__host__ __device__ constexpr int ws_tile_id(int wid, int j) {
  return wid * SLOTS + j < NT ? wid * SLOTS + j : -1;
}

// slot j of consumer warp WID: A = X_0 block bi scaled by sc (0: 1, 1 + v: V_v, 1 + NV + v: V_v^2),
// B = X_0 block bj; packed as A offset | B offset << 12 | sc << 24
template <int NB, int NV, int WID, int SLOTS>
__host__ __device__ constexpr uint32_t ws_slot(int j) {
  constexpr int NT = (1 + 2 * NV) * NB * (NB + 1) / 2;
  const int id = ws_tile_id<NT, SLOTS>(WID, j);
  if (id < 0) return kNoTile;
  int pa = 0, pb = 0, pair = 0, bi = 0, bj = 0;
  fused_tile<NB, NV>(id, pa, pb, pair, bi, bj);
  return (uint32_t)(8 * bi) | ((uint32_t)(8 * bj) << 12) | ((uint32_t)pair << 24);
}

template <int NB, int NV, int WID, int SLOTS>
__device__ __forceinline__ void ws_mma_warp(const double *buf, int lane, double (&acc)[SLOTS][2]) {
  using W = WsL<NB, NV>;
  const double *scb = buf + kWsRT * W::S;
#pragma unroll (kWsUnroll)
  for (int ks = 0; ks < kWsRT / 4; ++ks) {
    const int r = ks * 4 + (lane & 3);
    const double *row = buf + r * W::S + (lane >> 2);
    double sc[1 + 2 * NV];
    sc[0] = 1.0;
#pragma unroll
    for (int v = 0; v < 2 * NV; ++v) sc[1 + v] = scb[r * W::SCS + v];
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      constexpr uint32_t kNo = kNoTile;
      const uint32_t off = ws_slot<NB, NV, WID, SLOTS>(j);
      if (off != kNo) {
        const int pr = (int)(off >> 24);
        const double a = row[off & 0xfff];
        dmma_8x8x4(acc[j][0], acc[j][1], pr == 0 ? a : a * sc[pr], row[(off >> 12) & 0xfff]);
      }
    }
  }
}

template <int NB, int NV>
__global__ void __launch_bounds__(kWsThreads, 1) k_gram_ws(FusedArgs a) {
  using L = FL<NB, NV>;
  using W = WsL<NB, NV>;
  constexpr int SLOTS = (L::NT + kWsMW - 1) / kWsMW;
  extern __shared__ __align__(16) double fsm[];
  const GramBasis &B = *a.basis;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *sX = fsm;  // [kWsNS][W::XB]

  // slabs of whole 32-row tiles (tile starts are 16-byte aligned in X, V and S)
  const int64_t ntiles = (a.K + kWsRT - 1) / kWsRT;
  const int64_t r_begin = kWsRT * (ntiles * blockIdx.x / gridDim.x);
  const int64_t r_end_t = kWsRT * (ntiles * (blockIdx.x + 1) / gridDim.x);
  const int64_t r_end = r_end_t < a.K ? r_end_t : a.K;
  const int ntr = (int)((r_end - r_begin + kWsRT - 1) / kWsRT);
  // input ring after the producers' scratch: [kWsIS][INB] doubles + 2 kWsIS mbarriers
  const int INB = kWsRT * (B.n + NV + 1);
  double *sIn = fsm + ws_in_off<NB, NV>(B.n, B.maxdeg + 1);
  uint64_t *inFull = reinterpret_cast<uint64_t *>(sIn + kWsIS * INB), *inEmpty = inFull + kWsIS;
  for (int i = threadIdx.x; i < kWsNS * W::XB; i += blockDim.x) sX[i] = 0.0;  // pads stay zero
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsIS; ++i) {
      mbar_init(inFull + i, 1);        // the issuing thread's expect_tx arrival (+ the bytes)
      mbar_init(inEmpty + i, kWsPW);   // every producer warp has read its inputs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid >= kWsMW) {
    // ---- producers: 8 rows per warp per tile --------------------------------------------------
    // The inputs of the warp's 8 rows, [X (8 n) | V (8 NV) | S (8)], are loaded into registers one
    // tile ahead (2 values per lane), so the HBM latency is off the staging path.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RP_WS_PREG));
    const int pw = wid - kWsMW;
    const int n = B.n, m = B.n_num, pwr = B.maxdeg + 1;
    const int nXv = 8 * n, nVv = 8 * NV, nIn = nXv + nVv + (a.S ? 8 : 0);
    double *sPow = sX + kWsNS * W::XB + pw * (8 * n * pwr + 16);  // [8][n][pwr]
    double *sSw = sPow + 8 * n * pwr;                              // [8]   row scales
    uint32_t *sExp = reinterpret_cast<uint32_t *>(sX + kWsNS * W::XB + kWsPW * (8 * n * pwr + 16)) + pw * 3 * L::M8;
    uint32_t *sInfo = sExp + L::M8;                 // tree: parent | var << 16 of column j
    uint32_t *sLv = sInfo + L::M8;                  // tree: the columns level by level
    double *sU = sPow;                              // tree: u of the 8 rows [8][n] (aliases sPow)
    double *sK = sPow + 8 * n;                      // tree: the constant column of the 8 rows
    const bool tree = B.tree != 0;
    for (int j = lane; j < m; j += 32) {
      sExp[j] = B.pexp[j];
      sInfo[j] = (uint32_t)(uint16_t)B.parent[j] | ((uint32_t)(uint8_t)B.pvar[j] << 16);
      sLv[j] = (uint32_t)B.lv_cols[j];
    }
    const double xc = lane < nXv ? B.xc[lane % n] : 0.0, xs = lane < nXv ? ldexp(1.0, -B.xe[lane % n]) : 0.0;
    auto fetch = [&](int tr, int i) -> double {  // input i of the warp's rows of tile tr (0 past the slab)
      const int64_t r0 = r_begin + (int64_t)tr * kWsRT + 8 * pw;
      if (tr >= ntr || i >= nIn) return 0.0;
      if (i < nXv) return r0 + i / n < r_end ? a.X[(r0 + i / n) * n + i % n] : 0.0;
      i -= nXv;
      if (i < nVv) return r0 + i % 8 < r_end ? a.V[(int64_t)(i / 8) * a.K + r0 + i % 8] : 0.0;
      i -= nVv;
      return r0 + i < r_end ? a.S[r0 + i] : 0.0;
    };
    // TMA path: tile tr's raw inputs [X (32 n) | V (NV x 32) | S (32)] land in input stage
    // tr % kWsIS by bulk copies that one thread issues kWsIS - 1 tiles ahead; a partial tail
    // tile (and any launch whose rows are not 16-byte aligned) takes the register path below.
    const bool tma = a.tma != 0;
    auto full_tile = [&](int tr) { return r_begin + (int64_t)(tr + 1) * kWsRT <= r_end; };
    auto issue = [&](int tr) {  // one thread: the bulk copies of tile tr into its input stage
      const int st = tr % kWsIS;
      double *dst = sIn + st * INB;
      const int64_t r0 = r_begin + (int64_t)tr * kWsRT;
      const unsigned bx = kWsRT * n * 8, bv = kWsRT * 8;
      mbar_expect_tx(inFull + st, bx + NV * bv + (a.S ? bv : 0));
      bulk_g2s(dst, a.X + r0 * n, bx, inFull + st);
#pragma unroll
      for (int v = 0; v < NV; ++v) bulk_g2s(dst + kWsRT * n + v * kWsRT, a.V + (int64_t)v * a.K + r0, bv, inFull + st);
      if (a.S) bulk_g2s(dst + kWsRT * (n + NV), a.S + r0, bv, inFull + st);
    };
    auto from_stage = [&](const double *src, int i) -> double {  // input i of the warp's rows
      if (i >= nIn) return 0.0;
      if (i < nXv) return src[8 * pw * n + i];
      i -= nXv;
      if (i < nVv) return src[kWsRT * n + (i / 8) * kWsRT + 8 * pw + i % 8];
      i -= nVv;
      return src[kWsRT * (n + NV) + 8 * pw + i];
    };
    if (tma && pw == 0 && lane == 0)
      for (int t = 0; t < kWsIS - 1 && t < ntr; ++t)
        if (full_tile(t)) issue(t);
    double v0 = tma ? 0.0 : fetch(0, lane), v1 = tma ? 0.0 : fetch(0, lane + 32);
    __syncwarp();
    for (int tr = 0; tr < ntr; ++tr) {
      const int b = tr % kWsNS;
      double *buf = sX + b * W::XB;
      double *scb = buf + kWsRT * W::S + 8 * pw * W::SCS;  // scales of the warp's 8 rows
      const int64_t r0 = r_begin + (int64_t)tr * kWsRT + 8 * pw;
      const int nvalid = (int)((r_end - r0) < 8 ? (r_end - r0) : 8);  // rows of the warp in the slab
      double cv0, cv1;
      if (tma) {
        if (full_tile(tr)) {
          const int st = tr % kWsIS;
          mbar_wait(inFull + st, (tr / kWsIS) & 1);
          const double *src = sIn + st * INB;
          cv0 = from_stage(src, lane);
          cv1 = from_stage(src, lane + 32);
          __syncwarp();
          if (lane == 0) mbar_arrive1(inEmpty + st);
        } else {
          cv0 = fetch(tr, lane);
          cv1 = fetch(tr, lane + 32);
        }
        // refill the stage of tile tr - 1 with tile tr + kWsIS - 1 once every producer read it
        const int tn = tr + kWsIS - 1;
        if (pw == 0 && lane == 0 && tn < ntr && full_tile(tn)) {
          if (tn >= kWsIS) mbar_wait(inEmpty + tn % kWsIS, ((tn / kWsIS) - 1) & 1);
          issue(tn);
        }
      } else {
        cv0 = v0;
        cv1 = v1;
        v0 = fetch(tr + 1, lane);  // the next tile's inputs: in flight while this one is built
        v1 = fetch(tr + 1, lane + 32);
      }
      {  // row scales S
        const int i0 = lane - nXv - nVv, i1 = lane + 32 - nXv - nVv;
        if (i0 >= 0 && i0 < 8) sSw[i0] = cv0;
        if (i1 >= 0 && i1 < 8) sSw[i1] = cv1;
      }
      __syncwarp();
      // a10: u = (x - c) 2^-e (X lanes: row lane / n, variable lane % n); the tree needs u and the
      // constant column, the general path the power table
      if (tree) {
        if (lane < nXv) sU[lane] = (cv0 - xc) * xs;
        if (lane < 8) sK[lane] = lane < nvalid ? (a.S ? sSw[lane] : 1.0) : 0.0;  // weighted rows: s_r
      } else if (lane < nXv) {
        const int r = lane / n, k = lane % n;
        const double u = (cv0 - xc) * xs;
        double p = r < nvalid ? ((a.S && k == 0) ? sSw[r] : 1.0) : 0.0;  // weighted rows: s_r via u_0
        double *dst = sPow + (r * n + k) * pwr;
        for (int e = 0; e < pwr; ++e) {
          dst[e] = p;
          p *= u;
        }
      }
      if (tr >= kWsNS) named_sync(1 + kWsNS + b, kWsThreads);  // EMPTY[b]: consumers done with tile tr - NS
      {  // per-row scales V_v, V_v^2 (V inputs: index i = v * 8 + r)
        const int i0 = lane - nXv, i1 = lane + 32 - nXv;
        if (i0 >= 0 && i0 < nVv) scb[(i0 % 8) * W::SCS + i0 / 8] = cv0, scb[(i0 % 8) * W::SCS + NV + i0 / 8] = cv0 * cv0;
        if (i1 >= 0 && i1 < nVv) scb[(i1 % 8) * W::SCS + i1 / 8] = cv1, scb[(i1 % 8) * W::SCS + NV + i1 / 8] = cv1 * cv1;
      }
      __syncwarp();
      // a11: X_0 = M(u) for the warp's 8 rows (the design row is [X_0 | -V X_0])
      if (tree) {
        // a11 by the monomial tree: level d columns are parent (level d - 1) times one u
        for (int d = 0; d < B.n_lv; ++d) {
          const int l0 = B.lv_start[d], cnt = B.lv_start[d + 1] - l0;
          const float rc = 1.0f / (float)cnt;
          for (int e = lane; e < 8 * cnt; e += 32) {
            const int r = (int)(((float)e + 0.5f) * rc), col = (int)sLv[l0 + e - r * cnt];
            double *row = buf + (8 * pw + r) * W::S;
            if (d == 0) {
              row[col] = sK[r];
            } else {
              const uint32_t inf = sInfo[col];
              row[col] = row[inf & 0xffff] * sU[r * n + (inf >> 16)];
            }
          }
          __syncwarp();
        }
      }
      // entries j = lane + 32 it of the 8 m, two per iteration (independent chains)
      int r = lane / m, col = lane % m;
      int r2 = (lane + 32) / m, col2 = (lane + 32) % m;
      if (!tree)
      for (int j = lane; j < 8 * m; j += 64) {
        const bool two = j + 32 < 8 * m;
        const uint32_t w = sExp[col], w2 = sExp[two ? col2 : col];
        const double *pr = sPow + r * n * pwr, *pr2 = sPow + (two ? r2 : r) * n * pwr;
        double x = pr[w & 15], y = pr2[w2 & 15];
        if (n == 4) {  // the BASELINE bases: a product tree, depth 2
          x = (x * pr[pwr + ((w >> 4) & 15)]) * (pr[2 * pwr + ((w >> 8) & 15)] * pr[3 * pwr + ((w >> 12) & 15)]);
          y = (y * pr2[pwr + ((w2 >> 4) & 15)]) * (pr2[2 * pwr + ((w2 >> 8) & 15)] * pr2[3 * pwr + ((w2 >> 12) & 15)]);
        } else {
          for (int k = 1; k < n; ++k) {
            x *= pr[k * pwr + ((w >> (4 * k)) & 15)];
            y *= pr2[k * pwr + ((w2 >> (4 * k)) & 15)];
          }
        }
        buf[(8 * pw + r) * W::S + col] = x;
        if (two) buf[(8 * pw + r2) * W::S + col2] = y;
        col += 64;
        while (col >= m) col -= m, ++r;
        col2 += 64;
        while (col2 >= m) col2 -= m, ++r2;
      }
      __threadfence_block();
      named_arrive(1 + b, kWsThreads);  // FULL[b]
      __syncwarp();
    }
    return;
  }

  // ---- consumers: the upper tiles of the 1 + 2 NV blocks ----------------------------------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RP_WS_CREG));
  double acc[SLOTS][2];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) acc[j][0] = acc[j][1] = 0.0;
  double *part = a.part + (int64_t)blockIdx.x * L::NT * 64;
  bool first = true;
  for (int tr = 0; tr < ntr; ++tr) {
    const int b = tr % kWsNS;
    named_sync(1 + b, kWsThreads);  // FULL[b]
    const double *cur = sX + b * W::XB;
    switch (wid) {
#define RP_W(w) \
  case w: ws_mma_warp<NB, NV, w, SLOTS>(cur, lane, acc); break;
      RP_W(0) RP_W(1) RP_W(2) RP_W(3) RP_W(4) RP_W(5) RP_W(6) RP_W(7) RP_W(8) RP_W(9) RP_W(10) RP_W(11)
#if RP_WS_MW > 12
      RP_W(12) RP_W(13) RP_W(14) RP_W(15)
#endif
#undef RP_W
    }
    named_arrive(1 + kWsNS + b, kWsThreads);  // EMPTY[b]
    if (((tr + 1) % kWsFlush) == 0 || tr + 1 == ntr) {
#pragma unroll
      for (int j = 0; j < SLOTS; ++j) {
        const int id = ws_tile_id<L::NT, SLOTS>(wid, j);
        if (id >= 0) {
          int pa, pb, pair, bi, bj;
          fused_tile<NB, NV>(id, pa, pb, pair, bi, bj);
          double *dst = part + (int64_t)(pair * L::T + upper_index(NB, bi, bj)) * 64 + lane * 2;
          if (first) {
            dst[0] = acc[j][0];
            dst[1] = acc[j][1];
          } else {
            dst[0] += acc[j][0];
            dst[1] += acc[j][1];
          }
          acc[j][0] = acc[j][1] = 0.0;
        }
      }
      first = false;
    }
  }
  if (ntr == 0)  // empty slab: zero partial
    for (int i = threadIdx.x; i < L::NT * 64; i += kWsMW * 32) part[i] = 0.0;
}

template <int NB, int NV>
static size_t ws_smem(int n, int pw) {
  return sizeof(double) * (ws_in_off<NB, NV>(n, pw) + (size_t)kWsIS * kWsRT * (n + NV + 1)) +
         sizeof(uint64_t) * 2 * kWsIS;
}

// The per-CTA partials summed over CTAs in a fixed order: 4 quarter sums per element (CTAs
// q, q + 4, ...; each warp reads 32 consecutive elements of one CTA's partial), added as
// (q0 + q1) + (q2 + q3).  red[e] for the NT * 64 unique accumulator elements.
__global__ void __launch_bounds__(256) k_gram_fused_sum(const double *part, int nblk, int n_el, double *red) {
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

// G_v (v < n_v) assembled from the summed partials (red: NT * 64 elements).
__global__ void k_gram_fused_reduce(const double *red, int NB, int NV, int m, double *G) {
  const int T = NB * (NB + 1) / 2, nc = 2 * m;
  const int64_t total = (int64_t)NV * nc * nc;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(idx / ((int64_t)nc * nc));
    const int rc = (int)(idx % ((int64_t)nc * nc));
    const int row = rc / nc, col = rc % nc;
    const int qa = row >= m, qb = col >= m;
    int x = row - qa * m, y = col - qb * m;
    const int pair = (!qa && !qb) ? 0 : (qa != qb ? 1 + v : 1 + NV + v);
    const double sign = (qa != qb) ? -1.0 : 1.0;
    if (x / 8 > y / 8) {  // symmetric block: use the transposed element of the upper tile
      const int t = x;
      x = y;
      y = t;
    }
    const int bi = x / 8, bj = y / 8, mr = x % 8, nn = y % 8;
    const int can = pair * T + upper_index(NB, bi, bj);
    const int e = (mr * 4 + nn / 2) * 2 + (nn & 1);
    G[idx] = sign * red[(int64_t)can * 64 + e];
  }
}

template <int NB, int NV>
static size_t fused_smem(int n, int pw) {
  using L = FL<NB, NV>;
  return sizeof(double) * ((size_t)L::NX * kFRT * L::S + kFRT * kMaxVars + (size_t)kFRT * n * pw + NV * kFRT +
                            kFRT) +
         sizeof(uint32_t) * L::M8;
}

static int fused_grid_x(int64_t K) {
  int64_t want = (K + kFRT - 1) / kFRT;
  int64_t cap = num_sms();
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

template <int NB, int NV>
static cudaError_t launch_fused_t(const GramBasis *d_basis, const GramBasis &h, const double *X,
                                  const double *V, const double *S, int64_t K, double *G,
                                  double *d_part, size_t part_elems, cudaStream_t s) {
  using L = FL<NB, NV>;
  const int gx = fused_grid_x(K);
  if ((size_t)(gx + 1) * L::NT * 64 > part_elems) return cudaErrorInvalidValue;
  FusedArgs fa{d_basis, X, V, S, K, d_part};
  // bulk copies need 16-byte aligned sources: X rows and V / S tile starts (K even)
  fa.tma = ((uintptr_t)X % 16 == 0) && ((uintptr_t)V % 16 == 0) && (!S || (uintptr_t)S % 16 == 0) && (K % 2 == 0);
#ifdef RP_WS_NOTMA  // measurement: the register-prefetch path only
  fa.tma = 0;
#endif
  cudaError_t e;
  const char *gk = getenv("RP_GRAM_KERNEL");  // "fused": the single-role kernel (tests, measurements)
  const bool ws = !(gk && strcmp(gk, "fused") == 0);
  if (ws) {  // warp-specialised (default)
    const size_t smem = ws_smem<NB, NV>(h.n, h.maxdeg + 1);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(k_gram_ws<NB, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gram_ws<NB, NV><<<gx, kWsThreads, smem, s>>>(fa);
  } else {
    const size_t smem = fused_smem<NB, NV>(h.n, h.maxdeg + 1);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(k_gram_fused<NB, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gram_fused<NB, NV><<<gx, kFW * 32, smem, s>>>(fa);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int n_el = L::NT * 64;
  double *red = d_part + (size_t)gx * n_el;  // fused_partial_elems reserves it after the partials
  k_gram_fused_sum<<<(n_el + 63) / 64, 256, 0, s>>>(d_part, gx, n_el, red);
  const int64_t total = (int64_t)NV * 4 * h.n_num * h.n_num;
  const int rb = (int)((total + 255) / 256);
  k_gram_fused_reduce<<<rb, 256, 0, s>>>(red, NB, NV, h.n_num, G);
  return cudaGetLastError();
}

// which (NB, NV) pairs are compiled for the fused path
static bool fused_supported(const GramBasis &h, int n_v) {
  if (!h.fused || h.n > kMaxVars || h.maxdeg > 15) return false;
  const int nb = (h.n_num + 7) / 8;
  return (n_v == 1 || n_v == 3) && (nb == 2 || nb == 5 || nb == 9);
}

static size_t fused_partial_elems(const GramBasis &h, int n_v, int64_t K) {
  const int nb = (h.n_num + 7) / 8;
  const int NT = (1 + 2 * n_v) * nb * (nb + 1) / 2;
  return (size_t)(fused_grid_x(K) + 1) * NT * 64;  // partials + their sum
}

static cudaError_t launch_fused(const GramBasis *d_basis, const GramBasis &h, const double *X,
                                const double *V, const double *S, int64_t K, int n_v, double *G,
                                double *d_part, size_t part_elems, cudaStream_t s) {
  const int nb = (h.n_num + 7) / 8;
#define RP_FUSED_CASE(NB_, NV_)                                                                \
  if (nb == NB_ && n_v == NV_)                                                               \
    return launch_fused_t<NB_, NV_>(d_basis, h, X, V, S, K, G, d_part, part_elems, s);
  RP_FUSED_CASE(2, 1) RP_FUSED_CASE(2, 3) RP_FUSED_CASE(5, 1) RP_FUSED_CASE(5, 3)
  RP_FUSED_CASE(9, 1) RP_FUSED_CASE(9, 3)
#undef RP_FUSED_CASE
  return cudaErrorInvalidValue;
}

static int gram_grid_x(int64_t K) {
  int64_t want = (K + kRT - 1) / kRT;
  int64_t cap = num_sms();
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// RP_GRAM_KERNEL: unset or "mom" -> the moment contraction where supported (rp_moments.cu);
// "ws" / "fused" -> the outer-product kernels below (A/B measurements, tests)
static bool use_moments(const GramBasis &h, int n_v, bool weighted) {
  const char *gk = getenv("RP_GRAM_KERNEL");
  return (!gk || strcmp(gk, "mom") == 0) && mom_supported(h, n_v, weighted);
}

static size_t gram_partial_elems_op(const GramBasis &h, int n_v, int64_t K, bool weighted);
size_t gram_partial_elems(const GramBasis &h, int n_v, int64_t K, int nsm, bool weighted) {
  (void)nsm;
  const size_t op = gram_partial_elems_op(h, n_v, K, weighted), mo = mom_partial_elems(h, n_v, K, weighted);
  return op > mo ? op : mo;
}

static size_t gram_partial_elems_op(const GramBasis &h, int n_v, int64_t K, bool weighted) {
  if (weighted && fused_supported(h, 1)) return fused_partial_elems(h, 1, K);
  if (!weighted && fused_supported(h, n_v)) return fused_partial_elems(h, n_v, K);
  const int nb = (h.nc + 7) / 8;
  const int ntiles = nb * (nb + 1) / 2;
  const int groups = (ntiles + kTilesPerGroup - 1) / kTilesPerGroup;
  return (size_t)n_v * groups * gram_grid_x(K) * kTilesPerGroup * 64;
}

cudaError_t launch_gram(const GramBasis *d_basis, const GramBasis &h, const double *X,
                        const double *V, const double *S, int64_t K, int n_v, double *G,
                        double *d_part, size_t part_elems, cudaStream_t s) {
  if (use_moments(h, n_v, S != nullptr)) return launch_gram_mom(d_basis, h, X, V, S, K, n_v, G, d_part, part_elems, s);
  if (S && fused_supported(h, 1)) {  // weighted rows: one fused launch per metric
    for (int v = 0; v < n_v; ++v) {
      cudaError_t e = launch_fused(d_basis, h, X, V + (int64_t)v * K, S + (int64_t)v * K, K, 1,
                                   G + (int64_t)v * h.nc * h.nc, d_part, part_elems, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (!S && fused_supported(h, n_v)) return launch_fused(d_basis, h, X, V, nullptr, K, n_v, G, d_part, part_elems, s);
  const int nb = (h.nc + 7) / 8;
  const int ntiles = nb * (nb + 1) / 2;
  const int groups = (ntiles + kTilesPerGroup - 1) / kTilesPerGroup;
  const int gx = gram_grid_x(K);
  if (gram_partial_elems_op(h, n_v, K, false) > part_elems) return cudaErrorInvalidValue;
  const int stride = gram_stride(nb);
  GramArgs a{d_basis, X, V, S, K, n_v, nb, ntiles, stride, d_part};
  const size_t smem = (size_t)kRT * stride * 8 + (size_t)kTilesPerGroup * 64 * 8 +
                      2 * kRT * kMaxVars * 8 + 2 * kRT * 8 + kRT * kMaxVars * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_gram<<<dim3(gx, groups, n_v), kGramThreads, smem, s>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int rb = (int)((ntiles * 64 + 255) / 256);
  k_gram_reduce<<<dim3(rb, n_v), 256, 0, s>>>(d_part, gx, groups, nb, ntiles, h.nc, G);
  return cudaGetLastError();
}

}  // namespace rp

namespace rp {

// f4: S[v][r] = 1 / q_v(x_r), q_v the denominator of metric v with device coefficients coef
// [n_v][n_c] in the u-basis of the device GramBasis (repeated multiplication per monomial)
__global__ void k_den_weights(const GramBasis *gb, const double *X, int64_t K, int n_v,
                              const double *coef, double *S) {
  const GramBasis &B = *gb;
  const int n = B.n, n_num = B.n_num, n_den = B.n_den, nc = B.nc;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < K;
       r += (int64_t)gridDim.x * blockDim.x) {
    double u[kMaxVars];
    for (int k = 0; k < n; ++k) u[k] = (X[r * n + k] - B.xc[k]) * ldexp(1.0, -B.xe[k]);
    for (int v = 0; v < n_v; ++v) {
      double q = 0.0;
      for (int j = 0; j < n_den; ++j) {
        double m = 1.0;
        for (int k = 0; k < n; ++k)
          for (int e = 0; e < B.exp[n_num + j][k]; ++e) m *= u[k];
        q = fma(coef[(int64_t)v * nc + n_num + j], m, q);
      }
      S[(int64_t)v * K + r] = 1.0 / q;
    }
  }
}

// a13, deterministic form: out = ((p_0 + p_1) + p_2) + ... elementwise, partials in rank order
// (the all_gather'ed partial Grams of the K shards; bit-reproducible whatever the collective)
__global__ void k_sum_ordered(const double *parts, int n_parts, int64_t elems, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < elems; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = parts[i];
    for (int r = 1; r < n_parts; ++r) acc += parts[(int64_t)r * elems + i];
    out[i] = acc;
  }
}

cudaError_t launch_sum_ordered(const double *parts, int n_parts, int64_t elems, double *out, cudaStream_t s) {
  if (elems == 0) return cudaSuccess;
  const int64_t b = (elems + 255) / 256;
  const int grid = (int)(b < 4 * num_sms() ? b : 4 * num_sms());
  k_sum_ordered<<<grid, 256, 0, s>>>(parts, n_parts, elems, out);
  return cudaGetLastError();
}

cudaError_t launch_den_weights(const GramBasis *d_basis, const double *X, int64_t K, int n_v,
                               const double *d_coef, double *S, cudaStream_t s) {
  if (K == 0) return cudaSuccess;
  int64_t b = (K + 255) / 256;
  const int cap = 8 * num_sms();
  k_den_weights<<<(int)(b > cap ? cap : b), 256, 0, s>>>(d_basis, X, K, n_v, d_coef, S);
  return cudaGetLastError();
}

}  // namespace rp
