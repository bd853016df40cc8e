// rp_svd.cu -- NEXT row f1: the homogeneous least-squares problem by singular value decomposition.
//
// "Due to the fact that the system is very ill-conditioned ... we use the computationally more
// intensive yet more numerically stable method of singular value decomposition" (PAPER.md:
// 2601-2615); the linearised system p(x) - V q(x) = 0 is homogeneous (draft footnote PAPER.md:
// 2595-2598), so its least-squares solution is the right singular vector of the smallest
// singular value of A = [M(u) | -V N(u)], scaled so that beta_0 = 1 (reading R12).
//
// B200 design:
//   1. k_tsqr -- Householder TSQR of A without ever writing A to HBM.  One CTA per SM owns a
//      contiguous slab of rows and keeps its triangular factor R packed in shared memory; it
//      absorbs 128-row chunks of design rows generated on chip: every quad of threads owns one
//      column of the chunk in registers (32 rows per lane), so a reflector step reads only the
//      broadcast Householder vector from shared memory (one barrier per column).  The slab
//      factors are merged by a binary tree inside the same launch: the second CTA to reach a
//      tree node stacks [R_left; R_right] (fixed order: deterministic) and re-triangularises;
//      the root writes R.
//   2. k_svd_jacobi -- one-sided (Hestenes) Jacobi SVD of R, one CTA per metric: R lives in
//      shared memory (column-major, 157 KB at n_c = 140), the accumulated rotations V in L2;
//      each round of the round-robin ordering (all pairs disjoint) gives one pair per warp,
//      whose V columns are fetched before the dot products so that their latency overlaps.
//      Singular values are the final column norms.
#include "rp_internal.cuh"

namespace rp {

constexpr int kSvdMaxCols = 144;      // two columns per octet of lanes, 4 octets per warp -> 576 threads
constexpr int kRPL = 12;              // chunk rows per lane (rows l8 + 8 i)
constexpr int kChunk = 8 * kRPL;      // rows per chunk (96)
constexpr int kSD = 36;               // staging stride (32 rows + pad, = 4 mod 16)
constexpr int kTsqrMaxThreads = 576;
constexpr int kJacThreads = 1024;
constexpr int kJacMaxSweeps = 40;

__host__ __device__ inline int64_t packed_off(int i, int nc) {  // start of row i of packed R
  return (int64_t)i * nc - (int64_t)i * (i - 1) / 2;
}
__host__ __device__ inline int64_t packed_size(int nc) { return (int64_t)nc * (nc + 1) / 2; }

struct TsqrArgs {
  const GramBasis *basis;  // design rows from (X, V, S) when `rows` is null
  const double *X, *V, *S;
  const double *rows;      // or dense rows [n_v][K][nc]
  int64_t K;               // rows per metric
  int nc, n, leaves, P;    // P = leaves rounded up to a power of two
  double *slots;           // [n_v][2P][packed]  tree-node factors
  unsigned *counters;      // [n_v][2P]          arrival counters (zero on entry, zero on exit)
  double *R_out;           // [n_v][nc][nc]      final R (upper, zeros below the diagonal)
};

// One chunk of kChunk rows is absorbed into the packed R in shared memory by Householder
// reflectors j = j0 .. nc-1 acting on [R; chunk].  Thread layout: octet o = tid / 8 owns
// columns 2o and 2o + 1 of the chunk in registers (c[h][i] = row l8 + 8 i of column 2o + h,
// l8 = tid % 8).  Reflector j is published by the octet owning column j once it has applied
// reflectors 0 .. j-1 to that column: the scaled vector into RV[j], tau into par[j], beta onto
// the diagonal of R, then flags[j] = seq (release).  Every octet applies the reflectors in order
// as soon as they are published (acquire), so a chunk proceeds as a wavefront over the warps,
// with no block-wide barrier per column.
__device__ __forceinline__ void householder_params(double a, double sub, double &tau, double &beta,
                                                   double &s) {
  // H = I - tau v v^T with v = (1, s * x_sub): H (a, x_sub) = (beta, 0)
  if (sub == 0.0) {
    tau = 0.0;
    beta = a;
    s = 0.0;
  } else {
    const double nrm = sqrt(fma(a, a, sub));
    beta = a >= 0.0 ? -nrm : nrm;
    s = 1.0 / (a - beta);
    tau = (beta - a) / beta;
  }
}

// sum over the 8 lanes of an octet (conditions on the octet's columns keep octets convergent,
// so the mask names only this octet's lanes)
__device__ __forceinline__ double oct_sum(double x) {
  const unsigned m = 0xFFu << (threadIdx.x & 24);
  x += __shfl_xor_sync(m, x, 1);
  x += __shfl_xor_sync(m, x, 2);
  x += __shfl_xor_sync(m, x, 4);
  return x;
}

// Householder vector layout in RV[j]: lane l8's kRPL rows contiguous at l8 * kVS (kVS = 14: the
// eight 16-byte lane segments of a LDS.128 fall in distinct banks, one wavefront per load)
constexpr int kVS = kRPL + 2;
constexpr int kVBuf = 8 * kVS;

__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void publish(double *Rp, double *RV, double *par, int *flags, const double (&c)[kRPL],
                                        int k, int nc, int seq) {
  const int l8 = threadIdx.x & 7;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int i = 0; i < kRPL; i += 2) {
    s0 = fma(c[i], c[i], s0);
    s1 = fma(c[i + 1], c[i + 1], s1);
  }
  const double sub = oct_sum(s0 + s1);
  double *rkk = Rp + packed_off(k, nc);
  double tau, beta, sc;
  householder_params(*rkk, sub, tau, beta, sc);
  double *vn = RV + k * kVBuf + l8 * kVS;
#pragma unroll
  for (int i = 0; i < kRPL; i += 2) *(double2 *)(vn + i) = make_double2(sc * c[i], sc * c[i + 1]);
  __syncwarp(0xFFu << (threadIdx.x & 24));  // the octet's eight slices are written (and ordered)
  if (l8 == 0) {
    par[k] = tau;
    *rkk = beta;
    st_release(flags + k, seq);
  }
}

// reflector j applied to column k (entries c): R[j][k] and c updated
__device__ __forceinline__ void apply_col(double *Rp, double (&c)[kRPL], const double (&v)[kRPL], double tau,
                                          int j, int k, int nc) {
  double d0 = 0.0, d1 = 0.0;
#pragma unroll
  for (int i = 0; i < kRPL; i += 2) {
    d0 = fma(v[i], c[i], d0);
    d1 = fma(v[i + 1], c[i + 1], d1);
  }
  const double dot = oct_sum(d0 + d1);
  double *rjk = Rp + packed_off(j, nc) + (k - j);
  const double tw = tau * (*rjk + dot);
#pragma unroll
  for (int i = 0; i < kRPL; ++i) c[i] = fma(-tw, v[i], c[i]);
  if ((threadIdx.x & 7) == 0) *rjk -= tw;
}

__device__ __forceinline__ void absorb_chunk(double *Rp, double *RV, double *par, int *flags,
                                             double (&c)[2][kRPL], int nc, int j0, int seq) {
  const int o = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int k0 = 2 * o, k1 = 2 * o + 1;
  const int w0 = (threadIdx.x >> 5) * 8;  // first column of this warp
  __syncthreads();                        // RV aliases the staging buffer of the chunk fill
  if (w0 < nc && w0 + 7 >= j0) {
    if (k0 == j0 && k0 < nc) publish(Rp, RV, par, flags, c[0], k0, nc, seq);
    if (k1 == j0 && k1 < nc) publish(Rp, RV, par, flags, c[1], k1, nc, seq);
    const int jend = min(w0 + 7, nc - 1);  // reflectors this warp needs: j < its last column
    for (int j = j0; j < jend; ++j) {
      if (j < w0) {
        // warps far behind the wavefront front back off longer: spinning steals issue slots
        // from the warp on the critical path (the owner of column j + 1)
        const unsigned ns = (w0 - j) > 16 ? 256u : 16u;
        while (ld_acquire(flags + j) != seq) __nanosleep(ns);
      } else {
        __syncwarp();  // published by an octet of this warp at iteration j - 1
      }
      const bool a0 = k0 > j && k0 < nc, a1 = k1 > j && k1 < nc;
      if (a1) {  // k1 > j whenever k0 > j
        double v[kRPL];
        const double *vs = RV + j * kVBuf + l8 * kVS;
#pragma unroll
        for (int i = 0; i < kRPL; i += 2) {
          const double2 t = *(const double2 *)(vs + i);
          v[i] = t.x;
          v[i + 1] = t.y;
        }
        const double tau = par[j];
        if (a0) apply_col(Rp, c[0], v, tau, j, k0, nc);
        apply_col(Rp, c[1], v, tau, j, k1, nc);
        if (k0 == j + 1 && a0) publish(Rp, RV, par, flags, c[0], k0, nc, seq);
        if (k1 == j + 1) publish(Rp, RV, par, flags, c[1], k1, nc, seq);
      }
    }
  }
  __syncthreads();
}

// rows [r0, r0 + kChunk) of R2 (packed, global) as chunk entries of columns 2o, 2o + 1
__device__ __forceinline__ void fill_from_packed(double (&c)[2][kRPL], const double *R2, int nc, int r0) {
  const int o = threadIdx.x >> 3, l8 = threadIdx.x & 7;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = 2 * o + h;
#pragma unroll
    for (int i = 0; i < kRPL; ++i) {
      const int rho = r0 + l8 + 8 * i;
      c[h][i] = (k < nc && rho < nc && k >= rho) ? __ldcg(R2 + packed_off(rho, nc) + (k - rho)) : 0.0;
    }
  }
}

__device__ __forceinline__ void absorb_packed(double *Rp, double *RV, double *par, int *flags, const double *R2,
                                              int nc, int &seq) {
  double c[2][kRPL];
  for (int r0 = 0; r0 < nc; r0 += kChunk) {
    fill_from_packed(c, R2, nc, r0);
    absorb_chunk(Rp, RV, par, flags, c, nc, r0, ++seq);  // rows >= r0 are zero left of column r0
  }
}

__host__ __device__ inline int64_t tsqr_rv_elems(int nc) {  // reflector store, aliased by sD
  const int64_t rv = (int64_t)nc * kVBuf, sd = (int64_t)kSD * kSvdMaxCols;
  return rv > sd ? rv : sd;
}

// Shared memory: Rp [packed] | RV [nc][kVBuf] (aliased by sD [144][kSD] during the fill) |
// par [144] | sU [8][kChunk] | flags [144] | flag
__global__ void __maxnreg__(96) k_tsqr(TsqrArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nc = a.nc, n = a.n;
  const int64_t psz = packed_size(nc);
  double *Rp = sm;
  double *RV = Rp + ((psz + 1) & ~1ll);
  double *sD = RV;
  double *par = RV + tsqr_rv_elems(nc);
  double *sU = par + kSvdMaxCols;
  int *flags = (int *)(sU + kChunk * kMaxVars);
  int *flag = flags + kSvdMaxCols;
  int seq = 0;
  const int metric = blockIdx.y;
  const int leaf = blockIdx.x;
  const int o = threadIdx.x >> 3, l8 = threadIdx.x & 7;

  for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) Rp[i] = 0.0;
  for (int i = threadIdx.x; i < kSvdMaxCols; i += blockDim.x) flags[i] = 0;
  __syncthreads();

  // ---- leaf: the slab's rows ----------------------------------------------------------------
  const int64_t r_begin = a.K * leaf / a.leaves, r_end = a.K * (leaf + 1) / a.leaves;
  const double *V = a.V ? a.V + (int64_t)metric * a.K : nullptr;
  const double *S = a.S ? a.S + (int64_t)metric * a.K : nullptr;
  const double *rows = a.rows ? a.rows + (int64_t)metric * a.K * nc : nullptr;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kChunk) {
    const int cnt = (int)((r_end - r0) < kChunk ? (r_end - r0) : kChunk);
    if (!rows) {
      // a10: u = (x - c) 2^-e of the chunk's rows (variable-major: conflict-free reads below)
      for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
        const int r = i / n, t = i % n;
        sU[t * kChunk + r] = (a.X[(r0 + r) * n + t] - a.basis->xc[t]) * ldexp(1.0, -a.basis->xe[t]);
      }
    }
    // the chunk's entries are staged through sD in passes of 32 rows (column-major, stride
    // kSD = 36: the octet-row read pattern is conflict-free), then picked up into registers
    double c[2][kRPL];
#pragma unroll
    for (int ps = 0; ps < kChunk / 32; ++ps) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < nc * 32; idx += blockDim.x) {
        const int col = idx >> 5, rr = idx & 31, r = ps * 32 + rr;
        double m = 0.0;
        if (r < cnt) {
          if (rows) {
            m = rows[(r0 + r) * nc + col];
          } else {
            // a11: design row entry: M_col(u), or -V N_col(u) (times the row scale S)
            m = 1.0;
            for (int t = 0; t < n; ++t) {
              const double u = sU[t * kChunk + r];
              for (int e = 0; e < a.basis->exp[col][t]; ++e) m *= u;
            }
            if (col >= a.basis->n_num) m *= -V[r0 + r];
            if (S) m *= S[r0 + r];
          }
        }
        sD[col * kSD + rr] = m;
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
          c[h][ps * 4 + ii] = 2 * o + h < nc ? sD[(2 * o + h) * kSD + l8 + 8 * ii] : 0.0;
    }
    absorb_chunk(Rp, RV, par, flags, c, nc, 0, ++seq);
  }

  // ---- tree merge (heap numbering: leaves P .. P + leaves - 1, root 1) -------------------------
  double *slots = a.slots + (int64_t)metric * 2 * a.P * psz;
  unsigned *cnt = a.counters + (int64_t)metric * 2 * a.P;
  int node = a.P + leaf, h = 0;
  while (node > 1) {
    const int sib = node ^ 1;
    if ((int64_t)(sib << h) - a.P >= a.leaves) {  // no leaf under the sibling: pass through
      node >>= 1;
      ++h;
      continue;
    }
    double *mine = slots + (int64_t)node * psz;
    for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) mine[i] = Rp[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned old = atomicAdd(&cnt[node >> 1], 1u);
      if (old == 1u) {
        cnt[node >> 1] = 0u;  // both children arrived: reset for the next call
        __threadfence();
      }
      *flag = (int)old;
    }
    __syncthreads();
    if (*flag == 0) return;  // first to arrive: the sibling's CTA continues
    const double *other = slots + (int64_t)sib * psz;
    if (node & 1) {  // right child: R := R_left, then absorb my own rows
      for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) Rp[i] = __ldcg(other + i);
      __syncthreads();
      absorb_packed(Rp, RV, par, flags, mine, nc, seq);
    } else {
      absorb_packed(Rp, RV, par, flags, other, nc, seq);
    }
    node >>= 1;
    ++h;
  }
  // root: the factor of all K rows
  double *Ro = a.R_out + (int64_t)metric * nc * nc;
  for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) {
    const int r = i / nc, col = i % nc;
    Ro[i] = col >= r ? Rp[packed_off(r, nc) + (col - r)] : 0.0;
  }
}

// ============================================================================================
// one-sided Jacobi SVD of R (one CTA per metric)
// ============================================================================================
struct JacArgs {
  const double *R;  // [n_v][nc][nc] row-major (any square matrix works)
  int nc, n_num;
  double *V;        // [n_v][nc][nc] workspace: accumulated rotations, column-major (L2-resident)
  double *coef;     // [n_v][nc]
  double *sigma;    // [n_v][nc] ascending
  double *info;     // [n_v][6]: status, rank, resid2, sigma_min, sigma_max / sigma_min, sweeps
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

constexpr int kJacPer16 = (kSvdMaxCols + 15) / 16;  // column entries per lane of a 16-lane pair group

// Shared memory: A [nc][ld] column-major (ld odd) | sched [np-1][np/2] (p, q as uint8 pairs) |
// sig [nc] | ctl[4]
__global__ void __launch_bounds__(kJacThreads, 1) k_svd_jacobi(JacArgs a) {
  extern __shared__ __align__(16) double sj[];
  const int nc = a.nc, ld = nc | 1;
  const int np = (nc + 1) & ~1;  // players (a dummy when nc is odd)
  const int npairs = np / 2, nrounds = np - 1;
  double *A = sj;
  uint16_t *sched = (uint16_t *)(A + (int64_t)nc * ld);
  double *sig = (double *)(sched + ((nrounds * npairs + 3) & ~3));
  int *ctl = (int *)(sig + kSvdMaxCols);
  const int metric = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double *R = a.R + (int64_t)metric * nc * nc;
  double *V = a.V + (int64_t)metric * nc * nc;

  for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) {
    const int r = i / nc, col = i % nc;
    A[col * ld + r] = R[i];
    V[i] = (i % (nc + 1)) == 0 ? 1.0 : 0.0;  // V = I (column-major == row-major for I)
  }
  // round-robin tournament: position 0 fixed, the others rotate; pair m of round t is
  // (pos m, pos np-1-m).  Stored as (min, max) so every rotation acts on (p < q).
  for (int i = threadIdx.x; i < nrounds * npairs; i += blockDim.x) {
    const int t = i / npairs, m = i % npairs;
    const int pm = m == 0 ? 0 : 1 + (m - 1 + t) % (np - 1);
    const int pq = 1 + (np - 2 - m + t) % (np - 1);
    const int p = pm < pq ? pm : pq, q = pm < pq ? pq : pm;
    sched[i] = (uint16_t)(p | (q << 8));
  }
  if (threadIdx.x < 4) ctl[threadIdx.x] = 0;
  __syncthreads();

  const double tol = 1e-15 * sqrt((double)nc);
  int sweep = 0;
  for (; sweep < kJacMaxSweeps; ++sweep) {
    const int flag = sweep & 1;  // ctl[flag]: something rotated in this sweep
    for (int t = 0; t < nrounds; ++t) {
      // 16 lanes per pair, 2 pairs per warp: the scalar rotation math is shared by half a warp
      // instead of repeated by all 32 lanes (the FP64 pipe is the bottleneck of a round)
      for (int m0 = wid * 2; m0 < npairs; m0 += nw * 2) {
        const int m = m0 + (lane >> 4), l16 = lane & 15;
        const unsigned pqv = m < npairs ? sched[t * npairs + m] : 0xffffu;
        const int p = pqv & 0xff, q = pqv >> 8;
        const bool valid = q < nc;
        double *ap = A + (valid ? p : 0) * ld, *aq = A + (valid ? q : 0) * ld;
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int i = 0; i < kJacPer16; ++i) {
          const int r = l16 + 16 * i;
          const double x = (valid && r < nc) ? ap[r] : 0.0;
          const double y = (valid && r < nc) ? aq[r] : 0.0;
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (valid && ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          double *vp = V + (int64_t)p * nc, *vq = V + (int64_t)q * nc;
          double xv[kJacPer16], yv[kJacPer16];
#pragma unroll
          for (int i = 0; i < kJacPer16; ++i) {  // issued before the rotation math: latency overlap
            const int r = l16 + 16 * i;
            xv[i] = r < nc ? __ldcg(vp + r) : 0.0;
            yv[i] = r < nc ? __ldcg(vq + r) : 0.0;
          }
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double cs = 1.0 / sqrt(fma(tt, tt, 1.0));
          const double sn = cs * tt;
#pragma unroll
          for (int i = 0; i < kJacPer16; ++i) {
            const int r = l16 + 16 * i;
            if (r < nc) {  // A re-read from shared memory (fewer live registers)
              const double x = ap[r], y = aq[r];
              ap[r] = cs * x - sn * y;
              aq[r] = sn * x + cs * y;
              __stcg(vp + r, cs * xv[i] - sn * yv[i]);
              __stcg(vq + r, sn * xv[i] + cs * yv[i]);
            }
          }
          if (l16 == 0) ctl[flag] = 1;
        }
      }
      __syncthreads();
    }
    const int rotated = ctl[flag];
    if (threadIdx.x == 0) ctl[flag ^ 1] = 0;  // next sweep's flag (nobody writes it before the barrier)
    __syncthreads();
    if (!rotated) break;
  }

  // ---- singular values = column norms; the vector of the smallest -------------------------------
  for (int col = wid; col < nc; col += nw) {
    double s2 = 0.0;
    for (int r = lane; r < nc; r += 32) s2 = fma(A[col * ld + r], A[col * ld + r], s2);
    s2 = warp_sum(s2);
    if (lane == 0) sig[col] = sqrt(s2);
  }
  __syncthreads();
  double *so = a.sigma + (int64_t)metric * nc;
  for (int col = threadIdx.x; col < nc; col += blockDim.x) {  // ascending by rank counting
    const double v = sig[col];
    int rank = 0;
    for (int o = 0; o < nc; ++o) rank += (sig[o] < v) || (sig[o] == v && o < col);
    so[rank] = v;
    if (rank == 0) ctl[2] = col;
  }
  __syncthreads();
  const int jm = ctl[2];
  const double *vm = V + (int64_t)jm * nc;
  const double b0 = __ldcg(vm + a.n_num);
  const bool bad = !(fabs(b0) > 1e-300);
  for (int r = threadIdx.x; r < nc; r += blockDim.x)
    a.coef[(int64_t)metric * nc + r] = bad ? __longlong_as_double(0x7ff8000000000000ll) : __ldcg(vm + r) / b0;
  if (threadIdx.x == 0) {
    const double smin = sig[jm];
    double smax = sig[0];
    for (int o = 1; o < nc; ++o) smax = fmax(smax, sig[o]);
    int rank = 0;
    for (int o = 0; o < nc; ++o) rank += sig[o] > 1e-13 * smax;
    double *inf = a.info + metric * 6;
    inf[0] = bad ? (double)RP_ERR_DEGENERATE : 0.0;
    inf[1] = rank;
    inf[2] = (smin / b0) * (smin / b0);  // ||A coef||^2 with coef = v / v[beta_0], ||v|| = 1
    inf[3] = smin;
    inf[4] = smax / smin;
    inf[5] = sweep + 1;
  }
}

// ============================================================================================
// launchers
// ============================================================================================
static int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

int tsqr_leaves(int64_t K, int n_v) {
  const int64_t want = (K + kChunk - 1) / kChunk;
  int cap = num_sms() / (n_v > 0 ? n_v : 1);
  if (cap < 1) cap = 1;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

size_t tsqr_workspace_bytes(int nc, int n_v, int leaves) {
  const int P = pow2_ceil(leaves);
  return (size_t)n_v * 2 * P * packed_size(nc) * 8 + (size_t)n_v * 2 * P * sizeof(unsigned) + 64;
}

static size_t tsqr_smem(int nc) {
  return (size_t)((packed_size(nc) + 1) & ~1ll) * 8 + (size_t)tsqr_rv_elems(nc) * 8 + kSvdMaxCols * 8 +
         (size_t)kChunk * kMaxVars * 8 + (kSvdMaxCols + 4) * 4;
}

cudaError_t launch_tsqr(const GramBasis *d_basis, const double *X, const double *V, const double *S,
                        const double *rows, int64_t K, int n, int nc, int n_v, void *ws, size_t ws_bytes,
                        double *R_out, cudaStream_t s) {
  if (nc < 1 || nc > kSvdMaxCols) return cudaErrorInvalidValue;
  const int leaves = tsqr_leaves(K, n_v);
  const int P = pow2_ceil(leaves);
  if (tsqr_workspace_bytes(nc, n_v, leaves) > ws_bytes) return cudaErrorInvalidValue;
  TsqrArgs a{};
  a.basis = d_basis;
  a.X = X;
  a.V = V;
  a.S = S;
  a.rows = rows;
  a.K = K;
  a.nc = nc;
  a.n = n;
  a.leaves = leaves;
  a.P = P;
  a.slots = (double *)ws;
  a.counters = (unsigned *)((char *)ws + (size_t)n_v * 2 * P * packed_size(nc) * 8);
  a.R_out = R_out;
  cudaError_t e = cudaMemsetAsync(a.counters, 0, (size_t)n_v * 2 * P * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  const size_t smem = tsqr_smem(nc);
  e = cudaFuncSetAttribute(k_tsqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = 32 * ((nc + 7) / 8);  // 4 octets (8 columns) per warp
  k_tsqr<<<dim3(leaves, n_v), threads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_svd_jacobi(const double *R, int nc, int n_num, int n_v, double *V_ws, double *coef,
                              double *sigma, double *info, cudaStream_t s) {
  if (nc < 2 || nc > kSvdMaxCols) return cudaErrorInvalidValue;
  const int np = (nc + 1) & ~1;
  const size_t smem = (size_t)nc * (nc | 1) * 8 + (size_t)(((np - 1) * (np / 2) + 3) & ~3) * 2 +
                      kSvdMaxCols * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(k_svd_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  JacArgs a{R, nc, n_num, V_ws, coef, sigma, info};
  k_svd_jacobi<<<n_v, kJacThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rp
