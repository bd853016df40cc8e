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
//   2. k_svd_gk (default) -- the SVD of R by Householder bidiagonalisation, bisection on the
//      Golub-Kahan tridiagonal for every singular value and inverse iteration for the vector of
//      the smallest (one CTA per metric, R in shared memory; below).  k_svd_jacobi
//      (RP_SVD_SOLVER=jacobi) -- one-sided (Hestenes) Jacobi SVD of R, R in shared memory
//      (column-major, 157 KB at n_c = 140), the accumulated rotations V in L2; each round of the
//      round-robin ordering (all pairs disjoint) gives one pair per warp.  Singular values are the
//      final column norms.
#include <cstdlib>
#include <cstring>

#include "rp_internal.cuh"
#include "rp_umma.cuh"
#include "rp_device.cuh"

namespace rp {

constexpr int kSvdMaxCols = 144;      // two columns per octet of lanes, 4 octets per warp -> 576 threads
constexpr int kRPL = 12;              // chunk rows per lane (rows l8 + 8 i)
constexpr int kChunk = 8 * kRPL;      // rows per chunk (96)
constexpr int kSD = 36;               // staging stride (32 rows + pad, = 4 mod 16)
constexpr int kTsqrMaxThreads = 576;
constexpr int kJacThreads = 1024;
constexpr int kJacMaxSweeps = 40;
constexpr int kGkThreads = 512;  // k_svd_gk

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
  // (on the wavefront's critical path: MUFU seeds with Newton steps instead of IEEE sqrt and
  // division, ~1 ulp; the reflector stays exactly orthogonal in exact arithmetic for any s)
  if (sub == 0.0) {
    tau = 0.0;
    beta = a;
    s = 0.0;
  } else {
    const double x = fma(a, a, sub);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-0.5 * x * y, y, 0.5), y);  // y <- y (3 - x y^2) / 2, twice
    y = fma(y, fma(-0.5 * x * y, y, 0.5), y);
    double nrm = x * y;
    nrm = fma(0.5 * y, fma(-nrm, nrm, x), nrm);  // one Newton step on the root itself
    beta = a >= 0.0 ? -nrm : nrm;
    const double den = a - beta;  // |den| = |a| + nrm > 0
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    double ee = fma(-den, r, 1.0);
    r = fma(r, fma(ee, ee, ee), r);
    s = r;
    double rb;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rb) : "d"(beta));
    ee = fma(-beta, rb, 1.0);
    rb = fma(rb, fma(ee, ee, ee), rb);
    tau = (beta - a) * rb;
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

// ============================================================================================
// k_tsqr_b -- the blocked form of k_tsqr (RP_TSQR_KERNEL=blocked; measured 44.2 ms for fit_svd
// against 34.2 with the wavefront k_tsqr: the one-warp panel factorisation, ~6-8k cycles per
// 8 columns, is the critical path and the other warps wait at the panel barrier).
// Same slabs, chunks and tree as k_tsqr, but each chunk C (96 design rows, row-major in shared
// memory) is absorbed into [R; C] panel by panel (8 columns): one warp factors the panel with
// its 96 x 8 entries in registers (the column chain runs inside the warp: shuffle reductions,
// no cross-warp hand-off), forms the compact-WY factor T (H_0 ... H_7 = I - V T V^T, the unit
// parts of the reflectors on R's rows c0 .. c0 + 7, their C parts in V), and the block reflector
// goes to the trailing columns on DMMA, one 8-column tile per warp: Y = V^T [R; C], Z = T^T Y,
// [R; C] -= V Z (LAPACK's dlarft / dlarfb, forward columnwise), with a one-panel look-ahead.
// ============================================================================================
constexpr int kTbThreads = 512;
constexpr int kTbPW = 8;                 // panel width
constexpr int kTbLdC = (kSvdMaxCols + 8) | 1;  // C row stride (odd; room for a last column tile)

__host__ __device__ inline size_t tsqr_b_smem(int nc) {
  return (size_t)((packed_size(nc) + 1) & ~1ll) * 8 + (size_t)kChunk * kTbLdC * 8 + 2 * (size_t)kChunk * kTbPW * 8 +
         2 * kTbPW * kTbPW * 8 + 64;
}

// batched sum over the warp of NV values (xor butterfly: every lane gets every sum)
template <int NV>
__device__ __forceinline__ void warp_sum_n(double (&x)[NV]) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i] += __shfl_xor_sync(0xffffffffu, x[i], o);
}

// Panel factorisation by one warp: columns c0 .. c0 + w - 1 of [R; C] (lane: C rows lane + 32 t
// in registers).  Writes V (the reflectors' C parts, zero beyond w), tau, T (compact WY,
// row-major 8 x 8) and R's panel rows at the panel's columns.
__device__ void tb_panel(double *Rp, const double *sC, double *sV, double *sT, int nc, int c0, int w) {
  const int lane = threadIdx.x & 31;
  double pc[3][kTbPW];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int j = 0; j < kTbPW; ++j) pc[t][j] = j < w ? sC[(lane + 32 * t) * kTbLdC + c0 + j] : 0.0;
  double tauv[kTbPW];
#pragma unroll
  for (int j = 0; j < kTbPW; ++j) {
    tauv[j] = 0.0;
    if (j >= w) continue;
    double *rr = Rp + packed_off(c0 + j, nc) - (c0 + j);  // rr[c] = R[c0 + j][c]
    double rk[kTbPW];
#pragma unroll
    for (int k = 0; k < kTbPW; ++k) rk[k] = (k >= j && k < w) ? rr[c0 + k] : 0.0;  // (issued early)
    double s2[1] = {0.0};
#pragma unroll
    for (int t = 0; t < 3; ++t) s2[0] = fma(pc[t][j], pc[t][j], s2[0]);
    warp_sum_n<1>(s2);
    double tau, beta, sc;
    householder_params(rk[j], s2[0], tau, beta, sc);
    tauv[j] = tau;
#pragma unroll
    for (int t = 0; t < 3; ++t) pc[t][j] *= sc;
    // reflector j on the panel's columns k > j: dot_k = R[c0+j][c0+k] + v^T C[:, c0+k]
    double d[kTbPW];
#pragma unroll
    for (int k = 0; k < kTbPW; ++k) {
      d[k] = 0.0;
      if (k > j)
#pragma unroll
        for (int t = 0; t < 3; ++t) d[k] = fma(pc[t][j], pc[t][k], d[k]);
    }
    warp_sum_n<kTbPW>(d);
    double tw[kTbPW];
#pragma unroll
    for (int k = 0; k < kTbPW; ++k) {
      tw[k] = (k > j && k < w) ? tau * (rk[k] + d[k]) : 0.0;
#pragma unroll
      for (int t = 0; t < 3; ++t) pc[t][k] = fma(-tw[k], pc[t][j], pc[t][k]);
    }
    __syncwarp();  // every lane has read R[c0 + j][.]
    if (lane == j) rr[c0 + j] = beta;
#pragma unroll
    for (int k = 0; k < kTbPW; ++k)
      if (lane == k && k > j && k < w) rr[c0 + k] = rk[k] - tw[k];
  }
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int j = 0; j < kTbPW; ++j) sV[(lane + 32 * t) * kTbPW + j] = j < w ? pc[t][j] : 0.0;
  // T (dlarft, forward columnwise): G[m][i] = v_m^T v_i (the unit parts sit on distinct R rows),
  // T[i][i] = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] G[0:i, i]; lane jr keeps row jr of T
  double g[kTbPW * (kTbPW - 1) / 2];
  {
    int q = 0;
#pragma unroll
    for (int i = 1; i < kTbPW; ++i)
#pragma unroll
      for (int m = 0; m < i; ++m, ++q) {
        g[q] = 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) g[q] = fma(pc[t][m], pc[t][i], g[q]);
      }
  }
  warp_sum_n<kTbPW * (kTbPW - 1) / 2>(g);
  double trow[kTbPW];
#pragma unroll
  for (int i = 0; i < kTbPW; ++i) trow[i] = 0.0;
  {
    int q = 0;
#pragma unroll
    for (int i = 0; i < kTbPW; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < kTbPW; ++m)
        if (m < i) acc = fma(lane <= m ? trow[m] : 0.0, g[q + m], acc);  // T[jr][m] = 0 for m < jr
      trow[i] = lane == i ? tauv[i] : (lane < i ? -tauv[i] * acc : 0.0);
      q += i;
    }
  }
  if (lane < kTbPW)
#pragma unroll
    for (int i = 0; i < kTbPW; ++i) sT[lane * kTbPW + i] = trow[i];
}

// One 8-column trailing tile (columns col0 .. col0 + 7) by one warp, with the panel's V and T:
// Y = V^T C + R_panel (DMMA, two chains), Z = T^T Y (shuffles), R_panel -= Z, C -= V Z (DMMA).
__device__ void tb_tile(double *Rp, double *sC, const double *sV, const double *sT, int nc, int c0, int w, int col0) {
  const int lane = threadIdx.x & 31, r = lane >> 2, q = lane & 3;
  const int ca = col0 + 2 * q, cb = ca + 1;  // this lane's accumulator columns
  double y0 = 0.0, y1 = 0.0, u0 = 0.0, u1 = 0.0;
  if (r < w) {
    const double *rr = Rp + packed_off(c0 + r, nc) - (c0 + r);
    if (ca < nc) y0 = rr[ca];
    if (cb < nc) y1 = rr[cb];
  }
#pragma unroll 4
  for (int ks = 0; ks < kChunk / 4; ks += 2) {
    const double a0 = sV[(ks * 4 + q) * kTbPW + r], b0 = sC[(ks * 4 + q) * kTbLdC + col0 + r];
    const double a1 = sV[(ks * 4 + 4 + q) * kTbPW + r], b1 = sC[(ks * 4 + 4 + q) * kTbLdC + col0 + r];
    dmma(y0, y1, a0, b0);
    dmma(u0, u1, a1, b1);
  }
  y0 += u0;
  y1 += u1;
  // Z[r][c] = sum_{j <= r} T[j][r] Y[j][c]: Y[j][2q..2q+1] sits in lane 4 j + q
  double z0 = 0.0, z1 = 0.0;
#pragma unroll
  for (int jj = 0; jj < kTbPW; ++jj) {
    const double yj0 = __shfl_sync(0xffffffffu, y0, 4 * jj + q);
    const double yj1 = __shfl_sync(0xffffffffu, y1, 4 * jj + q);
    if (jj <= r) {
      const double t = sT[jj * kTbPW + r];
      z0 = fma(t, yj0, z0);
      z1 = fma(t, yj1, z1);
    }
  }
  if (r < w) {
    double *rr = Rp + packed_off(c0 + r, nc) - (c0 + r);
    if (ca < nc) rr[ca] -= z0;
    if (cb < nc) rr[cb] -= z1;
  }
  // B fragments of Z for C -= V Z: lane (r, q) needs Z[4 h + q][r], held by lane
  // 4 (4 h + q) + r / 2 in slot r % 2
  double bz[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int src = 4 * (4 * h + q) + (r >> 1);
    const double s0 = __shfl_sync(0xffffffffu, z0, src), s1 = __shfl_sync(0xffffffffu, z1, src);
    bz[h] = (r & 1) ? s1 : s0;
  }
#pragma unroll 2
  for (int mt = 0; mt < kChunk / 8; ++mt) {
    double *cr = sC + (mt * 8 + r) * kTbLdC + col0 + 2 * q;
    double d0 = cr[0], d1 = cr[1];
    const double va = -sV[(mt * 8 + r) * kTbPW + q], vb = -sV[(mt * 8 + r) * kTbPW + 4 + q];
    dmma(d0, d1, va, bz[0]);
    dmma(d0, d1, vb, bz[1]);
    cr[0] = d0;
    cr[1] = d1;
  }
}

// absorb C (rows 0 .. kChunk-1 of sC; zero rows beyond the data) into the packed R, with a
// look-ahead of one panel: while warps 1.. apply panel p to the trailing tiles 1.., warp 0
// applies it to tile 0 (panel p + 1's columns) and factors panel p + 1 (V, T double-buffered)
__device__ void absorb_chunk_b(double *Rp, double *sC, double *sV, double *sT, int nc) {
  const int wid = threadIdx.x >> 5, nw = kTbThreads / 32;
  if (wid == 0) tb_panel(Rp, sC, sV, sT, nc, 0, min(kTbPW, nc));
  __syncthreads();
  for (int p = 0, c0 = 0; c0 < nc; ++p, c0 += kTbPW) {
    const int w = min(kTbPW, nc - c0), c1 = c0 + w;
    const double *V = sV + (p & 1) * kChunk * kTbPW, *T = sT + (p & 1) * kTbPW * kTbPW;
    const int ntile = (nc - c1 + 7) / 8;
    if (wid == 0) {
      if (ntile > 0) {
        tb_tile(Rp, sC, V, T, nc, c0, w, c1);
        __syncwarp();
        tb_panel(Rp, sC, sV + ((p + 1) & 1) * kChunk * kTbPW, sT + ((p + 1) & 1) * kTbPW * kTbPW, nc, c1,
                 min(kTbPW, nc - c1));
      }
    } else {
      for (int tt = wid; tt < ntile; tt += nw - 1) tb_tile(Rp, sC, V, T, nc, c0, w, c1 + 8 * tt);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kTbThreads, 1) k_tsqr_b(TsqrArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nc = a.nc, n = a.n;
  const int64_t psz = packed_size(nc);
  double *Rp = sm;
  double *sC = Rp + ((psz + 1) & ~1ll);
  double *sV = sC + (size_t)kChunk * kTbLdC;      // [2][kChunk][8]  V of the current / next panel
  double *sT = sV + 2 * (size_t)kChunk * kTbPW;   // [2][8][8]
  int *flag = (int *)(sT + 2 * kTbPW * kTbPW);
  const int metric = blockIdx.y;
  const int leaf = blockIdx.x;

  for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) Rp[i] = 0.0;
  __syncthreads();
  const int64_t r_begin = a.K * leaf / a.leaves, r_end = a.K * (leaf + 1) / a.leaves;
  const double *V = a.V ? a.V + (int64_t)metric * a.K : nullptr;
  const double *S = a.S ? a.S + (int64_t)metric * a.K : nullptr;
  const double *rows = a.rows ? a.rows + (int64_t)metric * a.K * nc : nullptr;
  const GramBasis *B = a.basis;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kChunk) {
    const int cnt = (int)((r_end - r0) < kChunk ? (r_end - r0) : kChunk);
    // a10 + a11: the chunk's design rows (one thread per entry; rows beyond cnt are zero)
    for (int idx = threadIdx.x; idx < kChunk * nc; idx += blockDim.x) {
      const int r = idx / nc, col = idx % nc;
      double m = 0.0;
      if (r < cnt) {
        const int64_t row = r0 + r;
        if (rows) {
          m = rows[row * nc + col];
        } else {
          m = 1.0;
          for (int t = 0; t < n; ++t) {
            const int e = B->exp[col][t];
            if (e) {
              const double u = (a.X[row * n + t] - B->xc[t]) * ldexp(1.0, -B->xe[t]);
              for (int q = 0; q < e; ++q) m *= u;
            }
          }
          if (col >= B->n_num) m *= -V[row];
          if (S) m *= S[row];
        }
      }
      sC[r * kTbLdC + col] = m;
    }
    __syncthreads();
    absorb_chunk_b(Rp, sC, sV, sT, nc);
  }
  // ---- tree merge (as k_tsqr) ---------------------------------------------------------------
  double *slots = a.slots + (int64_t)metric * 2 * a.P * psz;
  unsigned *cntr = a.counters + (int64_t)metric * 2 * a.P;
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
      const unsigned old = atomicAdd(&cntr[node >> 1], 1u);
      if (old == 1u) {
        cntr[node >> 1] = 0u;  // both children arrived: reset for the next call
        __threadfence();
      }
      *flag = (int)old;
    }
    __syncthreads();
    if (*flag == 0) return;  // first to arrive: the sibling's CTA continues
    const double *other = slots + (int64_t)sib * psz;
    const double *R2 = other;
    if (node & 1) {  // right child: R := R_left, then absorb my own rows
      for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) Rp[i] = __ldcg(other + i);
      R2 = mine;
    }
    __syncthreads();
    for (int r0 = 0; r0 < nc; r0 += kChunk) {  // R2's rows as chunks
      for (int idx = threadIdx.x; idx < kChunk * nc; idx += blockDim.x) {
        const int r = idx / nc, col = idx % nc, rho = r0 + r;
        sC[r * kTbLdC + col] = (rho < nc && col >= rho) ? __ldcg(R2 + packed_off(rho, nc) + (col - rho)) : 0.0;
      }
      __syncthreads();
      absorb_chunk_b(Rp, sC, sV, sT, nc);
    }
    node >>= 1;
    ++h;
  }
  double *Ro = a.R_out + (int64_t)metric * nc * nc;
  for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) {
    const int r = i / nc, col = i % nc;
    Ro[i] = col >= r ? Rp[packed_off(r, nc) + (col - r)] : 0.0;
  }
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
  const char *kv = getenv("RP_TSQR_KERNEL");
  if (kv && strcmp(kv, "blocked") == 0) {
    const size_t smb = tsqr_b_smem(nc);
    e = cudaFuncSetAttribute(k_tsqr_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    if (e != cudaSuccess) return e;
    k_tsqr_b<<<dim3(leaves, n_v), kTbThreads, smb, s>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = tsqr_smem(nc);
  e = cudaFuncSetAttribute(k_tsqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = 32 * ((nc + 7) / 8);  // 4 octets (8 columns) per warp
  k_tsqr<<<dim3(leaves, n_v), threads, smem, s>>>(a);
  return cudaGetLastError();
}

__global__ void k_svd_gk(JacArgs a);
static bool svd_use_jacobi();

cudaError_t launch_svd_jacobi(const double *R, int nc, int n_num, int n_v, double *V_ws, double *coef,
                              double *sigma, double *info, cudaStream_t s) {
  if (nc < 2 || nc > kSvdMaxCols) return cudaErrorInvalidValue;
  if (!svd_use_jacobi()) {
    const size_t smem = ((size_t)nc * (nc | 1) + 20 * (size_t)nc + 16) * 8;
    cudaError_t e = cudaFuncSetAttribute(k_svd_gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    JacArgs a{R, nc, n_num, V_ws, coef, sigma, info};
    k_svd_gk<<<n_v, kGkThreads, smem, s>>>(a);
    return cudaGetLastError();
  }
  const int np = (nc + 1) & ~1;
  const size_t smem = (size_t)nc * (nc | 1) * 8 + (size_t)(((np - 1) * (np / 2) + 3) & ~3) * 2 +
                      kSvdMaxCols * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(k_svd_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  JacArgs a{R, nc, n_num, V_ws, coef, sigma, info};
  k_svd_jacobi<<<n_v, kJacThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================================
// k_svd_gk -- the SVD of R by Householder bidiagonalisation, bisection on the Golub-Kahan
// tridiagonal and inverse iteration (default; RP_SVD_SOLVER=jacobi keeps k_svd_jacobi).
//
//   1. R = U B V^T, B upper bidiagonal (d, e): left and right Householder reflectors alternately,
//      A in shared memory (column-major, odd stride); the right reflectors stay in A's rows.
//   2. All singular values by bisection on T_GK, the 2n x 2n symmetric tridiagonal with zero
//      diagonal and off-diagonal (d0, e0, d1, e1, ..., d_{n-1}), whose eigenvalues are
//      +-sigma_i: sigma_i is where the Sturm count (eigenvalues < x) passes n + i.  Four threads
//      per value (quadrisection), 30 rounds: absolute accuracy ~ u ||B||.
//   3. The vector of sigma_min by inverse iteration on T_GK - sigma_min I (tridiagonal LU with
//      partial pivoting): the even entries of the eigenvector are B's right singular vector (the
//      +-sigma_min pair shares them, so a tiny sigma_min does not matter), then V applies the right
//      reflectors in reverse.  Clustered sigma_min: any vector of the cluster (reading R30).
// Same outputs as k_svd_jacobi: coef = v / v[n_num], sigma ascending, info[6] (sweeps = 0).
// ============================================================================================

__device__ __forceinline__ double gk_rcp(double x) {  // ~1 ulp reciprocal (MUFU seed + cubic step)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// number of eigenvalues of T_GK below x (a2[j] = a_j^2, j < 2n - 1)
__device__ int gk_count(const double *a2, int m2, double x, double pivmin) {
  int cnt = 0;
  double q = -x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int j = 1; j < m2; ++j) {
    q = -x - a2[j - 1] * gk_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

__global__ void __launch_bounds__(kGkThreads, 1) k_svd_gk(JacArgs a) {
  extern __shared__ __align__(16) double sg[];
  const int n = a.nc, ld = n | 1, m2 = 2 * n;
  double *A = sg;                     // [n][ld] column-major: A[c * ld + r]
  double *d = A + (int64_t)n * ld;    // [n]    diagonal of B
  double *e = d + n;                  // [n]    superdiagonal of B (e[n-1] = 0)
  double *tauR = e + n;               // [n]    right reflectors
  double *a2 = tauR + n;              // [2n]   squared off-diagonal of T_GK
  double *sig = a2 + m2;              // [n]    singular values, ascending
  double *z = sig + n;                // [2n]   inverse iteration vector
  double *w = z + m2;                 // [n]    the singular vector
  double *Ud = w + n;                 // [2n]   inverse iteration: U's diagonal,
  double *Uo1 = Ud + m2;              // [2n]   first and
  double *Uo2 = Uo1 + m2;             // [2n]   second superdiagonals,
  double *Lm = Uo2 + m2;              // [2n]   multipliers,
  int *piv = (int *)(Lm + m2);        // [2n]   row interchanges
  __shared__ double s_par[4];
  const int metric = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double *R = a.R + (int64_t)metric * n * n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) A[(i % n) * ld + i / n] = R[i];
  __syncthreads();

  // ---- 1. bidiagonalisation ------------------------------------------------------------------
  for (int k = 0; k < n; ++k) {
    // left reflector of column k (rows k..n-1): one warp forms it
    if (wid == 0) {
      double s2 = 0.0;
      for (int r = k + 1 + lane; r < n; r += 32) s2 = fma(A[k * ld + r], A[k * ld + r], s2);
      s2 = warp_sum(s2);
      const double al = A[k * ld + k];
      double tau = 0.0, beta = al, sc = 0.0;
      if (s2 != 0.0) {
        const double nrm = sqrt(fma(al, al, s2));
        beta = al >= 0.0 ? -nrm : nrm;
        sc = 1.0 / (al - beta);
        tau = (beta - al) / beta;
      }
      for (int r = k + 1 + lane; r < n; r += 32) A[k * ld + r] *= sc;  // v (v_k = 1 implicit)
      if (lane == 0) {
        d[k] = beta;
        s_par[0] = tau;
      }
    }
    __syncthreads();
    const double tl = s_par[0];
    if (tl != 0.0)
      for (int j = k + 1 + wid; j < n; j += nw) {  // columns j > k: A_j -= tau (v^T A_j) v
        double t = lane == 0 ? A[j * ld + k] : 0.0;
        for (int r = k + 1 + lane; r < n; r += 32) t = fma(A[k * ld + r], A[j * ld + r], t);
        t = tl * warp_sum(t);
        if (lane == 0) A[j * ld + k] -= t;
        for (int r = k + 1 + lane; r < n; r += 32) A[j * ld + r] = fma(-t, A[k * ld + r], A[j * ld + r]);
      }
    __syncthreads();
    if (k + 1 >= n) break;
    // right reflector of row k (columns k+1..n-1)
    if (wid == 0) {
      double s2 = 0.0;
      for (int c = k + 2 + lane; c < n; c += 32) s2 = fma(A[c * ld + k], A[c * ld + k], s2);
      s2 = warp_sum(s2);
      const double al = A[(k + 1) * ld + k];
      double tau = 0.0, beta = al, sc = 0.0;
      if (s2 != 0.0) {
        const double nrm = sqrt(fma(al, al, s2));
        beta = al >= 0.0 ? -nrm : nrm;
        sc = 1.0 / (al - beta);
        tau = (beta - al) / beta;
      }
      for (int c = k + 2 + lane; c < n; c += 32) A[c * ld + k] *= sc;  // v (v_{k+1} = 1 implicit)
      if (lane == 0) {
        e[k] = beta;
        tauR[k] = tau;
        s_par[1] = tau;
      }
    }
    __syncthreads();
    const double tr = s_par[1];
    if (tr != 0.0)
      for (int i = k + 1 + wid; i < n; i += nw) {  // rows i > k: A^i -= tau (A^i v) v^T
        double t = lane == 0 ? A[(k + 1) * ld + i] : 0.0;
        for (int c = k + 2 + lane; c < n; c += 32) t = fma(A[c * ld + i], A[c * ld + k], t);
        t = tr * warp_sum(t);
        if (lane == 0) A[(k + 1) * ld + i] -= t;
        for (int c = k + 2 + lane; c < n; c += 32) A[c * ld + i] = fma(-t, A[c * ld + k], A[c * ld + i]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    e[n - 1] = 0.0;
    tauR[n - 1] = 0.0;
    if (n >= 2) tauR[n - 2] = 0.0;  // row n-2 has a single entry right of the diagonal: no reflector
  }
  __syncthreads();

  // ---- 2. singular values: bisection on T_GK --------------------------------------------------
  for (int j = threadIdx.x; j < m2 - 1; j += blockDim.x) {
    const double v = (j & 1) ? e[j >> 1] : d[j >> 1];
    a2[j] = v * v;
  }
  if (threadIdx.x == 0) {  // Gershgorin bound of T_GK and the pivot floor
    double b = 0.0, amax = 0.0;
    for (int j = 0; j < m2; ++j) {
      const double lo = j > 0 ? fabs((j - 1) & 1 ? e[(j - 1) >> 1] : d[(j - 1) >> 1]) : 0.0;
      const double hi = j < m2 - 1 ? fabs(j & 1 ? e[j >> 1] : d[j >> 1]) : 0.0;
      b = fmax(b, lo + hi);
      amax = fmax(amax, hi);
    }
    s_par[2] = b * (1.0 + 1e-14) + 1e-300;
    s_par[3] = fmax(amax * amax * 1e-300, 1e-300);  // LAPACK-style safe minimum pivot
  }
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x >> 2) {
    const double bound = s_par[2], pivmin = s_par[3];
    const int i = base + (threadIdx.x >> 2), q = threadIdx.x & 3;  // value i, quadrisection point q
    double lo = 0.0, hi = bound;
    for (int it = 0; it < 30; ++it) {  // 5^30 > 2^69: the interval ends below u ||B||
      const double h = (hi - lo) * 0.2;
      const double x = lo + h * (q + 1);
      // sigma_i >= x  <=>  at most n + i eigenvalues of T_GK lie below x
      const int below = i < n ? gk_count(a2, m2, x, pivmin) <= n + i : 0;
      // the quad's answers form a prefix: sigma_i lies in sub-interval nb
      const unsigned b = __ballot_sync(0xffffffffu, below);
      const int nb = __popc((b >> (lane & 28)) & 0xFu);
      const double nlo = lo + h * nb;
      hi = nb < 4 ? lo + h * (nb + 1) : hi;
      lo = nlo;
    }
    if (i < n && q == 0) sig[i] = 0.5 * (lo + hi);
  }
  __syncthreads();

  // ---- 3. the right singular vector of sigma_min --------------------------------------------
  if (threadIdx.x == 0) {
    // inverse iteration on M = T - lam I by Gaussian elimination with row interchanges (the
    // factor U has two superdiagonals); a zero pivot is replaced by eps ||T||
    const double lam = sig[0];
    const double eps = 2.220446049250313e-16 * fmax(s_par[2], 1e-300);
    auto aj = [&](int j) { return (j & 1) ? e[j >> 1] : d[j >> 1]; };  // off-diagonal j of T_GK
    double D = -lam, U1 = m2 > 1 ? aj(0) : 0.0, U2 = 0.0;
    for (int j = 0; j < m2; ++j) {
      if (j + 1 < m2) {
        const double L = aj(j), nd = -lam, nu = j + 2 < m2 ? aj(j + 1) : 0.0;
        if (fabs(D) >= fabs(L)) {  // keep row j
          const double dv = fabs(D) > 0.0 ? D : eps;
          const double mlt = L / dv;
          Ud[j] = dv; Uo1[j] = U1; Uo2[j] = U2; Lm[j] = mlt; piv[j] = 0;
          D = nd - mlt * U1;
          U1 = nu - mlt * U2;
        } else {                   // row j + 1 becomes the pivot row
          const double mlt = D / L;
          Ud[j] = L; Uo1[j] = nd; Uo2[j] = nu; Lm[j] = mlt; piv[j] = 1;
          D = U1 - mlt * nd;
          U1 = U2 - mlt * nu;
        }
        U2 = 0.0;
      } else {
        Ud[j] = fabs(D) >= eps ? D : (D < 0.0 ? -eps : eps);
        Uo1[j] = 0.0;
        Uo2[j] = 0.0;
      }
    }
    for (int j = 0; j < m2; ++j) z[j] = 1.0 + 0.01 * (double)(j % 7);  // fixed start: deterministic
    for (int iter = 0; iter < 3; ++iter) {
      for (int j = 0; j + 1 < m2; ++j) {
        if (piv[j]) {
          const double t = z[j];
          z[j] = z[j + 1];
          z[j + 1] = t - Lm[j] * z[j];
        } else {
          z[j + 1] -= Lm[j] * z[j];
        }
      }
      for (int j = m2 - 1; j >= 0; --j) {
        double t = z[j];
        if (j + 1 < m2) t -= Uo1[j] * z[j + 1];
        if (j + 2 < m2) t -= Uo2[j] * z[j + 2];
        z[j] = t / Ud[j];
      }
      double mx = 0.0;
      for (int j = 0; j < m2; ++j) mx = fmax(mx, fabs(z[j]));
      const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
      for (int j = 0; j < m2; ++j) z[j] *= sc;
    }
    // B's right singular vector: the even entries, normalised, into w
    double nv = 0.0;
    for (int i = 0; i < n; ++i) nv = fma(z[2 * i], z[2 * i], nv);
    nv = nv > 0.0 ? 1.0 / sqrt(nv) : 0.0;
    for (int i = 0; i < n; ++i) w[i] = z[2 * i] * nv;
  }
  __syncthreads();
  // v = H_0 H_1 ... H_{n-3} v_B: the right reflectors in reverse (the reflector of row k acts on
  // entries k+1..n-1 with vector (1, A[k][k+2..n-1]))
  for (int k = n - 3; k >= 0; --k) {
    const double tr = tauR[k];
    if (tr != 0.0 && wid == 0) {
      double t = lane == 0 ? w[k + 1] : 0.0;
      for (int c = k + 2 + lane; c < n; c += 32) t = fma(A[c * ld + k], w[c], t);
      t = tr * warp_sum(t);
      if (lane == 0) w[k + 1] -= t;
      for (int c = k + 2 + lane; c < n; c += 32) w[c] = fma(-t, A[c * ld + k], w[c]);
    }
    __syncwarp();
  }
  __syncthreads();
  double *so = a.sigma + (int64_t)metric * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) so[i] = sig[i];
  const double b0 = w[a.n_num];
  const bool bad = !(fabs(b0) > 1e-300);
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    a.coef[(int64_t)metric * n + r] = bad ? __longlong_as_double(0x7ff8000000000000ll) : w[r] / b0;
  if (threadIdx.x == 0) {
    const double smin = sig[0], smax = sig[n - 1];
    int rank = 0;
    for (int o = 0; o < n; ++o) rank += sig[o] > 1e-13 * smax;
    double *inf = a.info + metric * 6;
    inf[0] = bad ? (double)RP_ERR_DEGENERATE : 0.0;
    inf[1] = rank;
    inf[2] = (smin / b0) * (smin / b0);
    inf[3] = smin;
    inf[4] = smax / smin;
    inf[5] = 0;
  }
}

static bool svd_use_jacobi() {
  const char *v = getenv("RP_SVD_SOLVER");
  return v && strcmp(v, "jacobi") == 0;
}

}  // namespace rp
