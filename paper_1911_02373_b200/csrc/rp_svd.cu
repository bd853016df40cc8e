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
//   2. k_svd_jacobi -- one-sided (Hestenes) Jacobi SVD of R on a 2-CTA thread-block cluster
//      per metric: CTA 0 holds R (column-major, 157 KB at n_c = 140) and computes the
//      rotations of one round-robin round (all pairs disjoint, one warp per pair); it writes
//      them into CTA 1's shared memory (DSMEM), and CTA 1 applies them to the accumulated V
//      while CTA 0 computes the next round.  Singular values are the final column norms.
#include <cooperative_groups.h>

#include "rp_internal.cuh"

namespace cg = cooperative_groups;

namespace rp {

constexpr int kSvdMaxCols = 144;      // one quad per column, 8 quads per warp -> 576 threads
constexpr int kRPL = 24;              // chunk rows per lane
constexpr int kChunk = 4 * kRPL;      // rows per chunk (128)
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
  int zero;                // 0 (opaque to the compiler; see opaque_zero)
};

// One chunk absorbed into the packed R in shared memory: reflector steps j = j0 .. nc-1.
// Thread layout: quad q owns column k = q, lane l4 = lane & 3 owns chunk rows l4 + 4 i.
// c[] holds this thread's chunk entries; vbuf[2][kChunk] the scaled Householder vector of the
// current column (double-buffered), par[2][2] = (tau, beta).
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

// sum over the 4 lanes of a quad; conditions on the quad's column keep quads convergent, so
// the mask names only this quad's lanes
__device__ __forceinline__ double quad_sum(double x) {
  const unsigned m = 0xFu << (threadIdx.x & 28);
  x += __shfl_xor_sync(m, x, 1);
  x += __shfl_xor_sync(m, x, 2);
  return x;
}

// Householder vector layout in vbuf: lane l4's 32 rows contiguous at l4 * kVS (kVS = 34: the
// four 16-byte lane segments of a LDS.128 fall in distinct banks)
constexpr int kVS = kRPL + 2;
constexpr int kVBuf = 4 * kVS;

// shared-memory 2 x f64 load that the compiler may not cache in registers (the update pass
// re-reads v instead of keeping 32 more doubles live)
__device__ __forceinline__ double2 lds2(const double *p) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return r;
}

// 0, computed from x in a way the compiler cannot see through: a data dependency that orders
// shared-memory loads after the arithmetic producing x
__device__ __forceinline__ int opaque_zero(double x, int zero) {
  return __double2loint(x) & zero;  // `zero` is a kernel argument (0): nothing to fold
}

__device__ __forceinline__ void publish(double *vbuf, double *par, const double (&c)[kRPL], double a_kk,
                                        int slot) {
  const int l4 = threadIdx.x & 3;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int i = 0; i < kRPL; i += 2) {
    s0 = fma(c[i], c[i], s0);
    s1 = fma(c[i + 1], c[i + 1], s1);
  }
  const double sub = quad_sum(s0 + s1);
  double tau, beta, sc;
  householder_params(a_kk, sub, tau, beta, sc);
  double *vn = vbuf + slot * kVBuf + l4 * kVS;
#pragma unroll
  for (int i = 0; i < kRPL; i += 2) *(double2 *)(vn + i) = make_double2(sc * c[i], sc * c[i + 1]);
  if (l4 == 0) {
    par[slot * 2 + 0] = tau;
    par[slot * 2 + 1] = beta;
  }
}

__device__ __forceinline__ void absorb_chunk(double *Rp, double *vbuf, double *par, double (&c)[kRPL], int nc,
                                             int j0, int zero) {
  const int k = threadIdx.x >> 2, l4 = threadIdx.x & 3;
  const bool own = k < nc;
  // the owner of column j0 publishes its reflector
  if (own && k == j0) publish(vbuf, par, c, Rp[packed_off(k, nc)], j0 & 1);
  for (int j = j0; j < nc; ++j) {
    __syncthreads();
    const double *v = vbuf + (j & 1) * kVBuf + l4 * kVS;
    const double tau = par[(j & 1) * 2 + 0];
    if (own && k > j) {
      double d0 = 0.0, d1 = 0.0;
      int z = 0;
#pragma unroll
      for (int i = 0; i < kRPL; i += 2) {
        // groups of 8 rows: the next group's loads wait for this group's FMAs (an opaque zero
        // offset), so at most 8 v values are live next to the 2 kRPL registers of c
        if ((i & 7) == 0 && i > 0) z = opaque_zero(d0, zero);
        const double2 vv = lds2(v + i + z);
        d0 = fma(vv.x, c[i], d0);
        d1 = fma(vv.y, c[i + 1], d1);
      }
      const double dot = quad_sum(d0 + d1);
      double *rjk = Rp + packed_off(j, nc) + (k - j);
      const double w = *rjk + dot;
      const double tw = tau * w;
#pragma unroll
      for (int i = 0; i < kRPL; i += 2) {
        if ((i & 7) == 0 && i > 0) z = opaque_zero(c[i - 1], zero);
        const double2 vv = lds2(v + i + z);
        c[i] = fma(-tw, vv.x, c[i]);
        c[i + 1] = fma(-tw, vv.y, c[i + 1]);
      }
      if (l4 == 0) *rjk -= tw;
      if (k == j + 1) publish(vbuf, par, c, Rp[packed_off(k, nc)], (j + 1) & 1);  // look-ahead
    }
    if (own && k == j && l4 == 0) Rp[packed_off(j, nc)] = par[(j & 1) * 2 + 1];
  }
  __syncthreads();
}

// rows [r0, r0 + kChunk) of R2 (packed, global) as chunk entries of column k
__device__ __forceinline__ void fill_from_packed(double (&c)[kRPL], const double *R2, int nc, int r0) {
  const int k = threadIdx.x >> 2, l4 = threadIdx.x & 3;
#pragma unroll
  for (int i = 0; i < kRPL; ++i) {
    const int rho = r0 + l4 + 4 * i;
    c[i] = (k < nc && rho < nc && k >= rho) ? __ldcg(R2 + packed_off(rho, nc) + (k - rho)) : 0.0;
  }
}

__device__ __forceinline__ void absorb_packed(double *Rp, double *vbuf, double *par, const double *R2, int nc,
                                              int zero) {
  double c[kRPL];
  for (int r0 = 0; r0 < nc; r0 += kChunk) {
    fill_from_packed(c, R2, nc, r0);
    absorb_chunk(Rp, vbuf, par, c, nc, r0, zero);  // rows >= r0 are zero left of column r0
  }
}

// Shared memory: Rp [packed] | vbuf [2][kVBuf] | par [4] | sU [kChunk][8] | sD [160][kSD] | flag
__global__ void __maxnreg__(96) k_tsqr(TsqrArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nc = a.nc, n = a.n;
  const int64_t psz = packed_size(nc);
  double *Rp = sm;
  double *vbuf = Rp + ((psz + 1) & ~1ll);
  double *par = vbuf + 2 * kVBuf;
  double *sU = par + 4;
  double *sD = sU + kChunk * kMaxVars;
  int *flag = (int *)(sD + kSD * kSvdMaxCols);
  const int metric = blockIdx.y;
  const int leaf = blockIdx.x;
  const int k = threadIdx.x >> 2, l4 = threadIdx.x & 3;

  for (int64_t i = threadIdx.x; i < psz; i += blockDim.x) Rp[i] = 0.0;
  __syncthreads();

  // ---- leaf: the slab's rows ----------------------------------------------------------------
  const int64_t r_begin = a.K * leaf / a.leaves, r_end = a.K * (leaf + 1) / a.leaves;
  const double *V = a.V ? a.V + (int64_t)metric * a.K : nullptr;
  const double *S = a.S ? a.S + (int64_t)metric * a.K : nullptr;
  const double *rows = a.rows ? a.rows + (int64_t)metric * a.K * nc : nullptr;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kChunk) {
    const int cnt = (int)((r_end - r0) < kChunk ? (r_end - r0) : kChunk);
    if (!rows) {
      // a10: u = (x - c) 2^-e of the chunk's rows
      for (int i = threadIdx.x; i < cnt * n; i += blockDim.x) {
        const int r = i / n, t = i % n;
        sU[r * kMaxVars + t] = (a.X[(r0 + r) * n + t] - a.basis->xc[t]) * ldexp(1.0, -a.basis->xe[t]);
      }
    }
    // the chunk's entries are staged through sD in 4 passes of 32 rows (column-major, stride
    // kSD = 36: a quad-row read pattern is conflict-free), then picked up into registers
    double c[kRPL];
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
              const double u = sU[r * kMaxVars + t];
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
      for (int ii = 0; ii < 8; ++ii) c[ps * 8 + ii] = k < nc ? sD[k * kSD + l4 + 4 * ii] : 0.0;
    }
    absorb_chunk(Rp, vbuf, par, c, nc, 0, a.zero);
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
      absorb_packed(Rp, vbuf, par, mine, nc, a.zero);
    } else {
      absorb_packed(Rp, vbuf, par, other, nc, a.zero);
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
// one-sided Jacobi SVD of R on a 2-CTA cluster
// ============================================================================================
struct JacArgs {
  const double *R;  // [n_v][nc][nc] row-major (any square matrix works)
  int nc, n_num;
  double *coef;     // [n_v][nc]
  double *sigma;    // [n_v][nc] ascending
  double *info;     // [n_v][6]: status, rank, resid2, sigma_min, sigma_max / sigma_min, sweeps
};

__device__ __forceinline__ int rr_player(int pos, int t, int np) {  // round-robin tournament
  return pos == 0 ? 0 : 1 + (pos - 1 + t) % (np - 1);
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Shared memory (each CTA): M [nc][ld] column-major (CTA 0: A = R, CTA 1: V) | rot [2][kSvdMaxCols/2][2]
// | ctl[4]
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kJacThreads, 1) k_svd_jacobi(JacArgs a) {
  extern __shared__ __align__(16) double sj[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  const int nc = a.nc, ld = nc | 1;  // odd stride: row-wise scans stay conflict-free
  const int np = (nc + 1) & ~1;      // players (a dummy when nc is odd)
  const int npairs = np / 2;
  double *M = sj;
  double *rot = M + (int64_t)nc * ld;
  int *ctl = (int *)(rot + 2 * (kSvdMaxCols / 2) * 2);  // [0] rotated this sweep, [1] continue, [2] jmin
  double *rot1 = cluster.map_shared_rank(rot, 1);
  int *ctl1 = cluster.map_shared_rank(ctl, 1);
  const int metric = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double *R = a.R + (int64_t)metric * nc * nc;

  if (crank == 0) {
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) {
      const int r = i / nc, col = i % nc;
      M[col * ld + r] = R[i];
    }
  } else {
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) {
      const int r = i / nc, col = i % nc;
      M[col * ld + r] = r == col ? 1.0 : 0.0;
    }
  }
  if (threadIdx.x == 0) ctl[0] = ctl[1] = 0;
  cluster.sync();

  const double tol = 1e-15 * sqrt((double)nc);
  int sweep = 0;
  for (; sweep < kJacMaxSweeps; ++sweep) {
    for (int t = 0; t <= np - 1; ++t) {  // rounds 0 .. np-2 computed, round t-1 applied
      if (crank == 0 && t < np - 1) {
        for (int m = wid; m < npairs; m += nw) {
          int p = rr_player(m, t, np), q = rr_player(np - 1 - m, t, np);
          if (p > q) {
            const int x = p;
            p = q;
            q = x;
          }
          double cs = 1.0, sn = 0.0;
          if (q < nc) {
            double *ap = M + p * ld, *aq = M + q * ld;
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int r = lane; r < nc; r += 32) {
              const double x = ap[r], y = aq[r];
              al = fma(x, x, al);
              be = fma(y, y, be);
              ga = fma(x, y, ga);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (ga != 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
              const double zeta = (be - al) / (2.0 * ga);
              const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              cs = 1.0 / sqrt(fma(tt, tt, 1.0));
              sn = cs * tt;
              for (int r = lane; r < nc; r += 32) {
                const double x = ap[r], y = aq[r];
                ap[r] = cs * x - sn * y;
                aq[r] = sn * x + cs * y;
              }
              if (lane == 0) ctl[0] = 1;
            }
          }
          if (lane == 0) {
            rot1[((t & 1) * (kSvdMaxCols / 2) + m) * 2 + 0] = cs;
            rot1[((t & 1) * (kSvdMaxCols / 2) + m) * 2 + 1] = sn;
          }
        }
      }
      if (crank == 1 && t > 0) {  // apply round t-1 to V
        const int tp = t - 1;
        for (int m = wid; m < npairs; m += nw) {
          int p = rr_player(m, tp, np), q = rr_player(np - 1 - m, tp, np);
          if (p > q) {
            const int x = p;
            p = q;
            q = x;
          }
          const double cs = rot[((tp & 1) * (kSvdMaxCols / 2) + m) * 2 + 0];
          const double sn = rot[((tp & 1) * (kSvdMaxCols / 2) + m) * 2 + 1];
          if (q < nc && sn != 0.0) {
            double *vp = M + p * ld, *vq = M + q * ld;
            for (int r = lane; r < nc; r += 32) {
              const double x = vp[r], y = vq[r];
              vp[r] = cs * x - sn * y;
              vq[r] = sn * x + cs * y;
            }
          }
        }
      }
      cluster.sync();
    }
    // sweep done: CTA 0 tells CTA 1 whether anything rotated
    if (crank == 0 && threadIdx.x == 0) {
      const int cont = ctl[0];
      ctl[1] = cont;
      ctl1[1] = cont;
      ctl[0] = 0;
    }
    cluster.sync();
    if (!ctl[1]) break;
  }

  // ---- singular values (CTA 0), the vector of the smallest (CTA 1) -----------------------------
  double *sig = rot;  // reuse (CTA 0): sigma per column; needs nc <= kSvdMaxCols doubles
  if (crank == 0) {
    for (int col = wid; col < nc; col += nw) {
      double s2 = 0.0;
      for (int r = lane; r < nc; r += 32) s2 = fma(M[col * ld + r], M[col * ld + r], s2);
      s2 = warp_sum(s2);
      if (lane == 0) sig[col] = sqrt(s2);
    }
    __syncthreads();
    // ascending order by rank counting (ties by column index), smallest -> jmin
    double *so = a.sigma + (int64_t)metric * nc;
    for (int col = threadIdx.x; col < nc; col += blockDim.x) {
      const double v = sig[col];
      int rank = 0;
      for (int o = 0; o < nc; ++o) rank += (sig[o] < v) || (sig[o] == v && o < col);
      so[rank] = v;
      if (rank == 0) ctl1[2] = col;
    }
  }
  cluster.sync();
  double *rot0 = cluster.map_shared_rank(rot, 0);
  if (crank == 1) {
    const int jm = ctl[2];
    const double *vm = M + jm * ld;
    const double b0 = vm[a.n_num];
    const bool bad = !(fabs(b0) > 1e-300);
    for (int r = threadIdx.x; r < nc; r += blockDim.x)
      a.coef[(int64_t)metric * nc + r] = bad ? __longlong_as_double(0x7ff8000000000000ll) : vm[r] / b0;
    if (threadIdx.x == 0) rot0[2 * (kSvdMaxCols / 2) * 2 - 1] = b0;  // to CTA 0 (DSMEM)
  }
  cluster.sync();
  if (crank == 0 && threadIdx.x == 0) {
    double smin = sig[0], smax = sig[0];
    for (int o = 1; o < nc; ++o) {
      smin = fmin(smin, sig[o]);
      smax = fmax(smax, sig[o]);
    }
    int rank = 0;
    for (int o = 0; o < nc; ++o) rank += sig[o] > 1e-13 * smax;
    const double b0 = rot[2 * (kSvdMaxCols / 2) * 2 - 1];
    const bool bad = !(fabs(b0) > 1e-300);
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
  return (size_t)((packed_size(nc) + 1) & ~1ll) * 8 + 2 * kVBuf * 8 + 4 * 8 +
         (size_t)kChunk * kMaxVars * 8 + (size_t)kSD * kSvdMaxCols * 8 + 16;
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
  const int threads = 32 * ((nc + 7) / 8);
  k_tsqr<<<dim3(leaves, n_v), threads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_svd_jacobi(const double *R, int nc, int n_num, int n_v, double *coef, double *sigma,
                              double *info, cudaStream_t s) {
  if (nc < 2 || nc > kSvdMaxCols) return cudaErrorInvalidValue;
  const size_t smem = (size_t)nc * (nc | 1) * 8 + 2 * (kSvdMaxCols / 2) * 2 * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(k_svd_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  JacArgs a{R, nc, n_num, coef, sigma, info};
  k_svd_jacobi<<<dim3(2, n_v), kJacThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rp
