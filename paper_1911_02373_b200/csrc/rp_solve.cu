// rp_solve.cu -- a14: normalise beta_0 = 1 and solve the normal equations on the device.
//
// PAPER.md:2578-2584 solves the over-determined linearised system "by the method of linear
// least squares"; the draft footnote notes the system is homogeneous.
// Reading R12 fixes the constant denominator coefficient beta_0 = 1, turning it into
// G_ff z = -G_{f,beta0} with G = A^T A (reading R13: normal equations, as the north star asks;
// the paper's SVD is the f1 NEXT row).  The matrix is at most 160 x 160, so one CTA per metric
// does it on chip:
//   1. Jacobi equilibration  S = D G_ff D, D = diag(1/sqrt(G_ii))   (conditioning, R14);
//   2. Cholesky S = L L^T (pivot <= 1e-13 -> RP_ERR_DEGENERATE): by default blocked (k_solve_b:
//      8-column panels factored by one warp with a one-panel look-ahead, the rank-8 trailing
//      updates on DMMA); RP_SOLVE_KERNEL=reg keeps the register-resident right-looking k_solve
//      (2-D cyclic over the 512 threads, one block barrier per column);
//   3. two triangular solves by one warp (unknowns in registers, shuffle broadcasts);
//   4. one step of iterative refinement with the residual b - G_ff z accumulated in
//      double-double from the unrounded Gram entries, which removes the solve's own rounding
//      error and leaves only the Gram's.
#include <cstdlib>
#include <cstring>

#include "rp_internal.cuh"
#include "rp_device.cuh"

namespace rp {

constexpr int kSolveThreads = 512;

__device__ __forceinline__ void dd_add(double &hi, double &lo, double a) {
  const double s = hi + a;
  const double bb = s - hi;
  const double err = (hi - (s - bb)) + (a - bb);
  hi = s;
  lo += err;
}
__device__ __forceinline__ void dd_fma(double &hi, double &lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  dd_add(hi, lo, p);
  lo += pe;
}

// 1/x and 1/sqrt(x) for x > 0: MUFU seeds plus Newton steps (a few ulp; the refinement step
// below removes the solve's own rounding error anyway)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int it = 0; it < 2; ++it) {  // y <- y (3 - x y^2) / 2
    const double h = 0.5 * x * y;
    y = fma(y, fma(-h, y, 0.5), y);
  }
  return y;
}

// Register-resident Cholesky (one block barrier per column; measured phases with
// -DRP_SOLVE_TS at m = 139: load 11k cycles, factorisation 165k, each triangular solve pair 42k,
// residuals 18k): thread (ty, tx) = (tid / 32, tid % 32) of 512 owns the entries
// (i, j) = (ty + 16 a, tx + 32 b) of the equilibrated matrix (m <= 16 kRA, m <= 32 kCB).
constexpr int kRA = 10, kCB = 5;
// slot (a, b) can hold a lower-triangle entry (j <= i) for some thread: only those 30 of the 50
// are ever touched, so the compiler keeps 60 registers of the matrix per thread
__host__ __device__ constexpr bool live(int a, int b) { return 32 * b <= 16 * a + 15; }

// x <- (L L^T)^{-1} x by warp 0: lane owns x_i, i = lane + 32 k, in registers; L (lower, sL,
// stride ld odd: conflict-free column reads) and rd[j] = 1 / L_jj from shared memory; each
// step broadcasts the finished unknown by one shuffle.
__device__ void chol_solve_warp(const double *sL, const double *rd, int ld, int m, double *x) {
  const int lane = threadIdx.x;
  double v[kCB];
#pragma unroll
  for (int k = 0; k < kCB; ++k) v[k] = (lane + 32 * k < m) ? x[lane + 32 * k] : 0.0;
#pragma unroll
  for (int kb = 0; kb < kCB; ++kb) {  // forward: L y = x
    if (32 * kb >= m) break;
    const int jn = (m - 32 * kb) < 32 ? (m - 32 * kb) : 32;
    for (int jj = 0; jj < jn; ++jj) {
      const int j = 32 * kb + jj;
      const double yj = __shfl_sync(0xffffffffu, v[kb], jj) * rd[j];
      if (lane == jj) v[kb] = yj;
#pragma unroll
      for (int k = kb; k < kCB; ++k) {
        const int i = lane + 32 * k;
        if (i > j && i < m) v[k] = fma(-sL[i * ld + j], yj, v[k]);
      }
    }
  }
#pragma unroll
  for (int kb = kCB - 1; kb >= 0; --kb) {  // backward: L^T z = y
    if (32 * kb >= m) continue;
    const int jn = (m - 32 * kb) < 32 ? (m - 32 * kb) : 32;
    for (int jj = jn - 1; jj >= 0; --jj) {
      const int j = 32 * kb + jj;
      const double zj = __shfl_sync(0xffffffffu, v[kb], jj) * rd[j];
      if (lane == jj) v[kb] = zj;
#pragma unroll
      for (int k = 0; k <= kb; ++k) {
        const int i = lane + 32 * k;
        if (i < j) v[k] = fma(-sL[j * ld + i], zj, v[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kCB; ++k)
    if (lane + 32 * k < m) x[lane + 32 * k] = v[k];
}

// double-double sum of a warp's (hi, lo) pairs (fixed butterfly order)
__device__ __forceinline__ void dd_warp_sum(double &hi, double &lo) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    dd_add(hi, lo, h2);
    lo += l2;
  }
}

__global__ void __launch_bounds__(kSolveThreads, 1) k_solve(const double *G, int nc, int beta0,
                                                            double *coef_out, double *info_out) {
  extern __shared__ __align__(16) double sm[];
  const int m = nc - 1, ld = m | 1;
  double *sL = sm;            // [m][ld]  the factor L (lower)
  double *dsc = sL + m * ld;  // [m]
  double *b0 = dsc + m;       // -G_{f,beta0}
  double *x = b0 + m;         // work vector
  double *z = x + m;          // solution, unequilibrated
  double *rd = z + m;         // 1 / L_jj
  double *cb = rd + m;        // [2][m]  published column of the factorisation step (double buffer)
  double *csc = cb + 2 * m;   // [m]  1 / sqrt(pivot) of each column
  __shared__ int s_status;
  __shared__ double s_pmin, s_pmax;
#ifdef RP_SOLVE_TS  // phase timestamps (debug builds): written over coef[1..6] of metric 0
  unsigned long long ts[8];
#define RP_TS(k) ts[k] = clock64()
  RP_TS(0);
#else
#define RP_TS(k)
#endif
  const double *Gm = G + (int64_t)blockIdx.x * nc * nc;
  auto col = [beta0](int i) { return i < beta0 ? i : i + 1; };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ty = wid, tx = lane;

  if (threadIdx.x == 0) {
    s_status = 0;
    s_pmin = __longlong_as_double(0x7ff0000000000000ll);
    s_pmax = 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double di = Gm[(int64_t)col(i) * nc + col(i)];
    if (!(di > 0.0)) s_status = RP_ERR_DEGENERATE;
    dsc[i] = di > 0.0 ? 1.0 / sqrt(di) : 0.0;
    b0[i] = -Gm[(int64_t)col(i) * nc + beta0];
  }
  __syncthreads();
  // owned entries of S = D G_ff D (Jacobi equilibration), column 0 published
  double A[kRA][kCB];
#pragma unroll
  for (int a = 0; a < kRA; ++a)
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      if (!live(a, b)) continue;
      const int i = ty + 16 * a, j = tx + 32 * b;
      A[a][b] = (i < m && j < m && j <= i) ? Gm[(int64_t)col(i) * nc + col(j)] * dsc[i] * dsc[j] : 0.0;
      if (j == 0 && i < m) cb[i] = A[a][b];
    }
  __syncthreads();
  RP_TS(1);
  // right-looking Cholesky, one column per step and one block barrier per step: every thread
  // reads the published column c (its pivot included), applies the rank-1 update to the entries
  // it owns, finishes column c, and the owners of column c + 1 publish it into the other buffer
  int status = s_status;
  double pmin = __longlong_as_double(0x7ff0000000000000ll), pmax = 0.0;
  for (int c = 0; c < m && status == 0; ++c) {
    const double *bc = cb + (c & 1) * m;
    double *bn = cb + ((c + 1) & 1) * m;
    const double piv = bc[c];
    pmin = fmin(pmin, piv);
    pmax = fmax(pmax, piv);
    if (!(piv > 1e-13)) {  // uniform: every thread reads the same pivot
      status = RP_ERR_DEGENERATE;
      break;
    }
    const double rp = rcp_nr(piv);
    if (threadIdx.x == 0) csc[c] = rsqrt_nr(piv);  // L_ic = S_ic / sqrt(piv), applied at the end
    // rank-1 update S_ij -= S_ic S_jc / piv of the owned entries with j > c (cj = 0 elsewhere:
    // the FMA leaves those unchanged) in rows i > c (warp-uniform: ty is the warp id)
    double cj[kCB];
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      const int j = tx + 32 * b;
      cj[b] = (j > c && j < m) ? bc[j] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < kRA; ++a) {
      const int i = ty + 16 * a;
      if (i > c && i < m) {
        const double sa = bc[i] * rp;
#pragma unroll
        for (int b = 0; b < kCB; ++b)
          if (live(a, b)) A[a][b] = fma(-sa, cj[b], A[a][b]);
      }
    }
    // the owners of column c + 1 (lane (c + 1) % 32 of every warp, slot b = (c + 1) / 32:
    // uniform) publish it, its pivot included
    if (tx == ((c + 1) & 31)) {
      switch ((c + 1) >> 5) {
#define RP_PUB(B)                                                   \
  case B:                                                           \
    _Pragma("unroll") for (int a = 0; a < kRA; ++a) {               \
      const int i = ty + 16 * a;                                    \
      if (live(a, B) && i > c && i < m) bn[i] = A[a][B];            \
    }                                                               \
    break;
        RP_PUB(0) RP_PUB(1) RP_PUB(2) RP_PUB(3) RP_PUB(4)
#undef RP_PUB
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s_status = status;
    s_pmin = pmin;
    s_pmax = pmax;
  }
#pragma unroll
  for (int a = 0; a < kRA; ++a)
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      const int i = ty + 16 * a, j = tx + 32 * b;
      if (live(a, b) && i < m && j <= i) sL[i * ld + j] = A[a][b] * csc[j];
    }
  __syncthreads();
  RP_TS(2);
  double *cf = coef_out + (int64_t)blockIdx.x * nc;
  double *inf = info_out + (int64_t)blockIdx.x * 5;
  if (s_status != 0) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) cf[i] = __longlong_as_double(0x7ff8000000000000ll);
    if (threadIdx.x == 0) {
      inf[0] = (double)s_status;
      inf[1] = 0;
      inf[2] = __longlong_as_double(0x7ff8000000000000ll);
      inf[3] = s_pmin;
      inf[4] = __longlong_as_double(0x7ff0000000000000ll);
    }
    return;
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    rd[i] = 1.0 / sL[i * ld + i];
    x[i] = dsc[i] * b0[i];
  }
  __syncthreads();
  if (wid == 0) chol_solve_warp(sL, rd, ld, m, x);
  __syncthreads();
  RP_TS(3);
  for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] = dsc[i] * x[i];
  __syncthreads();
  // one refinement step: r = b0 - G_ff z in double-double from the original Gram (a warp per
  // row, lanes over columns: coalesced reads of G)
  for (int i = wid; i < m; i += nw) {
    const double *Gi = Gm + (int64_t)col(i) * nc;
    double hi = 0.0, lo = 0.0;
    for (int j = lane; j < m; j += 32) dd_fma(hi, lo, -Gi[col(j)], z[j]);
    dd_warp_sum(hi, lo);
    if (lane == 0) {
      dd_add(hi, lo, b0[i]);
      x[i] = dsc[i] * (hi + lo);
    }
  }
  __syncthreads();
  RP_TS(4);
  if (wid == 0) chol_solve_warp(sL, rd, ld, m, x);
  __syncthreads();
  RP_TS(5);
  for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] += dsc[i] * x[i];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) cf[col(i)] = z[i];
  if (threadIdx.x == 0) cf[beta0] = 1.0;
  // resid2 = coef^T G coef (double-double): a warp per row, then the warp partials in order
  __shared__ double s_rh[32], s_rl[32];
  {
    double wh = 0.0, wl = 0.0;
    for (int i = wid; i < nc; i += nw) {
      const double ci = (i == beta0) ? 1.0 : z[i < beta0 ? i : i - 1];
      double rh = 0.0, rl = 0.0;
      for (int j = lane; j < nc; j += 32) {
        const double cj = (j == beta0) ? 1.0 : z[j < beta0 ? j : j - 1];
        dd_fma(rh, rl, Gm[(int64_t)i * nc + j], cj);
      }
      dd_warp_sum(rh, rl);
      dd_fma(wh, wl, ci, rh);
      dd_fma(wh, wl, ci, rl);
    }
    if (lane == 0) {
      s_rh[wid] = wh;
      s_rl[wid] = wl;
    }
  }
  __syncthreads();
  RP_TS(6);
  if (threadIdx.x == 0) {
    double hi = 0.0, lo = 0.0;
    for (int w = 0; w < nw; ++w) {
      dd_add(hi, lo, s_rh[w]);
      lo += s_rl[w];
    }
#ifdef RP_SOLVE_TS
    for (int k = 1; k <= 6; ++k) cf[k] = (double)(ts[k] - ts[k - 1]);
#endif
    inf[0] = 0;
    inf[1] = (double)m;
    inf[2] = hi + lo;
    inf[3] = s_pmin;
    inf[4] = s_pmax / s_pmin;
  }
}

// ============================================================================================
// k_solve_b -- the same solve with a blocked Cholesky (default; RP_SOLVE_KERNEL=reg keeps k_solve).
// The equilibrated matrix S (padded to a multiple of 8 with an identity block) lives in shared
// memory (row-major, odd stride).  Per 8-column panel: warp 0 factors the panel with its rows in
// registers (pivots broadcast by shuffles, no block barrier inside the panel), then every warp
// applies the rank-8 update S22 -= L21 L21^T to its lower 8 x 8 tiles on DMMA.  So the block
// barriers drop from one per column to two per 8 columns, and the trailing update runs on the
// tensor pipe.  Triangular solves: one warp, column-oriented forward / row-oriented backward
// (unknowns in registers, one shuffle per step); then the same double-double refinement step.
// ============================================================================================
constexpr int kSbMaxM = 160;  // padded unknowns (m <= 160)

__global__ void __launch_bounds__(kSolveThreads, 1) k_solve_b(const double *G, int nc, int beta0,
                                                              double *coef_out, double *info_out) {
  extern __shared__ __align__(16) double sm[];
  const int m = nc - 1, M8 = (m + 7) & ~7, ld = M8 | 1;
  double *S = sm;               // [M8][ld]  S, then L (lower)
  double *dsc = S + M8 * ld;    // [M8]
  double *b0 = dsc + M8;        // [M8]  -G_{f,beta0}
  double *x = b0 + M8;          // [M8]
  double *z = x + M8;           // [M8]
  double *rd = z + M8;          // [M8]  1 / L_jj
  __shared__ int s_status;
  __shared__ double s_pmin, s_pmax;
  const double *Gm = G + (int64_t)blockIdx.x * nc * nc;
  auto col = [beta0](int i) { return i < beta0 ? i : i + 1; };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#ifdef RP_SOLVE_TS
  unsigned long long tsb[8];
  tsb[0] = clock64();
#define RP_TSB(k) tsb[k] = clock64()
#else
#define RP_TSB(k)
#endif
  if (threadIdx.x == 0) {
    s_status = 0;
    s_pmin = __longlong_as_double(0x7ff0000000000000ll);
    s_pmax = 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < M8; i += blockDim.x) {
    if (i < m) {
      const double di = Gm[(int64_t)col(i) * nc + col(i)];
      if (!(di > 0.0)) s_status = RP_ERR_DEGENERATE;
      dsc[i] = di > 0.0 ? 1.0 / sqrt(di) : 0.0;
      b0[i] = -Gm[(int64_t)col(i) * nc + beta0];
    } else {
      dsc[i] = 0.0;
      b0[i] = 0.0;
    }
  }
  __syncthreads();
  // S = D G_ff D, lower triangle only (the factorisation never reads above the diagonal),
  // identity padding; a warp per row, coalesced reads of G's row
  for (int i = wid; i < M8; i += nw)
    for (int j = lane; j <= i; j += 32) {
      double v;
      if (i < m && j < m) v = Gm[(int64_t)col(i) * nc + col(j)] * dsc[i] * dsc[j];
      else v = (i == j) ? 1.0 : 0.0;
      S[i * ld + j] = v;
    }
  __syncthreads();
  RP_TSB(1);
  // ---- blocked Cholesky with a one-panel look-ahead ------------------------------------------
  // panel(c): warp 0 factors columns c .. c+7 (rows in registers, pivots by shuffles)
  auto panel = [&](int c) {
    double P[5][8];  // rows c + lane + 32 k of the panel's 8 columns
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = c + lane + 32 * k;
        P[k][j] = r < M8 ? S[r * ld + c + j] : 0.0;
      }
    int st = 0;
    double pmin = s_pmin, pmax = s_pmax;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double piv = __shfl_sync(0xffffffffu, P[0][j], j);  // S[c+j][c+j] sits in lane j
      if (c + j < m) {
        pmin = fmin(pmin, piv);
        pmax = fmax(pmax, piv);
      }
      if (!(piv > 1e-13)) st = RP_ERR_DEGENERATE;  // (uniform)
      const double rs = rsqrt_nr(piv > 1e-13 ? piv : 1.0);
      if (lane == 0) rd[c + j] = rs;
#pragma unroll
      for (int k = 0; k < 5; ++k) P[k][j] *= rs;  // L[., c+j] (rows below the diagonal matter)
#pragma unroll
      for (int kk = j + 1; kk < 8; ++kk) {
        const double lk = __shfl_sync(0xffffffffu, P[0][j], kk);  // L[c+kk][c+j] in lane kk
#pragma unroll
        for (int k = 0; k < 5; ++k) P[k][kk] = fma(-P[k][j], lk, P[k][kk]);
      }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = c + lane + 32 * k;
        if (r < M8 && r >= c + j) S[r * ld + c + j] = P[k][j];
      }
    if (lane == 0) {
      s_pmin = pmin;
      s_pmax = pmax;
      if (st) s_status = st;
    }
  };
  // tile(c, I, J): S[I block][J block] -= L[I][c..c+7] L[J][c..c+7]^T (DMMA, K = 8)
  const int r8 = lane >> 2, q4 = lane & 3;
  auto tile = [&](int c, int ri, int rj) {
    double *acc = S + (ri + r8) * ld + rj + 2 * q4;
    double d0 = acc[0], d1 = acc[1];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double a = -S[(ri + r8) * ld + c + 4 * h + q4];  // -L[ri + r][c + 4h + q]
      const double b = S[(rj + r8) * ld + c + 4 * h + q4];   //  L[rj + r][c + 4h + q] = B[q][r]
      dmma(d0, d1, a, b);
    }
    acc[0] = d0;
    acc[1] = d1;
  };
  if (wid == 0) panel(0);
  __syncthreads();
  for (int c = 0; c < M8 && s_status == 0; c += 8) {
    const int c1 = c + 8;
    if (c1 >= M8) break;
    const int nb = M8 / 8 - c1 / 8;  // block rows / columns below the panel
    // A: the next panel's block column (J = c1 / 8), every warp
    for (int I = wid; I < nb; I += nw) tile(c, c1 + 8 * I, c1);
    __syncthreads();
    // B: warp 0 factors the next panel while the others update the remaining lower tiles
    if (wid == 0) {
      panel(c1);
    } else {
      const int nrest = nb * (nb + 1) / 2 - nb;  // tiles (I, J) with I >= J >= 1 (relative)
      for (int tt = wid - 1; tt < nrest; tt += nw - 1) {
        // tt -> (I, J), 1 <= J <= I < nb, row-major over that triangle
        int I = (int)((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
        while ((I + 1) * (I + 2) / 2 <= tt) ++I;
        while (I * (I + 1) / 2 > tt) --I;
        const int J = tt - I * (I + 1) / 2;
        tile(c, c1 + 8 * (I + 1), c1 + 8 * (J + 1));
      }
    }
    __syncthreads();
  }
  RP_TSB(2);
  double *cf = coef_out + (int64_t)blockIdx.x * nc;
  double *inf = info_out + (int64_t)blockIdx.x * 5;
  if (s_status != 0) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) cf[i] = __longlong_as_double(0x7ff8000000000000ll);
    if (threadIdx.x == 0) {
      inf[0] = (double)s_status;
      inf[1] = 0;
      inf[2] = __longlong_as_double(0x7ff8000000000000ll);
      inf[3] = s_pmin;
      inf[4] = __longlong_as_double(0x7ff0000000000000ll);
    }
    return;
  }
  // ---- (L L^T) z = D b0 by warp 0, twice (the second on the double-double residual) ---------
  // (L L^T)^{-1} in place by warp 0: the register solver of k_solve (L lower, odd stride)
  auto chol_solve = [&](double *v) {
    if (wid == 0) chol_solve_warp(S, rd, ld, M8, v);
  };
  for (int i = threadIdx.x; i < M8; i += blockDim.x) x[i] = dsc[i] * b0[i];
  __syncthreads();
  chol_solve(x);
  __syncthreads();
  RP_TSB(3);
  for (int i = threadIdx.x; i < M8; i += blockDim.x) z[i] = dsc[i] * x[i];
  __syncthreads();
  // one refinement step: r = b0 - G_ff z in double-double from the original Gram
  for (int i = wid; i < m; i += nw) {
    const double *Gi = Gm + (int64_t)col(i) * nc;
    double hi = 0.0, lo = 0.0;
    double gv[kSbMaxM / 32];  // the row's entries, loaded together (one L2 round trip)
#pragma unroll
    for (int k = 0; k < kSbMaxM / 32; ++k) gv[k] = lane + 32 * k < m ? Gi[col(lane + 32 * k)] : 0.0;
#pragma unroll
    for (int k = 0; k < kSbMaxM / 32; ++k)
      if (lane + 32 * k < m) dd_fma(hi, lo, -gv[k], z[lane + 32 * k]);
    dd_warp_sum(hi, lo);
    if (lane == 0) {
      dd_add(hi, lo, b0[i]);
      x[i] = dsc[i] * (hi + lo);
    }
  }
  for (int i = m + threadIdx.x; i < M8; i += blockDim.x) x[i] = 0.0;
  __syncthreads();
  RP_TSB(4);
  chol_solve(x);
  __syncthreads();
  RP_TSB(5);
  for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] += dsc[i] * x[i];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) cf[col(i)] = z[i];
  if (threadIdx.x == 0) cf[beta0] = 1.0;
  // resid2 = coef^T G coef (double-double): a warp per row, then the warp partials in order
  __shared__ double s_rh[32], s_rl[32];
  {
    double wh = 0.0, wl = 0.0;
    for (int i = wid; i < nc; i += nw) {
      const double ci = (i == beta0) ? 1.0 : z[i < beta0 ? i : i - 1];
      double rh = 0.0, rl = 0.0;
      double gv[(kSbMaxM + 32) / 32];  // loaded together (one L2 round trip)
#pragma unroll
      for (int k = 0; k < (kSbMaxM + 32) / 32; ++k) {
        const int j = lane + 32 * k;
        gv[k] = j < nc ? Gm[(int64_t)i * nc + j] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < (kSbMaxM + 32) / 32; ++k) {
        const int j = lane + 32 * k;
        if (j < nc) dd_fma(rh, rl, gv[k], (j == beta0) ? 1.0 : z[j < beta0 ? j : j - 1]);
      }
      dd_warp_sum(rh, rl);
      dd_fma(wh, wl, ci, rh);
      dd_fma(wh, wl, ci, rl);
    }
    if (lane == 0) {
      s_rh[wid] = wh;
      s_rl[wid] = wl;
    }
  }
  __syncthreads();
  RP_TSB(6);
  if (threadIdx.x == 0) {
    double hi = 0.0, lo = 0.0;
    for (int w = 0; w < nw; ++w) {
      dd_add(hi, lo, s_rh[w]);
      lo += s_rl[w];
    }
#ifdef RP_SOLVE_TS
    for (int k = 1; k <= 6; ++k) cf[k] = (double)(tsb[k] - tsb[k - 1]);
#endif
    inf[0] = 0;
    inf[1] = (double)m;
    inf[2] = hi + lo;
    inf[3] = s_pmin;
    inf[4] = s_pmax / s_pmin;
  }
}

cudaError_t launch_solve(const double *G, int n_v, int nc, int beta0, double *coef_out,
                         double *info_out, cudaStream_t s) {
  const int m = nc - 1;
  if (m > 16 * kRA || m > 32 * kCB) return cudaErrorInvalidValue;
  const char *kv = getenv("RP_SOLVE_KERNEL");
  if (!(kv && strcmp(kv, "reg") == 0) && m <= kSbMaxM) {
    const int M8 = (m + 7) & ~7;
    const size_t smb = ((size_t)M8 * (M8 | 1) + 5 * (size_t)M8) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_solve_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    if (e != cudaSuccess) return e;
    k_solve_b<<<n_v, kSolveThreads, smb, s>>>(G, nc, beta0, coef_out, info_out);
    return cudaGetLastError();
  }
  const size_t smem = ((size_t)m * (m | 1) + 8 * (size_t)m) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_solve<<<n_v, kSolveThreads, smem, s>>>(G, nc, beta0, coef_out, info_out);
  return cudaGetLastError();
}

}  // namespace rp
