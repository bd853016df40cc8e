// rp_solve.cu -- a14: normalise beta_0 = 1 and solve the normal equations on the device.
//
// PAPER.md:2578-2584 solves the over-determined linearised system "by the method of linear
// least squares"; the draft footnote notes the system is homogeneous.
// Reading R12 fixes the constant denominator coefficient beta_0 = 1, turning it into
// G_ff z = -G_{f,beta0} with G = A^T A (reading R13: normal equations, as the north star asks;
// the paper's SVD is the f1 NEXT row).  The matrix is at most 160 x 160, so one CTA per metric
// does it in shared memory:
//   1. Jacobi equilibration  S = D G_ff D, D = diag(1/sqrt(G_ii))   (conditioning, R14);
//   2. right-looking Cholesky S = L L^T  (pivot <= 1e-13 -> RP_ERR_DEGENERATE);
//   3. two triangular solves;
//   4. one step of iterative refinement with the residual b - G_ff z accumulated in
//      double-double from the unrounded Gram entries, which removes the solve's own rounding
//      error and leaves only the Gram's.
#include "rp_internal.cuh"

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

// x <- (L L^T)^{-1} x, L lower triangular in sL (stride ld), rd[j] = 1 / L_jj.  One warp does
// both triangular solves (warp-synchronous steps instead of block-wide barriers).
__device__ void chol_solve(const double *sL, const double *rd, int ld, int m, double *x) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int j = 0; j < m; ++j) {  // forward: L y = x
      const double xj = x[j] * rd[j];
      __syncwarp();
      if (lane == 0) x[j] = xj;
      for (int i = j + 1 + lane; i < m; i += 32) x[i] -= sL[i * ld + j] * xj;
      __syncwarp();
    }
    for (int j = m - 1; j >= 0; --j) {  // backward: L^T z = y
      const double xj = x[j] * rd[j];
      __syncwarp();
      if (lane == 0) x[j] = xj;
      for (int i = lane; i < j; i += 32) x[i] -= sL[j * ld + i] * xj;
      __syncwarp();
    }
  }
  __syncthreads();
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

__global__ void __launch_bounds__(kSolveThreads) k_solve(const double *G, int nc, int beta0,
                                                         double *coef_out, double *info_out) {
  extern __shared__ __align__(16) double sm[];
  const int m = nc - 1, ld = m + 1;
  double *sL = sm;            // [m][ld]
  double *dsc = sL + m * ld;  // [m]
  double *b0 = dsc + m;       // -G_{f,beta0}
  double *x = b0 + m;         // work vector
  double *z = x + m;          // solution, unequilibrated
  double *rd = z + m;         // 1 / L_jj
  __shared__ int s_status;
  __shared__ double s_pmin, s_pmax;
  const double *Gm = G + (int64_t)blockIdx.x * nc * nc;
  auto col = [beta0](int i) { return i < beta0 ? i : i + 1; };

  if (threadIdx.x == 0) {
    s_status = 0;
    s_pmin = __longlong_as_double(0x7ff0000000000000ll);
    s_pmax = 0.0;
  }
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int i = t / m, j = t % m;
    sL[i * ld + j] = Gm[(int64_t)col(i) * nc + col(j)];
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) b0[i] = -Gm[(int64_t)col(i) * nc + beta0];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double di = sL[i * ld + i];
    if (!(di > 0.0)) s_status = RP_ERR_DEGENERATE;
    dsc[i] = di > 0.0 ? 1.0 / sqrt(di) : 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int i = t / m, j = t % m;
    sL[i * ld + j] *= dsc[i] * dsc[j];
  }
  __syncthreads();
  // Cholesky, lower triangle, blocked right-looking: an 8-column panel is factorised by warp 0
  // (warp-synchronous), then every warp applies the rank-8 update to its rows of the trailing
  // matrix (2 block barriers per panel)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int kb = 0; kb < m; kb += 8) {
    const int nb = (m - kb) < 8 ? (m - kb) : 8;
    if (wid == 0 && s_status == 0) {
      for (int c = kb; c < kb + nb; ++c) {
        const double piv = sL[c * ld + c];
        if (lane == 0) {
          if (!(piv > 1e-13)) s_status = RP_ERR_DEGENERATE;
          s_pmin = fmin(s_pmin, piv);
          s_pmax = fmax(s_pmax, piv);
        }
        const double lcc = sqrt(fmax(piv, 1e-300));
        const double rlcc = 1.0 / lcc;
        __syncwarp();
        if (lane == 0) sL[c * ld + c] = lcc;
        for (int i = c + 1 + lane; i < m; i += 32) sL[i * ld + c] *= rlcc;
        __syncwarp();
        for (int j = c + 1; j < kb + nb; ++j) {
          const double ljc = sL[j * ld + c];
          for (int i = j + lane; i < m; i += 32) sL[i * ld + j] -= sL[i * ld + c] * ljc;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (s_status != 0) break;
    const int j0 = kb + nb;
    for (int i = j0 + wid; i < m; i += nw) {
      double li[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) li[c] = c < nb ? sL[i * ld + kb + c] : 0.0;
      for (int j = j0 + lane; j <= i; j += 32) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nb) acc = fma(li[c], sL[j * ld + kb + c], acc);
        sL[i * ld + j] -= acc;
      }
    }
    __syncthreads();
  }
  __syncthreads();
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
  for (int i = threadIdx.x; i < m; i += blockDim.x) rd[i] = 1.0 / sL[i * ld + i];
  // solve
  for (int i = threadIdx.x; i < m; i += blockDim.x) x[i] = dsc[i] * b0[i];
  chol_solve(sL, rd, ld, m, x);
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
  chol_solve(sL, rd, ld, m, x);
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
  if (threadIdx.x == 0) {
    double hi = 0.0, lo = 0.0;
    for (int w = 0; w < nw; ++w) {
      dd_add(hi, lo, s_rh[w]);
      lo += s_rl[w];
    }
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
  const size_t smem = ((size_t)m * (m + 1) + 5 * (size_t)m) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_solve<<<n_v, kSolveThreads, smem, s>>>(G, nc, beta0, coef_out, info_out);
  return cudaGetLastError();
}

}  // namespace rp
