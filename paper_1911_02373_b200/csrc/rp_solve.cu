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

// x <- (L L^T)^{-1} x, L lower triangular in sL (stride ld); y is scratch.
__device__ void chol_solve(const double *sL, int ld, int m, double *x) {
  for (int j = 0; j < m; ++j) {  // forward: L y = x
    if (threadIdx.x == 0) x[j] /= sL[j * ld + j];
    __syncthreads();
    const double xj = x[j];
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) x[i] -= sL[i * ld + j] * xj;
    __syncthreads();
  }
  for (int j = m - 1; j >= 0; --j) {  // backward: L^T z = y
    if (threadIdx.x == 0) x[j] /= sL[j * ld + j];
    __syncthreads();
    const double xj = x[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) x[i] -= sL[j * ld + i] * xj;
    __syncthreads();
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
  // Cholesky, lower triangle
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      const double piv = sL[k * ld + k];
      if (!(piv > 1e-13)) s_status = RP_ERR_DEGENERATE;
      s_pmin = fmin(s_pmin, piv);
      s_pmax = fmax(s_pmax, piv);
      sL[k * ld + k] = sqrt(fmax(piv, 1e-300));
    }
    __syncthreads();
    if (s_status != 0) break;
    const double lkk = sL[k * ld + k];
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) sL[i * ld + k] /= lkk;
    __syncthreads();
    const int w = m - k - 1;
    for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
      const int i = k + 1 + t / w, j = k + 1 + t % w;
      if (j <= i) sL[i * ld + j] -= sL[i * ld + k] * sL[j * ld + k];
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
  // solve
  for (int i = threadIdx.x; i < m; i += blockDim.x) x[i] = dsc[i] * b0[i];
  __syncthreads();
  chol_solve(sL, ld, m, x);
  for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] = dsc[i] * x[i];
  __syncthreads();
  // one refinement step: r = b0 - G_ff z in double-double from the original Gram
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double hi = b0[i], lo = 0.0;
    const double *Gi = Gm + (int64_t)col(i) * nc;
    for (int j = 0; j < m; ++j) dd_fma(hi, lo, -Gi[col(j)], z[j]);
    x[i] = dsc[i] * (hi + lo);
  }
  __syncthreads();
  chol_solve(sL, ld, m, x);
  for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] += dsc[i] * x[i];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) cf[col(i)] = z[i];
  if (threadIdx.x == 0) cf[beta0] = 1.0;
  __syncthreads();
  // resid2 = coef^T G coef (double-double), from the original Gram
  if (threadIdx.x < 32) {
    double hi = 0.0, lo = 0.0;
    for (int i = threadIdx.x; i < nc; i += 32) {
      const double ci = (i == beta0) ? 1.0 : z[i < beta0 ? i : i - 1];
      double rh = 0.0, rl = 0.0;
      for (int j = 0; j < nc; ++j) {
        const double cj = (j == beta0) ? 1.0 : z[j < beta0 ? j : j - 1];
        dd_fma(rh, rl, Gm[(int64_t)i * nc + j], cj);
      }
      dd_fma(hi, lo, ci, rh);
      dd_fma(hi, lo, ci, rl);
    }
    for (int o = 16; o >= 1; o >>= 1) {
      const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
      dd_add(hi, lo, h2);
      lo += l2;
    }
    if (threadIdx.x == 0) {
      inf[0] = 0;
      inf[1] = (double)m;
      inf[2] = hi + lo;
      inf[3] = s_pmin;
      inf[4] = s_pmax / s_pmin;
    }
  }
}

cudaError_t launch_solve(const double *G, int n_v, int nc, int beta0, double *coef_out,
                         double *info_out, cudaStream_t s) {
  const int m = nc - 1;
  const size_t smem = ((size_t)m * (m + 1) + 4 * (size_t)m) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_solve<<<n_v, kSolveThreads, smem, s>>>(G, nc, beta0, coef_out, info_out);
  return cudaGetLastError();
}

}  // namespace rp
