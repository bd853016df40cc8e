// Do DMMA (FP64 tensor) and DFMA share the FP64 datapath on sm_100a?  Runs DFMA-only, DMMA-only
// and interleaved kernels with the same per-warp instruction counts and compares times.
// Also: IEEE double division vs rcp.approx + Newton division throughput.
#include <cstdio>
#include <cuda_runtime.h>
template <bool DO_FMA, bool DO_MMA>
__global__ void k_mix(double* out, int iters, double a, double b) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  double c[8][2];
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0;
  double av = threadIdx.x * 1e-3, bv = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (DO_FMA) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
      }
      if (DO_MMA)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(av), "d"(bv));
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j] + c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ double fast_div(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0); r = fma(r, e, r);
  e = fma(-b, r, 1.0); r = fma(r, e, r);
  double q = a * r;
  double rem = fma(-b, q, a);
  return fma(rem, r, q);
}
template <int MODE>
__global__ void k_div(double* out, int iters, double bb) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) { x0 = bb / x0 + 1.0; x1 = bb / x1 + 1.0; x2 = bb / x2 + 1.0; x3 = bb / x3 + 1.0; }
      else { x0 = fast_div(bb, x0) + 1.0; x1 = fast_div(bb, x1) + 1.0; x2 = fast_div(bb, x2) + 1.0; x3 = fast_div(bb, x3) + 1.0; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
template <class K> float timeit(K k, int blocks, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k(blocks, threads); cudaDeviceSynchronize();
  cudaEventRecord(e0); k(blocks, threads); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int B = 148 * 4, T = 512, it = 2000;
  float t_f = timeit([&](int b, int t) { k_mix<true, false><<<b, t>>>(out, it, 0.999, 1e-3); }, B, T);
  float t_m = timeit([&](int b, int t) { k_mix<false, true><<<b, t>>>(out, it, 0.999, 1e-3); }, B, T);
  float t_b = timeit([&](int b, int t) { k_mix<true, true><<<b, t>>>(out, it, 0.999, 1e-3); }, B, T);
  double fma_flop = 2.0 * 64 * it * (double)B * T;           // 64 DFMA per thread per iter
  double mma_flop = 2.0 * 256 * 8 * it * (double)B * (T / 32);  // 8 DMMA per warp per iter
  printf("{\"dfma_only_ms\":%.3f,\"dmma_only_ms\":%.3f,\"both_ms\":%.3f,\"dfma_tf\":%.2f,\"dmma_tf\":%.2f,\"both_tf\":%.2f",
         t_f, t_m, t_b, fma_flop / t_f / 1e9, mma_flop / t_m / 1e9, (fma_flop + mma_flop) / t_b / 1e9);
  float d0 = timeit([&](int b, int t) { k_div<0><<<b, t>>>(out, 500, 3.0); }, B, T);
  float d1 = timeit([&](int b, int t) { k_div<1><<<b, t>>>(out, 500, 3.0); }, B, T);
  double nd = 32.0 * 500 * (double)B * T;
  printf(",\"ieee_div_gops\":%.1f,\"fast_div_gops\":%.1f}\n", nd / d0 / 1e6, nd / d1 / 1e6);
  return 0;
}
