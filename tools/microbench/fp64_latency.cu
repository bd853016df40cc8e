// Dependent-chain latencies on one warp (clock64): DFMA, DADD, 64-bit SHFL, IEEE sqrt / div,
// MUFU.RCP64H, LDS.64, bar.sync (1 warp + 18 warps).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, double seed, int n) {
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  __shared__ double sm[1024];
  sm[threadIdx.x] = x;
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // 64-bit shuffle + add chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 3.0 / (x + 1.5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // rcp.approx chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x + 1.5));
    x = r;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // LDS chain (pointer chase through smem index)
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x += sm[idx];
    idx = ((int)x & 0) + ((idx + 1) & 1023);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // __syncthreads back to back
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  out[threadIdx.x] = x;
}

int main() {
  double *out;
  long long *cyc, h[8];
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8 * 8);
  const int n = 1000;
  const char *names[8] = {"DFMA", "SHFL64+DADD", "sqrt(f64)", "div(f64)", "rcp.approx.f64", "LDS.64+DADD", "bar.sync", "DMUL"};
  for (int threads : {32, 576}) {
    lat<<<1, threads>>>(out, cyc, 1.5, n);
    lat<<<1, threads>>>(out, cyc, 1.5, n);
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("{\"threads\": %d, \"op\": \"%s\", \"cycles\": %.1f}\n", threads, names[i], h[i] / (double)n);
  }
  return 0;
}
