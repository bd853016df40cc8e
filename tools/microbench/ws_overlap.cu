// Do DMMA.8x8x4 and FP32 FFMA overlap when issued by *different* warps of a sub-partition
// (warp specialisation), sm_100a?  512-thread CTAs, one per SM: warps with (wid & 1) == 0 issue
// DMMAs (6 chains), odd warps FFMAs (8 chains); compared with the same warps doing one kind only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ws_overlap ws_overlap.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool DM, bool FF, int NFF>
__global__ void k(double* out, int iters) {
  const int wid = threadIdx.x >> 5;
  double c[6][2];
#pragma unroll
  for (int t = 0; t < 6; ++t) c[t][0] = c[t][1] = 0;
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  if ((wid & 1) == 0) {
    if (DM)
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 24; ++t)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[t % 6][0]), "+d"(c[t % 6][1]) : "d"(a), "d"(b));
      }
  } else {
    if (FF)
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int f = 0; f < NFF; ++f) x[f % 8] = fmaf(x[f % 8], 0.999f, 1e-3f);
      }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 6; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool DM, bool FF, int NFF>
float run(int blocks, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<DM, FF, NFF><<<blocks, 512>>>(out, 1000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  return ms;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)nsm * 512 * 8);
  const float td = run<true, false, 448>(nsm, out), tf = run<false, true, 448>(nsm, out), tb = run<true, true, 448>(nsm, out);
  printf("{\"dmma_warps_only_ms\":%.3f,\"ffma_warps_only_ms\":%.3f,\"both_ms\":%.3f,\"both_over_max\":%.3f,\"both_over_sum\":%.3f}\n",
         td, tf, tb, tb / (td > tf ? td : tf), tb / (td + tf));
  return 0;
}
