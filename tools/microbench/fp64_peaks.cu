// FP64 pipe microbenchmarks on sm_100a: DFMA, DMMA.8x8x4 (mma.sync f64), IEEE double division,
// MUFU.RCP64H. Used once to derive the sweep/Gram roofline denominators.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ddiv(double* out, int iters, double b) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { x0 = b / x0 + 1.0; x1 = b / x1 + 1.0; x2 = b / x2 + 1.0; x3 = b / x3 + 1.0; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

__global__ void k_rcp(double* out, int iters) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x0)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x1));
      asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x2)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

int main() {
  int dev = 0, nsm = 0, clk = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d", p.name, nsm, clk);
  double* out; CK(cudaMalloc(&out, 148 * 64 * 1024 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int blocks = nsm * 4, threads = 512;
  // DFMA
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4000;
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 128 * iters * (double)blocks * threads;
    if (rep) printf(",\"dfma_tflops\":%.3f", flop / (ms * 1e-3) / 1e12);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 2000;
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    if (rep) printf(",\"dmma_tflops\":%.3f", flop / (ms * 1e-3) / 1e12);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1000;
    cudaEventRecord(e0); k_ddiv<<<blocks, threads>>>(out, iters, 3.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = 32.0 * iters * (double)blocks * threads;
    if (rep) printf(",\"ddiv_gops\":%.3f", n / (ms * 1e-3) / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 2000;
    cudaEventRecord(e0); k_rcp<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = 32.0 * iters * (double)blocks * threads;
    if (rep) printf(",\"rcp64_gops\":%.3f", n / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
