// DMMA.8x8x4 throughput versus warps per SM sub-partition and operand source, sm_100a.
// Question behind it: can 4 warps per SMSP (one 512-thread CTA per SM, the Gram kernel's shape)
// keep the FP64 tensor pipe busy, with register operands and with shared-memory fragments?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_occ dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC, bool SMEM>
__global__ void k(double* out, int iters) {
  __shared__ double sA[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) sA[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int t = 0; t < NACC; ++t) c[t][0] = c[t][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double* row = sA + (ks * 4 + (lane & 3)) * 36 + (lane >> 2);
#pragma unroll
      for (int t = 0; t < NACC; ++t) {
        double av = a, bv = b;
        if (SMEM) {
          av = row[8 * (t % 4)];
          bv = row[8 * ((t / 4) % 4) + 2 * 36 * 4];
        }
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(av), "d"(bv));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NACC; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC, bool SMEM>
void run(int nsm, int threads, int bps, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 400, blocks = nsm * bps;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<NACC, SMEM><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double flop = 2.0 * 256 * NACC * 2 * (double)iters * blocks * (threads / 32);
  printf("{\"nacc\":%d,\"smem\":%d,\"threads\":%d,\"blocks_per_sm\":%d,\"warps_per_smsp\":%d,\"tflops\":%.2f}\n", NACC,
         (int)SMEM, threads, bps, threads / 32 * bps / 4, flop / (ms * 1e-3) / 1e12);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)nsm * 2048 * 8);
  for (int bps : {1, 2}) {
    for (int th : {128, 256, 512}) {
      run<8, false>(nsm, th, bps, out);
      run<20, false>(nsm, th, bps, out);
      run<20, true>(nsm, th, bps, out);
    }
  }
  return 0;
}
