// DMMA.8x8x4 latency on sm_100a: one warp, a chain of NCH independent accumulators each advanced
// by a dependent DMMA per step; cycles per step / NCH -> issue interval, cycles per step -> the
// dependent latency once NCH chains no longer hide it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_latency dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[NCH][2];
#pragma unroll
  for (int t = 0; t < NCH; ++t) c[t][0] = c[t][1] = 0;
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < NCH; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int t = 0; t < NCH; ++t) s += c[t][0] + c[t][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int NCH>
void run(double* out, long long* dc) {
  const int iters = 10000;
  long long c = 0;
  for (int rep = 0; rep < 2; ++rep) {
    k<NCH><<<1, 32>>>(out, dc, iters);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  }
  printf("{\"chains\":%d,\"cycles_per_step\":%.1f,\"cycles_per_dmma\":%.1f}\n", NCH, (double)c / iters,
         (double)c / iters / NCH);
}

int main() {
  double* out;
  long long* dc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&dc, 8);
  run<1>(out, dc);
  run<2>(out, dc);
  run<4>(out, dc);
  run<6>(out, dc);
  run<8>(out, dc);
  run<12>(out, dc);
  return 0;
}
