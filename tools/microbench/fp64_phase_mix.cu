// FP64 datapath utilisation for the sweep's instruction mix on sm_100a: per loop iteration a warp
// issues NM DMMA.8x8x4 (6 accumulator chains) followed by NF scalar DFMAs (8 independent chains),
// as k_sweep does (24 DMMAs per config octet, then ~112 scalar FP64 ops of E for 2 pairs per lane).
// Reports the time against the sum of the DMMA-only and DFMA-only times of the same counts: a
// ratio of 1 means the two share the datapath without switching cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_phase_mix fp64_phase_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF, int PHASED, typename FT = double>
__global__ void k(double* out, int iters) {
  double c[6][2];
#pragma unroll
  for (int t = 0; t < 6; ++t) c[t][0] = c[t][1] = 0;
  FT x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = (FT)(threadIdx.x + j);
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
    if (PHASED) {
#pragma unroll
      for (int t = 0; t < NM; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t % 6][0]), "+d"(c[t % 6][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int f = 0; f < NF; ++f) x[f % 8] = fma(x[f % 8], (FT)0.999, (FT)1e-3);
    } else {  // interleaved: the same counts spread evenly
#pragma unroll
      for (int t = 0; t < NM; ++t) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t % 6][0]), "+d"(c[t % 6][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int f = 0; f < NF / (NM ? NM : 1); ++f)
          x[(t * (NF / (NM ? NM : 1)) + f) % 8] = fma(x[(t * (NF / (NM ? NM : 1)) + f) % 8], (FT)0.999, (FT)1e-3);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 6; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int j = 0; j < 8; ++j) s += (double)x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NM, int NF, int PH, typename FT = double>
float run(int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<NM, NF, PH, FT><<<blocks, threads>>>(out, 1000);
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
  cudaMalloc(&out, (size_t)nsm * 8 * 1024 * 8);
  for (int wps : {4, 8}) {  // warps per SM sub-partition
    const int blocks = nsm * wps / 4, threads = 512;
    const float tm = run<24, 0, 1>(blocks, threads, out);
    const float tf = run<0, 112, 1>(blocks, threads, out);
    const float tp = run<24, 112, 1>(blocks, threads, out);
    const float ti = run<24, 96, 0>(blocks, threads, out);
    const float tf96 = run<0, 96, 1>(blocks, threads, out);
    printf("{\"warps_per_smsp\":%d,\"dmma_only_ms\":%.3f,\"dfma_only_ms\":%.3f,\"phased_ms\":%.3f,\"phased_ratio\":%.3f,"
           "\"interleaved_ms\":%.3f,\"interleaved_ratio\":%.3f}\n",
           wps, tm, tf, tp, tp / (tm + tf), ti, ti / (tm + tf96));
    // FP32 FFMA (a different pipe) mixed with the DMMAs: does the DMMA rate survive?
    const float tf32 = run<0, 224, 1, float>(blocks, threads, out);
    const float tp32 = run<24, 224, 1, float>(blocks, threads, out);
    const float ti32 = run<24, 216, 0, float>(blocks, threads, out);
    printf("{\"warps_per_smsp\":%d,\"ffma224_only_ms\":%.3f,\"dmma24+ffma224_phased_ms\":%.3f,\"interleaved_ms\":%.3f,"
           "\"vs_max\":%.3f}\n", wps, tf32, tp32, ti32, tp32 / (tm > tf32 ? tm : tf32));
  }
  return 0;
}
