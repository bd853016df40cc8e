// umma_tf32.cu -- check the tcgen05 kind::tf32 building blocks of rp_umma.cuh and measure the
// accuracy of a 3-term split-tf32 product (hi*hi + hi*lo + lo*hi, FP32 accumulation in TMEM)
// against FP64, in units of u = 2^-24 of sum |a||b|; also the |a_hi||b_hi| bound GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1911_02373_b200/csrc tools/microbench/umma_tf32.cu -o tools/microbench/umma_tf32
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "rp_umma.cuh"

using namespace rp;

constexpr int M = 128, N = 32, K = 16;
constexpr uint32_t LBO = 128, SBO = 512;  // 4 core matrices along K per 8-row group
constexpr uint32_t A_BYTES = (M / 8) * SBO, B_BYTES = (N / 8) * SBO;

__global__ void k_test(const double *A, const double *B, float *out_val, float *out_bnd, int reps, long long *cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char *sAh = sm, *sAl = sm + A_BYTES, *sAa = sm + 2 * A_BYTES;
  unsigned char *sBh = sm + 3 * A_BYTES, *sBl = sBh + B_BYTES, *sBa = sBh + 2 * B_BYTES;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const double a = A[i];
    const float h = to_tf32((float)a), l = to_tf32((float)(a - (double)h));
    const uint32_t o = umma_off(r, k, LBO, SBO);
    *(float *)(sAh + o) = h;
    *(float *)(sAl + o) = l;
    *(float *)(sAa + o) = fabsf(h);
  }
  for (int i = t; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const double b = B[i];
    const float h = to_tf32((float)b), l = to_tf32((float)(b - (double)h));
    const uint32_t o = umma_off(r, k, LBO, SBO);
    *(float *)(sBh + o) = h;
    *(float *)(sBl + o) = l;
    *(float *)(sBa + o) = fabsf(h);
  }
  fence_async_smem();
  if (w == 0) tmem_alloc(smem_u32(&tbase), 64);
  if (t == 0) mbar_init(smem_u32(&bar), 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t idesc = umma_idesc_tf32(M, N);
  long long c0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (t == 0) {
      const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), aa = smem_u32(sAa);
      const uint32_t bh = smem_u32(sBh), bl = smem_u32(sBl), ba = smem_u32(sBa);
#pragma unroll
      for (int kk = 0; kk < K / 8; ++kk) {
        const uint32_t ko = kk * 2 * LBO;
        umma_tf32(tm, umma_sdesc(ah + ko, LBO, SBO), umma_sdesc(bh + ko, LBO, SBO), idesc, kk > 0);
        umma_tf32(tm, umma_sdesc(ah + ko, LBO, SBO), umma_sdesc(bl + ko, LBO, SBO), idesc, 1);
        umma_tf32(tm, umma_sdesc(al + ko, LBO, SBO), umma_sdesc(bh + ko, LBO, SBO), idesc, 1);
        umma_tf32(tm + N, umma_sdesc(aa + ko, LBO, SBO), umma_sdesc(ba + ko, LBO, SBO), idesc, kk > 0);
      }
      umma_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), rep & 1);
  }
  long long c1 = clock64();
  tc_fence_after();
  // thread t = TMEM lane t = row t
  const uint32_t lane_addr = tm + ((uint32_t)(w * 32) << 16);
  float v[16];
  for (int c = 0; c < N; c += 16) {
    tmem_ld16(lane_addr + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out_val[t * N + c + j] = v[j];
    tmem_ld16(lane_addr + N + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out_bnd[t * N + c + j] = v[j];
  }
  if (t == 0) *cyc = c1 - c0;
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tm, 64);
}

// issue throughput: `iters` x 48 MMAs (M = 128, N = NN, K = 8) back to back, one commit at the end
template <int NN>
__global__ void k_thru(int iters, long long *cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 40960 / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
  fence_async_smem();
  if (w == 0) tmem_alloc(smem_u32(&tbase), 512);
  if (t == 0) mbar_init(smem_u32(&bar), 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, idesc = umma_idesc_tf32(128, NN);
  if (t == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int j = 0; j < 48; ++j)
        umma_tf32(tm + (j % 12) * NN % 384, umma_sdesc(a + (j & 1) * 256, LBO, SBO), umma_sdesc(b + (j & 1) * 256, LBO, SBO),
                  idesc, j > 1);
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    *cyc = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tm, 512);
}

int main(int argc, char **argv) {
  if (argc > 2) {  // throughput mode: umma_tf32 <iters> <N>
    const int iters = atoi(argv[1]), nn = atoi(argv[2]);
    long long *dc, cyc = 0;
    cudaMalloc(&dc, 8);
    auto kern = nn == 16 ? k_thru<16> : nn == 32 ? k_thru<32> : k_thru<64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
    kern<<<148, 128, 40960>>>(iters, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("{\"N\": %d, \"iters\": %d, \"cycles_per_mma\": %.2f, \"err\": \"%s\"}\n", nn, iters,
           (double)cyc / (48.0 * iters), cudaGetErrorString(e));
    return 0;
  }
  const int reps = argc > 1 ? atoi(argv[1]) : 1000;
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(-1, 1), E(-6, 6);
  std::vector<double> A(M * K), B(N * K);
  for (auto &x : A) x = U(g) * pow(10.0, E(g) / 3);
  for (auto &x : B) x = U(g) * pow(10.0, E(g) / 3);
  double *dA, *dB;
  float *dv, *db;
  long long *dc;
  cudaMalloc(&dA, A.size() * 8);
  cudaMalloc(&dB, B.size() * 8);
  cudaMalloc(&dv, M * N * 4);
  cudaMalloc(&db, M * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  const int smem = 3 * A_BYTES + 3 * B_BYTES;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_test<<<1, 128, smem>>>(dA, dB, dv, db, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> v(M * N), b(M * N);
  long long cyc;
  cudaMemcpy(v.data(), dv, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), db, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double worst = 0, worst_bnd = 1e300, mean = 0;
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ex = 0, S = 0;
      for (int k = 0; k < K; ++k) {
        ex += A[i * K + k] * B[j * K + k];
        S += fabs(A[i * K + k] * B[j * K + k]);
      }
      const double err = fabs((double)v[i * N + j] - ex) / S / ldexp(1.0, -24);
      worst = fmax(worst, err);
      mean += err;
      worst_bnd = fmin(worst_bnd, (double)b[i * N + j] / S);
      if (!(err < 1e6)) ++bad;
    }
  printf("{\"M\": %d, \"N\": %d, \"K\": %d, \"max_err_u_of_S\": %.3f, \"mean_err_u_of_S\": %.3f, "
         "\"min_bound_over_S\": %.9f, \"bad\": %d, \"cycles_per_rep_4mma_x2k\": %.1f}\n",
         M, N, K, worst, mean / (M * N), worst_bnd, bad, (double)cyc / reps);
  return 0;
}
