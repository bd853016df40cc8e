// rp_pipeline.cu -- host-fed fit -> plan update -> sweep, pipelined over steps (C ABI).
//
// The paper's driver re-fits and re-evaluates the rational program as new profiles and new data
// sizes arrive (the program is evaluated "immediately preceding the launch of a
// kernel"; the metrics are re-estimated from measured samples).  A caller who
// feeds those batches from host memory pays two copies per step: the samples X, V and the tuples D
// in, the per-D winners out.  rp_pipeline overlaps them with the neighbouring steps' computation:
// step i+1's inputs stream in on one copy stream and step i-1's winners stream out on another while
// step i fits, refreshes the plan and sweeps on the compute stream.  Only copies, events and the
// library's own stream-ordered calls (rp_fit_dev, rp_plan_update_program, rp_plan_eval_argmin)
// happen here; device buffers are allocated once per in-flight slot.
//
// Per slot s (depth slots in flight):
//   h2d:     wait out_done[s] (the slot's previous step is retired), X, V, D -> s, in_ready[s]
//   compute: wait in_ready[s], fit (a10-a14), plan refresh, sweep (a1-a8), comp_done[s]
//   d2h:     wait comp_done[s], winners -> the caller's host arrays, out_done[s]
#include <cstdlib>
#include <vector>

#include "rp_internal.cuh"

struct rp_pipeline_s {
  rp_plan plan = nullptr;
  int prog = 0, n_v = 0, n = 0, nc = 0, d = 0, depth = 0;
  int64_t K = 0, nD = 0, n_out = 0;
  std::vector<int16_t> num, den;
  rp_basis basis{};
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  struct Slot {
    double *X = nullptr, *V = nullptr, *coef = nullptr, *xf = nullptr, *E = nullptr;
    int32_t *D = nullptr, *idx = nullptr;
    cudaEvent_t in_ready = nullptr, comp_done = nullptr, out_done = nullptr;
    bool used = false;
  };
  std::vector<Slot> slots;
  int64_t submitted = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // rp_pipeline_timer_*
};

static void pipeline_free(rp_pipeline p) {
  if (!p) return;
  if (p->h2d) cudaStreamSynchronize(p->h2d);
  if (p->comp) cudaStreamSynchronize(p->comp);
  if (p->d2h) cudaStreamSynchronize(p->d2h);
  for (auto &s : p->slots) {
    cudaFree(s.X);
    cudaFree(s.V);
    cudaFree(s.coef);
    cudaFree(s.xf);
    cudaFree(s.E);
    cudaFree(s.D);
    cudaFree(s.idx);
    if (s.in_ready) cudaEventDestroy(s.in_ready);
    if (s.comp_done) cudaEventDestroy(s.comp_done);
    if (s.out_done) cudaEventDestroy(s.out_done);
  }
  rp::plan_forget_stream(p->plan, p->comp);  // the plan outlives the pipeline's streams
  if (p->t0) cudaEventDestroy(p->t0);
  if (p->t1) cudaEventDestroy(p->t1);
  if (p->h2d) cudaStreamDestroy(p->h2d);
  if (p->comp) cudaStreamDestroy(p->comp);
  if (p->d2h) cudaStreamDestroy(p->d2h);
  delete p;
}

extern "C" {

rp_status rp_pipeline_create(rp_plan plan, int32_t prog, const rp_basis *basis, int32_t n_v, int64_t K,
                             int32_t d, int64_t nD, int32_t depth, rp_pipeline *out) {
  RP_REQUIRE(out, RP_ERR_INVALID_ARG, "null pipeline out");
  *out = nullptr;
  RP_REQUIRE(plan && basis && basis->num_exp && basis->den_exp, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(n_v >= 1 && n_v <= RP_MAX_METRICS && K >= 1 && nD >= 1 && d >= 1 && d <= RP_MAX_VARS &&
                 depth >= 1 && depth <= 4,
             RP_ERR_INVALID_ARG, "n_v %d, K %lld, d %d, nD %lld, depth %d", n_v, (long long)K, d, (long long)nD,
             depth);
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  RP_REQUIRE(n >= 1 && n <= RP_MAX_VARS && basis->n_num >= 1 && basis->n_den >= 1, RP_ERR_INVALID_ARG,
             "basis shape");
  RP_REQUIRE(rp::plan_num_programs(plan) == 1 && prog == 0, RP_ERR_INVALID_ARG,
             "a pipeline drives a single-program plan (prog 0)");
  RP_REQUIRE(rp::plan_num_data_params(plan) == d, RP_ERR_INVALID_ARG, "d %d != the plan's %d", d,
             rp::plan_num_data_params(plan));
  rp_pipeline p = new rp_pipeline_s;
  p->plan = plan;
  p->prog = prog;
  p->n_v = n_v;
  p->n = n;
  p->nc = nc;
  p->d = d;
  p->depth = depth;
  p->K = K;
  p->nD = nD;
  p->num.assign(basis->num_exp, basis->num_exp + (size_t)basis->n_num * n);
  p->den.assign(basis->den_exp, basis->den_exp + (size_t)basis->n_den * n);
  p->basis = *basis;
  p->basis.num_exp = p->num.data();
  p->basis.den_exp = p->den.data();
  auto fail = [&](cudaError_t e, const char *w) {
    rp_status r = rp::cuda_fail(e, w, __FILE__, __LINE__);
    pipeline_free(p);
    return r;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
  if ((e = cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
  if ((e = cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
  if ((e = cudaEventCreate(&p->t0)) != cudaSuccess) return fail(e, "event");
  if ((e = cudaEventCreate(&p->t1)) != cudaSuccess) return fail(e, "event");
  p->slots.resize(depth);
  for (auto &s : p->slots) {
    if ((e = cudaMalloc((void **)&s.X, sizeof(double) * K * n)) != cudaSuccess) return fail(e, "alloc X");
    if ((e = cudaMalloc((void **)&s.V, sizeof(double) * K * n_v)) != cudaSuccess) return fail(e, "alloc V");
    if ((e = cudaMalloc((void **)&s.coef, sizeof(double) * n_v * nc)) != cudaSuccess) return fail(e, "alloc coef");
    if ((e = cudaMalloc((void **)&s.xf, sizeof(double) * 2 * RP_MAX_VARS)) != cudaSuccess) return fail(e, "alloc xf");
    if ((e = cudaMalloc((void **)&s.D, sizeof(int32_t) * nD * d)) != cudaSuccess) return fail(e, "alloc D");
    if ((e = cudaMalloc((void **)&s.idx, sizeof(int32_t) * nD)) != cudaSuccess) return fail(e, "alloc idx");
    if ((e = cudaMalloc((void **)&s.E, sizeof(double) * nD)) != cudaSuccess) return fail(e, "alloc E");
    if ((e = cudaEventCreateWithFlags(&s.in_ready, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreateWithFlags(&s.comp_done, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "event");
  }
  *out = p;
  return RP_OK;
}

rp_status rp_pipeline_submit(rp_pipeline p, const double *X, const double *V, const int32_t *D, int32_t *best_idx,
                             double *best_E) {
  RP_REQUIRE(p && X && V && D && best_idx && best_E, RP_ERR_INVALID_ARG, "null argument");
  const int si = (int)(p->submitted % p->depth);
  auto &s = p->slots[si];
  // h2d: the slot's previous step must have left the device (its winners copied out)
  if (s.used) RP_CUDA(cudaStreamWaitEvent(p->h2d, s.out_done, 0));
  RP_CUDA(cudaMemcpyAsync(s.X, X, sizeof(double) * p->K * p->n, cudaMemcpyHostToDevice, p->h2d));
  RP_CUDA(cudaMemcpyAsync(s.V, V, sizeof(double) * p->K * p->n_v, cudaMemcpyHostToDevice, p->h2d));
  RP_CUDA(cudaMemcpyAsync(s.D, D, sizeof(int32_t) * p->nD * p->d, cudaMemcpyHostToDevice, p->h2d));
  RP_CUDA(cudaEventRecord(s.in_ready, p->h2d));
  s.used = true;
  // compute: fit (a10-a14) -> plan refresh -> sweep (a1-a8), all stream-ordered on the device
  RP_CUDA(cudaStreamWaitEvent(p->comp, s.in_ready, 0));
  rp_status st = rp_fit_dev(s.X, s.V, p->K, p->n_v, &p->basis, s.coef, s.xf, nullptr, p->comp);
  if (st != RP_OK) return st;
  if ((st = rp_plan_update_program(p->plan, p->prog, s.coef, p->nc, s.xf, p->comp)) != RP_OK) return st;
  if ((st = rp_plan_eval_argmin(p->plan, s.D, p->nD, s.idx, s.E, nullptr, p->comp)) != RP_OK) return st;
  RP_CUDA(cudaEventRecord(s.comp_done, p->comp));
  // d2h: the winners into the caller's host arrays
  RP_CUDA(cudaStreamWaitEvent(p->d2h, s.comp_done, 0));
  RP_CUDA(cudaMemcpyAsync(best_idx, s.idx, sizeof(int32_t) * p->nD, cudaMemcpyDeviceToHost, p->d2h));
  RP_CUDA(cudaMemcpyAsync(best_E, s.E, sizeof(double) * p->nD, cudaMemcpyDeviceToHost, p->d2h));
  RP_CUDA(cudaEventRecord(s.out_done, p->d2h));
  ++p->submitted;
  return RP_OK;
}

rp_status rp_pipeline_sync(rp_pipeline p) {
  RP_REQUIRE(p, RP_ERR_INVALID_ARG, "null pipeline");
  RP_CUDA(cudaStreamSynchronize(p->h2d));
  RP_CUDA(cudaStreamSynchronize(p->comp));
  RP_CUDA(cudaStreamSynchronize(p->d2h));
  return RP_OK;
}

rp_status rp_pipeline_timer_start(rp_pipeline p) {
  RP_REQUIRE(p, RP_ERR_INVALID_ARG, "null pipeline");
  RP_CUDA(cudaEventRecord(p->t0, p->h2d));
  return RP_OK;
}

rp_status rp_pipeline_timer_stop(rp_pipeline p, float *ms) {
  RP_REQUIRE(p && ms, RP_ERR_INVALID_ARG, "null argument");
  RP_CUDA(cudaEventRecord(p->t1, p->d2h));  // after the last submitted step's D2H
  RP_CUDA(cudaEventSynchronize(p->t1));
  RP_CUDA(cudaEventElapsedTime(ms, p->t0, p->t1));
  return RP_OK;
}

rp_status rp_pipeline_destroy(rp_pipeline p) {
  pipeline_free(p);
  return RP_OK;
}

}  // extern "C"
