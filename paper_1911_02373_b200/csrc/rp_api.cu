// rp_api.cu -- the C ABI of librp (include/rp.h): argument checks, host/device staging,
// program marshalling, plans.  All arithmetic of the method happens in the kernels of
// rp_sweep.cu, rp_gram.cu and rp_solve.cu.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "rp_internal.cuh"
#include "rp_decide.cuh"

namespace rp {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

rp_status cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
  set_error("CUDA error %d (%s) in %s at %s:%d", (int)e, cudaGetErrorString(e), what, file, line);
  cudaGetLastError();
  return RP_ERR_CUDA;
}

static bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static rp_status ensure_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device available (librp has no CPU fallback)");
    return RP_ERR_CUDA;
  }
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  return RP_OK;
}

// Stream-ordered temporary device buffer (cudaMallocAsync pool).
struct Tmp {
  void *p = nullptr;
  cudaStream_t s = nullptr;
  ~Tmp() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(&p, bytes ? bytes : 16, st);
  }
};

// Input that may be host or device: returns a device pointer (staging host data on `s`).
template <class T>
static rp_status stage_in(const T *src, size_t count, Tmp &tmp, const T **out, cudaStream_t s) {
  if (count == 0 || is_device_ptr(src)) {
    *out = src;
    return RP_OK;
  }
  RP_CUDA(tmp.alloc(count * sizeof(T), s));
  RP_CUDA(cudaMemcpyAsync(tmp.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  *out = (const T *)tmp.p;
  return RP_OK;
}
// Output that may be host or device: returns a device pointer; `host` is set if a copy back
// (and a synchronisation) is needed.
template <class T>
static rp_status stage_out(T *dst, size_t count, Tmp &tmp, T **out, bool *host, cudaStream_t s) {
  *host = false;
  if (!dst || count == 0 || is_device_ptr(dst)) {
    *out = dst;
    return RP_OK;
  }
  RP_CUDA(tmp.alloc(count * sizeof(T), s));
  *out = (T *)tmp.p;
  *host = true;
  return RP_OK;
}

// ---------------------------------------------------------------------------------------------
// program marshalling (layout only)
// ---------------------------------------------------------------------------------------------
static rp_status check_basis(const rp_basis &b, int n, const char *what, bool fit) {
  RP_REQUIRE(b.n_vars == n, RP_ERR_INVALID_ARG, "%s: basis n_vars %d != %d", what, b.n_vars, n);
  RP_REQUIRE(b.n_num >= 1 && b.n_den >= 1, RP_ERR_INVALID_ARG, "%s: empty numerator/denominator basis", what);
  RP_REQUIRE(b.num_exp && b.den_exp, RP_ERR_INVALID_ARG, "%s: null exponent table", what);
  for (int j = 0; j < b.n_num * n; ++j)
    RP_REQUIRE(b.num_exp[j] >= 0 && b.num_exp[j] <= 64, RP_ERR_INVALID_ARG, "%s: exponent out of [0,64]", what);
  for (int j = 0; j < b.n_den * n; ++j)
    RP_REQUIRE(b.den_exp[j] >= 0 && b.den_exp[j] <= 64, RP_ERR_INVALID_ARG, "%s: exponent out of [0,64]", what);
  if (fit)
    for (int k = 0; k < n; ++k)
      RP_REQUIRE(b.den_exp[k] == 0, RP_ERR_UNSUPPORTED,
                 "%s: den_exp[0] must be the zero vector (beta_0 = 1 normalisation)", what);
  return RP_OK;
}

rp_status compile_program(const rp_program *prog, DevProg *o) {
  RP_REQUIRE(prog, RP_ERR_INVALID_ARG, "null program");
  const int d = prog->d, p = prog->p, n = d + p, nm = prog->n_metrics;
  RP_REQUIRE(d >= 1 && p >= 1 && p <= 3 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG,
             "program: need d >= 1, 1 <= p <= 3, d + p <= %d (got d=%d p=%d)", RP_MAX_VARS, d, p);
  RP_REQUIRE(nm >= 1 && nm <= RP_MAX_METRICS, RP_ERR_INVALID_ARG, "program: n_metrics %d", nm);
  RP_REQUIRE(prog->e_template == RP_TEMPLATE_MWPCWP || prog->e_template == RP_TEMPLATE_G1,
             RP_ERR_INVALID_ARG, "program: unknown template %d", prog->e_template);
  RP_REQUIRE(prog->e_template != RP_TEMPLATE_MWPCWP || nm == 3, RP_ERR_INVALID_ARG,
             "program: the MWP-CWP template needs 3 metrics (comp, coal, uncoal)");
  const rp_hw &h = prog->hw;
  RP_REQUIRE(h.n_sm >= 1 && h.w_max >= 1 && h.b_max >= 1 && h.t_max >= 1 && h.r_max >= 1 && h.z_max >= 1,
             RP_ERR_INVALID_ARG, "program: hardware limits must be >= 1");
  RP_REQUIRE(h.n_sm < kRSMTab, RP_ERR_UNSUPPORTED, "program: n_sm = %d >= %d", h.n_sm, kRSMTab);
  RP_REQUIRE(prog->regs_per_thread >= 0 && prog->smem_words_base >= 0 && prog->smem_words_per_thread >= 0,
             RP_ERR_INVALID_ARG, "program: negative resource usage");
  for (int k = 0; k < 3; ++k)
    RP_REQUIRE(prog->grid_map[k] >= -1 && prog->grid_map[k] < d, RP_ERR_INVALID_ARG,
               "program: grid_map[%d] = %d out of range", k, prog->grid_map[k]);
  for (int k = 0; k < n; ++k)
    RP_REQUIRE(prog->xform.e[k] > -1000 && prog->xform.e[k] < 1000, RP_ERR_INVALID_ARG, "program: xform exponent");

  memset(o, 0, sizeof *o);
  o->d = d;
  o->p = p;
  o->nm = nm;
  o->tmpl = prog->e_template;
  o->npoly = 2 * nm;
  for (int k = 0; k < 3; ++k) o->grid_map[k] = prog->grid_map[k];
  o->n_sm = h.n_sm;
  o->w_max = h.w_max;
  o->b_max = h.b_max;
  o->t_max = h.t_max;
  o->r_max = h.r_max;
  o->z_max = h.z_max;
  o->R = prog->regs_per_thread;
  o->Z0 = prog->smem_words_base;
  o->Z1 = prog->smem_words_per_thread;
  o->freq = h.freq_hz;
  o->mem_bw = h.mem_bw;
  o->lbpw = h.load_bytes_per_warp;
  o->mem_ld = h.mem_ld;
  o->dd_coal = h.dd_coal;
  o->dd_unc = h.dd_unc;
  o->U = h.uncoal_per_mw;
  o->issue = h.issue_cycles;
  for (int k = 0; k < n; ++k) {
    o->xc[k] = prog->xform.c[k];
    o->xe[k] = prog->xform.e[k];
  }
  struct Term {
    int k;
    std::vector<int> eD, eP;
    double c;
    int src;
  };
  std::vector<Term> terms;
  for (int i = 0; i < nm; ++i) {
    rp_status st = check_basis(prog->basis[i], n, "program", false);
    if (st != RP_OK) return st;
    const rp_basis &b = prog->basis[i];
    RP_REQUIRE(prog->coef[i], RP_ERR_INVALID_ARG, "program: null coef[%d]", i);
    RP_REQUIRE(b.n_num + b.n_den < kMaxSrc, RP_ERR_UNSUPPORTED, "program: basis too large");
    for (int h2 = 0; h2 < 2; ++h2) {
      const int cnt = h2 ? b.n_den : b.n_num;
      const int16_t *ex = h2 ? b.den_exp : b.num_exp;
      for (int j = 0; j < cnt; ++j) {
        Term t;
        t.k = 2 * i + h2;
        t.eD.assign(ex + j * n, ex + j * n + d);
        t.eP.assign(ex + j * n + d, ex + j * n + n);
        t.c = prog->coef[i][(h2 ? b.n_num : 0) + j];
        t.src = i * kMaxSrc + (h2 ? b.n_num : 0) + j;
        terms.push_back(t);
      }
    }
  }
  auto graded_less = [](const std::vector<int> &a, const std::vector<int> &b) {
    int sa = 0, sb = 0;
    for (int v : a) sa += v;
    for (int v : b) sb += v;
    return sa != sb ? sa < sb : a < b;
  };
  std::vector<std::vector<int>> PE, DE;
  for (auto &t : terms) {
    PE.push_back(t.eP);
    DE.push_back(t.eD);
  }
  std::sort(PE.begin(), PE.end(), graded_less);
  PE.erase(std::unique(PE.begin(), PE.end()), PE.end());
  std::sort(DE.begin(), DE.end(), graded_less);
  DE.erase(std::unique(DE.begin(), DE.end()), DE.end());
  RP_REQUIRE((int)PE.size() <= kMaxPE, RP_ERR_UNSUPPORTED,
             "program: %d distinct program-part monomials > %d", (int)PE.size(), kMaxPE);
  RP_REQUIRE((int)DE.size() <= kMaxDE, RP_ERR_UNSUPPORTED,
             "program: %d distinct data-part monomials > %d", (int)DE.size(), kMaxDE);
  RP_REQUIRE((int)terms.size() <= kMaxTerms, RP_ERR_UNSUPPORTED, "program: %d terms > %d",
             (int)terms.size(), kMaxTerms);
  o->nPE = (int)PE.size();
  o->nDE = (int)DE.size();
  o->nterm = (int)terms.size();
  for (int a = 0; a < o->nPE; ++a)
    for (int k = 0; k < p; ++k) o->pe_exp[a][k] = (int8_t)PE[a][k];
  for (int a = 0; a < o->nDE; ++a)
    for (int k = 0; k < d; ++k) o->de_exp[a][k] = (int8_t)DE[a][k];
  // rows r = k * nPE + pe; terms grouped by row keeping basis order within a row
  const int nrows = o->npoly * o->nPE;
  std::vector<std::vector<const Term *>> rows(nrows);
  std::vector<int> tde(terms.size());
  for (size_t i = 0; i < terms.size(); ++i) {
    const Term &t = terms[i];
    const int pe = (int)(std::lower_bound(PE.begin(), PE.end(), t.eP, graded_less) - PE.begin());
    tde[i] = (int)(std::lower_bound(DE.begin(), DE.end(), t.eD, graded_less) - DE.begin());
    rows[t.k * o->nPE + pe].push_back(&t);
  }
  int pos = 0;
  for (int r = 0; r < nrows; ++r) {
    o->row_start[r] = (int16_t)pos;
    for (const Term *t : rows[r]) {
      o->term_de[pos] = (int16_t)tde[t - terms.data()];
      o->term_coef[pos] = t->c;
      o->term_src[pos] = (int16_t)t->src;
      ++pos;
    }
  }
  o->row_start[nrows] = (int16_t)pos;
  return RP_OK;
}

static int npe_pad_for(int nPE) {
  const int opts[] = {4, 8, 16, 20, 24, 36};
  for (int v : opts)
    if (nPE <= v) return v;
  return -1;
}

static rp_status build_gram_basis(const rp_basis *basis, const rp_xform *xf, GramBasis *gb) {
  RP_REQUIRE(basis, RP_ERR_INVALID_ARG, "null basis");
  const int n = basis->n_vars;
  RP_REQUIRE(n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "basis: n_vars %d", n);
  rp_status st = check_basis(*basis, n, "fit", true);
  if (st != RP_OK) return st;
  const int nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc <= 176, RP_ERR_UNSUPPORTED, "fit: n_c = %d > 176 columns", nc);
  memset(gb, 0, sizeof *gb);
  gb->n = n;
  gb->n_num = basis->n_num;
  gb->n_den = basis->n_den;
  gb->nc = nc;
  int maxdeg = 0;
  for (int j = 0; j < nc; ++j)
    for (int k = 0; k < n; ++k) {
      const int e = j < basis->n_num ? basis->num_exp[j * n + k] : basis->den_exp[(j - basis->n_num) * n + k];
      gb->exp[j][k] = (int8_t)e;
      maxdeg = std::max(maxdeg, e);
    }
  gb->maxdeg = maxdeg;
  // the fused weighted-Gram path needs identical numerator / denominator exponent lists
  bool same = basis->n_num == basis->n_den && maxdeg <= 15;
  for (int j = 0; same && j < basis->n_num * n; ++j) same = basis->num_exp[j] == basis->den_exp[j];
  gb->fused = same ? 1 : 0;
  for (int j = 0; j < basis->n_num; ++j) {
    uint32_t w = 0;
    for (int k = 0; k < n; ++k) w |= (uint32_t)(basis->num_exp[j * n + k] & 15) << (4 * k);
    gb->pexp[j] = w;
  }
  // monomial tree (layout only): parent = the column with one unit less of the first variable
  // that has a nonzero exponent
  {
    const int m = basis->n_num;
    bool tree = same && m <= 256;
    int nconst = 0, maxd = 0;
    std::vector<int> deg(m, 0);
    for (int j = 0; tree && j < m; ++j) {
      const int16_t *e = basis->num_exp + j * n;
      for (int k = 0; k < n; ++k) deg[j] += e[k];
      maxd = std::max(maxd, deg[j]);
      if (deg[j] == 0) {
        ++nconst;
        gb->parent[j] = -1;
        gb->pvar[j] = 0;
        continue;
      }
      int k0 = 0;
      while (e[k0] == 0) ++k0;
      int par = -1;
      for (int i = 0; i < m && par < 0; ++i) {
        const int16_t *f = basis->num_exp + i * n;
        bool eq = true;
        for (int k = 0; k < n && eq; ++k) eq = f[k] == e[k] - (k == k0 ? 1 : 0);
        if (eq) par = i;
      }
      if (par < 0) tree = false;
      gb->parent[j] = (int16_t)par;
      gb->pvar[j] = (int8_t)k0;
    }
    tree = tree && nconst == 1 && maxd <= 16;
    gb->tree = tree ? 1 : 0;
    if (tree) {
      int pos = 0;
      for (int d = 0; d <= maxd; ++d) {
        gb->lv_start[d] = (int16_t)pos;
        for (int j = 0; j < m; ++j)
          if (deg[j] == d) gb->lv_cols[pos++] = (int16_t)j;
      }
      gb->lv_start[maxd + 1] = (int16_t)pos;
      gb->n_lv = maxd + 1;
    }
  }
  if (xf)
    for (int k = 0; k < n; ++k) {
      gb->xc[k] = xf->c[k];
      gb->xe[k] = xf->e[k];
    }
  return RP_OK;
}

}  // namespace rp

using namespace rp;

// =============================================================================================
// plans
// =============================================================================================
struct rp_plan_s {
  int device = 0;
  int n_prog = 0, nF = 0, d = 0, p = 0, npe_pad = 0;
  bool mwp = true;
  int nde_max = 1, n_sm_max = 1;
  int kb = 1;  // D1 bucket bound: kb^2 > max T_max >= P1 P2 of any feasible configuration
  DevProg *d_progs = nullptr;
  int32_t *buf_i = nullptr;
  double *buf_d = nullptr;
  unsigned char *buf_g = nullptr;  // the sweep's tile schedule (CfgTable grec, gmP, ghv, gdesc, gcnt)
  int32_t *d_F = nullptr;  // F kept on the device (rp_plan_update_program re-runs a1 / a5)
  std::vector<int> nc_of;  // per program: max n_c over its metrics (coefficient row stride check)
  CfgTable tab{};
  cudaStream_t stream = nullptr;
  HistTable hist;
  int n_deciders = 0;  // live rp_decider objects whose captured graph holds hist.slots
  // rp_plan_enable_timing: events around the phases of the last rp_plan_eval_argmin
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // start, sweep, refine, end
};

namespace rp {
int plan_num_programs(rp_plan plan) { return plan ? plan->n_prog : 0; }
int plan_num_data_params(rp_plan plan) { return plan ? plan->d : 0; }
// a stream the plan was last used on is about to be destroyed: later stream-ordered frees of the
// plan go to the legacy default stream instead
void plan_forget_stream(rp_plan plan, cudaStream_t s) {
  if (plan && plan->stream == s) plan->stream = nullptr;
}
}  // namespace rp

static void plan_free(rp_plan pl) {
  if (!pl) return;
  // stream-ordered frees on the stream the plan was last used on (rp.h: rp_plan_destroy)
  if (pl->d_progs) cudaFreeAsync(pl->d_progs, pl->stream);
  if (pl->buf_i) cudaFreeAsync(pl->buf_i, pl->stream);
  if (pl->buf_d) cudaFreeAsync(pl->buf_d, pl->stream);
  if (pl->buf_g) cudaFreeAsync(pl->buf_g, pl->stream);
  if (pl->d_F) cudaFreeAsync(pl->d_F, pl->stream);
  if (pl->hist.slots) {
    cudaStreamSynchronize(pl->stream);
    cudaFree(pl->hist.slots);
    cudaFree(pl->hist.counters);
  }
  for (cudaEvent_t &e : pl->ev)
    if (e) cudaEventDestroy(e);
  delete pl;
}

static rp_status plan_create(const rp_program *progs, int32_t n_prog, const int32_t *F, int32_t nF,
                             rp_plan *out, cudaStream_t s, bool async_free) {
  RP_REQUIRE(out, RP_ERR_INVALID_ARG, "null plan out");
  *out = nullptr;
  RP_REQUIRE(progs && n_prog >= 1 && n_prog <= 65535, RP_ERR_INVALID_ARG, "n_prog %d", n_prog);
  RP_REQUIRE(F && nF >= 1 && nF <= 65536, RP_ERR_UNSUPPORTED, "nF = %d outside [1, 65536]", nF);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  std::vector<DevProg> hp(n_prog);
  int npe_max = 0;
  for (int g = 0; g < n_prog; ++g) {
    st = compile_program(&progs[g], &hp[g]);
    if (st != RP_OK) return st;
    RP_REQUIRE(progs[g].d == progs[0].d && progs[g].p == progs[0].p &&
                   progs[g].e_template == progs[0].e_template,
               RP_ERR_INVALID_ARG, "batched programs must share d, p and the E template");
    npe_max = std::max(npe_max, hp[g].nPE);
  }
  const int npe_pad = npe_pad_for(npe_max);
  RP_REQUIRE(npe_pad > 0, RP_ERR_UNSUPPORTED, "too many program-part monomials");
  rp_plan pl = new rp_plan_s;
  pl->n_prog = n_prog;
  pl->nF = nF;
  pl->d = progs[0].d;
  pl->p = progs[0].p;
  pl->npe_pad = npe_pad;
  pl->stream = s;
  (void)async_free;
  cudaGetDevice(&pl->device);
  auto fail = [&](cudaError_t e, const char *w) {
    rp_status r = cuda_fail(e, w, __FILE__, __LINE__);
    plan_free(pl);
    return r;
  };
  pl->mwp = progs[0].e_template == RP_TEMPLATE_MWPCWP;
  cudaError_t e;
  const int nFp = (nF + 7) & ~7;
  for (int g = 0; g < n_prog; ++g) {
    pl->nde_max = std::max(pl->nde_max, hp[g].nDE);
    pl->n_sm_max = std::max(pl->n_sm_max, hp[g].n_sm);
    int kb = 1;
    while ((int64_t)kb * kb <= (int64_t)hp[g].t_max) ++kb;
    pl->kb = std::max(pl->kb, kb);
  }
  const int nde_pad = std::max(4, (pl->nde_max + 3) & ~3);
  const size_t nrec = (size_t)n_prog * nFp;                               // CfgRec (64 B)
  const size_t ncm = (size_t)n_prog * kMaxPolys * npe_pad * nde_pad;      // Cmat
  const size_t nrt = (size_t)n_prog * npe_pad * nde_pad;                  // refinement terms
  const size_t nd = 2 * (size_t)n_prog * nFp * npe_pad + (size_t)n_prog * kRSMTab + ncm +  // mP x2, rSM, Cmat,
                    nrt * kMaxPolys + (size_t)n_prog * 8 +                                  // rcoef, rinfo,
                    2 * (size_t)n_prog * nFp * npe_pad;                                     // mPdd
  const size_t ni = 2 * nrec * sizeof(CfgRec) + n_prog * 8 + 16 + nrt * 4 + nrec * 4;  // rec, srec, nFc, rterm, inv
  // stream-ordered pool allocations (a synchronous cudaMalloc/cudaFree per plan costs ms)
  if ((e = cudaMallocAsync((void **)&pl->d_progs, sizeof(DevProg) * n_prog, s)) != cudaSuccess) return fail(e, "alloc");
  if ((e = cudaMallocAsync((void **)&pl->buf_i, ni, s)) != cudaSuccess) return fail(e, "alloc");
  if ((e = cudaMallocAsync((void **)&pl->buf_d, nd * 8, s)) != cudaSuccess) return fail(e, "alloc");
  // zero padding entries: padded configurations read as m_pe = 0 by the DMMA tiles
  if ((e = cudaMemsetAsync(pl->buf_i, 0, ni, s)) != cudaSuccess) return fail(e, "memset");
  if ((e = cudaMemsetAsync(pl->buf_d, 0, nd * 8, s)) != cudaSuccess) return fail(e, "memset");
  pl->tab.nFp = nFp;
  pl->tab.rec = reinterpret_cast<CfgRec *>(pl->buf_i);
  pl->tab.srec = pl->tab.rec + nrec;
  pl->tab.nFc = reinterpret_cast<int32_t *>(pl->tab.srec + nrec);
  pl->tab.mP = pl->buf_d;
  pl->tab.smP = pl->buf_d + (size_t)n_prog * nFp * npe_pad;
  pl->tab.rSM = pl->tab.smP + (size_t)n_prog * nFp * npe_pad;
  pl->tab.Cmat = pl->tab.rSM + (size_t)n_prog * kRSMTab;
  pl->tab.nde_pad = nde_pad;
  pl->tab.rcoef = pl->tab.Cmat + ncm;  // even offset (ncm and kRSMTab even): 16-byte aligned
  pl->tab.rinfo = pl->tab.rcoef + nrt * kMaxPolys;
  pl->tab.mPdd = reinterpret_cast<double2 *>(pl->tab.rinfo + (size_t)n_prog * 8);  // (16-byte aligned)
  pl->tab.rterm = pl->tab.nFc + 2 * n_prog + 4;
  pl->tab.inv = pl->tab.rterm + nrt;
  pl->tab.nrt_max = 1;
  {  // tile schedule: factored tiles are full, the dense part pads once (slots <= nFc + 7)
    const int nGp = nFp + 8;
    const size_t b_rec = (size_t)n_prog * nGp * sizeof(CfgRec), b_mp = (size_t)n_prog * npe_pad * nGp * 8,
                 b_hv = (size_t)n_prog * nGp * 4, b_gd = (size_t)n_prog * kMaxGroups * sizeof(GroupDesc),
                 b_cnt = (size_t)n_prog * 16;
    const size_t nb = b_rec + b_mp + b_hv + b_gd + b_cnt;
    if ((e = cudaMallocAsync((void **)&pl->buf_g, nb, s)) != cudaSuccess) return fail(e, "alloc");
    if ((e = cudaMemsetAsync(pl->buf_g, 0, nb, s)) != cudaSuccess) return fail(e, "memset");
    pl->tab.nGp = nGp;
    pl->tab.grec = reinterpret_cast<CfgRec *>(pl->buf_g);
    pl->tab.gmP = reinterpret_cast<double *>(pl->buf_g + b_rec);
    pl->tab.gdesc = reinterpret_cast<GroupDesc *>(pl->buf_g + b_rec + b_mp);
    pl->tab.ghv = reinterpret_cast<int32_t *>(pl->buf_g + b_rec + b_mp + b_gd);
    pl->tab.gcnt = pl->tab.ghv + (size_t)n_prog * nGp;
  }
  for (int g = 0; g < n_prog; ++g) {  // distinct (pe, de) pairs over the polynomials' terms
    std::vector<char> seen((size_t)npe_pad * nde_pad, 0);
    int cnt = 0;
    for (int r = 0; r < hp[g].npoly * hp[g].nPE; ++r)
      for (int j = hp[g].row_start[r]; j < hp[g].row_start[r + 1]; ++j) {
        char &c = seen[(size_t)(r % hp[g].nPE) * nde_pad + hp[g].term_de[j]];
        cnt += c == 0;
        c = 1;
      }
    pl->tab.nrt_max = std::max(pl->tab.nrt_max, cnt);
  }
  // the DevProg blob is staged through pinned-free pageable memory: copy synchronously w.r.t.
  // the host buffer lifetime (cudaMemcpyAsync from pageable memory returns after staging)
  if ((e = cudaMemcpyAsync(pl->d_progs, hp.data(), sizeof(DevProg) * n_prog, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return fail(e, "H2D program");
  if ((e = cudaMallocAsync((void **)&pl->d_F, (size_t)nF * pl->p * sizeof(int32_t), s)) != cudaSuccess)
    return fail(e, "alloc");
  if ((e = cudaMemcpyAsync(pl->d_F, F, (size_t)nF * pl->p * sizeof(int32_t), cudaMemcpyDefault, s)) != cudaSuccess)
    return fail(e, "F");
  for (int g = 0; g < n_prog; ++g) {
    int m = 0;
    for (int i = 0; i < progs[g].n_metrics; ++i) m = std::max(m, progs[g].basis[i].n_num + progs[g].basis[i].n_den);
    pl->nc_of.push_back(m);
  }
  if ((e = launch_plan_configs(pl->d_progs, n_prog, pl->d_F, nF, npe_pad, pl->tab, s)) != cudaSuccess)
    return fail(e, "k_plan_configs");
  *out = pl;
  return RP_OK;
}

static rp_status plan_eval(rp_plan pl, const int32_t *D, int64_t nD, int32_t *best_idx,
                           double *best_E, double *second_E, cudaStream_t s) {
  RP_REQUIRE(pl, RP_ERR_INVALID_ARG, "null plan");
  RP_REQUIRE(nD >= 0, RP_ERR_INVALID_ARG, "nD < 0");
  if (nD == 0) return RP_OK;
  RP_REQUIRE(D && best_idx && best_E, RP_ERR_INVALID_ARG, "null D / outputs");
  RP_REQUIRE((nD + 7) / 8 <= 0x7fffffffll, RP_ERR_UNSUPPORTED, "nD too large");
  pl->stream = s;
  Tmp tD, ti, tb, ts;
  const int32_t *dD;
  rp_status st = stage_in(D, (size_t)nD * pl->d, tD, &dD, s);
  if (st != RP_OK) return st;
  const size_t no = (size_t)pl->n_prog * nD;
  int32_t *di;
  double *db, *ds;
  bool hi, hb, hs;
  if ((st = stage_out(best_idx, no, ti, &di, &hi, s)) != RP_OK) return st;
  if ((st = stage_out(best_E, no, tb, &db, &hb, s)) != RP_OK) return st;
  if ((st = stage_out(second_E, no, ts, &ds, &hs, s)) != RP_OK) return st;
  // group tuples by D1 (only D1 < kb, kb^2 > T_max >= P1 P2, can fail the D rule) so whole
  // configuration octets are skipped by the sweep's early exit; pays off on large batches
  if (pl->timing) RP_CUDA(cudaEventRecord(pl->ev[0], s));
  Tmp tperm;
  const int32_t *perm = nullptr;
  if (nD >= 4096 && nD <= 0x7fffffffll && pl->kb < 255) {
    const int kb = pl->kb;
    RP_CUDA(tperm.alloc((size_t)nD * 4 + (size_t)(kb + 1) * 4 + 16, s));
    int32_t *p = (int32_t *)tperm.p;
    RP_CUDA(launch_bucket_perm(dD, nD, pl->d, kb, (unsigned *)(p + nD), p, s));
    perm = p;
  }
  // the runner-ups' indices, for the refinement of the runner-up (rp_sweep.cu k_refine)
  Tmp tidx2;
  int32_t *idx2 = nullptr;
  if (ds) {
    RP_CUDA(tidx2.alloc(no * 4, s));
    idx2 = (int32_t *)tidx2.p;
  }
  RP_CUDA(launch_sweep(pl->d_progs, pl->n_prog, pl->mwp, pl->tab, pl->npe_pad, pl->nde_max, pl->n_sm_max,
                       pl->d, dD, nD, di, db, ds, perm, idx2, pl->timing ? pl->ev : nullptr, s));
  if (pl->timing) RP_CUDA(cudaEventRecord(pl->ev[3], s));

  if (hi) RP_CUDA(cudaMemcpyAsync(best_idx, di, no * 4, cudaMemcpyDeviceToHost, s));
  if (hb) RP_CUDA(cudaMemcpyAsync(best_E, db, no * 8, cudaMemcpyDeviceToHost, s));
  if (hs) RP_CUDA(cudaMemcpyAsync(second_E, ds, no * 8, cudaMemcpyDeviceToHost, s));
  if (hi || hb || hs) RP_CUDA(cudaStreamSynchronize(s));
  return RP_OK;
}

namespace rp {
rp_status check_program(const rp_program *prog) {
  std::vector<DevProg> t(1);
  return compile_program(prog, t.data());
}

rp_status jit_stage_and_launch(rp_jit jit, const int32_t *D, int64_t nD, const int32_t *F, int32_t nF,
                                   int32_t *best_idx, double *best_E, double *second_E, cudaStream_t s) {
  if (nD == 0) return RP_OK;
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  const int d = rp_jit_dims(jit, 0), p = rp_jit_dims(jit, 1);
  Tmp tD, tF, ti, tb, ts;
  const int32_t *dD, *dF;
  if ((st = stage_in(D, (size_t)nD * d, tD, &dD, s)) != RP_OK) return st;
  if ((st = stage_in(F, (size_t)nF * p, tF, &dF, s)) != RP_OK) return st;
  int32_t *di;
  double *db, *ds;
  bool hi, hb, hs;
  if ((st = stage_out(best_idx, (size_t)nD, ti, &di, &hi, s)) != RP_OK) return st;
  if ((st = stage_out(best_E, (size_t)nD, tb, &db, &hb, s)) != RP_OK) return st;
  if ((st = stage_out(second_E, (size_t)nD, ts, &ds, &hs, s)) != RP_OK) return st;
  RP_CUDA(launch_jit(jit, dD, nD, dF, nF, di, db, ds, s));
  if (hi) RP_CUDA(cudaMemcpyAsync(best_idx, di, (size_t)nD * 4, cudaMemcpyDeviceToHost, s));
  if (hb) RP_CUDA(cudaMemcpyAsync(best_E, db, (size_t)nD * 8, cudaMemcpyDeviceToHost, s));
  if (hs) RP_CUDA(cudaMemcpyAsync(second_E, ds, (size_t)nD * 8, cudaMemcpyDeviceToHost, s));
  if (hi || hb || hs) RP_CUDA(cudaStreamSynchronize(s));
  return RP_OK;
}
}  // namespace rp

// =============================================================================================
// ABI
// =============================================================================================
extern "C" {

int32_t rp_abi_version(void) { return RP_ABI_VERSION; }
const char *rp_last_error(void) { return g_err; }
int32_t rp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

rp_status rp_xform_from_box(int32_t n, const double *lo, const double *hi, rp_xform *out) {
  RP_REQUIRE(n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "n = %d", n);
  RP_REQUIRE(lo && hi && out, RP_ERR_INVALID_ARG, "null argument");
  for (int k = 0; k < n; ++k) RP_REQUIRE(lo[k] <= hi[k], RP_ERR_INVALID_ARG, "hi < lo at %d", k);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  double hlohi[2 * RP_MAX_VARS], hout[2 * RP_MAX_VARS];
  for (int k = 0; k < n; ++k) {
    hlohi[2 * k] = lo[k];
    hlohi[2 * k + 1] = hi[k];
  }
  Tmp t;
  RP_CUDA(t.alloc(4 * RP_MAX_VARS * sizeof(double), nullptr));
  double *d = (double *)t.p;
  RP_CUDA(cudaMemcpyAsync(d, hlohi, 2 * n * sizeof(double), cudaMemcpyHostToDevice, nullptr));
  RP_CUDA(launch_xform(d, n, d + 2 * RP_MAX_VARS, nullptr));
  RP_CUDA(cudaMemcpyAsync(hout, d + 2 * RP_MAX_VARS, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, nullptr));
  RP_CUDA(cudaStreamSynchronize(nullptr));
  memset(out, 0, sizeof *out);
  for (int k = 0; k < n; ++k) {
    out->c[k] = hout[2 * k];
    out->e[k] = (int32_t)hout[2 * k + 1];
  }
  return RP_OK;
}

rp_status rp_minmax(const double *X, int64_t K, int32_t n, double *lo, double *hi, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(X && lo && hi, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 1 && n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "K = %lld, n = %d", (long long)K, n);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  Tmp tX, tw;
  const double *dX;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  const int nblk = minmax_blocks(K);
  RP_CUDA(tw.alloc(((size_t)nblk * n * 2 + 2 * RP_MAX_VARS) * sizeof(double), s));
  double *part = (double *)tw.p, *res = part + (size_t)nblk * n * 2;
  RP_CUDA(launch_minmax(dX, K, n, part, nblk, res, s));
  double h[2 * RP_MAX_VARS];
  RP_CUDA(cudaMemcpyAsync(h, res, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < n; ++k) {
    lo[k] = h[2 * k];
    hi[k] = h[2 * k + 1];
  }
  return RP_OK;
}

static rp_status gram_impl(const double *X, const double *V, const double *S, int64_t K, int32_t n_v,
                           const rp_basis *basis, const rp_xform *xform, double *G, cudaStream_t s) {
  RP_REQUIRE(G && basis && xform, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 0 && n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "K = %lld, n_v = %d", (long long)K, n_v);
  RP_REQUIRE(K == 0 || (X && V), RP_ERR_INVALID_ARG, "null X / V");
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  GramBasis gb;
  if ((st = build_gram_basis(basis, xform, &gb)) != RP_OK) return st;
  const int nc = gb.nc, n = gb.n;
  Tmp tX, tV, tG, tb, tp;
  const double *dX = nullptr, *dV = nullptr;
  double *dG;
  bool hG;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_in(V, (size_t)K * n_v, tV, &dV, s)) != RP_OK) return st;
  Tmp tS;
  const double *dS = nullptr;
  if (S && (st = stage_in(S, (size_t)K * n_v, tS, &dS, s)) != RP_OK) return st;
  if ((st = stage_out(G, (size_t)n_v * nc * nc, tG, &dG, &hG, s)) != RP_OK) return st;
  if (K == 0) {
    RP_CUDA(cudaMemsetAsync(dG, 0, (size_t)n_v * nc * nc * 8, s));
  } else {
    RP_CUDA(tb.alloc(sizeof(GramBasis), s));
    RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
    const size_t pe = gram_partial_elems(gb, n_v, K, num_sms(), dS != nullptr);
    RP_CUDA(tp.alloc(pe * 8, s));
    RP_CUDA(launch_gram((const GramBasis *)tb.p, gb, dX, dV, dS, K, n_v, dG, (double *)tp.p, pe, s));
  }
  // (host sources of H2D copies from pageable memory are consumed before cudaMemcpyAsync
  // returns, so stack-resident staging data needs no synchronisation)
  if (hG) {
    RP_CUDA(cudaMemcpyAsync(G, dG, (size_t)n_v * nc * nc * 8, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
  return RP_OK;
}

rp_status rp_gram_accumulate(const double *X, const double *V, int64_t K, int32_t n_v,
                             const rp_basis *basis, const rp_xform *xform, double *G, rp_stream sv) {
  return gram_impl(X, V, nullptr, K, n_v, basis, xform, G, (cudaStream_t)sv);
}

rp_status rp_gram_accumulate_weighted(const double *X, const double *V, const double *S, int64_t K,
                                      int32_t n_v, const rp_basis *basis, const rp_xform *xform,
                                      double *G, rp_stream sv) {
  RP_REQUIRE(S || K == 0, RP_ERR_INVALID_ARG, "null row scales");
  return gram_impl(X, V, S, K, n_v, basis, xform, G, (cudaStream_t)sv);
}

static rp_status solve_impl(const double *dG, int32_t n_v, int nc, int beta0, double *coef_out,
                            rp_fit_info *info, cudaStream_t s) {
  Tmp tc;
  RP_CUDA(tc.alloc((size_t)n_v * (nc + 5) * 8, s));
  double *dc = (double *)tc.p, *di = dc + (size_t)n_v * nc;
  RP_CUDA(launch_solve(dG, n_v, nc, beta0, dc, di, s));
  std::vector<double> hinfo((size_t)n_v * 5);
  RP_CUDA(cudaMemcpyAsync(coef_out, dc, (size_t)n_v * nc * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaMemcpyAsync(hinfo.data(), di, (size_t)n_v * 5 * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  rp_status worst = RP_OK;
  for (int v = 0; v < n_v; ++v) {
    const int stv = (int)hinfo[v * 5];
    if (info) {
      info[v].status = stv;
      info[v].rank = (int32_t)hinfo[v * 5 + 1];
      info[v].resid2 = hinfo[v * 5 + 2];
      info[v].min_pivot = hinfo[v * 5 + 3];
      info[v].cond_est = hinfo[v * 5 + 4];
      info[v].iters = 1;
      info[v].reserved = 0;
    }
    if (stv != 0) worst = (rp_status)stv;
  }
  if (worst != RP_OK) set_error("normal equations are degenerate (non-SPD or pivot <= 1e-13)");
  return worst;
}

rp_status rp_solve_normal(const double *G, int32_t n_v, const rp_basis *basis, double *coef_out,
                          rp_fit_info *info, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(G && basis && coef_out, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "n_v = %d", n_v);
  rp_status st = check_basis(*basis, basis->n_vars, "solve", true);
  if (st != RP_OK) return st;
  const int nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc >= 2 && nc <= 161, RP_ERR_UNSUPPORTED, "solve: n_c = %d outside [2, 161]", nc);
  if ((st = ensure_device()) != RP_OK) return st;
  Tmp tG;
  const double *dG;
  if ((st = stage_in(G, (size_t)n_v * nc * nc, tG, &dG, s)) != RP_OK) return st;
  return solve_impl(dG, n_v, nc, basis->n_num, coef_out, info, s);
}

rp_status rp_fit(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                 double *coef_out, rp_xform *xform_out, rp_fit_info *info, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(X && V && basis && coef_out, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 1 && n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "K = %lld, n_v = %d", (long long)K, n_v);
  rp_status st = check_basis(*basis, basis->n_vars, "fit", true);
  if (st != RP_OK) return st;
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc <= 161, RP_ERR_UNSUPPORTED, "fit: n_c = %d > 161", nc);
  if ((st = ensure_device()) != RP_OK) return st;
  Tmp tX, tV, tw, tG, tb, tp;
  const double *dX, *dV;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_in(V, (size_t)K * n_v, tV, &dV, s)) != RP_OK) return st;
  // a10 on the device: min / max, then the transform
  const int nblk = minmax_blocks(K);
  RP_CUDA(tw.alloc(((size_t)nblk * n * 2 + 4 * RP_MAX_VARS) * sizeof(double), s));
  double *part = (double *)tw.p, *lohi = part + (size_t)nblk * n * 2, *xf = lohi + 2 * RP_MAX_VARS;
  RP_CUDA(launch_minmax(dX, K, n, part, nblk, lohi, s));
  RP_CUDA(launch_xform(lohi, n, xf, s));
  // the Gram reads the transform from the device copy of the basis: no host round trip
  GramBasis gb;
  if ((st = build_gram_basis(basis, nullptr, &gb)) != RP_OK) return st;
  RP_CUDA(tG.alloc((size_t)n_v * nc * nc * 8, s));
  RP_CUDA(tb.alloc(sizeof(GramBasis), s));
  RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
  RP_CUDA(launch_xform_to_basis(xf, n, (GramBasis *)tb.p, s));
  const size_t pe = gram_partial_elems(gb, n_v, K, num_sms(), false);
  RP_CUDA(tp.alloc(pe * 8, s));
  RP_CUDA(launch_gram((const GramBasis *)tb.p, gb, dX, dV, nullptr, K, n_v, (double *)tG.p, (double *)tp.p, pe, s));
  rp_status sst = solve_impl((const double *)tG.p, n_v, nc, basis->n_num, coef_out, info, s);  // synchronises
  double hxf[2 * RP_MAX_VARS];
  RP_CUDA(cudaMemcpyAsync(hxf, xf, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  if (xform_out) {
    memset(xform_out, 0, sizeof *xform_out);
    for (int k = 0; k < n; ++k) {
      xform_out->c[k] = hxf[2 * k];
      xform_out->e[k] = (int32_t)hxf[2 * k + 1];
    }
  }
  return sst;
}

// ---- stream-ordered (device-resident) forms ---------------------------------------------------
static rp_status require_dev(const void *p, const char *what) {
  RP_REQUIRE(p && is_device_ptr(p), RP_ERR_INVALID_ARG, "%s must be a device pointer", what);
  return RP_OK;
}

rp_status rp_minmax_dev(const double *X, int64_t K, int32_t n, double *lohi, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(K >= 1 && n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "K = %lld, n = %d", (long long)K, n);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  if ((st = require_dev(X, "X")) != RP_OK || (st = require_dev(lohi, "lohi")) != RP_OK) return st;
  const int nblk = minmax_blocks(K);
  Tmp tw;
  RP_CUDA(tw.alloc((size_t)nblk * n * 2 * sizeof(double), s));
  RP_CUDA(launch_minmax(X, K, n, (double *)tw.p, nblk, lohi, s));
  return RP_OK;
}

rp_status rp_xform_dev(const double *lohi, int32_t n, double *xf, rp_stream sv) {
  RP_REQUIRE(n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "n = %d", n);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  if ((st = require_dev(lohi, "lohi")) != RP_OK || (st = require_dev(xf, "xf")) != RP_OK) return st;
  RP_CUDA(launch_xform(lohi, n, xf, (cudaStream_t)sv));
  return RP_OK;
}

rp_status rp_gram_sum_ordered(const double *parts, int32_t n_parts, int64_t elems, double *out, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(n_parts >= 1 && elems >= 0, RP_ERR_INVALID_ARG, "n_parts %d, elems %lld", n_parts, (long long)elems);
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  if (elems == 0) return RP_OK;
  if ((st = require_dev(parts, "parts")) != RP_OK || (st = require_dev(out, "out")) != RP_OK) return st;
  RP_CUDA(launch_sum_ordered(parts, n_parts, elems, out, s));
  return RP_OK;
}

rp_status rp_gram_accumulate_dev(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                                 const double *xf, double *G, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(basis && K >= 0 && n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "bad argument");
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  if ((st = require_dev(xf, "xf")) != RP_OK || (st = require_dev(G, "G")) != RP_OK) return st;
  if (K > 0 && ((st = require_dev(X, "X")) != RP_OK || (st = require_dev(V, "V")) != RP_OK)) return st;
  GramBasis gb;
  if ((st = build_gram_basis(basis, nullptr, &gb)) != RP_OK) return st;
  const int nc = gb.nc, n = gb.n;
  if (K == 0) {
    RP_CUDA(cudaMemsetAsync(G, 0, (size_t)n_v * nc * nc * 8, s));
    return RP_OK;
  }
  Tmp tb, tp;
  RP_CUDA(tb.alloc(sizeof(GramBasis), s));
  RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
  RP_CUDA(launch_xform_to_basis(xf, n, (GramBasis *)tb.p, s));
  const size_t pe = gram_partial_elems(gb, n_v, K, num_sms(), false);
  RP_CUDA(tp.alloc(pe * 8, s));
  RP_CUDA(launch_gram((const GramBasis *)tb.p, gb, X, V, nullptr, K, n_v, G, (double *)tp.p, pe, s));
  return RP_OK;
}

rp_status rp_solve_normal_dev(const double *G, int32_t n_v, const rp_basis *basis, double *coef, double *info,
                              rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(basis && n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "bad argument");
  rp_status st = check_basis(*basis, basis->n_vars, "solve", true);
  if (st != RP_OK) return st;
  const int nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc >= 2 && nc <= 161, RP_ERR_UNSUPPORTED, "solve: n_c = %d outside [2, 161]", nc);
  if ((st = ensure_device()) != RP_OK) return st;
  if ((st = require_dev(G, "G")) != RP_OK || (st = require_dev(coef, "coef")) != RP_OK) return st;
  if (info && (st = require_dev(info, "info")) != RP_OK) return st;
  Tmp ti;
  double *di = info;
  if (!di) {
    RP_CUDA(ti.alloc((size_t)n_v * 5 * 8, s));
    di = (double *)ti.p;
  }
  RP_CUDA(launch_solve(G, n_v, nc, basis->n_num, coef, di, s));
  return RP_OK;
}

rp_status rp_fit_dev(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis, double *coef,
                     double *xf_out, double *info, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(basis && K >= 1 && n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "bad argument");
  const int n = basis->n_vars;
  RP_REQUIRE(n >= 1 && n <= RP_MAX_VARS, RP_ERR_INVALID_ARG, "n_vars %d", n);
  const int nc = basis->n_num + basis->n_den;
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  Tmp tl, tx, tG;
  RP_CUDA(tl.alloc(2 * RP_MAX_VARS * sizeof(double), s));
  double *xf = xf_out;
  if (!xf) {
    RP_CUDA(tx.alloc(2 * RP_MAX_VARS * sizeof(double), s));
    xf = (double *)tx.p;
  } else if ((st = require_dev(xf, "xf_out")) != RP_OK) {
    return st;
  }
  if ((st = rp_minmax_dev(X, K, n, (double *)tl.p, sv)) != RP_OK) return st;
  if ((st = rp_xform_dev((const double *)tl.p, n, xf, sv)) != RP_OK) return st;
  RP_CUDA(tG.alloc((size_t)n_v * nc * nc * 8, s));
  if ((st = rp_gram_accumulate_dev(X, V, K, n_v, basis, xf, (double *)tG.p, sv)) != RP_OK) return st;
  return rp_solve_normal_dev((const double *)tG.p, n_v, basis, coef, info, sv);
}

rp_status rp_fit_sk(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                    int32_t iters, double *coef_out, rp_xform *xform_out, rp_fit_info *info, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(X && V && basis && coef_out, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 1 && n_v >= 1 && n_v <= 64 && iters >= 1 && iters <= 64, RP_ERR_INVALID_ARG,
             "K = %lld, n_v = %d, iters = %d", (long long)K, n_v, iters);
  rp_status st = check_basis(*basis, basis->n_vars, "fit", true);
  if (st != RP_OK) return st;
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc <= 161, RP_ERR_UNSUPPORTED, "fit: n_c = %d > 161", nc);
  if ((st = ensure_device()) != RP_OK) return st;
  Tmp tX, tV, tw, tG, tb, tp, tS, tc;
  const double *dX, *dV;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_in(V, (size_t)K * n_v, tV, &dV, s)) != RP_OK) return st;
  const int nblk = minmax_blocks(K);
  RP_CUDA(tw.alloc(((size_t)nblk * n * 2 + 4 * RP_MAX_VARS) * sizeof(double), s));
  double *part = (double *)tw.p, *lohi = part + (size_t)nblk * n * 2, *xf = lohi + 2 * RP_MAX_VARS;
  RP_CUDA(launch_minmax(dX, K, n, part, nblk, lohi, s));
  RP_CUDA(launch_xform(lohi, n, xf, s));
  GramBasis gb;
  if ((st = build_gram_basis(basis, nullptr, &gb)) != RP_OK) return st;
  RP_CUDA(tG.alloc((size_t)n_v * nc * nc * 8, s));
  RP_CUDA(tb.alloc(sizeof(GramBasis), s));
  RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
  RP_CUDA(launch_xform_to_basis(xf, n, (GramBasis *)tb.p, s));
  const size_t pe = std::max(gram_partial_elems(gb, n_v, K, num_sms(), false),
                             gram_partial_elems(gb, n_v, K, num_sms(), true));
  RP_CUDA(tp.alloc(pe * 8, s));
  RP_CUDA(tS.alloc((size_t)n_v * K * 8, s));
  RP_CUDA(tc.alloc((size_t)n_v * (nc + 5) * 8, s));
  double *dc = (double *)tc.p, *di = dc + (size_t)n_v * nc;
  for (int t = 0; t < iters; ++t) {
    if (t > 0) RP_CUDA(launch_den_weights((const GramBasis *)tb.p, dX, K, n_v, dc, (double *)tS.p, s));
    RP_CUDA(launch_gram((const GramBasis *)tb.p, gb, dX, dV, t > 0 ? (const double *)tS.p : nullptr, K, n_v,
                        (double *)tG.p, (double *)tp.p, pe, s));
    RP_CUDA(launch_solve((const double *)tG.p, n_v, nc, basis->n_num, dc, di, s));
  }
  std::vector<double> hinfo((size_t)n_v * 5);
  double hxf[2 * RP_MAX_VARS];
  RP_CUDA(cudaMemcpyAsync(coef_out, dc, (size_t)n_v * nc * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaMemcpyAsync(hinfo.data(), di, (size_t)n_v * 5 * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaMemcpyAsync(hxf, xf, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  if (xform_out) {
    memset(xform_out, 0, sizeof *xform_out);
    for (int k = 0; k < n; ++k) {
      xform_out->c[k] = hxf[2 * k];
      xform_out->e[k] = (int32_t)hxf[2 * k + 1];
    }
  }
  rp_status worst = RP_OK;
  for (int v = 0; v < n_v; ++v) {
    const int stv = (int)hinfo[v * 5];
    if (info) {
      info[v].status = stv;
      info[v].rank = (int32_t)hinfo[v * 5 + 1];
      info[v].resid2 = hinfo[v * 5 + 2];
      info[v].min_pivot = hinfo[v * 5 + 3];
      info[v].cond_est = hinfo[v * 5 + 4];
      info[v].iters = iters;
      info[v].reserved = 0;
    }
    if (stv != 0) worst = (rp_status)stv;
  }
  if (worst != RP_OK) set_error("weighted normal equations are degenerate");
  return worst;
}

// ---------------------------------------------------------------------------------------------
// f1: SVD of the homogeneous system
// ---------------------------------------------------------------------------------------------
static rp_status svd_finish(const double *dR, int32_t n_v, int nc, int n_num, double *coef_out,
                            double *sigma_out, rp_fit_info *info, cudaStream_t s) {
  Tmp to;
  RP_CUDA(to.alloc((size_t)n_v * (2 * nc + 6 + nc * nc) * 8, s));
  double *dc = (double *)to.p, *dsg = dc + (size_t)n_v * nc, *di = dsg + (size_t)n_v * nc;
  double *dV = di + (size_t)n_v * 6;
  RP_CUDA(launch_svd_jacobi(dR, nc, n_num, n_v, dV, dc, dsg, di, s));
  std::vector<double> hinfo((size_t)n_v * 6);
  RP_CUDA(cudaMemcpyAsync(coef_out, dc, (size_t)n_v * nc * 8, cudaMemcpyDeviceToHost, s));
  if (sigma_out) RP_CUDA(cudaMemcpyAsync(sigma_out, dsg, (size_t)n_v * nc * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaMemcpyAsync(hinfo.data(), di, (size_t)n_v * 6 * 8, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  rp_status worst = RP_OK;
  for (int v = 0; v < n_v; ++v) {
    const int stv = (int)hinfo[v * 6];
    if (info) {
      info[v].status = stv;
      info[v].rank = (int32_t)hinfo[v * 6 + 1];
      info[v].resid2 = hinfo[v * 6 + 2];
      info[v].min_pivot = hinfo[v * 6 + 3];
      info[v].cond_est = hinfo[v * 6 + 4];
      info[v].iters = (int32_t)hinfo[v * 6 + 5];
      info[v].reserved = 0;
    }
    if (stv != 0) worst = (rp_status)stv;
  }
  if (worst != RP_OK) set_error("SVD: beta_0 of the smallest right singular vector is zero");
  return worst;
}

static rp_status svd_checks(const rp_basis *basis, int32_t n_v) {
  RP_REQUIRE(basis, RP_ERR_INVALID_ARG, "null basis");
  RP_REQUIRE(n_v >= 1 && n_v <= 64, RP_ERR_INVALID_ARG, "n_v = %d", n_v);
  rp_status st = check_basis(*basis, basis->n_vars, "svd", true);
  if (st != RP_OK) return st;
  const int nc = basis->n_num + basis->n_den;
  RP_REQUIRE(nc >= 2 && nc <= 144, RP_ERR_UNSUPPORTED, "svd: n_c = %d outside [2, 144]", nc);
  return ensure_device();
}

rp_status rp_fit_svd(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                     double *coef_out, double *sigma_out, rp_xform *xform_out, rp_fit_info *info,
                     rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(X && V && coef_out, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 1, RP_ERR_INVALID_ARG, "K = %lld", (long long)K);
  rp_status st = svd_checks(basis, n_v);
  if (st != RP_OK) return st;
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  Tmp tX, tV, tw, tb, tws, tR;
  const double *dX, *dV;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_in(V, (size_t)K * n_v, tV, &dV, s)) != RP_OK) return st;
  const int nblk = minmax_blocks(K);
  RP_CUDA(tw.alloc(((size_t)nblk * n * 2 + 4 * RP_MAX_VARS) * sizeof(double), s));
  double *part = (double *)tw.p, *lohi = part + (size_t)nblk * n * 2, *xf = lohi + 2 * RP_MAX_VARS;
  RP_CUDA(launch_minmax(dX, K, n, part, nblk, lohi, s));
  RP_CUDA(launch_xform(lohi, n, xf, s));
  GramBasis gb;
  if ((st = build_gram_basis(basis, nullptr, &gb)) != RP_OK) return st;
  RP_CUDA(tb.alloc(sizeof(GramBasis), s));
  RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
  RP_CUDA(launch_xform_to_basis(xf, n, (GramBasis *)tb.p, s));
  RP_CUDA(tR.alloc((size_t)n_v * nc * nc * 8, s));
  if (gram_dd_supported(gb, n_v, K)) {  // R from the double-double Gram (rp_moments.cu)
    const size_t wsb = gram_dd_workspace_bytes(gb, n_v, K);
    RP_CUDA(tws.alloc(wsb, s));
    RP_CUDA(launch_gram_dd_chol((const GramBasis *)tb.p, gb, dX, dV, K, n_v, tws.p, wsb, (double *)tR.p, s));
  } else {  // Householder TSQR
    const size_t wsb = tsqr_workspace_bytes(nc, n_v, tsqr_leaves(K, n_v));
    RP_CUDA(tws.alloc(wsb, s));
    RP_CUDA(launch_tsqr((const GramBasis *)tb.p, dX, dV, nullptr, nullptr, K, n, nc, n_v, tws.p, wsb,
                        (double *)tR.p, s));
  }
  rp_status sst = svd_finish((const double *)tR.p, n_v, nc, basis->n_num, coef_out, sigma_out, info, s);
  if (sst == RP_ERR_CUDA) return sst;
  double hxf[2 * RP_MAX_VARS];
  RP_CUDA(cudaMemcpyAsync(hxf, xf, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  if (xform_out) {
    memset(xform_out, 0, sizeof *xform_out);
    for (int k = 0; k < n; ++k) {
      xform_out->c[k] = hxf[2 * k];
      xform_out->e[k] = (int32_t)hxf[2 * k + 1];
    }
  }
  return sst;
}

rp_status rp_tsqr_accumulate(const double *X, const double *V, int64_t K, int32_t n_v, const rp_basis *basis,
                             const rp_xform *xform, double *R, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(R && xform, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(K >= 0, RP_ERR_INVALID_ARG, "K = %lld", (long long)K);
  RP_REQUIRE(K == 0 || (X && V), RP_ERR_INVALID_ARG, "null X / V");
  rp_status st = svd_checks(basis, n_v);
  if (st != RP_OK) return st;
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  GramBasis gb;
  if ((st = build_gram_basis(basis, xform, &gb)) != RP_OK) return st;
  Tmp tX, tV, tR, tb, tws;
  const double *dX = nullptr, *dV = nullptr;
  double *dR;
  bool hR;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_in(V, (size_t)K * n_v, tV, &dV, s)) != RP_OK) return st;
  if ((st = stage_out(R, (size_t)n_v * nc * nc, tR, &dR, &hR, s)) != RP_OK) return st;
  if (K == 0) {
    RP_CUDA(cudaMemsetAsync(dR, 0, (size_t)n_v * nc * nc * 8, s));
  } else {
    RP_CUDA(tb.alloc(sizeof(GramBasis), s));
    RP_CUDA(cudaMemcpyAsync(tb.p, &gb, sizeof gb, cudaMemcpyHostToDevice, s));
    const size_t wsb = tsqr_workspace_bytes(nc, n_v, tsqr_leaves(K, n_v));
    RP_CUDA(tws.alloc(wsb, s));
    RP_CUDA(launch_tsqr((const GramBasis *)tb.p, dX, dV, nullptr, nullptr, K, n, nc, n_v, tws.p, wsb, dR, s));
  }
  if (hR) {
    RP_CUDA(cudaMemcpyAsync(R, dR, (size_t)n_v * nc * nc * 8, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
  return RP_OK;
}

rp_status rp_svd_rows(const double *rows, int64_t n_rows, int32_t n_v, const rp_basis *basis,
                      double *coef_out, double *sigma_out, rp_fit_info *info, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(rows && coef_out, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(n_rows >= 1, RP_ERR_INVALID_ARG, "n_rows = %lld", (long long)n_rows);
  rp_status st = svd_checks(basis, n_v);
  if (st != RP_OK) return st;
  const int n = basis->n_vars, nc = basis->n_num + basis->n_den;
  Tmp tr, tws, tR;
  const double *dr;
  if ((st = stage_in(rows, (size_t)n_v * n_rows * nc, tr, &dr, s)) != RP_OK) return st;
  const size_t wsb = tsqr_workspace_bytes(nc, n_v, tsqr_leaves(n_rows, n_v));
  RP_CUDA(tws.alloc(wsb, s));
  RP_CUDA(tR.alloc((size_t)n_v * nc * nc * 8, s));
  RP_CUDA(launch_tsqr(nullptr, nullptr, nullptr, nullptr, dr, n_rows, n, nc, n_v, tws.p, wsb, (double *)tR.p, s));
  return svd_finish((const double *)tR.p, n_v, nc, basis->n_num, coef_out, sigma_out, info, s);
}

rp_status rp_eval_metrics(const rp_program *prog, const double *X, int64_t K, double *out, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(prog && out && (X || K == 0) && K >= 0, RP_ERR_INVALID_ARG, "bad argument");
  rp_status st = ensure_device();
  if (st != RP_OK) return st;
  DevProg hp;
  if ((st = compile_program(prog, &hp)) != RP_OK) return st;
  if (K == 0) return RP_OK;
  const int n = prog->d + prog->p;
  Tmp tX, to, tp;
  const double *dX;
  double *dout;
  bool ho;
  if ((st = stage_in(X, (size_t)K * n, tX, &dX, s)) != RP_OK) return st;
  if ((st = stage_out(out, (size_t)K * prog->n_metrics, to, &dout, &ho, s)) != RP_OK) return st;
  RP_CUDA(tp.alloc(sizeof(DevProg), s));
  RP_CUDA(cudaMemcpyAsync(tp.p, &hp, sizeof hp, cudaMemcpyHostToDevice, s));
  RP_CUDA(launch_eval_metrics((const DevProg *)tp.p, prog->n_metrics, dX, K, dout, s));
  if (ho) {
    RP_CUDA(cudaMemcpyAsync(out, dout, (size_t)K * prog->n_metrics * 8, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
  return RP_OK;
}

rp_status rp_plan_create(const rp_program *progs, int32_t n_prog, const int32_t *F, int32_t nF,
                         rp_plan *out, rp_stream sv) {
  rp_status st = plan_create(progs, n_prog, F, nF, out, (cudaStream_t)sv, false);
  if (st == RP_OK) {
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)sv);
    if (e != cudaSuccess) {
      plan_free(*out);
      *out = nullptr;
      return cuda_fail(e, "plan create", __FILE__, __LINE__);
    }
  }
  return st;
}

rp_status rp_plan_eval_argmin(rp_plan plan, const int32_t *D, int64_t nD, int32_t *best_idx,
                              double *best_E, double *second_E, rp_stream sv) {
  return plan_eval(plan, D, nD, best_idx, best_E, second_E, (cudaStream_t)sv);
}

rp_status rp_plan_update_program(rp_plan plan, int32_t prog, const double *coef, int32_t stride,
                                 const double *xform, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(plan && coef && prog >= 0 && prog < plan->n_prog, RP_ERR_INVALID_ARG, "bad argument");
  RP_REQUIRE(stride >= plan->nc_of[prog], RP_ERR_INVALID_ARG, "stride %d < n_c %d", stride, plan->nc_of[prog]);
  RP_REQUIRE(is_device_ptr(coef) && (!xform || is_device_ptr(xform)), RP_ERR_INVALID_ARG,
             "coef / xform must be device pointers (stream-ordered update)");
  plan->stream = s;
  RP_CUDA(launch_plan_refresh(plan->d_progs + prog, prog, coef, stride, xform, plan->npe_pad, plan->tab, s));
  if (plan->hist.enabled) {  // decisions of the old program are stale
    RP_CUDA(cudaMemsetAsync(plan->hist.slots, 0, ((size_t)plan->hist.mask + 1) * sizeof(HistSlot), s));
    RP_CUDA(cudaMemsetAsync(plan->hist.counters, 0, 3 * sizeof(unsigned long long), s));
  }
  return RP_OK;
}

rp_status rp_plan_static_feasible(rp_plan plan, int32_t prog, int32_t *n_static_feasible) {
  RP_REQUIRE(plan && n_static_feasible && prog >= 0 && prog < plan->n_prog, RP_ERR_INVALID_ARG, "bad argument");
  int32_t v = 0;
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  RP_CUDA(cudaMemcpy(&v, plan->tab.nFc + 2 * prog, 4, cudaMemcpyDeviceToHost));
  *n_static_feasible = v;
  return RP_OK;
}

rp_status rp_plan_decide(rp_plan plan, int32_t prog, const int32_t *D, int64_t n, double margin,
                         rp_decision *out, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(plan, RP_ERR_INVALID_ARG, "null plan");
  RP_REQUIRE(prog >= 0 && prog < plan->n_prog, RP_ERR_INVALID_ARG, "prog %d out of range", prog);
  RP_REQUIRE(n >= 0 && margin >= 0.0, RP_ERR_INVALID_ARG, "n < 0 or margin < 0 / NaN");
  RP_REQUIRE(plan->nF <= kDecideMaxF, RP_ERR_UNSUPPORTED, "decide: nF = %d > %d", plan->nF, kDecideMaxF);
  if (plan->hist.enabled)
    RP_REQUIRE(plan->hist.prog == prog && plan->hist.margin == margin, RP_ERR_INVALID_ARG,
               "the runtime history was enabled for program %d, margin %g", plan->hist.prog, plan->hist.margin);
  if (n == 0) return RP_OK;
  RP_REQUIRE(D && out, RP_ERR_INVALID_ARG, "null D / out");
  plan->stream = s;
  Tmp tD, to;
  const int32_t *dD;
  rp_decision *dout;
  bool ho;
  rp_status st = stage_in(D, (size_t)n * plan->d, tD, &dD, s);
  if (st != RP_OK) return st;
  if ((st = stage_out(out, (size_t)n, to, &dout, &ho, s)) != RP_OK) return st;
  DecideArgs a{plan->d_progs, plan->tab, plan->npe_pad, prog, dD, n, margin, dout, plan->hist};
  RP_CUDA(launch_decide(a, plan->mwp, s));
  if (ho) {
    RP_CUDA(cudaMemcpyAsync(out, dout, (size_t)n * sizeof(rp_decision), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
  return RP_OK;
}

// ---- single-launch decider: mapped pinned buffers + a captured graph of the decide kernel ------
struct rp_decider_s {
  rp_plan plan = nullptr;
  int32_t *hD = nullptr, *dD = nullptr;            // d ints, host-mapped
  rp_decision *hout = nullptr, *dout = nullptr;    // one decision, host-mapped
  cudaStream_t s = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int d = 0;
};

static void decider_free(rp_decider dc) {
  if (!dc) return;
  if (dc->s) cudaStreamSynchronize(dc->s);
  if (dc->exec) cudaGraphExecDestroy(dc->exec);
  if (dc->graph) cudaGraphDestroy(dc->graph);
  if (dc->s) cudaStreamDestroy(dc->s);
  if (dc->hD) cudaFreeHost(dc->hD);
  if (dc->hout) cudaFreeHost(dc->hout);
  delete dc;
}

rp_status rp_decider_create(rp_plan plan, int32_t prog, double margin, rp_decider *out) {
  RP_REQUIRE(out, RP_ERR_INVALID_ARG, "null decider out");
  *out = nullptr;
  RP_REQUIRE(plan, RP_ERR_INVALID_ARG, "null plan");
  RP_REQUIRE(prog >= 0 && prog < plan->n_prog, RP_ERR_INVALID_ARG, "prog %d out of range", prog);
  RP_REQUIRE(margin >= 0.0, RP_ERR_INVALID_ARG, "margin < 0 / NaN");
  RP_REQUIRE(plan->nF <= kDecideMaxF, RP_ERR_UNSUPPORTED, "decide: nF = %d > %d", plan->nF, kDecideMaxF);
  if (plan->hist.enabled)
    RP_REQUIRE(plan->hist.prog == prog && plan->hist.margin == margin, RP_ERR_INVALID_ARG,
               "the runtime history was enabled for program %d, margin %g", plan->hist.prog, plan->hist.margin);
  rp_decider dc = new rp_decider_s;
  dc->plan = plan;
  dc->d = plan->d;
  auto fail = [&](cudaError_t e, const char *w) {
    rp_status r = cuda_fail(e, w, __FILE__, __LINE__);
    decider_free(dc);
    return r;
  };
  cudaError_t e;
  if ((e = cudaStreamSynchronize(plan->stream)) != cudaSuccess) return fail(e, "plan stream");
  if ((e = cudaHostAlloc((void **)&dc->hD, sizeof(int32_t) * kMaxVars, cudaHostAllocMapped)) != cudaSuccess)
    return fail(e, "mapped D");
  if ((e = cudaHostAlloc((void **)&dc->hout, sizeof(rp_decision), cudaHostAllocMapped)) != cudaSuccess)
    return fail(e, "mapped out");
  if ((e = cudaHostGetDevicePointer((void **)&dc->dD, dc->hD, 0)) != cudaSuccess) return fail(e, "map D");
  if ((e = cudaHostGetDevicePointer((void **)&dc->dout, dc->hout, 0)) != cudaSuccess) return fail(e, "map out");
  for (int k = 0; k < kMaxVars; ++k) dc->hD[k] = 1;
  if ((e = cudaStreamCreateWithFlags(&dc->s, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
  DecideArgs a{plan->d_progs, plan->tab, plan->npe_pad, prog, dc->dD, 1, margin, dc->dout, plan->hist};
  // warm-up outside the capture (kernel attributes, module load); a history insert of D = 1...
  // would be a real decision, so the history is cleared afterwards when it is on
  if ((e = launch_decide(a, plan->mwp, dc->s)) != cudaSuccess) return fail(e, "warm-up");
  if ((e = cudaStreamSynchronize(dc->s)) != cudaSuccess) return fail(e, "warm-up sync");
  if (plan->hist.enabled) {
    if ((e = cudaMemsetAsync(plan->hist.slots, 0, ((size_t)plan->hist.mask + 1) * sizeof(HistSlot), dc->s)) != cudaSuccess)
      return fail(e, "history clear");
    if ((e = cudaMemsetAsync(plan->hist.counters, 0, 3 * sizeof(unsigned long long), dc->s)) != cudaSuccess)
      return fail(e, "history clear");
    if ((e = cudaStreamSynchronize(dc->s)) != cudaSuccess) return fail(e, "history clear");
  }
  if ((e = cudaStreamBeginCapture(dc->s, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return fail(e, "capture");
  e = launch_decide(a, plan->mwp, dc->s);
  cudaError_t e2 = cudaStreamEndCapture(dc->s, &dc->graph);
  if (e != cudaSuccess) return fail(e, "capture launch");
  if (e2 != cudaSuccess) return fail(e2, "end capture");
  if ((e = cudaGraphInstantiate(&dc->exec, dc->graph, 0)) != cudaSuccess) return fail(e, "instantiate");
  ++plan->n_deciders;
  *out = dc;
  return RP_OK;
}

rp_status rp_decider_decide(rp_decider dc, const int32_t *D, rp_decision *out) {
  RP_REQUIRE(dc && D && out, RP_ERR_INVALID_ARG, "null argument");
  for (int k = 0; k < dc->d; ++k) dc->hD[k] = D[k];
  RP_CUDA(cudaGraphLaunch(dc->exec, dc->s));
  RP_CUDA(cudaStreamSynchronize(dc->s));
  *out = *dc->hout;
  return RP_OK;
}

rp_status rp_decider_destroy(rp_decider dc) {
  if (dc && dc->exec && dc->plan) --dc->plan->n_deciders;
  decider_free(dc);
  return RP_OK;
}

rp_status rp_plan_history_enable(rp_plan plan, int32_t prog, int32_t log2_capacity, double margin) {
  RP_REQUIRE(plan, RP_ERR_INVALID_ARG, "null plan");
  RP_REQUIRE(prog >= 0 && prog < plan->n_prog, RP_ERR_INVALID_ARG, "prog %d out of range", prog);
  RP_REQUIRE(log2_capacity >= 4 && log2_capacity <= 24 && margin >= 0.0, RP_ERR_INVALID_ARG,
             "log2_capacity in [4, 24], margin >= 0");
  const size_t cap = (size_t)1 << log2_capacity;
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  if (plan->hist.slots && (size_t)plan->hist.mask + 1 == cap) {
    // same capacity: clear in place, so the table a live decider's graph captured stays valid
    RP_REQUIRE(plan->n_deciders == 0 || (plan->hist.prog == prog && plan->hist.margin == margin),
               RP_ERR_INVALID_ARG, "%d decider(s) use the history of program %d, margin %g",
               plan->n_deciders, plan->hist.prog, plan->hist.margin);
    RP_CUDA(cudaMemset(plan->hist.slots, 0, cap * sizeof(HistSlot)));
    RP_CUDA(cudaMemset(plan->hist.counters, 0, 3 * sizeof(unsigned long long)));
    plan->hist.prog = prog;
    plan->hist.margin = margin;
    return RP_OK;
  }
  // a new allocation would leave a live decider's captured graph with a freed table
  RP_REQUIRE(plan->n_deciders == 0, RP_ERR_INVALID_ARG,
             "cannot resize the runtime history while %d decider(s) use it", plan->n_deciders);
  if (plan->hist.slots) {
    cudaFree(plan->hist.slots);
    cudaFree(plan->hist.counters);
    plan->hist = HistTable();
  }
  RP_CUDA(cudaMalloc((void **)&plan->hist.slots, cap * sizeof(HistSlot)));
  RP_CUDA(cudaMalloc((void **)&plan->hist.counters, 3 * sizeof(unsigned long long)));
  RP_CUDA(cudaMemset(plan->hist.slots, 0, cap * sizeof(HistSlot)));
  RP_CUDA(cudaMemset(plan->hist.counters, 0, 3 * sizeof(unsigned long long)));
  plan->hist.mask = (uint32_t)(cap - 1);
  plan->hist.enabled = 1;
  plan->hist.prog = prog;
  plan->hist.margin = margin;
  return RP_OK;
}

rp_status rp_plan_history_stats(rp_plan plan, int64_t *hits, int64_t *misses, int64_t *entries) {
  RP_REQUIRE(plan && hits && misses && entries, RP_ERR_INVALID_ARG, "null argument");
  *hits = *misses = *entries = 0;
  if (!plan->hist.enabled) return RP_OK;
  unsigned long long c[3];
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  RP_CUDA(cudaMemcpy(c, plan->hist.counters, sizeof c, cudaMemcpyDeviceToHost));
  *hits = (int64_t)c[0];
  *misses = (int64_t)c[1];
  *entries = (int64_t)c[2];
  return RP_OK;
}

rp_status rp_plan_history_clear(rp_plan plan, rp_stream sv) {
  RP_REQUIRE(plan, RP_ERR_INVALID_ARG, "null plan");
  if (!plan->hist.enabled) return RP_OK;
  cudaStream_t s = (cudaStream_t)sv;
  RP_CUDA(cudaMemsetAsync(plan->hist.slots, 0, ((size_t)plan->hist.mask + 1) * sizeof(HistSlot), s));
  RP_CUDA(cudaMemsetAsync(plan->hist.counters, 0, 3 * sizeof(unsigned long long), s));
  return RP_OK;
}

rp_status rp_plan_enable_timing(rp_plan plan, int32_t on) {
  RP_REQUIRE(plan, RP_ERR_INVALID_ARG, "null plan");
  if (on && !plan->ev[0])
    for (cudaEvent_t &e : plan->ev) RP_CUDA(cudaEventCreate(&e));
  plan->timing = on != 0;
  return RP_OK;
}

rp_status rp_plan_last_timing(rp_plan plan, float *ms) {
  RP_REQUIRE(plan && ms, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(plan->timing, RP_ERR_INVALID_ARG, "timing not enabled (rp_plan_enable_timing)");
  RP_CUDA(cudaEventSynchronize(plan->ev[3]));
  RP_CUDA(cudaEventElapsedTime(&ms[0], plan->ev[0], plan->ev[1]));
  RP_CUDA(cudaEventElapsedTime(&ms[1], plan->ev[1], plan->ev[2]));
  RP_CUDA(cudaEventElapsedTime(&ms[2], plan->ev[2], plan->ev[3]));
  return RP_OK;
}

rp_status rp_plan_destroy(rp_plan plan) {
  plan_free(plan);
  return RP_OK;
}

rp_status rp_eval_argmin_batched(const rp_program *progs, int32_t n_prog, const int32_t *D, int64_t nD,
                                 const int32_t *F, int32_t nF, int32_t *best_idx, double *best_E,
                                 double *second_E, rp_stream sv) {
  cudaStream_t s = (cudaStream_t)sv;
  RP_REQUIRE(nD >= 0, RP_ERR_INVALID_ARG, "nD < 0");
  rp_plan pl = nullptr;
  rp_status st = plan_create(progs, n_prog, F, nF, &pl, s, true);
  if (st != RP_OK) return st;
  st = plan_eval(pl, D, nD, best_idx, best_E, second_E, s);
  plan_free(pl);  // stream-ordered frees
  return st;
}

rp_status rp_eval_argmin(const rp_program *prog, const int32_t *D, int64_t nD, const int32_t *F,
                         int32_t nF, int32_t *best_idx, double *best_E, double *second_E, rp_stream s) {
  return rp_eval_argmin_batched(prog, 1, D, nD, F, nF, best_idx, best_E, second_E, s);
}

}  // extern "C"

// =============================================================================================
// persistence: the rational program and the runtime history (byte layout only; no arithmetic)
// =============================================================================================
namespace {
struct Writer {
  std::vector<unsigned char> b;
  template <class T>
  void put(const T &v) {
    const unsigned char *p = reinterpret_cast<const unsigned char *>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void put_bytes(const void *p, size_t n) {
    const unsigned char *c = reinterpret_cast<const unsigned char *>(p);
    b.insert(b.end(), c, c + n);
  }
};
struct Reader {
  const unsigned char *p;
  size_t n, off = 0;
  bool ok = true;
  template <class T>
  T get() {
    T v{};
    if (off + sizeof(T) > n) {
      ok = false;
      return v;
    }
    memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
  bool get_bytes(void *dst, size_t k) {
    if (off + k > n) return ok = false;
    memcpy(dst, p + off, k);
    off += k;
    return true;
  }
};
uint64_t fnv64(const unsigned char *b, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}
const char kProgMagic[8] = {'R', 'P', 'P', 'R', 'O', 'G', '0', '1'};
const char kHistMagic[8] = {'R', 'P', 'H', 'I', 'S', 'T', '0', '1'};
// hand the bytes out: buf null -> size only; too small -> INVALID_ARG (size still written)
rp_status emit(const Writer &w, void *buf, int64_t cap, int64_t *size) {
  *size = (int64_t)w.b.size();
  if (!buf) return RP_OK;
  RP_REQUIRE(cap >= (int64_t)w.b.size(), RP_ERR_INVALID_ARG, "buffer of %lld bytes < %lld", (long long)cap,
             (long long)w.b.size());
  memcpy(buf, w.b.data(), w.b.size());
  return RP_OK;
}
}  // namespace

struct rp_program_blob_s {
  rp_program prog{};
  std::vector<int16_t> exps[RP_MAX_METRICS][2];
  std::vector<double> coef[RP_MAX_METRICS];
};

extern "C" {

rp_status rp_program_save(const rp_program *prog, void *buf, int64_t cap, int64_t *size) {
  RP_REQUIRE(prog && size, RP_ERR_INVALID_ARG, "null argument");
  DevProg scratch;  // validates the program exactly as rp_plan_create would
  rp_status st = compile_program(prog, &scratch);
  if (st != RP_OK) return st;
  Writer w;
  w.put_bytes(kProgMagic, 8);
  w.put(prog->d);
  w.put(prog->p);
  w.put(prog->n_metrics);
  w.put(prog->e_template);
  w.put(prog->regs_per_thread);
  for (int k = 0; k < 3; ++k) w.put(prog->grid_map[k]);
  w.put(prog->smem_words_base);
  w.put(prog->smem_words_per_thread);
  w.put(prog->hw);
  w.put(prog->xform);
  for (int i = 0; i < prog->n_metrics; ++i) {
    const rp_basis &b = prog->basis[i];
    w.put(b.n_vars);
    w.put(b.n_num);
    w.put(b.n_den);
    w.put_bytes(b.num_exp, sizeof(int16_t) * b.n_num * b.n_vars);
    w.put_bytes(b.den_exp, sizeof(int16_t) * b.n_den * b.n_vars);
    w.put_bytes(prog->coef[i], sizeof(double) * (b.n_num + b.n_den));  // IEEE bits: exact
  }
  w.put(fnv64(w.b.data(), w.b.size()));
  return emit(w, buf, cap, size);
}

rp_status rp_program_load(const void *buf, int64_t size, rp_program_blob *out) {
  RP_REQUIRE(buf && out && size >= 16, RP_ERR_INVALID_ARG, "null argument or short buffer");
  *out = nullptr;
  const unsigned char *b = reinterpret_cast<const unsigned char *>(buf);
  uint64_t want;
  memcpy(&want, b + size - 8, 8);
  RP_REQUIRE(memcmp(b, kProgMagic, 8) == 0, RP_ERR_INVALID_ARG, "not a saved rp_program (magic)");
  RP_REQUIRE(fnv64(b, (size_t)size - 8) == want, RP_ERR_INVALID_ARG, "saved rp_program: checksum mismatch");
  Reader r{b + 8, (size_t)size - 16};
  rp_program_blob o = new rp_program_blob_s;
  rp_program &p = o->prog;
  p.d = r.get<int32_t>();
  p.p = r.get<int32_t>();
  p.n_metrics = r.get<int32_t>();
  p.e_template = r.get<int32_t>();
  p.regs_per_thread = r.get<int32_t>();
  for (int k = 0; k < 3; ++k) p.grid_map[k] = r.get<int32_t>();
  p.smem_words_base = r.get<int64_t>();
  p.smem_words_per_thread = r.get<int64_t>();
  p.hw = r.get<rp_hw>();
  p.xform = r.get<rp_xform>();
  bool ok = r.ok && p.n_metrics >= 1 && p.n_metrics <= RP_MAX_METRICS;
  for (int i = 0; ok && i < p.n_metrics; ++i) {
    rp_basis &bs = p.basis[i];
    bs.n_vars = r.get<int32_t>();
    bs.n_num = r.get<int32_t>();
    bs.n_den = r.get<int32_t>();
    ok = r.ok && bs.n_vars >= 1 && bs.n_vars <= RP_MAX_VARS && bs.n_num >= 0 && bs.n_den >= 1 &&
         bs.n_num + bs.n_den < kMaxSrc;
    if (!ok) break;
    o->exps[i][0].resize((size_t)bs.n_num * bs.n_vars);
    o->exps[i][1].resize((size_t)bs.n_den * bs.n_vars);
    o->coef[i].resize((size_t)bs.n_num + bs.n_den);
    ok = r.get_bytes(o->exps[i][0].data(), o->exps[i][0].size() * 2) &&
         r.get_bytes(o->exps[i][1].data(), o->exps[i][1].size() * 2) &&
         r.get_bytes(o->coef[i].data(), o->coef[i].size() * 8);
    bs.num_exp = o->exps[i][0].data();
    bs.den_exp = o->exps[i][1].data();
    p.coef[i] = o->coef[i].data();
  }
  ok = ok && r.off == r.n;
  if (!ok) {
    delete o;
    RP_REQUIRE(false, RP_ERR_INVALID_ARG, "saved rp_program: truncated or malformed");
  }
  DevProg scratch;
  const rp_status st = compile_program(&p, &scratch);
  if (st != RP_OK) {
    delete o;
    return st;
  }
  *out = o;
  return RP_OK;
}

const rp_program *rp_program_blob_program(rp_program_blob blob) { return blob ? &blob->prog : nullptr; }

rp_status rp_program_blob_free(rp_program_blob blob) {
  delete blob;
  return RP_OK;
}

// fingerprint of program `prog` of a plan as the device holds it now, and of the plan's F
static rp_status plan_fingerprint(rp_plan plan, int32_t prog, uint64_t *fp) {
  Tmp t;
  RP_CUDA(t.alloc(sizeof(unsigned long long), plan->stream));
  RP_CUDA(launch_fingerprint(plan->d_progs + prog, plan->d_F, (size_t)plan->nF * plan->p * sizeof(int32_t),
                             (unsigned long long *)t.p, plan->stream));
  RP_CUDA(cudaMemcpy(fp, t.p, 8, cudaMemcpyDeviceToHost));
  return RP_OK;
}

rp_status rp_plan_history_save(rp_plan plan, void *buf, int64_t cap, int64_t *size) {
  RP_REQUIRE(plan && size, RP_ERR_INVALID_ARG, "null argument");
  RP_REQUIRE(plan->hist.enabled, RP_ERR_INVALID_ARG, "the plan's runtime history is not enabled");
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  const int d = plan->d;
  const int64_t cap_slots = (int64_t)plan->hist.mask + 1;
  uint64_t fp = 0;
  rp_status st = plan_fingerprint(plan, plan->hist.prog, &fp);
  if (st != RP_OK) return st;
  Tmp t;
  const size_t kb = (size_t)cap_slots * d * 4, vb = (size_t)cap_slots * sizeof(rp_decision), sb = (size_t)cap_slots * 4;
  RP_CUDA(t.alloc(kb + vb + sb + 16, plan->stream));
  unsigned char *base = (unsigned char *)t.p;
  rp_decision *dv = (rp_decision *)base;  // 48-byte records first (alignment)
  int32_t *dk = (int32_t *)(base + vb);
  int32_t *ds = (int32_t *)(base + vb + kb);
  unsigned *dc = (unsigned *)(base + vb + kb + sb);
  RP_CUDA(launch_hist_export(plan->hist, d, dk, dv, ds, dc, plan->stream));
  unsigned n = 0;
  RP_CUDA(cudaMemcpyAsync(&n, dc, 4, cudaMemcpyDeviceToHost, plan->stream));
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  std::vector<int32_t> hk((size_t)n * d), hs(n);
  std::vector<rp_decision> hv(n);
  if (n) {
    RP_CUDA(cudaMemcpy(hk.data(), dk, (size_t)n * d * 4, cudaMemcpyDeviceToHost));
    RP_CUDA(cudaMemcpy(hv.data(), dv, (size_t)n * sizeof(rp_decision), cudaMemcpyDeviceToHost));
    RP_CUDA(cudaMemcpy(hs.data(), ds, (size_t)n * 4, cudaMemcpyDeviceToHost));
  }
  std::vector<unsigned> order(n);
  for (unsigned i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](unsigned a, unsigned b) { return hs[a] < hs[b]; });  // slot order
  Writer w;
  w.put_bytes(kHistMagic, 8);
  w.put((int32_t)d);
  w.put((int32_t)plan->hist.prog);
  w.put(plan->hist.margin);
  w.put(fp);
  w.put((int64_t)n);
  for (unsigned i : order) {
    w.put_bytes(hk.data() + (size_t)i * d, (size_t)d * 4);
    hv[i].from_history = 0;
    w.put(hv[i]);
  }
  w.put(fnv64(w.b.data(), w.b.size()));
  return emit(w, buf, cap, size);
}

rp_status rp_plan_history_load(rp_plan plan, const void *buf, int64_t size) {
  RP_REQUIRE(plan && buf && size >= 16, RP_ERR_INVALID_ARG, "null argument or short buffer");
  RP_REQUIRE(plan->hist.enabled, RP_ERR_INVALID_ARG, "enable the plan's runtime history before loading one");
  const unsigned char *b = reinterpret_cast<const unsigned char *>(buf);
  uint64_t want;
  memcpy(&want, b + size - 8, 8);
  RP_REQUIRE(memcmp(b, kHistMagic, 8) == 0, RP_ERR_INVALID_ARG, "not a saved runtime history (magic)");
  RP_REQUIRE(fnv64(b, (size_t)size - 8) == want, RP_ERR_INVALID_ARG, "saved runtime history: checksum mismatch");
  Reader r{b + 8, (size_t)size - 16};
  const int32_t d = r.get<int32_t>(), prog = r.get<int32_t>();
  const double margin = r.get<double>();
  const uint64_t fp = r.get<uint64_t>();
  const int64_t n = r.get<int64_t>();
  RP_REQUIRE(r.ok && d == plan->d && n >= 0 && r.n - r.off == (size_t)n * ((size_t)d * 4 + sizeof(rp_decision)),
             RP_ERR_INVALID_ARG, "saved runtime history: malformed or of another data arity");
  RP_REQUIRE(prog == plan->hist.prog && margin == plan->hist.margin, RP_ERR_INVALID_ARG,
             "saved runtime history of program %d, margin %g; the plan's is program %d, margin %g", prog, margin,
             plan->hist.prog, plan->hist.margin);
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  uint64_t mine = 0;
  rp_status st = plan_fingerprint(plan, prog, &mine);
  if (st != RP_OK) return st;
  RP_REQUIRE(mine == fp, RP_ERR_INVALID_ARG,
             "saved runtime history belongs to another program or configuration set (fingerprint)");
  if (n == 0) return RP_OK;
  std::vector<int32_t> hk((size_t)n * d);
  std::vector<rp_decision> hv(n);
  for (int64_t i = 0; i < n; ++i) {
    r.get_bytes(hk.data() + (size_t)i * d, (size_t)d * 4);
    hv[i] = r.get<rp_decision>();
  }
  Tmp t;
  const size_t vb = (size_t)n * sizeof(rp_decision), kb = (size_t)n * d * 4;
  RP_CUDA(t.alloc(vb + kb, plan->stream));
  RP_CUDA(cudaStreamSynchronize(plan->stream));  // the synchronous copies below use the allocation
  rp_decision *dv = (rp_decision *)t.p;
  int32_t *dk = (int32_t *)((unsigned char *)t.p + vb);
  RP_CUDA(cudaMemcpy(dv, hv.data(), vb, cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(dk, hk.data(), kb, cudaMemcpyHostToDevice));
  RP_CUDA(launch_hist_import(plan->hist, d, dk, dv, n, plan->stream));
  RP_CUDA(cudaStreamSynchronize(plan->stream));
  return RP_OK;
}

}  // extern "C"
