// rp_decide.cuh -- runtime decision service (NEXT row f2): history table and kernel arguments.
#pragma once

#include "rp_internal.cuh"

namespace rp {

constexpr int kHistProbes = 32;  // linear-probe window of the history table
constexpr int kDecideMaxF = 8192;

struct HistSlot {                // 96 B
  uint32_t state;                // 0 empty, 1 being written, 2 ready
  int32_t key[kMaxVars];         // the data tuple
  int32_t pad[3];
  rp_decision val;
};
static_assert(sizeof(rp_decision) == 48, "rp_decision layout");

struct HistTable {
  HistSlot *slots = nullptr;
  uint32_t mask = 0;
  unsigned long long *counters = nullptr;  // hits, misses, entries
  int enabled = 0;
  int prog = 0;
  double margin = 0.0;
};

struct DecideArgs {
  const DevProg *progs;
  CfgTable tab;
  int npe_pad;
  int prog;
  const int32_t *D;
  int64_t n;
  double margin;
  rp_decision *out;
  HistTable hist;
};

cudaError_t launch_decide(const DecideArgs &a, bool mwp, cudaStream_t s);
cudaError_t launch_hist_export(const HistTable &H, int d, int32_t *keys, rp_decision *vals, int32_t *slot_of,
                               unsigned *count, cudaStream_t s);
cudaError_t launch_hist_import(const HistTable &H, int d, const int32_t *keys, const rp_decision *vals, int64_t n,
                               cudaStream_t s);
cudaError_t launch_fingerprint(const DevProg *pg, const int32_t *F, size_t f_bytes, unsigned long long *out,
                               cudaStream_t s);

}  // namespace rp
