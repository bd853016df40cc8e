// rp_device.cuh -- device helpers shared by the sweep and the decision kernels.
#pragma once

#include "rp_internal.cuh"

namespace rp {

// ---- argmin state: exact lexicographic (E, index) with the runner-up E ----------------------
struct Best {
  double e;   // best E (+inf: none)
  int32_t i;  // its original config index (INT_MAX: none)
  double s;   // the runner-up's E: the second-smallest (E, index) key among the others
  int32_t j;  // the runner-up's original index (meaningful where s < +inf)
};
__device__ __forceinline__ bool key_less(double e1, int32_t i1, double e2, int32_t i2) {
  return e1 < e2 || (e1 == e2 && i1 < i2);
}
__device__ __forceinline__ Best merge(const Best &a, const Best &b) {
  const bool aw = key_less(a.e, a.i, b.e, b.i);
  const Best &w = aw ? a : b, &l = aw ? b : a;
  Best r;
  r.e = w.e;
  r.i = w.i;
  // runner-up: the better of the winner's runner-up and the loser's best
  const bool ls = key_less(l.e, l.i, w.s, w.j);
  r.s = ls ? l.e : w.s;
  r.j = ls ? l.i : w.j;
  return r;
}
__device__ __forceinline__ Best shfl_xor(const Best &a, int m) {
  Best r;
  r.e = __shfl_xor_sync(0xffffffffu, a.e, m);
  r.i = __shfl_xor_sync(0xffffffffu, a.i, m);
  r.s = __shfl_xor_sync(0xffffffffu, a.s, m);
  r.j = __shfl_xor_sync(0xffffffffu, a.j, m);
  return r;
}

#ifdef RP_DMMA_NV  // a pure function of its operands: let the scheduler move it
#define RP_DMMA_ASM asm
#else
#define RP_DMMA_ASM asm volatile
#endif
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  RP_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(c0), "+d"(c1)
              : "d"(a), "d"(b));
}

// D = A B + C with C given separately (the factored tiles start from w_{k,0})
__device__ __forceinline__ void dmma_c(double &d0, double &d1, double a, double b, double c0, double c1) {
  RP_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
              : "=d"(d0), "=d"(d1)
              : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// 1/x: MUFU.RCP64H seed r0 (relative error e0 < 2^-20) and one cubically convergent step
// r = r0 (1 + e + e^2), e = 1 - x r0 (exact 1/x = r0 / (1 - e)): relative error e^3 + rounding,
// ~1 ulp, in 3 DFMA instead of the 4 of two Newton steps.  0 and +-inf give NaN (e = NaN),
// which the final finiteness test masks, as the literal program's x/0 would.
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// 1/x with one Newton step, r = r0 (1 + e): relative error ~e0^2 (< 2^-40), 2 DFMA.  Used by the
// sweep when the winners are re-evaluated exactly afterwards (k_refine): its E only ranks, and a
// ~1e-12 error changes the ranking only between configurations tied within ~1e-11 (the idx gate
// excludes margins below 1e-9; the refined winner's E is exact either way).
__device__ __forceinline__ double frcp1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}
template <bool FAST>
__device__ __forceinline__ double rcp_t(double x) {
  return FAST ? frcp1(x) : frcp(x);
}

// positive finite doubles order like their bit patterns: the validity test and the argmin key
// compare run on the integer pipes instead of the (shared, saturated) FP64 datapath
__device__ __forceinline__ bool pos_finite(double x) {
  const long long b = __double_as_longlong(x);
  return b > 0 && b < 0x7ff0000000000000ll;
}

// exact ceil(D / P) = floor((D + P - 1) / P) for 1 <= D + P - 1 < 2^31 via the per-config
// multiply-shift (M, s) of k_plan_configs
__device__ __forceinline__ int64_t ceil_div_magic(int32_t D, int32_t Pm1, uint32_t M, uint32_t s) {
  const uint64_t n = (uint64_t)(uint32_t)(D + Pm1);
  return (int64_t)((n * (uint64_t)M) >> s);
}

// the same in 32 bits (the quotient is < 2^32): one IMAD.WIDE.U32 and one funnel shift
__device__ __forceinline__ uint32_t ceil_div32(int32_t D, int32_t Pm1, uint32_t M, uint32_t s) {
  const uint64_t n = (uint64_t)(uint32_t)(D + Pm1);
  return (uint32_t)((n * (uint64_t)M) >> s);
}

// E for one (D, P) pair from its 2l polynomial values (Appendix A in
// common-denominator form g_i = a_i / Q; every division is a Newton reciprocal).  Straight-line
// code: masked pairs are carried to the end and returned as +inf.
struct EConst {
  double Lunc, Lcoal, DdU, ddc, issue, Kbw, rKbw;
};
// per-program constants of Appendix A, folded once (lines 7, 9, 11, 13)
__device__ __forceinline__ EConst make_econst(const DevProg &pg) {
  EConst kc;
  kc.Lunc = pg.mem_ld + (pg.U - 1.0) * pg.dd_unc;  // line 7
  kc.Lcoal = pg.mem_ld;
  kc.DdU = pg.dd_unc * pg.U;  // line 9
  kc.ddc = pg.dd_coal;
  kc.issue = pg.issue;                       // line 13
  kc.Kbw = pg.mem_bw / (pg.freq * pg.lbpw);  // line 11: Mem_BW / (Freq LoadBytesPerWarp)
  kc.rKbw = (pg.freq * pg.lbpw) / pg.mem_bw;
  return kc;
}

template <bool FAST = false>
__device__ __forceinline__ double mwpcwp_E(double p1, double q1, double p2, double q2, double p3,
                                           double q3, double W, double Rep, double rSM,
                                           double SMact, const EConst &k) {
  const double q23 = q2 * q3, q13 = q1 * q3, q12 = q1 * q2;
  const double Q = q1 * q23;
  const double a1 = p1 * q23, a2 = p2 * q13, a3 = p3 * q12;  // g_i = a_i / Q
  const double s23 = a2 + a3;                                 // Mem Q          (line 5)
  const double s = a1 + s23;                                  // Tot Q          (line 5)
  const double mc = fma(k.Lunc, a3, k.Lcoal * a2);            // Mem_c Q        (line 13)
  const double dn = fma(k.DdU, a3, k.ddc * a2);               // Dep Mem Q      (lines 6, 9)
  const double cc = k.issue * s;                              // Comp_c Q       (line 13)
  const double rQ = rcp_t<FAST>(Q), r23 = rcp_t<FAST>(s23);
  const double Mem_c = mc * rQ, Comp_c = cc * rQ;
  const double MWP_nb = mc * rcp_t<FAST>(dn);  // line 10: Mem_L / Dep
  const double MWP_bw = k.Kbw * mc * r23 * rSM;  // line 11: Mem_BW / (BW_per_warp SM_act)
  const double CWPf = 1.0 + mc * rcp_t<FAST>(cc);  // line 14: (Mem_c + Comp_c) / Comp_c
  // line 12: MWP = min(MWP_nb, MWP_bw, W_act); each comparison is made once and its outcome
  // reused for the case tests (MWP == W_act <=> W_act <= min(MWP_nb, MWP_bw), also for NaN)
  const bool bw = MWP_bw < MWP_nb;
  const double mwp0 = bw ? MWP_bw : MWP_nb;
  const bool mwpW = W <= mwp0;
  const double mwp = mwpW ? W : mwp0;
  const bool cwpf = CWPf < W;  // line 14: CWP = min(CWPf, W_act); CWP == W_act <=> !cwpf
  const double cwp = cwpf ? CWPf : W;
  const double cpm = cc * r23;             // Comp_c / Mem
  const double tail = cpm * (mwp - 1.0);
  // Mem_c W / MWP for each operand of the min: W / W = 1; Mem_c / MWP_nb = Dep Mem = dn / Q;
  // Mem_c / MWP_bw = Mem SM_act / K_bw = s23 SM_act / (Q K_bw)  (MWP_nb NaN: tail is NaN)
  const double mcw = mwpW ? Mem_c : W * rQ * (bw ? s23 * SMact * k.rKbw : dn);
  const double E1 = Mem_c + Comp_c + tail;         // line 16
  const double E2 = mcw + tail;                    // line 17
  const double E3 = mc * r23 + Comp_c * W;         // line 18 (Mem_L = Mem_c / Mem)
  const bool c1 = mwpW && !cwpf;
  const bool c2 = (cwp >= mwp) || (Comp_c > Mem_c);
  return (c1 ? E1 : (c2 ? E2 : E3)) * Rep;
}

// ---- the screening estimate of the warp-specialised sweep: Appendix A in FP32, proven bound ----
// Every quantity below is a product, quotient or sum of positive values (the inputs are checked
// positive; MWP >= 2 makes MWP - 1 >= MWP / 2, so no subtraction cancels), which bounds the
// relative error of each by a count of roundings: ~70 u (u = 2^-24, ~4.2e-6) for E, ~25 u for
// every compared quantity.  A pair is flagged `unc` (its FP32 value
// is not trusted and it is re-evaluated in FP64) when an input lies outside [1e-9, 1e9],
// MWP < 2, a case comparison is within kScreenCmp relative, or E is not positive and finite.
constexpr float kScreenCmp = 1e-5f;  // comparisons closer than this are decided in FP64
constexpr double kScreenEta = 1e-5;  // |E32 - E| <= kScreenEta E for pairs not flagged

struct EConst32 {
  float Lunc, Lcoal, DdU, ddc, issue, Kbw, rKbw;
};
__device__ __forceinline__ EConst32 to_econst32(const EConst &k) {
  return EConst32{(float)k.Lunc, (float)k.Lcoal, (float)k.DdU, (float)k.ddc, (float)k.issue, (float)k.Kbw,
                  (float)k.rKbw};
}
__device__ __forceinline__ bool fclose(float x, float y, float tol = kScreenCmp) {  // |x - y| <= tol max(x, y)
  return fabsf(x - y) <= tol * fmaxf(x, y);
}
__device__ __forceinline__ float rcp32(float x) {  // MUFU.RCP: relative error <= 2^-23
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// x in [1e-9, 1e9] (positive, normal, not NaN) by one unsigned compare on the bit pattern
__device__ __forceinline__ bool in_range32(float x) {
  return (uint32_t)(__float_as_uint(x) - 0x3089705fu) <= (uint32_t)(0x4e6e6b28u - 0x3089705fu);
}

// tol: the relative closeness below which a case comparison is not trusted (kScreenCmp for inputs
// that are rounded FP64 values; the tensor-core screen passes its per-pair bound)
__device__ __forceinline__ float mwpcwp_E32(float p1, float q1, float p2, float q2, float p3, float q3, float W,
                                            float Rep, float rSM, float SMact, const EConst32 &k, bool &unc,
                                            float tol = kScreenCmp) {
  // inputs in [1e-9, 1e9]: every intermediate stays a normal float (products of three inputs and
  // the hardware constants lie within ~1e-30 .. 1e33)
  unc = !(in_range32(p1) & in_range32(q1) & in_range32(p2) & in_range32(q2) & in_range32(p3) & in_range32(q3));
  const float q23 = q2 * q3, q13 = q1 * q3, q12 = q1 * q2;
  const float Q = q1 * q23;
  const float a1 = p1 * q23, a2 = p2 * q13, a3 = p3 * q12;
  const float s23 = a2 + a3, s = a1 + s23;
  const float mc = fmaf(k.Lunc, a3, k.Lcoal * a2);
  const float dn = fmaf(k.DdU, a3, k.ddc * a2);
  const float cc = k.issue * s;
  const float rQ = rcp32(Q), r23 = rcp32(s23);
  const float Mem_c = mc * rQ, Comp_c = cc * rQ;
  const float MWP_nb = mc * rcp32(dn);
  const float MWP_bw = k.Kbw * mc * r23 * rSM;
  const float CWPf = fmaf(mc, rcp32(cc), 1.0f);
  const bool bw = MWP_bw < MWP_nb;
  const float mwp0 = bw ? MWP_bw : MWP_nb;
  const bool mwpW = W <= mwp0;
  const float mwp = mwpW ? W : mwp0;
  const bool cwpf = CWPf < W;
  const float cwp = cwpf ? CWPf : W;
  const float cpm = cc * r23;
  const float tail = cpm * (mwp - 1.0f);
  const float mcw = mwpW ? Mem_c : W * rQ * (bw ? s23 * SMact * k.rKbw : dn);
  const float E1 = Mem_c + Comp_c + tail;
  const float E2 = mcw + tail;
  const float E3 = mc * r23 + Comp_c * W;
  const bool c1 = mwpW && !cwpf;
  const bool c2 = (cwp >= mwp) || (Comp_c > Mem_c);
  const float E = (c1 ? E1 : (c2 ? E2 : E3)) * Rep;
  // a comparison is checked only where its outcome is used: W <= min(MWP_nb, MWP_bw) decides
  // MWP = W_act (case 1); which of MWP_nb, MWP_bw is smaller picks the formula of Mem_c W / MWP
  // (line 17) when MWP < W_act; CWPf < W_act decides case 1 when MWP = W_act; CWP >= MWP and then
  // Comp_c > Mem_c decide case 2 when case 1 does not hold.  (The values of the mins are accurate
  // whichever operand is smaller.)
  // (bitwise | and &: branch-free)
  unc = unc | !(mwp >= 2.0f) | fclose(W, mwp0, tol) | (!mwpW & fclose(MWP_bw, MWP_nb, tol)) |
        (mwpW & fclose(CWPf, W, tol)) | (!c1 & fclose(cwp, mwp, tol)) |
        (!c1 & !(cwp >= mwp) & fclose(Comp_c, Mem_c, tol)) | !(E > 0.f & E < 3.0e38f);
  return E;
}

}  // namespace rp
