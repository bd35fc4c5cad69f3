// small_step.cu -- host side of K3: shared-memory plan, cluster-size choice and dispatch of
// the cluster kernel (templates in small_step.cuh, one translation unit per eigen-block
// width BT so the build parallelises).
#include <cstdlib>

#include "small_step.cuh"

namespace wlr {

#define WLR_SS_EXTERN(B)                                                                   \
  extern template cudaError_t launch_ss<B>(const SmallArgs&, int, cudaStream_t);            \
  extern template int ss_max_clusters<B>(int, size_t);
WLR_SS_EXTERN(4)
WLR_SS_EXTERN(8)
WLR_SS_EXTERN(12)
WLR_SS_EXTERN(16)
WLR_SS_EXTERN(24)
WLR_SS_EXTERN(32)

static int bt_of(int b) { return b <= 4 ? 4 : b <= 8 ? 8 : b <= 12 ? 12 : b <= 16 ? 16 : b <= 24 ? 24 : 32; }
int small_step_bt(int b) { return bt_of(b); }

static int max_clusters(int bt, int CL, size_t smem) {
  switch (bt) {
    case 4: return ss_max_clusters<4>(CL, smem);
    case 8: return ss_max_clusters<8>(CL, smem);
    case 12: return ss_max_clusters<12>(CL, smem);
    case 16: return ss_max_clusters<16>(CL, smem);
    case 24: return ss_max_clusters<24>(CL, smem);
    default: return ss_max_clusters<32>(CL, smem);
  }
}

static constexpr int64_t kSmemLimit = 227 * 1024 / 8;   // doubles per CTA

// Lay out the shared memory of one CTA for cluster size CL.  Required regions first, then
// optional ones greedily in priority order (C' slice, Newton-Schulz mats, M' slice, gathered
// S-product operand -- for non-uniform W1: C' and M' slices, gathered operand, Newton-Schulz
// mats --, staged G/Gamma/Omega, C_in slice, CTA-0 tail staging); an optional
// region that does not fit gets offset -1 (the kernel then uses the global copy).
static bool plan_once(SmallArgs& a, int CL, int ccx) {
  SSPlan& p = a.pl;
  const int k = a.k, nk = a.nk, t = a.t, b = a.b, bt = bt_of(b);
  p.CL = CL;
  p.SL = (int)ceil_div(nk, CL);
  if (p.SL > 64 || p.SL < 1) return false;
  p.JS = bt <= 8 ? 1 : bt <= 16 ? 2 : 4;
  p.KS = 16 / p.JS;
  const int64_t SL = p.SL, kt = (int64_t)k * t, kk = (int64_t)k * k;
  // exchange bank: C X (k b), the Rayleigh-Ritz Grams (+ C'C'^T on the first pass), C'V' (k t)
  int64_t pl = std::max<int64_t>({(int64_t)k * b, 2LL * b * b + 2LL * t * b + (ccx ? kk : 0), (int64_t)t + kt});
  p.ccx = ccx;
  p.PL = (int)round_up(pl, 2);
  const FinOff fo(k, t);
  p.flen = fo.len;
  const SmallOff so(b, t, k);
  int64_t o = 0;
  auto take = [&](int64_t n) { const int64_t r = o; o += round_up(n, 2); return r; };
  p.oPart = take(2LL * p.PL);
  p.oBuf = take(4 * SL * b);
  p.oVp = take(SL * t);
  p.oE = take(SL * t);
  p.oSE = take(SL * t);
  p.oWk = take((int64_t)k * b);
  p.oCinE = take(t + kt);
  p.oSmall = take(so.len);
  p.oRed = take(std::max<int64_t>((int64_t)p.KS * SL * b, (SL + t) * (int64_t)k));   // also U rows, Qt
  if (o > kSmemLimit) return false;
  auto opt = [&](int64_t n) -> int64_t {
    if (o + round_up(n, 2) > kSmemLimit) return -1;
    return take(n);
  };
  p.oCs = opt((int64_t)k * (SL | 1));
  if (a.uniform) {       // (the K^{-1} refinement runs on the staged Newton-Schulz matrices every call)
    p.oGsq = opt(4 * kk);
    p.oMs = opt((int64_t)k * (SL | 1));
    p.oXf = opt((int64_t)nk * b);
  } else {               // (narrow gaps: many filter products per call, each gathers X)
    p.oMs = opt((int64_t)k * (SL | 1));
    p.oXf = opt((int64_t)nk * b);
    p.oGsq = opt(4 * kk);
  }
  p.oMat3 = opt(3 * kk + kt);
  p.oCin = opt((int64_t)k * (SL | 1));
  p.oTail = opt(p.flen + 3 * kt);
  p.total = o;
  p.gws_stride = p.oGsq >= 0 ? 0 : 4 * kk;
  return true;
}

// C'C'^T in the exchange bank (ccx) serves the uniform K^{-1}; for non-uniform W1 the bank space
// goes to the staged Newton-Schulz matrices first (C'C'^T is then summed through global memory,
// each CTA storing its share of the row solves' operand)
bool small_step_plan(SmallArgs& a, int CL) {
  if (!a.uniform) return plan_once(a, CL, 0) || plan_once(a, CL, 1);
  return plan_once(a, CL, 1) || plan_once(a, CL, 0);
}

// Largest cluster (<= 16 CTAs, >= 24 columns per CTA where possible) whose plan fits and
// which the device can co-schedule.
int small_step_cluster_size(SmallArgs& a) {
  const int lo = (int)std::max<int64_t>(1, ceil_div(a.nk, 64));
  if (lo > 16) return 0;                       // (n - k > 16 x 64: no cluster holds the slices)
  int want = (int)std::max<int64_t>(lo, std::min<int64_t>(16, ceil_div(a.nk, 24)));
  if (const char* e = std::getenv("WLR_K3_CL")) want = std::max(lo, std::min(16, std::atoi(e)));   // (A/B)
  for (int CL = want; CL >= lo; --CL) {
    if (!small_step_plan(a, CL)) continue;
    if (max_clusters(bt_of(a.b), CL, (size_t)a.pl.total * 8) >= 1) return CL;
  }
  return 0;
}

cudaError_t launch_small_step(const SmallArgs& a, int part, cudaStream_t st) {
  switch (bt_of(a.b)) {
    case 4: return launch_ss<4>(a, part, st);
    case 8: return launch_ss<8>(a, part, st);
    case 12: return launch_ss<12>(a, part, st);
    case 16: return launch_ss<16>(a, part, st);
    case 24: return launch_ss<24>(a, part, st);
    default: return launch_ss<32>(a, part, st);
  }
}

}  // namespace wlr
