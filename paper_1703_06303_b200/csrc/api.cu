// api.cu -- the C ABI of libwlr.so (include/wlr.h) and the host-side state machine.
//
// One wlr_init builds the initial canonical state X_0 (GHS / Theorem 1 when X1_0 = A1,
// PAPER.md:56-65).  Every iteration then enqueues, on the handle's stream:
//     K2a row pass  -> K2b Gram-increment GEMM -> K2c fixed-order reduce
//     -> [ncclAllReduce of the packed fp64 increments when rows are sharded]
//     -> K3 small step (one thread-block cluster)
// optionally captured once per buffer parity as a CUDA graph and replayed.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wlr.h"
#include "kernels.h"

using namespace wlr;

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    if (!getUniqueId || !commInitRank || !allReduce || !commDestroy) {
      err = "libnccl is missing symbols";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;

thread_local std::string g_err;

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct Profile {
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  double ms[6] = {0, 0, 0, 0, 0, 0};   // row pass, increments (or Gram propagation), reduce, K3a, K3b, row solves
  int64_t launches = 0, iters = 0;
  std::vector<int> groups;           // per profiled iteration: 1 if it launched a deferred K3b
};

}  // namespace

// Virtual ranks on one GPU (include/wlr.h wlr_vgroup): a host barrier between the members' threads,
// per-slot staging buffers and events; the sum is a fixed-order device reduce (vsum_kernel).
struct wlr_vgroup_s {
  int G = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  double* buf[2] = {nullptr, nullptr};   // slot s: G x cap doubles
  size_t cap = 0;
  std::vector<cudaEvent_t> ready, done[2];
  std::vector<char> done_valid[2];
  void barrier(const std::function<void()>& last = nullptr) {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t my = gen;
    if (++arrived == G) {
      if (last) last();
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

// f3 block-ALS state (R21; kernels in als.cu)
struct AlsSt {
  void* B = nullptr;            // m x kp (first r-k columns), storage dtype
  void* Wb = nullptr;           // B row map (KA + KX) x rpb
  double *C[2] = {}, *D[2] = {};
  double *inc1 = nullptr, *inc2 = nullptr, *scal = nullptr, *F = nullptr;
  double *cct = nullptr, *dct = nullptr, *part = nullptr;
  int nF = 0, nrec = 0;         // F capacity, states recorded
  CUtensorMap tmBx, tmAr, tmXr[2], tmWb;
  int rpb = 0, x = 0, c = 0;
  double F0 = 0.0;              // objective of the GHS state (host copy, staged to F[0])
};

struct wlr_ctx {
  // dimensions
  int64_t m = 0, n = 0, k = 0, r = 0, t = 0, nk = 0, kp = 0, k0 = 0;
  int64_t m_global = 0, row_offset = 0;
  int dtype = WLR_F32;
  size_t es = 4;
  bool uniform = true;
  double w1s = 1.0;
  int b = 0, rp = 0, rp_tr = 8, bm = 0, nz = 0, nsplit = 0, rp_grid = 0, KA = 0;
  int64_t rps = 0;
  SSPlan spl{};
  int nsm = 148;
  wlr_opts opts;
  // data
  const void* A = nullptr; int64_t lda = 0;
  const void* W1 = nullptr; int64_t ldw = 0;
  void* X[2] = {nullptr, nullptr};
  void* Dl = nullptr;          // Delta = X1_{p+1} - X1_p (m x kp, written by the row pass)
  CUtensorMap tmA{}, tmX[2]{}, tmW{};   // TMA descriptors of A, X1 (per buffer) and Wt
  // tensor-core row pass (uniform W1, fp32): 128-row boxes of A / X1 and the K-major W'^T
  bool tc_ok = false, tc_on = false;
  int tc_dbg = 0;                       // diagnostics only (WLR_TC_DBG)
  unsigned long long* tc_tstamp = nullptr;   // per-CTA timestamps (WLR_TC_DBG & 16)
  unsigned long long* itc_tstamp = nullptr;  // increments, per CTA (WLR_TC_DBG & 32)
  int tc_grid = 0;
  int64_t tc_m_main = 0;       // rows covered by tensor-core tiles
  int tc_extra = 0;            // leftover rows per CTA on the CUDA cores (one CTA per SM)
  bool tc_deep = false;        // 8-stage ring, one CTA per SM
  CUtensorMap tmA_x, tmX_x[2];  // leftover-row boxes (32 columns x 4 rows)
  void* WtT = nullptr; int KW = 0;
  CUtensorMap tmA_tc{}, tmX_tc[2]{}, tmWT{};
  int nwc = 8;                 // row-pass warps running per-row Cholesky
  void *Wt = nullptr, *CVop = nullptr, *Kop = nullptr;
  // W' double-buffered by iteration parity: row pass(p) and prop(p) read W'_p while K3a(p) writes
  // W'_{p+1} (buffer 0 is Wt / WtT / tmW / tmWT, also used by the block ALS)
  void *Wt1 = nullptr, *WtT1 = nullptr;
  CUtensorMap tmW1{}, tmWT1{};
  // Gram propagation (uniform W1, prop.cu): A^T A, Q_p = A^T X1_p (by parity), scratch
  bool prop = false;
  double *AtA = nullptr, *Qg[2] = {nullptr, nullptr}, *Hs = nullptr, *dgs = nullptr, *GAY[2] = {nullptr, nullptr};   // G_A Y by iteration parity
  double a1sq = 0.0;
  cudaStream_t st3 = nullptr;  // row-pass branch of a propagation iteration
  cudaStream_t st4 = nullptr;  // critical chain (prop -> K3a) of a propagation iteration, high priority
  cudaEvent_t ev_f3 = nullptr, ev_j3 = nullptr, ev_j4 = nullptr;
  float* Sop = nullptr;        // fp32 C C^T, ld round_up(k, 8): per-row solves (non-uniform fp32)
  double *inc_part = nullptr, *inc_part2 = nullptr, *fw_part = nullptr, *fw0 = nullptr;
  int ics = 1, ncl = 0;        // increment row splits per cluster, cluster partials
  // tensor-core increments (fp32, kp <= 32): own column layout (A part padded to 32)
  bool itc_ok = false, itc_on = false;
  int itc_nsplit = 0, itc_nA32 = 0, itc_nz = 0, itc_cs = 1, itc_kpd = 32;
  // non-uniform fp32: e rows -> warp-per-row shared-memory Cholesky (rowsolve.cu)
  void* Ebuf = nullptr; int rs_grid = 0;
  int64_t itc_rps = 0;
  CUtensorMap tmA32{}, tmX32[2]{}, tmD32{};
  double* inc[2] = {nullptr, nullptr};   // packed increments, by iteration parity
  double* GA = nullptr;
  double a2sq = 0.0;
  // small-step state S_p (Grams, C, G^{-1}, Ritz block) in slot p mod 3: K3a(p) writes slot
  // (p+1) mod 3 while the deferred K3b(p-1) still reads slots (p-1) and p mod 3
  double *G[3] = {}, *M[3] = {}, *C[3] = {};
  double *Gi[3] = {}, *Ki = nullptr, *gws = nullptr, *gws2 = nullptr;   // G^{-1}, K^{-1}, workspaces
  double *V[3] = {}, *CV[3] = {}, *th[3] = {};
  double *Y = nullptr, *k3x[2] = {nullptr, nullptr};
  double *xchg = nullptr, *xchg2 = nullptr, *red = nullptr, *scal = nullptr, *trace = nullptr;
  double* tdbg = nullptr;      // K3 phase timestamps (wlr_debug_state "ktime")
  int prop_nb = 0;             // prop1 CTAs (min(n, prop_nsm))
  int prop_nsm = 0;            // SMs prop1 spreads over: #SMs less those the K3b / shadow clusters hold
  unsigned long long* prop_ts = nullptr;   // (diagnostics: WLR_PROP_TS=1, prop1 phase stamps)
  bool k3b_early = true;       // K3b(p-1) forks at the iteration start (WLR_K3B_EARLY=0: after prop1)
  // shadow K3a (propagation mode): at the start of iteration p a rerun of K3a(p-1)
  // with every output redirected into these private buffers, so that its instruction fetches pull
  // K3a's code into L2 ahead of the real K3a(p) (the bench flushes L2 before every iteration).
  // Nothing reads what it writes; WLR_SHADOW=0 disables it.
  bool shadow = false;
  bool shadow_now = false;     // enqueue_prop_iteration launches the shadow (every iteration but p = 0)
                               // (every real K3a writes the snapshots, whatever path launched it)
  cudaStream_t st5 = nullptr;
  cudaEvent_t ev_j5 = nullptr;
  double *sh_G = nullptr, *sh_M = nullptr, *sh_C = nullptr, *sh_V = nullptr, *sh_CV = nullptr, *sh_th = nullptr;
  double *sh_k3x = nullptr, *sh_Gi = nullptr, *sh_gws = nullptr, *sh_xchg = nullptr;
  double *snapY[2] = {nullptr, nullptr}, *snapKi[2] = {nullptr, nullptr};   // K3a(p)'s Y, K^{-1} inputs, by parity
  double *sh_red = nullptr, *sh_scal = nullptr, *sh_trace = nullptr;
  void *sh_Wt = nullptr, *sh_WtT = nullptr, *sh_CVop = nullptr, *sh_Kop = nullptr;
  float* sh_Sop = nullptr;
  int* sh_flags = nullptr;
  SmallArgs last_ss{};         // arguments of the last small-step launch (diagnostics)
  bool ktime = false;
  int trace_cap = 4096;
  // device flags (8 ints): [0] first error (DevFlag), [1] input validation bits (1: W1 <= 0, 2: non-
  // finite), [2] converged (eps rule), [3] eigensolver restarts of the last small step (diagnostics),
  // [4] (spare), [5] tensor-core increments gate (X1
  // step small), [6] the iteration's latched stop flag (eps mode), [7] K3b(p-1) of the next graph
  // already ran (set by flush_pending / init, cleared by that K3b)
  int* flags = nullptr;
  int* h_flags = nullptr;
  double* h_scal = nullptr;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  int ph = 0;                  // phase of the current state (= p mod 6: X by p mod 2, state by p mod 3)
  int64_t p = 0;               // index of the current canonical state
  AlsSt* als = nullptr;        // f3 block ALS (consumes the sWLR state)
  // row-pass timing inside the graph (wlr_debug_state "rptime_on"): external event records around
  // the row pass only, read after each graph launch (bench.py's roofline pass)
  bool rp_time = false;
  cudaEvent_t rp_ev[2] = {};
  double rp_ms = 0.0;
  int64_t rp_n = 0;
  cudaGraphExec_t gexec[6][2] = {};   // [phase][deferred pending]
  cudaStream_t st2 = nullptr;  // side stream of the deferred small-step half
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool zero_defer = false;     // dalloc defers its zeroing to flush_zero (init allocation block)
  std::vector<std::pair<void*, int64_t>> zero_list;
  bool pending = false;        // deferred half of the last small step not launched yet
  // One graph per phase: it always holds K3b(p-1); when that half already ran (flush_pending, or
  // the GHS step at init) the host sets flags[7] and the graph's K3b clears it and returns
  // (halves the graphs instantiated at init).  Eager iterations launch K3b only when pending.
  bool capturing = false;
  SmallArgs pend{};
  ncclComm_t comm = nullptr;
  wlr_vgroup_s* vg = nullptr;  // virtual ranks (test hook), instead of comm
  int64_t vcalls = 0;
  bool prof = false;
  Profile pr;
  std::string err;
  std::vector<void*> allocs;
};

static wlr_status fail(wlr_ctx* h, wlr_status s, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return s;
}

#define CUDA_TRY(h, x)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return fail(h, e_ == cudaErrorMemoryAllocation ? WLR_ENOMEM : WLR_ECUDA,               \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                          \
  } while (0)

// Pinned 128-byte blocks for the per-handle status words (8 doubles + 8 ints), kept in a
// process-wide free list.
static std::mutex g_pin_mu;
static std::vector<void*> g_pin_free;
static void* pinned_take() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      void* p = g_pin_free.back();
      g_pin_free.pop_back();
      std::memset(p, 0, 128);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, 128) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  std::memset(p, 0, 128);
  return p;
}
static void pinned_give(void* p) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

// Device buffers come from the device's default stream-ordered memory pool with the release
// threshold raised, so that a new handle (e.g. one per solve) reuses the memory of a destroyed one
// instead of paying cudaMalloc / cudaFree (which synchronises the device) every time.
static cudaMemPool_t wlr_pool() {
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!pools[dev]) {
    cudaMemPool_t p = nullptr;
    if (cudaDeviceGetDefaultMemPool(&p, dev) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[dev] = p;
  }
  return pools[dev];
}

static wlr_status dalloc(wlr_ctx* h, void** p, size_t bytes) {
  cudaMemPool_t pool = wlr_pool();
  cudaError_t e = pool ? cudaMallocFromPoolAsync(p, bytes ? bytes : 16, pool, h->st)
                       : cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, WLR_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  }
  h->allocs.push_back(*p);
  if (h->zero_defer) {                         // (init: zeroed together by flush_zero)
    h->zero_list.push_back({*p, (int64_t)(bytes ? bytes : 16)});
    return WLR_OK;
  }
  e = cudaMemsetAsync(*p, 0, bytes ? bytes : 16, h->st);
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, cudaGetErrorString(e));
  return WLR_OK;
}
// Zero every allocation deferred since zero_defer was set, with one kernel per 64 buffers (the
// initialisation allocates ~80 buffers between its first kernels; one memset each cost ~0.3 ms of
// launch-bound host time)
static wlr_status flush_zero(wlr_ctx* h) {
  h->zero_defer = false;
  for (size_t i = 0; i < h->zero_list.size(); i += kZeroList) {
    ZeroList z{};
    z.n = (int)std::min<size_t>(kZeroList, h->zero_list.size() - i);
    for (int j = 0; j < z.n; ++j) { z.ptr[j] = h->zero_list[i + j].first; z.bytes[j] = h->zero_list[i + j].second; }
    CUDA_TRY(h, launch_zero_list(z, h->st));
  }
  h->zero_list.clear();
  return WLR_OK;
}
template <typename P>
static wlr_status dalloc_t(wlr_ctx* h, P** p, size_t count) {
  return dalloc(h, reinterpret_cast<void**>(p), count * sizeof(P));
}

// Sum of buf (count fp64 values) over the ranks, in place, ordered on st: NCCL across GPUs, or the
// virtual group's fixed-order device sum; a no-op on one rank.
static wlr_status group_allreduce(wlr_ctx* h, double* buf, size_t count, cudaStream_t st, const char* what) {
  if (h->comm) {
    ncclResult_t nr = g_nccl.allReduce(buf, buf, count, ncclFloat64, ncclSum, h->comm, st);
    if (nr != ncclSuccess) return fail(h, WLR_ENCCL, std::string("ncclAllReduce(") + what + "): " + g_nccl.errStr(nr));
    return WLR_OK;
  }
  wlr_vgroup_s* g = h->vg;
  if (!g) return WLR_OK;
  const int r = h->opts.rank, slot = (int)(h->vcalls++ & 1);
  cudaError_t ae = cudaSuccess;
  g->barrier([&] {                           // the last member to arrive sizes the staging buffers
    if (count > g->cap) {
      cudaDeviceSynchronize();
      for (auto& b : g->buf) { if (b) cudaFree(b); b = nullptr; }
      for (auto& b : g->buf)
        if (ae == cudaSuccess) ae = cudaMalloc(&b, (size_t)g->G * count * sizeof(double));
      g->cap = ae == cudaSuccess ? count : 0;
    }
  });
  if (ae != cudaSuccess || !g->buf[slot]) return fail(h, WLR_ENOMEM, "virtual group staging buffers");
  for (int j = 0; j < g->G; ++j)             // the previous use of this slot has been summed everywhere
    if (g->done_valid[slot][j]) CUDA_TRY(h, cudaStreamWaitEvent(st, g->done[slot][j], 0));
  CUDA_TRY(h, cudaMemcpyAsync(g->buf[slot] + (size_t)r * g->cap, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaEventRecord(g->ready[r], st));
  g->barrier();
  for (int j = 0; j < g->G; ++j) CUDA_TRY(h, cudaStreamWaitEvent(st, g->ready[j], 0));
  CUDA_TRY(h, launch_vsum(buf, g->buf[slot], g->G, g->cap, count, st));
  CUDA_TRY(h, cudaEventRecord(g->done[slot][r], st));
  g->done_valid[slot][r] = 1;
  return WLR_OK;
}

extern "C" wlr_status wlr_vgroup_create(int32_t G, wlr_vgroup* out) {
  if (!out || G < 1) return fail(nullptr, WLR_EINVAL, "wlr_vgroup_create: need G >= 1");
  wlr_vgroup_s* g = new wlr_vgroup_s();
  g->G = G;
  g->ready.resize(G);
  for (int s = 0; s < 2; ++s) { g->done[s].resize(G); g->done_valid[s].assign(G, 0); }
  for (int j = 0; j < G; ++j) {
    bool ok = cudaEventCreateWithFlags(&g->ready[j], cudaEventDisableTiming) == cudaSuccess;
    for (int s = 0; s < 2; ++s) ok = ok && cudaEventCreateWithFlags(&g->done[s][j], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { cudaGetLastError(); wlr_vgroup_destroy(g); return fail(nullptr, WLR_ECUDA, "wlr_vgroup_create: events"); }
  }
  *out = g;
  return WLR_OK;
}

extern "C" void wlr_vgroup_destroy(wlr_vgroup g) {
  if (!g) return;
  cudaDeviceSynchronize();
  for (auto e : g->ready) if (e) cudaEventDestroy(e);
  for (auto& v : g->done) for (auto e : v) if (e) cudaEventDestroy(e);
  for (auto b : g->buf) if (b) cudaFree(b);
  delete g;
}

static wlr_status flush_pending(wlr_ctx* h);
static wlr_status check_flags(wlr_ctx* h) {
  {
    wlr_status fs = flush_pending(h);
    if (fs != WLR_OK) return fs;
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->h_flags, h->flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(h, cudaMemcpyAsync(h->h_scal, h->scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  switch (h->h_flags[0]) {
    case DF_OK: break;
    case DF_RANK: return fail(h, WLR_ERANK, "X1 is numerically rank deficient (Cholesky of X1^T X1 failed)");
    case DF_EIG: return fail(h, WLR_EEIG, "top-(r-k) eigensolver exceeded its iteration budget");
    case DF_ROWSPD: return fail(h, WLR_EINTERNAL, "a row system diag(W1^2)+CC^T was not SPD");
    case DF_NONFINITE: return fail(h, WLR_ENONFINITE, "non-finite objective");
    default: return fail(h, WLR_EINTERNAL, "unknown device flag");
  }
  h->p = (int64_t)llround(h->h_scal[5]);
  h->ph = (int)(h->p % 6);
  return WLR_OK;
}

// ------------------------------------------------------------------------ one iteration
static cudaEvent_t prof_event(wlr_ctx* h) {
  if (h->pr.used == h->pr.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->pr.pool.push_back(e);
  }
  return h->pr.pool[h->pr.used++];
}

// L2 prefetch list for the row pass: the inputs the following small step reads first
static void set_prefetch(wlr_ctx* h, int ph, const void** ptr, int64_t* bytes) {
  const int cur = ph % 3;
  const int64_t k = h->k, nk = h->nk;
  ptr[0] = h->GA;       bytes[0] = nk * nk * 8;
  ptr[1] = h->M[cur];   bytes[1] = k * nk * 8;
  ptr[2] = h->C[cur];   bytes[2] = k * nk * 8;
  ptr[3] = h->Y;        bytes[3] = nk * h->b * 8;
  ptr[4] = h->V[cur];   bytes[4] = nk * h->t * 8;
  ptr[5] = h->Gi[cur];  bytes[5] = k * k * 8;
  // (prefetching K3b(p-1)'s inputs too -- previous state slot, last increments -- shortened K3b
  // by ~8 us but slowed the critical K3a by ~2 us: measured and left out)
  for (int i = 6; i < kPf; ++i) { ptr[i] = nullptr; bytes[i] = 0; }
}

// Small-step arguments of iteration p (phase ph = p mod 6): state slot p mod 3 -> (p+1) mod 3,
// increments / exchange block by p mod 2.
// prop1 computes G_A Y of the warm block (Y fragments in registers: b <= 8, n - k <= 768)
static bool gay_fits(const wlr_ctx* h) { return prop_gay_ok((int)h->n, (int)h->k, h->b, h->prop_nsm); }

static SmallArgs small_args(wlr_ctx* h, int ph, int mode) {
  const int cur = ph % 3, nxt = (ph + 1) % 3, par = ph & 1;
  SmallArgs s{};
  s.k = (int)h->k; s.nk = (int)h->nk; s.t = (int)h->t; s.b = h->b; s.kp = (int)h->kp;
  s.k0 = (int)h->k0; s.rp = h->rp; s.KA = h->KA; s.mode = mode; s.dtype = h->dtype == WLR_F64 ? 1 : 0;
  s.uniform = h->uniform ? 1 : 0; s.w2 = h->w1s * h->w1s;
  s.GA = h->GA; s.a2sq = h->a2sq; s.inc = mode ? h->inc[par] : h->fw0;
  s.G_in = h->G[cur]; s.G_out = h->G[nxt]; s.M_in = h->M[cur]; s.M_out = h->M[nxt];
  s.C_in = h->C[cur]; s.C_out = h->C[nxt];
  s.V_in = h->V[cur]; s.V_out = h->V[nxt]; s.CV_in = h->CV[cur]; s.CV_out = h->CV[nxt];
  s.th_in = h->th[cur]; s.th_out = h->th[nxt]; s.k3x = h->k3x[par];
  s.Y = h->Y;
  if (h->shadow && mode != 0) { s.snapY = h->snapY[ph & 1]; s.snapKi = h->snapKi[ph & 1]; }
  s.Gi_in = h->Gi[cur]; s.Gi_out = h->Gi[nxt]; s.Ki = h->Ki; s.gws = h->gws;
  s.xchg = h->xchg; s.red = h->red; s.scal = h->scal;
  s.trace = h->trace; s.trace_cap = h->trace_cap;
  const bool wb1 = ((ph + 1) & 1) != 0;     // K3(p) writes W'_{p+1}
  s.Wt = wb1 ? h->Wt1 : h->Wt; s.CVop = h->CVop; s.Kop = h->Kop; s.Sop = h->Sop; s.flags = h->flags;
  s.WtT = wb1 ? h->WtT1 : h->WtT; s.KW = h->KW;
  s.eps = h->opts.eps; s.tol = h->opts.eig_tol; s.max_outer = h->opts.eig_max_outer; s.max_deg = 16;
  s.stop = (mode != 0 && h->opts.eps > 0.0) ? h->flags + 6 : nullptr;   // eps mode: latched stop flag
  s.GAY = (mode != 0 && h->prop && gay_fits(h)) ? h->GAY[ph & 1] : nullptr;
  s.dg = (mode != 0 && h->prop) ? h->dgs : nullptr;   // f_w from prop2's diagonal terms
  s.a1sq = h->a1sq;                      // (computed by prop1)
  s.cold = 0;
  s.tdbg = h->ktime ? h->tdbg : nullptr;
  s.pl = h->spl;
  return s;
}

// Launch the deferred half of the previous small step (objective, step norm, trace) on the
// main stream: needed before the host reads F / the trace / the stopping flag.
// K3b has its own exchange block / workspace, so it can run beside the next K3a.
static cudaError_t launch_deferred(wlr_ctx* h, const SmallArgs& a, cudaStream_t st) {
  SmallArgs d = a;
  d.skip = h->capturing ? h->flags + 7 : nullptr;
  d.xchg = h->xchg2;
  d.gws = h->gws2;
  if (d.tdbg) d.tdbg += 64;                  // its own timestamp block
  return launch_small_step(d, 2, st);
}

// Shadow K3a (see wlr_ctx::shadow), launched at the start of iteration p: a rerun of K3a(p-1) --
// state p-1 (slot (p-1) mod 3, intact until K3a(p+1) writes it), iteration p-1's increments and
// G_A Y (the parity-(p-1) buffers, which prop(p) does not write), and the copies of its two
// in-place inputs (warm block Y, K^{-1}) that K3a(p-1) wrote as it read them (snapY / snapKi by
// parity; the shadow updates that copy in place, K3a(p) writes the other one).  Same inputs, same
// code path: its instruction fetches run ahead of the real K3a(p).  Nothing carries over from one
// shadow to the next.
static SmallArgs shadow_args(wlr_ctx* h, int ph) {
  SmallArgs a = small_args(h, (ph + 5) % 6, 1);
  a.pdl = 0;
  a.G_out = h->sh_G; a.M_out = h->sh_M; a.C_out = h->sh_C; a.V_out = h->sh_V; a.CV_out = h->sh_CV;
  const int pp = ((ph + 5) % 6) & 1;         // parity of p-1
  a.th_out = h->sh_th; a.k3x = h->sh_k3x; a.Y = h->snapY[pp]; a.Gi_out = h->sh_Gi; a.Ki = h->snapKi[pp];
  a.snapY = nullptr; a.snapKi = nullptr;
  a.gws = h->sh_gws; a.xchg = h->sh_xchg; a.red = h->sh_red; a.scal = h->sh_scal; a.trace = h->sh_trace;
  a.Wt = h->sh_Wt; a.WtT = a.WtT ? h->sh_WtT : nullptr; a.CVop = h->sh_CVop; a.Kop = h->sh_Kop;
  a.Sop = a.Sop ? h->sh_Sop : nullptr; a.flags = h->sh_flags;
  a.tdbg = nullptr;
  return a;
}

static wlr_status flush_pending(wlr_ctx* h) {
  if (!h->pending) return WLR_OK;
  // eps mode: re-latch, so that a convergence decided inside the last launched iteration also
  // stops this deferred half (the state stays at the converged one)
  cudaError_t e = h->opts.eps > 0.0 ? launch_stop_latch(h->flags, h->st) : cudaSuccess;
  if (e == cudaSuccess) e = launch_deferred(h, h->pend, h->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->flags + 7, 1, 1, h->st);   // the next graph's K3b: done
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (deferred): ") + cudaGetErrorString(e));
  h->pending = false;
  h->pr.launches += 1;
  return WLR_OK;
}

// One iteration.  Stream order:
//   K3b(p-1) => row pass(p) -> increments(p) -> reduce(p) -> allreduce -> K3a(p)
// (=> programmatic dependent launch: the row pass overlaps K3b(p-1), the objective / step
// norm of the previous state; K3b only reads state the row pass does not write, and the
// increments, which wait for both, are where K3b's inputs get rewritten.)
// Row pass of iteration p (phase ph) on stream st: X1_{p+1} from [A | X1_p] and W'_p.  light: the
// tensor-core pass writes X1_{p+1} only (Gram-propagation mode needs no Delta / f_w partials).
static cudaError_t launch_row_pass_iter(wlr_ctx* h, int ph, cudaStream_t st, bool light, bool pdl = false,
                                        cudaEvent_t mid = nullptr) {
  const int cur = ph & 1, nxt = cur ^ 1;      // X1 buffers
  const bool wb = cur != 0;                   // W'_p buffer
  const int* stop = h->opts.eps > 0.0 ? h->flags + 6 : nullptr;
  cudaError_t e;
  if (h->dtype == WLR_F32) {
    RowPassArgs<float> a{};
    a.A = (const float*)h->A; a.lda = h->lda; a.W1 = (const float*)h->W1; a.ldw = h->ldw;
    a.w2s = (float)(h->w1s * h->w1s);
    a.Xold = (const float*)h->X[cur]; a.Xnew = (float*)h->X[nxt]; a.Dnew = (float*)h->Dl; a.nwc = h->nwc;
    a.Wt = (const float*)(wb ? h->Wt1 : h->Wt); a.KA = h->KA; a.Kmat = (const float*)h->Kop;
    a.tmA = h->tmA; a.tmX = h->tmX[cur]; a.tmW = wb ? h->tmW1 : h->tmW;
    a.fw_part = h->fw_part; a.flags = h->flags;
    a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->kp;
    a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
    a.Ebuf = (float*)h->Ebuf;
    a.stop = stop;
    set_prefetch(h, ph, a.pf_ptr, a.pf_bytes);
    if (h->tc_on) {
      RowPassTcArgs q{};
      q.E = (float*)h->Ebuf; q.W1 = (const float*)h->W1; q.ldw = h->ldw;   // (non-uniform: e rows)
      q.tmA = h->tmA_tc; q.tmX = h->tmX_tc[cur]; q.tmW = wb ? h->tmWT1 : h->tmWT;
      q.A = a.A; q.lda = a.lda; q.Xold = a.Xold; q.Xnew = a.Xnew; q.Dnew = light ? nullptr : a.Dnew;
      q.w2s = a.w2s; q.fw_part = h->fw_part;
      for (int i = 0; i < kPf; ++i) { q.pf_ptr[i] = light ? nullptr : a.pf_ptr[i]; q.pf_bytes[i] = light ? 0 : a.pf_bytes[i]; }
      q.m = h->m; q.KA = h->KA; q.k = (int)h->k; q.kp = (int)h->kp; q.n = (int)h->n;
      q.m_main = h->tc_m_main; q.extra = h->tc_extra;
      q.tmAx = h->tmA_x; q.tmXx = h->tmX_x[cur];
      q.dbg = h->tc_dbg;
      q.tstamp = h->tc_tstamp;
      q.pdl = pdl ? 1 : 0;
      q.stop = stop;
      e = launch_row_pass_tc(q, h->rp, h->tc_grid, st, nullptr, h->tc_deep);
    } else {
      e = launch_row_pass<float>(a, h->rp, h->rp_tr, h->uniform, 0, h->rp_grid, st);
    }
    if (mid) cudaEventRecord(mid, st);           // (profiling: the row pass / per-row solve boundary)
    {
      if (e == cudaSuccess && h->Ebuf) {
        RowSolveArgs q{};
        q.E = (const float*)h->Ebuf; q.S = h->Sop;
        q.W1 = (const float*)h->W1; q.ldw = h->ldw; q.A = (const float*)h->A; q.lda = h->lda;
        q.Xold = a.Xold; q.Xnew = a.Xnew; q.Dnew = a.Dnew; q.fw_part = h->fw_part; q.flags = h->flags;
        q.m = h->m; q.k = (int)h->k; q.kp = (int)h->kp;
        q.stop = stop;
        q.e_lin = h->tc_on ? 1 : 0;              // (the tensor-core row pass writes the linear part)
        e = launch_row_solve(q, h->rs_grid, st);
      }
    }
  } else {
    RowPassArgs<double> a{};
    a.A = (const double*)h->A; a.lda = h->lda; a.W1 = (const double*)h->W1; a.ldw = h->ldw;
    a.w2s = h->w1s * h->w1s;
    a.Xold = (const double*)h->X[cur]; a.Xnew = (double*)h->X[nxt]; a.Dnew = (double*)h->Dl; a.nwc = h->nwc;
    a.Wt = (const double*)(wb ? h->Wt1 : h->Wt); a.KA = h->KA; a.Kmat = (const double*)h->Kop;
    a.tmA = h->tmA; a.tmX = h->tmX[cur]; a.tmW = wb ? h->tmW1 : h->tmW;
    a.fw_part = h->fw_part; a.flags = h->flags;
    a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->kp;
    a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
    a.stop = stop;
    set_prefetch(h, ph, a.pf_ptr, a.pf_bytes);
    e = launch_row_pass<double>(a, h->rp, h->rp_tr, h->uniform, 0, h->rp_grid, st);
    if (mid) cudaEventRecord(mid, st);           // (fp64: the solves run inside the row pass)
  }
  return e;
}

// One iteration in Gram-propagation mode (uniform W1):
//   st : prop1(p) -> prop2(p) -> K3a(p)                   (the critical chain, m-independent)
//   st3:   row pass(p)  (X1_{p+1} materialised beside it; joined at the end of the iteration)
//   st2:   K3b(p-1)     (deferred objective / step norm of the previous state)
static wlr_status enqueue_prop_iteration(wlr_ctx* h, int ph) {
  const int cur = ph & 1, nxt = cur ^ 1, slot = ph % 3;
  const bool prof = h->prof, pend = h->pending;
  PropArgs pa{};
  pa.AtA = h->AtA; pa.Wt = cur ? h->Wt1 : h->Wt; pa.RP = h->rp; pa.KA = h->KA;
  pa.Qp = h->Qg[cur]; pa.Qn = h->Qg[nxt]; pa.Gp = h->G[slot]; pa.part = h->Hs;
  pa.inc = h->inc[cur]; pa.dg = h->dgs;
  pa.w2 = h->w1s * h->w1s; pa.a1sq = h->a1sq;
  pa.n = (int)h->n; pa.k = (int)h->k;
  set_prefetch(h, ph, pa.pf_ptr, pa.pf_bytes);   // K3a(p)'s inputs, issued at prop1's entry
  pa.stop = h->opts.eps > 0.0 ? h->flags + 6 : nullptr;
  pa.Y = h->Y; pa.GAY = gay_fits(h) ? h->GAY[cur] : nullptr; pa.b = h->b;   // G_A Y of the warm block for K3a(p)'s first S-product
  pa.ts = h->prop_ts;
  pa.nb = h->prop_nb;
  SmallArgs sa = small_args(h, ph, 1);
  cudaError_t e;
  if (prof) {   // eager profiling pass: everything serial on st, one event group per kernel kind
    cudaEvent_t ev[9];
    for (int i = 0; i < 9; ++i) ev[i] = prof_event(h);
    cudaEventRecord(ev[0], h->st);
    if ((e = launch_row_pass_iter(h, ph, h->st, true, false, ev[8])) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("row pass: ") + cudaGetErrorString(e));
    cudaEventRecord(ev[1], h->st);
    if ((e = launch_prop(pa, false, 0, h->st)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("Gram propagation: ") + cudaGetErrorString(e));
    cudaEventRecord(ev[2], h->st);
    cudaEventRecord(ev[3], h->st);
    cudaEventRecord(ev[4], h->st);
    sa.pdl = 0;
    h->last_ss = sa;
    if ((e = launch_small_step(sa, 1, h->st)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step: ") + cudaGetErrorString(e));
    cudaEventRecord(ev[5], h->st);
    if (pend) {
      cudaEventRecord(ev[6], h->st);
      if ((e = launch_deferred(h, h->pend, h->st)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (deferred): ") + cudaGetErrorString(e));
      cudaEventRecord(ev[7], h->st);
    }
    h->pr.iters++;
    h->pr.groups.push_back(pend ? 1 : 0);
  } else {
    // critical chain on the high-priority st4: prop1 -> prop2 -> K3a, and the row pass as K3a's
    // programmatic dependent: K3a holds its cluster's SMs before the streaming pass fills the rest
    // of the GPU beside it.  K3b(p-1) on st2 once prop1 is done (it only needs to end with K3a).
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, h->st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->st4, h->ev_fork, 0));
    const bool shadow = h->shadow && h->shadow_now;   // (K3a(p-1) exists: p >= 1)
    if (shadow) {
      // K3b(p-1) and the shadow are clusters of whole SMs of one GPC: they must be resident before
      // prop1's CTAs spread over every GPC (prop1 leaves them prop_nsm's room), so they are
      // launched first and prop1 follows an empty kernel on st4 (its launch latency is the head start)
      if (pend) {
        CUDA_TRY(h, cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
        if ((e = launch_deferred(h, h->pend, h->st2)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (deferred): ") + cudaGetErrorString(e));
        CUDA_TRY(h, cudaEventRecord(h->ev_join, h->st2));
      }
      CUDA_TRY(h, cudaStreamWaitEvent(h->st5, h->ev_fork, 0));
      if ((e = launch_small_step(shadow_args(h, ph), 1, h->st5)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (shadow): ") + cudaGetErrorString(e));
      CUDA_TRY(h, cudaEventRecord(h->ev_j5, h->st5));
      if ((e = launch_noop(h->st4)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("no-op: ") + cudaGetErrorString(e));
    }
    if ((e = launch_prop(pa, false, 0, h->st4, h->ev_f3)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("Gram propagation: ") + cudaGetErrorString(e));
    if (pend && !shadow) {
      CUDA_TRY(h, cudaStreamWaitEvent(h->st2, h->k3b_early ? h->ev_fork : h->ev_f3, 0));
      if ((e = launch_deferred(h, h->pend, h->st2)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (deferred): ") + cudaGetErrorString(e));
      CUDA_TRY(h, cudaEventRecord(h->ev_join, h->st2));
    }
    sa.pdl = 1;                                // right behind prop2
    h->last_ss = sa;
    if ((e = launch_small_step(sa, 1, h->st4)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step: ") + cudaGetErrorString(e));
    const bool rpt = h->rp_time;
    if (rpt) CUDA_TRY(h, cudaEventRecordWithFlags(h->rp_ev[0], h->st4, cudaEventRecordExternal));
    if ((e = launch_row_pass_iter(h, ph, h->st4, true, !rpt)) != cudaSuccess) return fail(h, WLR_ECUDA, std::string("row pass: ") + cudaGetErrorString(e));
    if (rpt) CUDA_TRY(h, cudaEventRecordWithFlags(h->rp_ev[1], h->st4, cudaEventRecordExternal));
    CUDA_TRY(h, cudaEventRecord(h->ev_j4, h->st4));
    CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_j4, 0));
    if (pend) CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_join, 0));
    if (shadow) CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_j5, 0));
  }
  if (!pend && !h->capturing) CUDA_TRY(h, cudaMemsetAsync(h->flags + 7, 0, 1, h->st));   // (now pending)
  h->pend = sa;
  h->pending = true;
  h->pr.launches += (pend ? 5 : 4) + (h->shadow && h->shadow_now && !prof ? 2 : 0);   // (+ shadow, no-op)
  return WLR_OK;
}

static wlr_status enqueue_iteration(wlr_ctx* h, int ph) {
  if (h->opts.eps > 0.0) {                     // eps mode: latch the converged flag for this iteration
    cudaError_t le = launch_stop_latch(h->flags, h->st);
    if (le != cudaSuccess) return fail(h, WLR_ECUDA, std::string("stop latch: ") + cudaGetErrorString(le));
    h->pr.launches += 1;
  }
  if (h->prop) return enqueue_prop_iteration(h, ph);
  const int cur = ph & 1, nxt = cur ^ 1;      // X1 buffers
  cudaEvent_t ev[9] = {};
  const bool prof = h->prof;
  const bool pend = h->pending;
  if (prof) {
    for (int i = 0; i < 9; ++i) ev[i] = prof_event(h);
    cudaEventRecord(ev[0], h->st);
  }
  const bool rpt = h->rp_time && !prof;
  if (rpt) CUDA_TRY(h, cudaEventRecordWithFlags(h->rp_ev[0], h->st, cudaEventRecordExternal));
  cudaError_t e = launch_row_pass_iter(h, ph, h->st, false, false, prof ? ev[8] : nullptr);
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("row pass: ") + cudaGetErrorString(e));
  if (prof) cudaEventRecord(ev[1], h->st);
  if (rpt) CUDA_TRY(h, cudaEventRecordWithFlags(h->rp_ev[1], h->st, cudaEventRecordExternal));
  if (h->dtype == WLR_F32) {
    IncrArgs<float> a{};
    a.A = (const float*)h->A; a.lda = h->lda;
    a.Xold = (const float*)h->X[cur]; a.Dnew = (const float*)h->Dl;
    a.part = h->inc_part; a.part2 = h->inc_part2; a.cs = h->ics; a.m = h->m; a.rows_per_split = h->rps;
    a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.k0 = (int)h->k0; a.nz = h->nz; a.nsplit = h->nsplit;
    a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0) && (h->n % 4 == 0);
    // tensor-core layout: one kernel; the small step's gate (flags[5]) decides on the device
    // whether its pipeline feeds the tensor cores (small X1 step) or CUDA-core FMAs
    a.gate = nullptr;
    a.pdl = prof ? 0 : 1;
    if (h->itc_on && h->itc_kpd > 32) a.gate = h->flags + 5;   // (it computes only while the gate is off)
    if (!h->itc_on || h->itc_kpd > 32) e = launch_incr<float>(a, h->bm, h->st);
    if (h->itc_on && e == cudaSuccess) {
      IncrTcArgs q{};
      q.tmA = h->tmA32; q.tmX = h->tmX32[cur]; q.tmD = h->tmD32;
      q.part = h->inc_part; q.m = h->m; q.rows_per_split = h->itc_rps;
      q.k = (int)h->k; q.k0 = (int)h->k0; q.nA32 = h->itc_nA32; q.nz = h->itc_nz; q.kpd = h->itc_kpd;
      q.gate = h->flags + 5;
      q.cs = h->itc_cs;
      q.tstamp = h->itc_tstamp;
      e = launch_incr_tc(q, h->itc_nsplit, h->st);
    }
  } else {
    IncrArgs<double> a{};
    a.A = (const double*)h->A; a.lda = h->lda;
    a.Xold = (const double*)h->X[cur]; a.Dnew = (const double*)h->Dl;
    a.part = h->inc_part; a.part2 = h->inc_part2; a.cs = h->ics; a.m = h->m; a.rows_per_split = h->rps;
    a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.k0 = (int)h->k0; a.nz = h->nz; a.nsplit = h->nsplit;
    a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0) && (h->n % 4 == 0);
    e = launch_incr<double>(a, h->bm, h->st);
  }
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("increments: ") + cudaGetErrorString(e));
  if (prof) cudaEventRecord(ev[2], h->st);
  // fork (before the reduce, so that K3a can be the reduce's programmatic dependent): the
  // deferred half of the previous step runs beside reduce(p) and K3a(p) on its own SMs; it reads
  // state slots and increments that neither writes (inc[p-1 mod 2]); joined at the end
  if (pend) {
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, h->st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
    if (prof) cudaEventRecord(ev[6], h->st2);
    e = launch_deferred(h, h->pend, h->st2);
    if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (deferred): ") + cudaGetErrorString(e));
    if (prof) cudaEventRecord(ev[7], h->st2);
    CUDA_TRY(h, cudaEventRecord(h->ev_join, h->st2));
  }
  const int nfw = h->Ebuf ? h->rs_grid : (h->tc_on ? h->tc_grid : h->rp_grid);   // (the solver writes f_w)
  if (h->itc_on && h->itc_kpd == 32)   // tensor-core layout: A part padded to nA32, kp' = 32
    launch_reduce_incr(h->inc_part, (int)ceil_div(h->itc_nsplit, h->itc_cs), (int)h->k, (int)h->nk, h->itc_nz,
                       (int)(h->k - h->k0), h->itc_nA32, 32, h->fw_part, nfw, h->inc[cur], h->st, nullptr,
                       ReduceLayout{nullptr, 0, 0, 0, 0}, !prof && !pend);
  else if (h->itc_on)   // KPD > 32: the CUDA-core layout while the gate is off, the tensor-core one after
    launch_reduce_incr(h->ics > 1 ? h->inc_part2 : h->inc_part, h->ics > 1 ? h->ncl : h->nsplit, (int)h->k,
                       (int)h->nk, h->nz, (int)(h->k - h->k0), (int)(h->n - h->k0), (int)h->kp, h->fw_part,
                       nfw, h->inc[cur], h->st, h->flags + 5,
                       ReduceLayout{h->inc_part, h->itc_nsplit, h->itc_nz, h->itc_nA32, h->itc_kpd}, !prof && !pend);
  else
    launch_reduce_incr(h->ics > 1 ? h->inc_part2 : h->inc_part, h->ics > 1 ? h->ncl : h->nsplit, (int)h->k,
                       (int)h->nk, h->nz, (int)(h->k - h->k0), (int)(h->n - h->k0), (int)h->kp, h->fw_part,
                       nfw, h->inc[cur], h->st, nullptr, ReduceLayout{nullptr, 0, 0, 0, 0}, !prof && !pend);
  if (prof) cudaEventRecord(ev[3], h->st);
  {
    wlr_status gs = group_allreduce(h, h->inc[cur], (size_t)(h->k * h->nk + 2 * h->k * h->k + 1), h->st, "increments");
    if (gs != WLR_OK) return gs;
  }
  if (prof) cudaEventRecord(ev[4], h->st);
  SmallArgs s = small_args(h, ph, 1);
  s.pdl = (!h->comm && !h->vg && !prof) ? 1 : 0;   // right behind the reduce kernel (no allreduce between)
  h->last_ss = s;
  e = launch_small_step(s, 1, h->st);
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step: ") + cudaGetErrorString(e));
  if (pend) CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_join, 0));   // join
  if (prof) {
    cudaEventRecord(ev[5], h->st);
    h->pr.iters++;
    h->pr.groups.push_back(pend ? 1 : 0);
  }
  if (!pend && !h->capturing) CUDA_TRY(h, cudaMemsetAsync(h->flags + 7, 0, 1, h->st));   // (now pending)
  h->pend = s;
  h->pending = true;
  h->pr.launches += pend ? 5 : 4;
  return WLR_OK;
}

// Capture one iteration (phase ph, deferred half pending or not) into *out.
static wlr_status capture_graph(wlr_ctx* h, int ph, int pend, cudaGraph_t* out) {
  const bool keep_pend = h->pending;
  const SmallArgs keep_args = h->pend;
  h->pending = pend != 0;
  if (pend) h->pend = small_args(h, (ph + 5) % 6, 1);   // the previous iteration's step
  h->capturing = true;
  CUDA_TRY(h, cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  const int64_t l0 = h->pr.launches;
  h->shadow_now = h->shadow;                 // graphs serve p >= 1 (p = 0 launches eagerly with a shadow)
  wlr_status s = enqueue_iteration(h, ph);
  h->shadow_now = false;
  h->pr.launches = l0;
  cudaError_t e = cudaStreamEndCapture(h->st, out);
  h->capturing = false;
  h->pending = keep_pend;
  h->pend = keep_args;
  if (s != WLR_OK) return s;
  CUDA_TRY(h, e);
  return WLR_OK;
}

// Instantiated iteration graphs outlive their handle (process-wide pool, keyed by device, shape and
// launch-path choices): a later handle of the same shape captures its graphs and updates a pooled
// executable in place (cudaGraphExecUpdate) instead of instantiating one -- instantiation is ~0.1 ms
// of host time per graph, the largest part of wlr_init for repeated solves.  An update that the
// driver rejects (another topology) falls back to instantiation.  Not for NCCL / virtual-group
// handles (their graphs hold communicator state).
static std::mutex g_gpool_mu;
static std::map<std::string, std::vector<cudaGraphExec_t>> g_gpool;
static std::string gpool_key(const wlr_ctx* h, int ph, int pend) {
  int dev = 0;
  cudaGetDevice(&dev);
  char b[256];
  std::snprintf(b, sizeof b, "%d:%lld:%lld:%lld:%lld:%d:%d:%d:%d:%d:%d:%d:%d:%d", dev, (long long)h->m,
                (long long)h->n, (long long)h->k, (long long)h->r, h->dtype, h->uniform ? 1 : 0,
                h->prop ? 1 : 0, h->shadow ? 1 : 0, h->tc_on ? 1 : 0, h->itc_on ? 1 : 0,
                h->opts.eps > 0.0 ? 1 : 0, ph, pend);
  return b;
}
static bool gpool_ok(const wlr_ctx* h) { return !h->comm && !h->vg && !h->rp_time; }

static wlr_status build_graph(wlr_ctx* h, int ph, int pend) {
  cudaGraph_t g;
  wlr_status s = capture_graph(h, ph, pend, &g);
  if (s != WLR_OK) return s;
  if (gpool_ok(h)) {
    cudaGraphExec_t ex = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_gpool_mu);
      auto it = g_gpool.find(gpool_key(h, ph, pend));
      if (it != g_gpool.end() && !it->second.empty()) { ex = it->second.back(); it->second.pop_back(); }
    }
    if (ex) {
      cudaGraphExecUpdateResultInfo info{};
      if (cudaGraphExecUpdate(ex, g, &info) == cudaSuccess) {
        h->gexec[ph][pend] = ex;
        cudaGraphDestroy(g);
        return WLR_OK;
      }
      cudaGetLastError();
      cudaGraphExecDestroy(ex);
    }
  }
  CUDA_TRY(h, cudaGraphInstantiate(&h->gexec[ph][pend], g, 0));
  cudaGraphDestroy(g);
  return WLR_OK;
}

// Instantiate (and upload) every per-iteration graph up front, so that no capture or
// instantiation ever lands inside a timed region or the first iterations of a solve.
// (Instantiating on 6 host threads was measured slower: 1.9-2.0 ms against 1.3 ms serial.)
static wlr_status build_all_graphs(wlr_ctx* h) {
  if (!h->opts.use_graph || h->prof) return WLR_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (int ph = 0; ph < 6; ++ph) {
    if (h->gexec[ph][1]) continue;
    wlr_status s = build_graph(h, ph, 1);
    if (s != WLR_OK) return s;
    CUDA_TRY(h, cudaGraphUpload(h->gexec[ph][1], h->st));
  }
  if (std::getenv("WLR_INIT_TIMES"))   // (diagnostics: host time of the graph builds)
    std::fprintf(stderr, "[wlr] graphs %.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  return WLR_OK;
}

static wlr_status reset_graphs(wlr_ctx* h) {   // after a launch-shape switch (diagnostics)
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  for (auto& gp : h->gexec)
    for (auto& g : gp)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  return build_all_graphs(h);
}

static wlr_status launch_iteration(wlr_ctx* h) {
  wlr_status s;
  if (h->als) return fail(h, WLR_EINVAL, "the handle ran the block-ALS variant (wlr_als_iterate); sWLR state is gone");
  if (h->opts.use_graph && !h->prof && !(h->shadow && h->p == 0)) {
    const int pend = 1;                       // (K3b(p-1) skips itself when not pending, flags[7])
    if (!h->gexec[h->ph][pend]) {
      s = build_graph(h, h->ph, pend);
      if (s != WLR_OK) return s;
    }
    CUDA_TRY(h, cudaGraphLaunch(h->gexec[h->ph][pend], h->st));
    if (h->rp_time) {   // (timing pass only: one host synchronisation per iteration)
      CUDA_TRY(h, cudaEventSynchronize(h->rp_ev[1]));
      float ms = 0.f;
      CUDA_TRY(h, cudaEventElapsedTime(&ms, h->rp_ev[0], h->rp_ev[1]));
      h->rp_ms += ms;
      h->rp_n++;
    }
    h->pend = small_args(h, h->ph, 1);
    h->pending = true;
    h->pr.launches += 5 + (h->shadow ? 2 : 0);
  } else {
    h->shadow_now = h->p > 0;                 // (the first iteration has no K3a(p-1) to rerun)
    s = enqueue_iteration(h, h->ph);
    h->shadow_now = false;
    if (s != WLR_OK) return s;
  }
  h->ph = (h->ph + 1) % 6;
  h->p += 1;
  return WLR_OK;
}

// ------------------------------------------------------------------------------- init
extern "C" void wlr_opts_default(wlr_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->dtype = WLR_F32;
  o->init = WLR_INIT_GHS;
  o->w1_scalar = 1.0;
  o->nranks = 1;
  o->use_graph = 1;
}

static uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
static void gram_launch(wlr_ctx* h, const void* L, int64_t ldl, int nl, const void* R, int64_t ldr,
                        int nr, double* part, int nsplit, double* out) {
  launch_gram64<T>((const T*)L, ldl, nl, (const T*)R, ldr, nr, h->m, part, nsplit, out, h->st);
}

static wlr_status do_init(wlr_ctx* h, const void* A, const void* W1) {
  const wlr_opts& o = h->opts;
  const size_t es = h->es;
  // ---- stream
  if (o.stream) h->st = (cudaStream_t)o.stream;
  else {
    // a BLOCKING stream: it orders behind work on the legacy default stream, so device inputs a
    // caller produced there (e.g. a torch tensor on the default stream) are complete before the
    // handle reads them.  Callers passing their own stream order inputs themselves.
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->st, cudaStreamDefault));
    h->own_stream = true;
  }
  int dev = 0;
  CUDA_TRY(h, cudaGetDevice(&dev));
  CUDA_TRY(h, cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, dev));
  {   // pinned status words, recycled across handles (cudaMallocHost costs ~1.5 ms)
    void* blk = pinned_take();
    if (!blk) return fail(h, WLR_ENOMEM, "pinned host block");
    h->h_scal = reinterpret_cast<double*>(blk);
    h->h_flags = reinterpret_cast<int*>(reinterpret_cast<char*>(blk) + 8 * sizeof(double));
  }
  wlr_status s;
  // ---- data: borrow device buffers, copy host buffers
  // The streaming kernels read A through TMA: rows must start 16-byte aligned.  A borrowed
  // device A that is not (odd n) and every host A are copied into a padded buffer.
  const bool dev_a = is_device_ptr(A);
  if (dev_a && (h->lda * es) % 16 == 0 && (uintptr_t)A % 16 == 0) {
    h->A = A;
  } else {
    const int64_t ldp = round_up(h->n, (int64_t)(16 / es));
    void* d = nullptr;
    if ((s = dalloc(h, &d, (size_t)h->m * ldp * es)) != WLR_OK) return s;
    if (ldp == h->lda)   // contiguous on both sides: one linear copy
      CUDA_TRY(h, cudaMemcpyAsync(d, A, (size_t)h->m * ldp * es,
                                  dev_a ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
    else
      CUDA_TRY(h, cudaMemcpy2DAsync(d, ldp * es, A, h->lda * es, h->n * es, h->m,
                                    dev_a ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
    h->A = d;
    h->lda = ldp;
  }
  if (W1) {
    if (is_device_ptr(W1)) h->W1 = W1;
    else {
      void* d = nullptr;
      if ((s = dalloc(h, &d, (size_t)h->m * h->k * es)) != WLR_OK) return s;
      CUDA_TRY(h, cudaMemcpy2DAsync(d, h->k * es, W1, h->ldw * es, h->k * es, h->m, cudaMemcpyHostToDevice, h->st));
      h->W1 = d;
      h->ldw = h->k;
    }
  }
  if ((s = dalloc_t(h, &h->flags, 8)) != WLR_OK) return s;   // (zeroed)
  // ---- validation on device: W1 > 0, finite data into flags[1]; read
  // back (first) at the end of the initialisation, so that the host set-up below and the init
  // Grams overlap it instead of waiting on a synchronisation here
  if (h->dtype == WLR_F32) launch_validate<float>((const float*)h->A, h->lda, h->m, (int)h->n, (const float*)h->W1, h->ldw, (int)h->k, h->flags, h->st);
  else launch_validate<double>((const double*)h->A, h->lda, h->m, (int)h->n, (const double*)h->W1, h->ldw, (int)h->k, h->flags, h->st);
  h->zero_defer = true;                        // the allocations below are zeroed by flush_zero, before
                                               // the first kernel that reads them (init_x1 below)

  // ---- sizes of the per-iteration kernels
  const int64_t k = h->k, n = h->n, nk = h->nk, t = h->t, kp = h->kp;
  h->rp = row_pass_rp((int)kp);                  // row pass output: the k (padded) columns of X1
  if (h->rp < 0 || kp > 128 || t > 32) return fail(h, WLR_EINVAL, "this build supports k <= 128 and r - k <= 32");
  h->KA = (int)round_up(n, 32);
  // Row-pass tile height BM = RS * TR: the pass is throughput-bound per SM, so pick the TR whose
  // busiest SM streams the fewest rows (ceil(tiles / SMs) * BM), with a small penalty for the
  // lower operand reuse of short tiles; ties go to the taller tile.
  {
    double best = 1e300;
    int best_tr = -1, best_cps = 1;
    for (int tr : {8, 6, 4}) {
      if (!row_pass_tr_ok(h->rp, tr)) continue;
      const size_t sm = h->dtype == WLR_F32 ? row_pass_smem<float>(h->rp, tr, h->uniform, (int)k, (int)kp)
                                            : row_pass_smem<double>(h->rp, tr, h->uniform, (int)k, (int)kp);
      const int nw = h->dtype == WLR_F32 ? row_pass_chol_warps<float>(h->rp, tr, h->uniform, (int)k, (int)kp)
                                         : row_pass_chol_warps<double>(h->rp, tr, h->uniform, (int)k, (int)kp);
      if (sm > 227 * 1024 || nw < 1) continue;
      int cps = 0;
      cudaError_t e;
      if (h->dtype == WLR_F32) {
        RowPassArgs<float> q{}; q.k = (int)k; q.kp = (int)kp; q.nwc = nw;
        e = launch_row_pass<float>(q, h->rp, tr, h->uniform, 0, 0, h->st, &cps);
      } else {
        RowPassArgs<double> q{}; q.k = (int)k; q.kp = (int)kp; q.nwc = nw;
        e = launch_row_pass<double>(q, h->rp, tr, h->uniform, 0, 0, h->st, &cps);
      }
      if (e != cudaSuccess || cps < 1) continue;
      const int bmr = row_pass_bm(h->rp, tr);
      const double cost = (double)ceil_div(ceil_div(h->m, bmr), (int64_t)h->nsm) * bmr *
                          (tr == 8 ? 1.0 : tr == 6 ? 1.03 : 1.08);
      if (cost < best) { best = cost; best_tr = tr; best_cps = cps; }
    }
    if (best_tr < 0) return fail(h, WLR_EINVAL, "row-pass shared memory exceeds 227 KB for this (k, r)");
    h->rp_tr = best_tr;
    h->nwc = h->dtype == WLR_F32 ? row_pass_chol_warps<float>(h->rp, best_tr, h->uniform, (int)k, (int)kp)
                                 : row_pass_chol_warps<double>(h->rp, best_tr, h->uniform, (int)k, (int)kp);
    // all tiles co-resident when they fit, else a persistent grid of co-resident CTAs
    const int64_t ntiles = ceil_div(h->m, row_pass_bm(h->rp, best_tr));
    h->rp_grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)h->nsm * best_cps));
  }
  h->bm = incr_bm((int)kp);
  const int bn = incr_bn(h->bm, (int)es);
  h->nz = (int)((n - h->k0) + 2 * kp);
  const int ncol = (int)ceil_div(h->nz, bn);
  int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(h->m, 128), ceil_div(4 * h->nsm, ncol)));
  h->rps = round_up(ceil_div(h->m, nsplit), 32);
  h->nsplit = (int)std::max<int64_t>(1, ceil_div(h->m, h->rps));
  // clusters of 8 row splits pre-reduce their partials through DSMEM (8x fewer for K2c)
  h->ics = h->nsplit >= 8 && incr_cluster_ok() ? 8 : 1;
  h->ncl = (int)ceil_div(h->nsplit, h->ics);
  // tensor-core increments: 128-column blocks x row splits, one wave at 2 CTAs/SM
  h->itc_kpd = incr_tc_kpd((int)kp);
  h->itc_ok = h->dtype == WLR_F32 && h->itc_kpd > 0;
  if (h->itc_ok) {
    h->itc_nA32 = (int)round_up(n - h->k0, 32);
    h->itc_nz = h->itc_nA32 + 2 * h->itc_kpd;
    const int64_t ncb = ceil_div(h->itc_nz, 128);
    const char* cps_env = getenv("WLR_ITC_CPS");    // (experiments: CTAs per SM of the split grid)
    const int cps = cps_env ? std::max(1, atoi(cps_env)) : (h->itc_kpd > 32 ? 1 : 2);   // (smem: 1 CTA/SM above 32)
    const int64_t want = std::max<int64_t>(1, (cps * h->nsm) / ncb);
    h->itc_rps = round_up(ceil_div(h->m, want), 32);
    h->itc_nsplit = (int)ceil_div(h->m, h->itc_rps);
    // (2/4/8-CTA clusters pre-reducing the partials were measured no faster: profiles/r01_v10_itc_cs.log)
  }
  // eigen block width b
  // warm block: 2 spare Ritz vectors (one product per iteration at steady state at config 3,
  // profiles/r01_v7_eigblock.log; at config 4's narrow gaps a wider block saves few filter products
  // but makes each one dearer: b = 6..11 -> 1243..1400 us per iteration, profiles/r02_eigblock.log)
  int b = o.eig_block > 0 ? o.eig_block : (int)(t + 2);
  b = (int)std::min<int64_t>(std::max<int64_t>(b, t), nk);
  if (b > 32) b = 32;
  if (b < t) return fail(h, WLR_EINVAL, "r-k > 32 is not supported by this build");
  h->b = b;
  // small-step (K3) cluster plan: depends on the dimensions only
  {
    SmallArgs pa{};
    pa.k = (int)k; pa.nk = (int)nk; pa.t = (int)t; pa.b = b; pa.uniform = h->uniform ? 1 : 0;
    if (nk > 1024) return fail(h, WLR_EINVAL, "n - k > 1024 is not supported by this build (small step: one cluster of <= 16 CTAs x 64 columns)");
    if (small_step_cluster_size(pa) <= 0)
      return fail(h, WLR_ECUDA, "no schedulable cluster configuration for the small step");
    h->spl = pa.pl;
  }

  // ---- allocations
  const int64_t wt_rows = h->KA + round_up(kp, 32);    // [A | X1_p] rows of the linear update
  if ((s = dalloc(h, &h->X[0], (size_t)h->m * kp * es)) != WLR_OK) return s;
  if ((s = dalloc(h, &h->X[1], (size_t)h->m * kp * es)) != WLR_OK) return s;
  if ((s = dalloc(h, &h->Dl, (size_t)h->m * kp * es)) != WLR_OK) return s;
  if (h->dtype == WLR_F32 && !h->uniform && row_solve_ok((int)k)) {
    if ((s = dalloc(h, &h->Ebuf, (size_t)h->m * kp * es + 64)) != WLR_OK) return s;   // (8-float over-read)
    if ((s = dalloc_t(h, &h->Sop, (size_t)k * round_up(k, (int64_t)8))) != WLR_OK) return s;
    h->rs_grid = (int)std::max<int64_t>(1, std::min<int64_t>(row_solve_grid((int)k, h->nsm), h->m));
  }
  if ((s = dalloc(h, &h->Wt, (size_t)wt_rows * h->rp * es)) != WLR_OK) return s;
  if ((s = dalloc(h, &h->Wt1, (size_t)wt_rows * h->rp * es)) != WLR_OK) return s;
  {   // TMA tensor maps: 128-byte x BM boxes (SWIZZLE_128B) of A and X1, 32-row boxes of Wt
    const uint32_t pe = (uint32_t)(128 / es), bm = (uint32_t)row_pass_bm(h->rp, h->rp_tr);
    bool ok = make_tmap_2d(&h->tmA, h->A, (int)es, (uint64_t)n, (uint64_t)h->m, (uint64_t)h->lda * es, pe, bm, true);
    for (int i = 0; i < 2; ++i)
      ok = ok && make_tmap_2d(&h->tmX[i], h->X[i], (int)es, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * es, pe, bm, true);
    ok = ok && make_tmap_2d(&h->tmW, h->Wt, (int)es, (uint64_t)h->rp, (uint64_t)wt_rows, (uint64_t)h->rp * es,
                            (uint32_t)h->rp, 32u, false);
    ok = ok && make_tmap_2d(&h->tmW1, h->Wt1, (int)es, (uint64_t)h->rp, (uint64_t)wt_rows, (uint64_t)h->rp * es,
                            (uint32_t)h->rp, 32u, false);
    if (!ok) return fail(h, WLR_ECUDA, "cuTensorMapEncodeTiled failed (TMA descriptors)");
  }
  // tensor-core row pass (uniform W1, fp32): K-major W'^T written by the small step
  // tensor-core row pass: fp32, uniform W1 (X1_{p+1} directly) or non-uniform with the per-row
  // solver (E mode: the tile result plus A1 . W1^2 goes to the e rows)
  h->tc_ok = h->dtype == WLR_F32 && (h->uniform || h->Ebuf != nullptr);
  if (const char* dbg = std::getenv("WLR_TC_DBG")) h->tc_dbg = std::atoi(dbg);
  if (h->tc_dbg & 32) {
    void* p = nullptr;
    if ((s = dalloc(h, &p, 8 * 8 * 4096)) != WLR_OK) return s;
    h->itc_tstamp = (unsigned long long*)p;
  }
  if (h->tc_dbg & 16) {
    void* p = nullptr;
    if ((s = dalloc(h, &p, 8 * 8 * 2048)) != WLR_OK) return s;
    h->tc_tstamp = (unsigned long long*)p;
  }
  if (h->tc_ok) {
    h->KW = (int)wt_rows;
    if ((s = dalloc(h, &h->WtT, (size_t)2 * h->rp * wt_rows * es)) != WLR_OK) return s;   // W'^T | W'^T_lo
    if ((s = dalloc(h, &h->WtT1, (size_t)2 * h->rp * wt_rows * es)) != WLR_OK) return s;
    bool ok = make_tmap_2d(&h->tmA_tc, h->A, 4, (uint64_t)n, (uint64_t)h->m, (uint64_t)h->lda * 4, 32u, (uint32_t)kTcBM, true);
    for (int i = 0; i < 2; ++i)
      ok = ok && make_tmap_2d(&h->tmX_tc[i], h->X[i], 4, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * 4, 32u, (uint32_t)kTcBM, true);
    ok = ok && make_tmap_2d(&h->tmWT, h->WtT, 4, (uint64_t)wt_rows, (uint64_t)(2 * h->rp), (uint64_t)wt_rows * 4, 32u, (uint32_t)h->rp, true);
    ok = ok && make_tmap_2d(&h->tmWT1, h->WtT1, 4, (uint64_t)wt_rows, (uint64_t)(2 * h->rp), (uint64_t)wt_rows * 4, 32u, (uint32_t)h->rp, true);
    int occ = 0;
    RowPassTcArgs q{};
    if (ok && launch_row_pass_tc(q, h->rp, 0, h->st, &occ) == cudaSuccess && occ > 0) {
      occ = std::max(occ, row_pass_tc_ctas_per_sm(h->rp));   // shared-memory bound (carveout 100)
      const int64_t ntiles = ceil_div(h->m, kTcBM);
      h->tc_m_main = h->m;
      h->tc_extra = 0;
      h->tc_deep = false;
      const int tcmode = std::getenv("WLR_TC_MODE") ? std::atoi(std::getenv("WLR_TC_MODE")) : -1;   // (A/B)
      if (tcmode == 0) {
        h->tc_grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)h->nsm * occ));
      } else if (row_pass_tc_deep_ok(h->rp) && ntiles <= h->nsm) {
        // one tile per CTA, one CTA per SM: the 8-stage ring
        h->tc_deep = true;
        h->tc_grid = (int)ntiles;
      } else if (row_pass_tc_deep_ok(h->rp) && h->rp <= 32 && h->uniform && h->m <= (int64_t)h->nsm * (kTcBM + 4) &&
                 make_tmap_2d(&h->tmA_x, h->A, 4, (uint64_t)n, (uint64_t)h->m, (uint64_t)h->lda * 4, 32u, 4u, false) &&
                 make_tmap_2d(&h->tmX_x[0], h->X[0], 4, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * 4, 32u, 4u, false) &&
                 make_tmap_2d(&h->tmX_x[1], h->X[1], 4, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * 4, 32u, 4u, false)) {
        // slightly more rows than one tile per SM (config 3: 150 tiles, 148 SMs): every SM takes
        // one tile plus <= 4 leftover rows on the CUDA cores, instead of a second wave for 2 tiles
        h->tc_deep = true;
        h->tc_grid = h->nsm;
        h->tc_m_main = (int64_t)h->nsm * kTcBM;
        h->tc_extra = (int)ceil_div(h->m - h->tc_m_main, (int64_t)h->nsm);
      } else {
        h->tc_grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)h->nsm * occ));
      }
      h->tc_on = true;
    } else {
      h->tc_ok = false;
    }
  }
  if (h->itc_ok) {   // 32 x 32 boxes of A, X1 (per buffer) and Delta for the tensor-core increments
    bool ok = make_tmap_2d(&h->tmA32, h->A, 4, (uint64_t)n, (uint64_t)h->m, (uint64_t)h->lda * 4, 32u, 32u, true);
    for (int i = 0; i < 2; ++i)
      ok = ok && make_tmap_2d(&h->tmX32[i], h->X[i], 4, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * 4, 32u, 32u, true);
    ok = ok && make_tmap_2d(&h->tmD32, h->Dl, 4, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * 4, 32u, 32u, true);
    h->itc_ok = h->itc_on = ok;
  }
  if ((s = dalloc(h, &h->CVop, (size_t)std::max<int64_t>(k * t, 1) * es)) != WLR_OK) return s;
  if ((s = dalloc(h, &h->Kop, (size_t)k * k * es)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->inc_part, std::max((size_t)h->nsplit * k * h->nz,
                                                (size_t)h->itc_nsplit * k * h->itc_nz))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->inc_part2, (size_t)h->ncl * k * h->nz)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->fw_part, (size_t)std::max({h->rp_grid, h->rs_grid, h->tc_grid, 1184}))) != WLR_OK) return s;
  for (int i = 0; i < 2; ++i)
    if ((s = dalloc_t(h, &h->inc[i], (size_t)(k * nk + 2 * k * k + 1))) != WLR_OK) return s;
  {   // Gram propagation for the linear (uniform-W1) X1 half-step (prop.cu; WLR_PROP=0 disables, A/B)
    const char* pe = std::getenv("WLR_PROP");
    if (const char* ke = std::getenv("WLR_K3B_EARLY")) h->k3b_early = std::atoi(ke) != 0;
    // prop1 runs one CTA per SM; K3b(p-1) and the shadow K3a start beside it at the iteration start,
    // each a cluster of CL whole SMs, so prop1 leaves them room (WLR_PROP_RSV: SMs left out, A/B)
    const char* se = std::getenv("WLR_SHADOW");
    const bool want_shadow = !se || std::atoi(se) != 0;
    int rsv = (want_shadow ? 2 : 1) * h->spl.CL;
    if (const char* re = std::getenv("WLR_PROP_RSV")) rsv = std::atoi(re);
    h->prop_nsm = std::max(1, h->nsm - std::max(0, rsv));
    auto prop_fits = [&](int nsm) {
      return prop1_smem((int)n, (int)k, nsm, h->b) <= 227 * 1024 && prop1_rb((int)n, nsm) <= 8;
    };
    if (!prop_fits(h->prop_nsm)) h->prop_nsm = h->nsm;
    h->prop = h->uniform && h->dtype == WLR_F32 && (!pe || std::atoi(pe) != 0) && prop_fits(h->prop_nsm) &&
              16 * k * k <= 200 * 1024;
    h->prop_nb = (int)std::min<int64_t>(n, h->prop_nsm);
  }
  if (h->prop) {
    for (int i = 0; i < 2; ++i)
      if ((s = dalloc_t(h, &h->Qg[i], (size_t)n * k)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->Hs, prop_part_doubles(h->prop_nb, (int)k))) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->dgs, (size_t)k)) != WLR_OK) return s;
    if (const char* pt = std::getenv("WLR_PROP_TS"); pt && std::atoi(pt)) {
      void* q = nullptr;
      if ((s = dalloc(h, &q, (size_t)8 * 8 * (h->prop_nb + 3 * k))) != WLR_OK) return s;
      h->prop_ts = (unsigned long long*)q;
    }
    for (int i = 0; i < 2; ++i)
      if ((s = dalloc_t(h, &h->GAY[i], (size_t)nk * 32)) != WLR_OK) return s;   // (n-k) x b, b <= 32
  }
  if ((s = dalloc_t(h, &h->fw0, 2)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->GA, (size_t)nk * nk)) != WLR_OK) return s;
  for (int i = 0; i < 3; ++i) {
    if ((s = dalloc_t(h, &h->G[i], (size_t)k * k)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->M[i], (size_t)k * nk)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->C[i], (size_t)k * nk)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->Gi[i], (size_t)k * k)) != WLR_OK) return s;
  }
  if ((s = dalloc_t(h, &h->Ki, (size_t)k * k)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->gws, (size_t)std::max<int64_t>(1, h->spl.CL * h->spl.gws_stride))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->gws2, (size_t)std::max<int64_t>(1, h->spl.CL * h->spl.gws_stride))) != WLR_OK) return s;
  for (int i = 0; i < 3; ++i) {
    if ((s = dalloc_t(h, &h->V[i], (size_t)nk * t)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->CV[i], (size_t)k * t)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->th[i], 32)) != WLR_OK) return s;
  }
  for (int i = 0; i < 2; ++i)
    if ((s = dalloc_t(h, &h->k3x[i], (size_t)2 * t * t + 8)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->Y, (size_t)nk * b)) != WLR_OK) return s;
  {
    int lo = 0, hi = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st2, cudaStreamNonBlocking, hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st3, cudaStreamNonBlocking, lo));   // row pass branch
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_f3, cudaEventDisableTiming));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_j3, cudaEventDisableTiming));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st4, cudaStreamNonBlocking, hi));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_j4, cudaEventDisableTiming));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  }
  if ((s = dalloc_t(h, &h->xchg, (size_t)h->spl.CL * h->spl.flen)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->xchg2, (size_t)h->spl.CL * h->spl.flen)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->red, (size_t)h->spl.flen + 3 * k * t + 64)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->scal, 8)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &h->tdbg, 256)) != WLR_OK) return s;   // K3a marks, K3b marks, exchange stamps
  if ((s = dalloc_t(h, &h->trace, (size_t)h->trace_cap * 4)) != WLR_OK) return s;
  if (h->prop) {   // shadow K3a buffers (same shapes as the real outputs)
    const char* se = std::getenv("WLR_SHADOW");
    h->shadow = !se || std::atoi(se) != 0;
  }
  if (h->shadow) {
    const int64_t wt_rows = h->KA + round_up(kp, 32);
    if ((s = dalloc_t(h, &h->sh_G, (size_t)k * k)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_M, (size_t)k * nk)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_C, (size_t)k * nk)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_V, (size_t)nk * t)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_CV, (size_t)k * t)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_th, 32)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_k3x, (size_t)2 * t * t + 8)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_Gi, (size_t)k * k)) != WLR_OK) return s;
    for (int i = 0; i < 2; ++i) {
      if ((s = dalloc_t(h, &h->snapY[i], (size_t)nk * b)) != WLR_OK) return s;
      if ((s = dalloc_t(h, &h->snapKi[i], (size_t)k * k)) != WLR_OK) return s;
    }
    if ((s = dalloc_t(h, &h->sh_gws, (size_t)std::max<int64_t>(1, h->spl.CL * h->spl.gws_stride))) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_xchg, (size_t)h->spl.CL * h->spl.flen)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_red, (size_t)h->spl.flen + 3 * k * t + 64)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_scal, 8)) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_trace, (size_t)h->trace_cap * 4)) != WLR_OK) return s;
    if ((s = dalloc(h, &h->sh_Wt, (size_t)wt_rows * h->rp * h->es)) != WLR_OK) return s;
    if ((s = dalloc(h, &h->sh_WtT, (size_t)2 * h->rp * wt_rows * h->es)) != WLR_OK) return s;
    if ((s = dalloc(h, &h->sh_CVop, (size_t)std::max<int64_t>(k * t, 1) * h->es)) != WLR_OK) return s;
    if ((s = dalloc(h, &h->sh_Kop, (size_t)k * k * h->es)) != WLR_OK) return s;
    if (h->Sop && (s = dalloc_t(h, &h->sh_Sop, (size_t)k * round_up(k, (int64_t)8))) != WLR_OK) return s;
    if ((s = dalloc_t(h, &h->sh_flags, 8)) != WLR_OK) return s;
    int lo = 0, hi = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st5, cudaStreamNonBlocking, hi));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_j5, cudaEventDisableTiming));
  }

  // ---- NCCL communicator (rows sharded over ranks), or the virtual group (one GPU, test hook)
  if (o.vgroup) {
    h->vg = reinterpret_cast<wlr_vgroup_s*>(o.vgroup);
    if (h->vg->G != o.nranks) return fail(h, WLR_EINVAL, "opts.nranks must equal the virtual group's size");
  } else if (o.nranks > 1 || o.nccl_id) {   // (nranks = 1 with an id: a one-rank communicator, test hook)
    if (!o.nccl_id) return fail(h, WLR_EINVAL, "nranks > 1 needs opts.nccl_id");
    std::string e;
    if (!g_nccl.load(e)) return fail(h, WLR_ENCCL, e);
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_id, sizeof(id));
    ncclResult_t nr = g_nccl.commInitRank(&h->comm, o.nranks, id, o.rank);
    if (nr != ncclSuccess) return fail(h, WLR_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.errStr(nr));
  }

  // ---- one-time Grams in fp64 (a0/a1): A^T A (or X1_0^T [X1_0 | A2] and A2^T A2)
  // row splits: enough CTAs (tiles x splits) for several per SM -- the tiles are latency-bound
  const int gsplit = (int)std::max<int64_t>(1, std::min<int64_t>(24, ceil_div(h->m, 1024)));
  double* part = nullptr;
  double* gram = nullptr;
  if ((s = dalloc_t(h, &part, (size_t)gsplit * n * n)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &gram, (size_t)n * n)) != WLR_OK) return s;
  const char* A2 = (const char*)h->A + k * es;
  if ((s = flush_zero(h)) != WLR_OK) return s;
  if (h->dtype == WLR_F32) {
    if (o.init == WLR_INIT_GIVEN) launch_init_x1<float>((const float*)h->opts.x1_0, k, h->m, (int)k, (int)kp, (float*)h->X[0], h->st);
    else launch_init_x1<float>((const float*)h->A, h->lda, h->m, (int)k, (int)kp, (float*)h->X[0], h->st);
  } else {
    if (o.init == WLR_INIT_GIVEN) launch_init_x1<double>((const double*)h->opts.x1_0, k, h->m, (int)k, (int)kp, (double*)h->X[0], h->st);
    else launch_init_x1<double>((const double*)h->A, h->lda, h->m, (int)k, (int)kp, (double*)h->X[0], h->st);
  }
  auto run_gram = [&](const void* L, int64_t ldl, int nl, const void* R, int64_t ldr, int nr, double* out) {
    if (h->dtype == WLR_F32) gram_launch<float>(h, L, ldl, nl, R, ldr, nr, part, gsplit, out);
    else gram_launch<double>(h, L, ldl, nl, R, ldr, nr, part, gsplit, out);
  };
  // gram buffer layout: n x n; for INIT_GIVEN rows [0,k) are X1_0^T [X1_0 | A2]
  if (o.init == WLR_INIT_GIVEN) {
    double* tmp = nullptr;
    if ((s = dalloc_t(h, &tmp, (size_t)k * n)) != WLR_OK) return s;
    run_gram(h->X[0], kp, (int)k, h->X[0], kp, (int)k, tmp);                 // k x k
    CUDA_TRY(h, cudaMemcpy2DAsync(gram, n * 8, tmp, k * 8, k * 8, k, cudaMemcpyDeviceToDevice, h->st));
    run_gram(h->X[0], kp, (int)k, A2, h->lda, (int)nk, tmp);                 // k x nk
    CUDA_TRY(h, cudaMemcpy2DAsync(gram + k, n * 8, tmp, nk * 8, nk * 8, k, cudaMemcpyDeviceToDevice, h->st));
    run_gram(A2, h->lda, (int)nk, A2, h->lda, (int)nk, h->GA);               // nk x nk
    if (h->prop) {   // the full A^T A and Q_0 = A^T X1_0 for the propagation
      if ((s = dalloc_t(h, &h->AtA, (size_t)n * n)) != WLR_OK) return s;
      run_gram(h->A, h->lda, (int)n, h->A, h->lda, (int)n, h->AtA);
      run_gram(h->A, h->lda, (int)n, h->X[0], kp, (int)k, h->Qg[0]);
    }
  } else {
    run_gram(h->A, h->lda, (int)n, h->A, h->lda, (int)n, gram);
    h->AtA = gram;
  }
  // sum the per-rank Grams (rows are sharded, Grams are additive over rows)
  if ((s = group_allreduce(h, gram, (size_t)n * n, h->st, "init gram")) != WLR_OK) return s;
  if (o.init == WLR_INIT_GIVEN) {
    if ((s = group_allreduce(h, h->GA, (size_t)nk * nk, h->st, "init GA")) != WLR_OK) return s;
    if (h->prop) {
      if ((s = group_allreduce(h, h->AtA, (size_t)n * n, h->st, "init A^T A")) != WLR_OK) return s;
      if ((s = group_allreduce(h, h->Qg[0], (size_t)n * k, h->st, "init Q_0")) != WLR_OK) return s;
    }
  }
  CUDA_TRY(h, cudaMemcpy2DAsync(h->G[0], k * 8, gram, n * 8, k * 8, k, cudaMemcpyDeviceToDevice, h->st));
  CUDA_TRY(h, cudaMemcpy2DAsync(h->M[0], nk * 8, gram + k, n * 8, nk * 8, k, cudaMemcpyDeviceToDevice, h->st));
  if (o.init != WLR_INIT_GIVEN)
    CUDA_TRY(h, cudaMemcpy2DAsync(h->GA, nk * 8, gram + k * n + k, n * 8, nk * 8, nk, cudaMemcpyDeviceToDevice, h->st));
  if (h->prop && o.init != WLR_INIT_GIVEN)   // X1_0 = A1: Q_0 = A^T A1, the first k columns of A^T A
    CUDA_TRY(h, cudaMemcpy2DAsync(h->Qg[0], k * 8, h->AtA, n * 8, k * 8, n, cudaMemcpyDeviceToDevice, h->st));
  if (h->prop) {   // ||A1||_F^2 = tr(A^T A)(0:k, 0:k)
    std::vector<double> diag(k);
    CUDA_TRY(h, cudaMemcpy2DAsync(diag.data(), 8, h->AtA, (n + 1) * 8, 8, k, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    double a1 = 0.0;
    for (double v : diag) a1 += v;
    h->a1sq = a1;
  }
  // ||A2||_F^2 = tr(G_A)
  {
    std::vector<double> diag(nk);
    CUDA_TRY(h, cudaMemcpy2DAsync(diag.data(), 8, h->GA, (nk + 1) * 8, 8, nk, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    double a2 = 0.0;
    for (double v : diag) a2 += v;
    h->a2sq = a2;
  }
  // f_w(X1_0): 0 for the GHS start, otherwise computed
  if (o.init == WLR_INIT_GIVEN) {
    if (h->dtype == WLR_F32) launch_fw<float>((const float*)h->A, h->lda, (const float*)h->W1, h->ldw, h->w1s * h->w1s, (const float*)h->X[0], (int)kp, h->m, (int)k, h->fw_part, 1184, h->st);
    else launch_fw<double>((const double*)h->A, h->lda, (const double*)h->W1, h->ldw, h->w1s * h->w1s, (const double*)h->X[0], (int)kp, h->m, (int)k, h->fw_part, 1184, h->st);
    launch_reduce_incr(h->inc_part, 0, 0, 0, 1, 0, 0, 0, h->fw_part, 1184, h->fw0, h->st);
    if ((s = group_allreduce(h, h->fw0, 1, h->st, "fw0")) != WLR_OK) return s;
  }
  // cold-start block of the eigensolver: deterministic host PRNG (identical on all ranks)
  {
    std::vector<double> y((size_t)nk * b);
    uint64_t st = 0x5eed0000ull + (uint64_t)(uint32_t)o.seed;
    for (auto& v : y) v = (double)(splitmix(st) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    CUDA_TRY(h, cudaMemcpyAsync(h->Y, y.data(), y.size() * 8, cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
  }
  // small step configuration
  // initial (C, D) half-step: outputs into state slot 0 (phase 5 maps out -> 0)
  SmallArgs sa = small_args(h, 5, 0);
  sa.G_in = nullptr; sa.M_in = nullptr; sa.C_in = nullptr; sa.Gi_in = nullptr;
  sa.V_in = nullptr; sa.CV_in = nullptr; sa.th_in = nullptr;
  sa.G_out = h->G[0]; sa.M_out = h->M[0];        // mode 0 reads the init Grams from here
  sa.max_outer = 4 * o.eig_max_outer; sa.cold = 1;
  sa.tdbg = h->tdbg;
  cudaError_t e = launch_small_step(sa, 1, h->st);
  if (e == cudaSuccess) e = launch_deferred(h, sa, h->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->flags + 7, 1, 1, h->st);   // (no deferred half pending)
  if (e != cudaSuccess) return fail(h, WLR_ECUDA, std::string("small step (init): ") + cudaGetErrorString(e));
  h->pr.launches = 0;
  CUDA_TRY(h, cudaMemcpyAsync(h->h_flags, h->flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  if (h->h_flags[1] & 2) return fail(h, WLR_ENONFINITE, "non-finite entry in A or W1");
  if (h->h_flags[1] & 1) return fail(h, WLR_EINVAL, "W1 must be > 0 (PAPER.md:94)");
  s = check_flags(h);
  if (s != WLR_OK) return s;
  h->p = 0;
  h->ph = 0;
  return build_all_graphs(h);
}

extern "C" wlr_status wlr_init(wlr_handle* out, const void* A, int64_t lda, const void* W1,
                               int64_t ldw, int64_t m_local, int64_t n, int64_t k, int64_t r,
                               const wlr_opts* o) {
  if (!out) return fail(nullptr, WLR_EINVAL, "null handle pointer");
  *out = nullptr;
  wlr_opts def;
  wlr_opts_default(&def);
  const wlr_opts& op = o ? *o : def;
  if (!A) return fail(nullptr, WLR_EINVAL, "A is null");
  if (m_local < 1 || n < 2) return fail(nullptr, WLR_EINVAL, "need m >= 1, n >= 2");
  if (k < 1 || k >= n) return fail(nullptr, WLR_EINVAL, "need 1 <= k < n");
  const int64_t mg = op.m_global > 0 ? op.m_global : m_local;
  if (r <= k) return fail(nullptr, WLR_EINVAL, "need r > k (Theorem 2, PAPER.md:94)");
  if (r > std::min(mg, n)) return fail(nullptr, WLR_EINVAL, "need r <= min(m, n)");
  if (lda < n) return fail(nullptr, WLR_EINVAL, "lda < n");
  if (W1 && ldw < k) return fail(nullptr, WLR_EINVAL, "ldw < k");
  if (!W1 && !(op.w1_scalar > 0.0)) return fail(nullptr, WLR_EINVAL, "uniform weight must be > 0");
  if (op.dtype != WLR_F32 && op.dtype != WLR_F64) return fail(nullptr, WLR_EINVAL, "bad dtype");
  if (op.init == WLR_INIT_GIVEN && !op.x1_0) return fail(nullptr, WLR_EINVAL, "INIT_GIVEN needs x1_0");
  if (op.nranks < 1 || op.rank < 0 || op.rank >= op.nranks) return fail(nullptr, WLR_EINVAL, "bad rank");
  if (m_local < k && op.nranks == 1) return fail(nullptr, WLR_EINVAL, "need m >= k");
  wlr_ctx* h = new wlr_ctx();
  h->opts = op;
  if (op.vgroup) h->opts.use_graph = 0;      // (cross-member event waits cannot be captured)
  // eigensolver target (relative to lambda_1; the S-product rounding floor is added in K3):
  // fp64 mode 1e-12, fp32 mode 1e-7 (DESIGN.md §3 reading R17 "eigensolver tolerance")
  if (h->opts.eig_tol <= 0.0) h->opts.eig_tol = op.dtype == WLR_F64 ? 1e-12 : 1e-7;
  if (h->opts.eig_max_outer <= 0) h->opts.eig_max_outer = 60;
  h->m = m_local; h->n = n; h->k = k; h->r = r; h->t = r - k; h->nk = n - k;
  h->kp = round_up(k, 4); h->k0 = k & ~3LL;
  h->m_global = mg; h->row_offset = op.row_offset;
  h->dtype = op.dtype; h->es = op.dtype == WLR_F64 ? 8 : 4;
  h->uniform = W1 == nullptr; h->w1s = op.w1_scalar;
  h->A = A; h->lda = lda; h->W1 = W1; h->ldw = ldw;
  if (op.init == WLR_INIT_GIVEN && !is_device_ptr(op.x1_0)) {
    void* d = nullptr;
    if (cudaMalloc(&d, (size_t)m_local * k * h->es) != cudaSuccess) { delete h; return fail(nullptr, WLR_ENOMEM, "x1_0 copy"); }
    h->allocs.push_back(d);
    cudaMemcpy(d, op.x1_0, (size_t)m_local * k * h->es, cudaMemcpyHostToDevice);
    h->opts.x1_0 = d;
  }
  wlr_status s = do_init(h, A, W1);
  if (s != WLR_OK) {
    g_err = h->err;
    wlr_destroy(h);
    return s;
  }
  *out = h;
  return WLR_OK;
}

// --------------------------------------------------------------------------- iterate
extern "C" wlr_status wlr_iterate_async(wlr_handle h, int32_t n_iters) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  for (int32_t i = 0; i < n_iters; ++i) {
    wlr_status s = launch_iteration(h);
    if (s != WLR_OK) return s;
  }
  return WLR_OK;
}

extern "C" wlr_status wlr_sync(wlr_handle h) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  return check_flags(h);
}

extern "C" wlr_status wlr_iterate(wlr_handle h, int32_t max_iters, int32_t* iters_done,
                                  int32_t* converged) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  if (max_iters < 0) return fail(h, WLR_EINVAL, "max_iters < 0");
  const int64_t p0 = h->p;
  wlr_status s = WLR_OK;
  int done = 0;
  // eps mode: the stopping rule is applied on the device (kernels of every iteration after the
  // converged state skip their work), so the host only checks every check_every iterations
  const int chunk = h->opts.eps > 0.0 ? (h->opts.check_every > 0 ? h->opts.check_every : 8) : 64;
  while (done < max_iters) {
    const int n = std::min(chunk, max_iters - done);
    s = wlr_iterate_async(h, n);
    if (s != WLR_OK) break;
    done += n;
    s = check_flags(h);
    if (s != WLR_OK) break;
    if (h->h_flags[2]) break;
  }
  if (iters_done) *iters_done = (int32_t)(h->p - p0);
  if (converged) *converged = h->h_flags[2] ? 1 : 0;
  return s;
}

extern "C" wlr_status wlr_objective(wlr_handle h, double* F, double* step_norm, double* rel_error) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  wlr_status s = check_flags(h);
  if (s != WLR_OK) return s;
  if (F) *F = h->h_scal[2];
  if (step_norm) *step_norm = h->h_scal[3];
  if (rel_error) *rel_error = h->h_scal[4];
  return WLR_OK;
}

extern "C" wlr_status wlr_trace(wlr_handle h, double* out, int32_t cap, int32_t* count) {
  if (!h || !out) return fail(h, WLR_EINVAL, "null argument");
  wlr_status s = check_flags(h);
  if (s != WLR_OK) return s;
  std::vector<double> all((size_t)h->trace_cap * 4);
  CUDA_TRY(h, cudaMemcpy(all.data(), h->trace, all.size() * 8, cudaMemcpyDeviceToHost));
  const int64_t nstates = h->p + 1;
  const int64_t avail = std::min<int64_t>(nstates, h->trace_cap);
  const int64_t nout = std::min<int64_t>(avail, cap);
  const int64_t first = nstates - nout;
  for (int64_t i = 0; i < nout; ++i) {
    const int64_t q = (first + i) % h->trace_cap;
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = all[q * 4 + j];
  }
  if (count) *count = (int32_t)nout;
  return WLR_OK;
}

// copy a device buffer (rows x cols, ld_src) into dst (host or device, ld_dst)
static wlr_status copy_out(wlr_ctx* h, void* dst, int64_t ldd, const void* src, int64_t lds,
                           int64_t rows, int64_t cols, size_t es) {
  const bool dev = is_device_ptr(dst);
  CUDA_TRY(h, cudaMemcpy2DAsync(dst, ldd * es, src, lds * es, cols * es, rows,
                                dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
  return WLR_OK;
}

extern "C" wlr_status wlr_result(wlr_handle h, void* X1, int64_t ldx1, void* C, void* B,
                                 int64_t ldb, void* D, void* X2, int64_t ldx2) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  wlr_status s = check_flags(h);
  if (s != WLR_OK) return s;
  const int cx = h->ph & 1, cur = h->ph % 3;   // X1 buffer, state slot
  const size_t es = h->es;
  if (X1) {
    if (ldx1 < h->k) return fail(h, WLR_EINVAL, "ldx1 < k");
    if ((s = copy_out(h, X1, ldx1, h->X[cx], h->kp, h->m, h->k, es)) != WLR_OK) return s;
  }
  if (C) {
    if ((s = copy_out(h, C, h->nk, h->C[cur], h->nk, h->k, h->nk, 8)) != WLR_OK) return s;
  }
  if (D) {
    std::vector<double> v((size_t)h->nk * h->t), d((size_t)h->nk * h->t);
    CUDA_TRY(h, cudaMemcpyAsync(v.data(), h->V[cur], v.size() * 8, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    for (int64_t c = 0; c < h->nk; ++c)
      for (int64_t j = 0; j < h->t; ++j) d[j * h->nk + c] = v[c * h->t + j];
    if (is_device_ptr(D)) CUDA_TRY(h, cudaMemcpy(D, d.data(), d.size() * 8, cudaMemcpyHostToDevice));
    else std::memcpy(D, d.data(), d.size() * 8);
  }
  if (B || X2) {
    void* Bd = nullptr;
    CUDA_TRY(h, cudaMallocAsync(&Bd, (size_t)h->m * h->t * es + 16, h->st));
    // B = A2 V - X1 (C V) as the same streaming GEMM: Wb = [0; V; -C V]  (host-built, small)
    const int rpb = row_pass_rp((int)h->t);
    const int64_t wrows = h->KA + round_up(h->kp, 32);
    std::vector<double> v((size_t)h->nk * h->t), cv((size_t)h->k * h->t);
    CUDA_TRY(h, cudaMemcpyAsync(v.data(), h->V[cur], v.size() * 8, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(h, cudaMemcpyAsync(cv.data(), h->CV[cur], cv.size() * 8, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    std::vector<double> wb((size_t)wrows * rpb, 0.0);
    for (int64_t c = 0; c < h->nk; ++c)
      for (int64_t j = 0; j < h->t; ++j) wb[(size_t)(h->k + c) * rpb + j] = v[(size_t)c * h->t + j];
    for (int64_t q = 0; q < h->k; ++q)
      for (int64_t j = 0; j < h->t; ++j) wb[(size_t)(h->KA + q) * rpb + j] = -cv[(size_t)q * h->t + j];
    void* Wbd = nullptr;
    CUDA_TRY(h, cudaMallocAsync(&Wbd, wb.size() * es, h->st));
    if (h->dtype == WLR_F32) {
      std::vector<float> wf(wb.begin(), wb.end());
      CUDA_TRY(h, cudaMemcpy(Wbd, wf.data(), wf.size() * 4, cudaMemcpyHostToDevice));
    } else {
      CUDA_TRY(h, cudaMemcpy(Wbd, wb.data(), wb.size() * 8, cudaMemcpyHostToDevice));
    }
    // the result pass runs with TR = 8: its own A / X1 boxes (BM rows) and the Wb map
    CUtensorMap tmB{}, tmAr{}, tmXr{};
    const uint32_t pe = (uint32_t)(128 / es), bmr = (uint32_t)row_pass_bm(rpb, 8);
    if (!make_tmap_2d(&tmB, Wbd, (int)es, (uint64_t)rpb, (uint64_t)wrows, (uint64_t)rpb * es, (uint32_t)rpb, 32u, false) ||
        !make_tmap_2d(&tmAr, h->A, (int)es, (uint64_t)h->n, (uint64_t)h->m, (uint64_t)h->lda * es, pe, bmr, true) ||
        !make_tmap_2d(&tmXr, h->X[cx], (int)es, (uint64_t)h->kp, (uint64_t)h->m, (uint64_t)h->kp * es, pe, bmr, true)) {
      cudaFreeAsync(Wbd, h->st); cudaFreeAsync(Bd, h->st);
      return fail(h, WLR_ECUDA, "cuTensorMapEncodeTiled failed (result)");
    }
    cudaError_t e;
    if (h->dtype == WLR_F32) {
      RowPassArgs<float> a{};
      a.tmA = tmAr; a.tmX = tmXr; a.tmW = tmB;
      a.A = (const float*)h->A; a.lda = h->lda; a.W1 = (const float*)h->W1; a.ldw = h->ldw;
      a.Xold = (const float*)h->X[cx]; a.nwc = h->nwc;
      a.Wt = (const float*)Wbd; a.KA = h->KA;
      a.Bout = (float*)Bd; a.ldb = h->t; a.fw_part = h->fw_part; a.flags = h->flags;
      a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->t;
      a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
      e = launch_row_pass<float>(a, rpb, 8, true, 1, h->rp_grid, h->st);
    } else {
      RowPassArgs<double> a{};
      a.tmA = tmAr; a.tmX = tmXr; a.tmW = tmB;
      a.A = (const double*)h->A; a.lda = h->lda; a.W1 = (const double*)h->W1; a.ldw = h->ldw;
      a.Xold = (const double*)h->X[cx]; a.nwc = h->nwc;
      a.Wt = (const double*)Wbd; a.KA = h->KA;
      a.Bout = (double*)Bd; a.ldb = h->t; a.fw_part = h->fw_part; a.flags = h->flags;
      a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->t;
      a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
      e = launch_row_pass<double>(a, rpb, 8, true, 1, h->rp_grid, h->st);
    }
    cudaStreamSynchronize(h->st);
    cudaFreeAsync(Wbd, h->st);
    if (e != cudaSuccess) { cudaFreeAsync(Bd, h->st); return fail(h, WLR_ECUDA, std::string("result row pass: ") + cudaGetErrorString(e)); }
    if (B) {
      if (ldb < h->t) { cudaFreeAsync(Bd, h->st); return fail(h, WLR_EINVAL, "ldb < r-k"); }
      if ((s = copy_out(h, B, ldb, Bd, h->t, h->m, h->t, es)) != WLR_OK) { cudaFreeAsync(Bd, h->st); return s; }
    }
    if (X2) {
      if (ldx2 < h->nk) { cudaFreeAsync(Bd, h->st); return fail(h, WLR_EINVAL, "ldx2 < n-k"); }
      void* X2d = nullptr;
      const bool dev = is_device_ptr(X2);
      if (dev) X2d = X2;
      else if (cudaMallocAsync(&X2d, (size_t)h->m * h->nk * es, h->st) != cudaSuccess) { cudaFreeAsync(Bd, h->st); return fail(h, WLR_ENOMEM, "X2 staging"); }
      const int64_t ldo = dev ? ldx2 : h->nk;
      if (h->dtype == WLR_F32)
        launch_assemble_x2<float>((const float*)h->X[cx], (int)h->kp, (const float*)Bd, h->t, h->C[cur], h->V[cur], h->m, (int)h->k, (int)h->nk, (int)h->t, (float*)X2d, ldo, h->st);
      else
        launch_assemble_x2<double>((const double*)h->X[cx], (int)h->kp, (const double*)Bd, h->t, h->C[cur], h->V[cur], h->m, (int)h->k, (int)h->nk, (int)h->t, (double*)X2d, ldo, h->st);
      if (!dev) {
        s = copy_out(h, X2, ldx2, X2d, h->nk, h->m, h->nk, es);
        cudaStreamSynchronize(h->st);
        cudaFreeAsync(X2d, h->st);
        if (s != WLR_OK) { cudaFreeAsync(Bd, h->st); return s; }
      }
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    cudaFreeAsync(Bd, h->st);
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  return WLR_OK;
}

// ------------------------------------------------------------------ f3: one-sweep block ALS
// SURVEY.md §8(f3), R21.  Per sweep: W'' (als_w) -> X1 row map over [A | B_p] (the
// sWLR row pass / per-row solves) -> Grams X1'^T [A2 | B_p | X1'] (increment kernel with
// Delta := X1') -> C step + B map (als_c) -> B' = [A | X1'] Wb (result-mode row pass) -> Grams
// B'^T [A2 | X1' | B'] -> D step + objective (als_d).
template <typename T>
static cudaError_t als_row_x1(wlr_ctx* h, AlsSt* st) {
  const int x = st->x, nx = x ^ 1;
  RowPassArgs<T> a{};
  a.A = (const T*)h->A; a.lda = h->lda; a.W1 = (const T*)h->W1; a.ldw = h->ldw;
  a.w2s = (T)(h->w1s * h->w1s);
  a.Xold = (const T*)st->B; a.Xnew = (T*)h->X[nx]; a.Dnew = (T*)h->Dl; a.nwc = h->nwc;
  a.Wt = (const T*)h->Wt; a.KA = h->KA; a.Kmat = (const T*)h->Kop;
  a.tmA = h->tmA; a.tmX = st->tmBx; a.tmW = h->tmW;
  a.fw_part = h->fw_part; a.flags = h->flags;
  a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->kp;
  a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
  if constexpr (sizeof(T) == 4) a.Ebuf = (T*)h->Ebuf;
  cudaError_t e = launch_row_pass<T>(a, h->rp, h->rp_tr, h->uniform, 0, h->rp_grid, h->st);
  if constexpr (sizeof(T) == 4) {
    if (e == cudaSuccess && h->Ebuf) {
      RowSolveArgs q{};
      q.E = (const float*)h->Ebuf; q.S = h->Sop;
      q.W1 = (const float*)h->W1; q.ldw = h->ldw; q.A = (const float*)h->A; q.lda = h->lda;
      q.Xold = (const float*)a.Xold; q.Xnew = (float*)a.Xnew; q.Dnew = (float*)a.Dnew; q.fw_part = h->fw_part;
      q.flags = h->flags; q.m = h->m; q.k = (int)h->k; q.kp = (int)h->kp;
      e = launch_row_solve(q, h->rs_grid, h->st);
    }
  }
  return e;
}

// Grams D^T [A(:, k0:n) | Xo | D] of a kp-wide D (rows l < kd) into inc = [D^T A2 | D^T Xo (gk) |
// D^T D | f_w]
template <typename T>
static cudaError_t als_grams(wlr_ctx* h, const void* Xo, const void* Dd, int kd, int gk, double* inc) {
  IncrArgs<T> a{};
  a.A = (const T*)h->A; a.lda = h->lda;
  a.Xold = (const T*)Xo; a.Dnew = (const T*)Dd;
  a.part = h->inc_part; a.part2 = h->inc_part2; a.cs = h->ics; a.m = h->m; a.rows_per_split = h->rps;
  a.n = (int)h->n; a.k = kd; a.kp = (int)h->kp; a.k0 = (int)h->k0; a.nz = h->nz; a.nsplit = h->nsplit;
  a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0) && (h->n % 4 == 0);
  a.gate = nullptr;
  a.pdl = 0;
  cudaError_t e = launch_incr<T>(a, h->bm, h->st);
  if (e != cudaSuccess) return e;
  const int nfw = h->Ebuf ? h->rs_grid : h->rp_grid;
  launch_reduce_incr(h->ics > 1 ? h->inc_part2 : h->inc_part, h->ics > 1 ? h->ncl : h->nsplit, kd,
                     (int)h->nk, h->nz, (int)(h->k - h->k0), (int)(h->n - h->k0), (int)h->kp, h->fw_part,
                     nfw, inc, h->st, nullptr, ReduceLayout{nullptr, 0, 0, 0, 0}, false, gk);
  return cudaGetLastError();
}

// B = [A | X1] Wb (result-mode row pass: b = a2 D^T S^{-1} - x1 C D^T S^{-1})
template <typename T>
static cudaError_t als_row_b(wlr_ctx* h, AlsSt* st, int x) {
  RowPassArgs<T> a{};
  a.tmA = st->tmAr; a.tmX = st->tmXr[x]; a.tmW = st->tmWb;
  a.A = (const T*)h->A; a.lda = h->lda; a.W1 = (const T*)h->W1; a.ldw = h->ldw;
  a.Xold = (const T*)h->X[x]; a.nwc = h->nwc;
  a.Wt = (const T*)st->Wb; a.KA = h->KA;
  a.Bout = (T*)st->B; a.ldb = h->kp; a.fw_part = h->fw_part; a.flags = h->flags;
  a.m = h->m; a.n = (int)h->n; a.k = (int)h->k; a.kp = (int)h->kp; a.no = (int)h->t;
  a.vec_ok = (h->lda % 4 == 0) && ((uintptr_t)h->A % 16 == 0);
  return launch_row_pass<T>(a, st->rpb, 8, true, 1, h->rp_grid, h->st);
}

static AlsArgs als_args(wlr_ctx* h, AlsSt* st) {
  AlsArgs a{};
  a.k = (int)h->k; a.nk = (int)h->nk; a.t = (int)h->t; a.KA = h->KA; a.rp = h->rp; a.rpb = st->rpb;
  a.uniform = h->uniform ? 1 : 0; a.w2 = h->w1s * h->w1s; a.a2sq = h->a2sq;
  a.flags = h->flags; a.scal = st->scal; a.Kop = h->Kop; a.Sop = h->Sop; a.W = h->Wt; a.Wb = st->Wb;
  a.cct = st->cct; a.dct = st->dct; a.part = st->part;
  return a;
}

static wlr_status als_setup(wlr_ctx* h) {
  wlr_status s = check_flags(h);              // flushes the pending half: F_0 in h_scal
  if (s != WLR_OK) return s;
  if (h->p != 0) return fail(h, WLR_EINVAL, "wlr_als_iterate starts from the GHS state (p = 0)");
  if (h->comm || h->vg) return fail(h, WLR_EINVAL, "block ALS: single rank only");
  if (!als_ok((int)h->k, (int)h->t)) return fail(h, WLR_EINVAL, "block ALS: k too large for the small steps");
  // B shares the X1 buffers' kp-wide row layout (row pass, TMA boxes, Gram kernels): r - k must fit
  if (h->t > h->kp) return fail(h, WLR_EINVAL, "block ALS: needs r - k <= round_up(k, 4)");
  AlsSt* st = new AlsSt();
  h->als = st;
  const size_t es = h->es;
  const int64_t kp = h->kp, wt_rows = h->KA + round_up(kp, 32);
  st->rpb = row_pass_rp((int)h->t);
  if ((s = dalloc(h, &st->B, (size_t)h->m * kp * es)) != WLR_OK) return s;
  if ((s = dalloc(h, &st->Wb, (size_t)wt_rows * st->rpb * es)) != WLR_OK) return s;
  for (int i = 0; i < 2; ++i) {
    if ((s = dalloc_t(h, &st->C[i], (size_t)(h->k * h->nk))) != WLR_OK) return s;
    if ((s = dalloc_t(h, &st->D[i], (size_t)(h->t * h->nk))) != WLR_OK) return s;
  }
  if ((s = dalloc_t(h, &st->inc1, (size_t)(h->k * h->nk + 2 * h->k * h->k + 1))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &st->inc2, (size_t)(h->t * h->nk + h->t * h->k + h->t * h->t + 1))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &st->scal, 8)) != WLR_OK) return s;
  if ((s = dalloc_t(h, &st->cct, (size_t)(h->k * h->k))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &st->dct, (size_t)(h->t * h->k))) != WLR_OK) return s;
  if ((s = dalloc_t(h, &st->part, als_part_doubles((int)h->k, (int)h->t, (int)h->nk))) != WLR_OK) return s;
  CUDA_TRY(h, cudaMemsetAsync(st->B, 0, (size_t)h->m * kp * es, h->st));
  CUDA_TRY(h, cudaMemsetAsync(st->Wb, 0, (size_t)wt_rows * st->rpb * es, h->st));
  CUDA_TRY(h, cudaMemsetAsync(h->Wt, 0, (size_t)wt_rows * h->rp * es, h->st));   // sWLR operand reused
  const uint32_t pe = (uint32_t)(128 / es), bm = (uint32_t)row_pass_bm(h->rp, h->rp_tr);
  const uint32_t bmr = (uint32_t)row_pass_bm(st->rpb, 8);
  bool ok = make_tmap_2d(&st->tmBx, st->B, (int)es, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * es, pe, bm, true) &&
            make_tmap_2d(&st->tmAr, h->A, (int)es, (uint64_t)h->n, (uint64_t)h->m, (uint64_t)h->lda * es, pe, bmr, true) &&
            make_tmap_2d(&st->tmWb, st->Wb, (int)es, (uint64_t)st->rpb, (uint64_t)wt_rows, (uint64_t)st->rpb * es,
                         (uint32_t)st->rpb, 32u, false);
  for (int i = 0; i < 2 && ok; ++i)
    ok = make_tmap_2d(&st->tmXr[i], h->X[i], (int)es, (uint64_t)kp, (uint64_t)h->m, (uint64_t)kp * es, pe, bmr, true);
  if (!ok) return fail(h, WLR_ECUDA, "cuTensorMapEncodeTiled failed (block ALS)");
  // p = 0: C_0 and V_0 of the GHS state; D_0 = V_0^T; B_0 = (A2 - X1_0 C_0) V_0 (result map)
  const int cur = h->ph % 3;
  st->x = h->ph & 1;
  st->c = 0;
  CUDA_TRY(h, cudaMemcpyAsync(st->C[0], h->C[cur], (size_t)(h->k * h->nk) * 8, cudaMemcpyDeviceToDevice, h->st));
  CUDA_TRY(h, launch_als_transpose(h->V[cur], st->D[0], (int)h->nk, (int)h->t, h->st));
  AlsArgs a = als_args(h, st);
  a.C = st->C[0]; a.D = st->D[0]; a.c_given = 1;
  const bool f64 = h->dtype == WLR_F64;
  CUDA_TRY(h, launch_als(a, 1, f64, h->st));
  CUDA_TRY(h, f64 ? als_row_b<double>(h, st, st->x) : als_row_b<float>(h, st, st->x));
  st->F0 = h->h_scal[2];
  return check_flags(h);
}

static wlr_status als_sweep(wlr_ctx* h, double* Fdev) {
  AlsSt* st = h->als;
  const bool f64 = h->dtype == WLR_F64;
  const int x = st->x, nx = x ^ 1, c = st->c, nc = c ^ 1;
  AlsArgs a = als_args(h, st);
  a.C = st->C[c]; a.D = st->D[c];
  CUDA_TRY(h, launch_als(a, 0, f64, h->st));                                       // W''
  CUDA_TRY(h, f64 ? als_row_x1<double>(h, st) : als_row_x1<float>(h, st));          // X1'
  CUDA_TRY(h, f64 ? als_grams<double>(h, st->B, h->X[nx], (int)h->k, (int)h->k, st->inc1)
                  : als_grams<float>(h, st->B, h->X[nx], (int)h->k, (int)h->k, st->inc1));
  a.inc = st->inc1; a.Cout = st->C[nc]; a.c_given = 0;
  CUDA_TRY(h, launch_als(a, 1, f64, h->st));                                       // C', Wb
  CUDA_TRY(h, f64 ? als_row_b<double>(h, st, nx) : als_row_b<float>(h, st, nx));    // B'
  CUDA_TRY(h, f64 ? als_grams<double>(h, h->X[nx], st->B, (int)h->t, (int)h->k, st->inc2)
                  : als_grams<float>(h, h->X[nx], st->B, (int)h->t, (int)h->k, st->inc2));
  AlsArgs d = als_args(h, st);
  d.C = st->C[nc]; d.inc = st->inc2; d.Dout = st->D[nc]; d.Fout = Fdev;
  CUDA_TRY(h, launch_als(d, 2, f64, h->st));                                       // D', F, D'C'^T
  st->x = nx;
  st->c = nc;
  return WLR_OK;
}

extern "C" wlr_status wlr_als_iterate(wlr_handle h, int32_t n_iters, double* F, int32_t cap) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  if (n_iters < 0) return fail(h, WLR_EINVAL, "n_iters < 0");
  wlr_status s;
  if (!h->als && (s = als_setup(h)) != WLR_OK) return s;
  AlsSt* st = h->als;
  if (st->nF < st->nrec + n_iters + 1) {      // device objective trace
    double* nf = nullptr;
    const int cap2 = std::max(2 * st->nF, st->nrec + n_iters + 1);
    if ((s = dalloc_t(h, &nf, (size_t)cap2)) != WLR_OK) return s;
    if (st->F && st->nrec > 0) CUDA_TRY(h, cudaMemcpyAsync(nf, st->F, (size_t)st->nrec * 8, cudaMemcpyDeviceToDevice, h->st));
    st->F = nf;
    st->nF = cap2;
  }
  if (st->nrec == 0) {
    CUDA_TRY(h, cudaMemcpyAsync(st->F, &st->F0, 8, cudaMemcpyHostToDevice, h->st));
    st->nrec = 1;
  }
  for (int32_t i = 0; i < n_iters; ++i) {
    if ((s = als_sweep(h, st->F + st->nrec)) != WLR_OK) return s;
    ++st->nrec;
  }
  if (!F) return WLR_OK;                       // asynchronous: errors surface at the next sync
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  if ((s = check_flags(h)) != WLR_OK) return s;
  if (F && cap > 0) {
    const int n = std::min(cap, st->nrec);
    CUDA_TRY(h, cudaMemcpy(F, st->F, (size_t)n * 8, is_device_ptr(F) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  }
  return WLR_OK;
}

extern "C" wlr_status wlr_als_result(wlr_handle h, void* X1, int64_t ldx1, void* C, void* B, int64_t ldb, void* D) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  if (!h->als) return fail(h, WLR_EINVAL, "wlr_als_result before wlr_als_iterate");
  wlr_status s = check_flags(h);
  if (s != WLR_OK) return s;
  AlsSt* st = h->als;
  const size_t es = h->es;
  if (X1) {
    if (ldx1 < h->k) return fail(h, WLR_EINVAL, "ldx1 < k");
    if ((s = copy_out(h, X1, ldx1, h->X[st->x], h->kp, h->m, h->k, es)) != WLR_OK) return s;
  }
  if (C && (s = copy_out(h, C, h->nk, st->C[st->c], h->nk, h->k, h->nk, 8)) != WLR_OK) return s;
  if (D && (s = copy_out(h, D, h->nk, st->D[st->c], h->nk, h->t, h->nk, 8)) != WLR_OK) return s;
  if (B) {
    if (ldb < h->t) return fail(h, WLR_EINVAL, "ldb < r-k");
    if ((s = copy_out(h, B, ldb, st->B, h->kp, h->m, h->t, es)) != WLR_OK) return s;
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  return WLR_OK;
}

extern "C" wlr_status wlr_debug_state(wlr_handle h, const char* name, double* out, int64_t cap,
                                      int64_t* count) {
  if (!h || !name) return fail(h, WLR_EINVAL, "null argument");
  if (std::string(name) == "ktime") {          // timestamps of the last launched K3 half,
    CUDA_TRY(h, cudaStreamSynchronize(h->st)); // read without launching a pending one
    if (count) *count = 256;
    if (out) CUDA_TRY(h, cudaMemcpy(out, h->tdbg, (size_t)std::min<int64_t>(cap, 256) * 8, cudaMemcpyDeviceToHost));
    return WLR_OK;
  }
  wlr_status s = check_flags(h);
  if (s != WLR_OK) return s;
  const int cx = h->ph & 1, cur = h->ph % 3;   // X1 buffer, state slot
  const double* src = nullptr;
  int64_t cnt = 0;
  std::string nm(name);
  if (nm == "G") { src = h->G[cur]; cnt = h->k * h->k; }
  else if (nm == "M") { src = h->M[cur]; cnt = h->k * h->nk; }
  else if (nm == "C") { src = h->C[cur]; cnt = h->k * h->nk; }
  else if (nm == "V") { src = h->V[cur]; cnt = h->nk * h->t; }
  else if (nm == "lam") { src = h->th[cur]; cnt = h->t; }
  else if (nm == "theta") { src = h->th[cur]; cnt = h->b; }
  else if (nm == "GA") { src = h->GA; cnt = h->nk * h->nk; }
  else if (nm == "scal") { src = h->scal; cnt = 8; }
  else if (nm == "ktime") { src = h->tdbg; cnt = 256; }
  else if (nm == "rptime_on" || nm == "rptime_off") {   // row-pass events inside the graph
    h->rp_time = nm == "rptime_on";
    if (h->rp_time && !h->rp_ev[0]) {
      CUDA_TRY(h, cudaEventCreate(&h->rp_ev[0]));
      CUDA_TRY(h, cudaEventCreate(&h->rp_ev[1]));
    }
    h->rp_ms = 0.0;
    h->rp_n = 0;
    if ((s = reset_graphs(h)) != WLR_OK) return s;
    if (count) *count = 0;
    return WLR_OK;
  }
  else if (nm == "gate") {   // [tensor-core increments enabled, gate (flags[5]: on once the X1 step is small), KPD]
    int f = 0;
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    CUDA_TRY(h, cudaMemcpy(&f, h->flags + 5, sizeof(int), cudaMemcpyDeviceToHost));
    const double v[3] = {h->itc_on ? 1.0 : 0.0, (double)f, (double)h->itc_kpd};
    for (int i = 0; i < 3 && out && i < cap; ++i) out[i] = v[i];
    if (count) *count = 3;
    return WLR_OK;
  }
  else if (nm == "prop") {   // Gram-propagation path: [active, prop1 CTAs, rows per CTA, G_A Y in prop1,
                             //  SMs prop1 spreads over, shadow K3a on]
    const double v[6] = {h->prop ? 1.0 : 0.0, (double)h->prop_nb,
                         h->prop ? (double)prop1_rb((int)h->n, h->prop_nsm) : 0.0, h->prop && gay_fits(h) ? 1.0 : 0.0,
                         (double)h->prop_nsm, h->shadow ? 1.0 : 0.0};
    for (int i = 0; i < 6 && out && i < cap; ++i) out[i] = v[i];
    if (count) *count = 6;
    return WLR_OK;
  }
  else if (nm == "rptime") {
    if (out && cap >= 2) { out[0] = h->rp_ms; out[1] = (double)h->rp_n; }
    if (count) *count = 2;
    return WLR_OK;
  }
  else if (nm == "itctime") { src = (const double*)h->itc_tstamp; cnt = h->itc_tstamp ? 8 * 4096 : 0; }
  else if (nm == "proptime") { src = (const double*)h->prop_ts; cnt = h->prop_ts ? 8 * (h->prop_nb + 3 * h->k) : 0; }
  else if (nm == "tctime") { src = (const double*)h->tc_tstamp; cnt = h->tc_tstamp ? 16 * h->tc_grid : 0; }
  else if (nm == "ktime_on" || nm == "ktime_off") {   // enable/disable K3 phase timestamps
    h->ktime = nm == "ktime_on";
    if ((s = reset_graphs(h)) != WLR_OK) return s;
    if (count) *count = 0;
    return WLR_OK;
  }
  else if (nm == "incrtc_on" || nm == "incrtc_off") {   // tensor-core / CUDA-core increments (A/B)
    h->itc_on = h->itc_ok && nm == "incrtc_on";
    if ((s = reset_graphs(h)) != WLR_OK) return s;
    if (count) *count = h->itc_on ? 1 : 0;
    return WLR_OK;
  }
  else if (nm == "rowtc_on" || nm == "rowtc_off") {   // tensor-core / CUDA-core row pass (A/B)
    h->tc_on = h->tc_ok && nm == "rowtc_on";
    if ((s = reset_graphs(h)) != WLR_OK) return s;
    if (count) *count = h->tc_on ? 1 : 0;
    return WLR_OK;
  }
  else if (nm == "ss_rerun") {                 // relaunch the last small step twice (timing only;
    SmallArgs s2 = h->last_ss;                  // leaves the state inconsistent)
    s2.tdbg = h->tdbg;
    s2.pdl = 0;
    for (int rep = 0; rep < 2; ++rep) CUDA_TRY(h, launch_small_step(s2, 1, h->st));
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    if (count) *count = 0;
    return WLR_OK;
  }
  else if (nm == "outer") {                    // eigensolver restarts of the last small step
    int fl[8];
    CUDA_TRY(h, cudaMemcpy(fl, h->flags, sizeof(fl), cudaMemcpyDeviceToHost));
    if (count) *count = 1;
    if (out && cap >= 1) out[0] = fl[3];
    return WLR_OK;
  }
  else return fail(h, WLR_EINVAL, "unknown state name");
  if (count) *count = cnt;
  if (out) CUDA_TRY(h, cudaMemcpy(out, src, (size_t)std::min(cap, cnt) * 8, cudaMemcpyDeviceToHost));
  return WLR_OK;
}

extern "C" wlr_status wlr_profile(wlr_handle h, int32_t enable, int32_t reset, double* ms,
                                  int32_t nms, int64_t* launches, int64_t* timed_iters) {
  if (!h) return fail(nullptr, WLR_EINVAL, "null handle");
  CUDA_TRY(h, cudaStreamSynchronize(h->st));
  // fold recorded event groups (9 per iteration; 6, 7 = deferred K3b on the side stream; 8 = the
  // row pass / row solve boundary inside [0, 1])
  for (size_t g = 0, it = 0; g + 9 <= h->pr.used; g += 9, ++it) {
    float t01 = 0, t12 = 0, t23 = 0, t45 = 0, t67 = 0, t81 = 0;
    cudaEventElapsedTime(&t01, h->pr.pool[g], h->pr.pool[g + 8]);
    cudaEventElapsedTime(&t81, h->pr.pool[g + 8], h->pr.pool[g + 1]);
    cudaEventElapsedTime(&t12, h->pr.pool[g + 1], h->pr.pool[g + 2]);
    cudaEventElapsedTime(&t23, h->pr.pool[g + 2], h->pr.pool[g + 3]);
    cudaEventElapsedTime(&t45, h->pr.pool[g + 4], h->pr.pool[g + 5]);
    if (it < h->pr.groups.size() && h->pr.groups[it]) cudaEventElapsedTime(&t67, h->pr.pool[g + 6], h->pr.pool[g + 7]);
    h->pr.ms[0] += t01; h->pr.ms[1] += t12; h->pr.ms[2] += t23; h->pr.ms[3] += t45; h->pr.ms[4] += t67;
    h->pr.ms[5] += t81;
  }
  h->pr.groups.clear();
  h->pr.used = 0;
  if (ms)
    for (int i = 0; i < nms && i < 6; ++i) ms[i] = h->pr.ms[i];
  if (launches) *launches = h->pr.launches;
  if (timed_iters) *timed_iters = h->pr.iters;
  if (reset) {
    for (double& v : h->pr.ms) v = 0.0;
    h->pr.launches = 0;
    h->pr.iters = 0;
  }
  h->prof = enable != 0;
  return WLR_OK;
}

extern "C" wlr_status wlr_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, WLR_EINVAL, "null output");
  std::string e;
  if (!g_nccl.load(e)) return fail(nullptr, WLR_ENCCL, e);
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, WLR_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof(id));
  return WLR_OK;
}

extern "C" const char* wlr_last_error(wlr_handle h) { return h ? h->err.c_str() : g_err.c_str(); }

extern "C" const char* wlr_status_string(int32_t s) {
  switch (s) {
    case WLR_OK: return "WLR_OK";
    case WLR_EINVAL: return "WLR_EINVAL";
    case WLR_ERANK: return "WLR_ERANK";
    case WLR_EEIG: return "WLR_EEIG";
    case WLR_EINTERNAL: return "WLR_EINTERNAL";
    case WLR_ENONFINITE: return "WLR_ENONFINITE";
    case WLR_ECUDA: return "WLR_ECUDA";
    case WLR_ENCCL: return "WLR_ENCCL";
    case WLR_ENOMEM: return "WLR_ENOMEM";
  }
  return "WLR_UNKNOWN";
}

extern "C" void wlr_destroy(wlr_handle h) {
  if (!h) return;
  if (h->st) cudaStreamSynchronize(h->st);
  for (int ph = 0; ph < 6; ++ph)
    for (int pend = 0; pend < 2; ++pend) {
      cudaGraphExec_t g = h->gexec[ph][pend];
      if (!g) continue;
      bool kept = false;
      if (gpool_ok(h)) {                           // (see build_graph: a later handle updates it)
        std::lock_guard<std::mutex> lk(g_gpool_mu);
        auto& v = g_gpool[gpool_key(h, ph, pend)];
        if (v.size() < 4) { v.push_back(g); kept = true; }
      }
      if (!kept) cudaGraphExecDestroy(g);
    }
  if (h->comm && g_nccl.commDestroy) g_nccl.commDestroy(h->comm);
  if (h->st2) cudaStreamSynchronize(h->st2);
  for (void* p : h->allocs) {
    if (!h->st || cudaFreeAsync(p, h->st) != cudaSuccess) { cudaGetLastError(); cudaFree(p); }
  }
  if (h->st) cudaStreamSynchronize(h->st);
  for (auto e : h->pr.pool) cudaEventDestroy(e);
  if (h->h_scal) pinned_give(h->h_scal);
  if (h->st2) { cudaStreamSynchronize(h->st2); cudaStreamDestroy(h->st2); }
  if (h->st3) { cudaStreamSynchronize(h->st3); cudaStreamDestroy(h->st3); }
  if (h->ev_f3) cudaEventDestroy(h->ev_f3);
  if (h->ev_j3) cudaEventDestroy(h->ev_j3);
  if (h->st4) { cudaStreamSynchronize(h->st4); cudaStreamDestroy(h->st4); }
  if (h->st5) { cudaStreamSynchronize(h->st5); cudaStreamDestroy(h->st5); }
  if (h->ev_j5) cudaEventDestroy(h->ev_j5);
  if (h->ev_j4) cudaEventDestroy(h->ev_j4);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (auto ev : h->rp_ev) if (ev) cudaEventDestroy(ev);
  if (h->own_stream && h->st) cudaStreamDestroy(h->st);
  delete h->als;
  delete h;
}

extern "C" int32_t wlr_version(void) { return WLR_VERSION; }
