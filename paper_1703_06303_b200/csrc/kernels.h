// kernels.h -- internal launchers of libwlr (CUDA path only).
#pragma once
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "tma.cuh"

namespace wlr {

// ---------------------------------------------------------------- init (init_kernels.cu)
template <typename T>
void launch_gram64(const T* L, int64_t ldl, int nl, const T* R, int64_t ldr, int nr, int64_t m,
                   double* part, int nsplit, double* out, cudaStream_t st);
template <typename T>
void launch_init_x1(const T* src, int64_t lds, int64_t m, int k, int kp, T* x, cudaStream_t st);
template <typename T>
void launch_fw(const T* A, int64_t lda, const T* W1, int64_t ldw, double w2s, const T* x, int kp,
               int64_t m, int k, double* part, int nblk, cudaStream_t st);
template <typename T>
void launch_validate(const T* A, int64_t lda, int64_t m, int n, const T* W1, int64_t ldw, int k,
                     int* flags, cudaStream_t st);

// ---------------------------------------------------------------- row pass (rowpass.cu)
constexpr int kPf = 12;             // L2 prefetch slots of the row pass (see api.cu set_prefetch)
template <typename T>
struct RowPassArgs {
  // TMA tensor maps (SWIZZLE_128B for A and X1_p boxes of 128 B x BM rows; Wt plain)
  CUtensorMap tmA, tmX, tmW;
  const T* A; int64_t lda;          // m x n (this rank's rows)
  const T* W1; int64_t ldw;         // m x k or nullptr (uniform)
  T w2s;                            // uniform weight squared
  const T* Xold; T* Xnew;           // m x kp
  T* Dnew;                          // m x kp  Delta = Xnew - Xold (stored values)
  int nwc;                          // warps running per-row Cholesky (non-uniform W1)
  // Linear row update: out = [A | X1_p] Wt, Wt is (KA + KX) x RP with rows
  // [0, n) for the columns of A and [KA, KA + kp) for X1_p (KA = n rounded up to 32):
  //   uniform W1    : Wt = [w^2 K^{-1}; U K^{-1}; P K^{-1}]  -> out = X1_{p+1} rows
  //   non-uniform   : Wt = [0; U; P]                        -> out = e - A1 . W1^2
  //   MODE_RESULT   : Wt = [0; V; -C V]                      -> out = B rows
  // with U = C^T - V (C V)^T ((n-k) x k), P = (C V)(C V)^T, K = w^2 I + C C^T.
  const T* Wt;
  int KA;                           // row offset of the X1_p block in Wt
  const T* Kmat;                    // k x k C C^T (non-uniform) or unused
  T* Bout; int64_t ldb;             // MODE_RESULT output (m x t)
  T* Ebuf;                          // non-uniform: write e rows here and skip the per-row solve
  double* fw_part;                  // gridDim.x partials
  int* flags;
  const void* pf_ptr[kPf]; int64_t pf_bytes[kPf];   // L2 prefetch of the next small steps' inputs
  int64_t m; int n, k, kp, no;      // no = output columns (kp, or t for MODE_RESULT)
  int vec_ok;                       // A rows 16-byte aligned at multiples of 4 elements
  const int* stop;                  // eps mode: the iteration's latched stop flag (skip all work), or nullptr
};
int row_pass_rp(int r);
bool row_pass_tr_ok(int rp, int tr);     // rows per thread TR available for this width
int row_pass_bm(int rp, int tr);         // tile height BM (rows per CTA tile)
template <typename T> size_t row_pass_smem(int rp, int tr, bool uniform, int k, int kp);
template <typename T> int row_pass_chol_warps(int rp, int tr, bool uniform, int k, int kp);
template <typename T>
cudaError_t launch_row_pass(const RowPassArgs<T>& a, int rp, int tr, bool uniform, int mode, int grid,
                            cudaStream_t st, int* occ = nullptr,   // occ: only report CTAs/SM
                            bool pdl = false);   // programmatic dependent of the previous kernel

// ------------------------------------------------- row pass on tcgen05 (rowpass_tc.cu)
// Uniform-weight fp32 row update X1_{p+1} = [A | X1_p] W' on the 5th-generation tensor cores
// with 3xTF32: 128-row tiles, TMEM accumulator, K-major W'^T.
struct RowPassTcArgs {
  CUtensorMap tmA, tmX;             // boxes 32 columns (128 B, SWIZZLE_128B) x 128 rows
  CUtensorMap tmW;                  // W'^T (RP x KW, K-major): boxes 32 x RP, SWIZZLE_128B
  CUtensorMap tmAx, tmXx;           // leftover rows: boxes 32 columns x 4 rows, no swizzle
  const float* A; int64_t lda;
  const float* Xold; float* Xnew; float* Dnew;   // m x kp
  float w2s;
  double* fw_part;                  // gridDim.x partials of f_w
  // non-uniform W1 (E mode, E != nullptr): the tile result is E - A1 . W1^2 (the linear part of E,
  // W'' = [0; U; P]); the epilogue writes those rows (m x kp) for the per-row solves, which add
  // A1 . W1^2 (RowSolveArgs::e_lin), instead of X1_{p+1} / Delta / f_w
  float* E; const float* W1; int64_t ldw;
  const void* pf_ptr[kPf]; int64_t pf_bytes[kPf];
  int64_t m; int KA, k, kp, n;
  // tiles cover rows [0, m_main); with extra > 0 (one CTA per SM, one tile each) CTA i also
  // computes the rows m_main + extra i + e, e < extra, on the CUDA cores (no tail wave)
  int64_t m_main; int extra;
  unsigned long long* tstamp;       // diagnostics: 8 globaltimer stamps per CTA, or nullptr
  int dbg;                          // diagnostics: bit 2 skip W loads, bit 3 skip epilogue
  int pdl;                          // host: launch as a programmatic dependent (no griddepcontrol.wait inside)
  const int* stop;                  // eps mode: the iteration's latched stop flag, or nullptr
};
constexpr int kTcBM = 128;          // rows per tile (UMMA M)
// deep = true: 8-stage ring, one CTA per SM (grid <= #SMs); false: 4 stages, 2 CTAs per SM
cudaError_t launch_row_pass_tc(const RowPassTcArgs& a, int rp, int grid, cudaStream_t st, int* occ = nullptr,
                               bool deep = false);
int row_pass_tc_ctas_per_sm(int rp);   // co-resident CTAs by shared memory (228 KB per SM)
bool row_pass_tc_deep_ok(int rp);      // the 8-stage ring fits one CTA per SM


template <typename T>
struct IncrArgs {
  const T* A; int64_t lda;
  const T* Xold; const T* Dnew;     // m x kp  X1_p and Delta
  double* part;                     // nsplit x k x nz (per-CTA fp64 chunk sums, rows > 256 only)
  double* part2;                    // (grid.y / cs) x k x nz: one fp64 partial per cluster
  int64_t m; int64_t rows_per_split;
  int n, k, kp, k0, nz, nsplit;
  int cs;                           // row splits per thread-block cluster (DSMEM pre-reduction)
  int vec_ok;
  const int* gate;                  // non-null and *gate != 0: the tensor-core kernel runs instead
  int pdl;                          // launched as a programmatic dependent of the row pass
};
// per-row SPD solves of the non-uniform X1 half-step (rowsolve.cu), fp32: warp per row,
// reverse-packed shared-memory Cholesky
// Gram propagation (prop.cu): uniform W1, the linear X1 half-step's Grams from A^T A
struct PropArgs {
  const double* AtA;                // n x n fp64 (once, at init)
  const void* Wt;                   // W' (KA + KX) x RP row-major, storage dtype (A rows 0..n-1, X rows KA..)
  int RP, KA;
  const double* Qp; double* Qn;     // n x k  A^T X1_p, A^T X1_{p+1}
  const double* Gp;                 // k x k  X1_p^T X1_p (small-step state)
  double* part;                     // ceil(n/RB) x 2 x k x k per-block partials (scratch)
  double* inc;                      // packed [N | Gamma | Omega | f_w] for the small step
  double* dg;                       // k scratch: f_w's diagonal terms
  double w2, a1sq;                  // w^2, ||A1||_F^2
  int n, k;
  const void* pf_ptr[kPf]; int64_t pf_bytes[kPf];   // L2 prefetch of the small step's inputs (prop1 entry)
  const int* stop;                  // eps mode: the iteration's latched stop flag, or nullptr
  const double* Y; double* GAY;     // warm Ritz block Y ((n-k) x b) -> G_A Y for the small step's first S-product
  int b;
  int nb;                           // prop1 CTAs (= blocks of the partials): min(n, #SMs)
  unsigned long long* ts;           // (diagnostics, or nullptr) prop1 phase %globaltimer stamps, 8 per CTA
};
size_t prop1_smem(int n, int k, int nsm, int b);   // dynamic shared memory of prop1 (one CTA per SM)
int prop1_rb(int n, int nsm);               // rows per prop1 CTA (<= 8 supported)
size_t prop_part_doubles(int nb, int k);
bool prop_gay_ok(int n, int k, int b, int nsm);   // prop1 computes G_A Y of the warm block (Y fits in smem)
// virtual-group sum: out[i] = sum_{g < G} in[g * stride + i], g in order (fixed, deterministic)
// eps mode: flags[6] = flags[2] (the converged flag) at the start of an iteration, one thread, so that
// every kernel of the iteration (clusters included) sees one consistent value
cudaError_t launch_stop_latch(int* flags, cudaStream_t st);
constexpr int kZeroList = 64;
struct ZeroList { void* ptr[kZeroList]; int64_t bytes[kZeroList]; int n; };
cudaError_t launch_zero_list(const ZeroList& z, cudaStream_t st);   // zero n buffers in one launch
cudaError_t launch_noop(cudaStream_t st);    // an empty kernel (launch ordering, api.cu)
cudaError_t launch_vsum(double* out, const double* in, int G, size_t stride, size_t count, cudaStream_t st);
cudaError_t launch_prop(const PropArgs& a, bool f64, int pdl, cudaStream_t st, cudaEvent_t after1 = nullptr);

struct RowSolveArgs {
  const float* E;                   // m x kp  e_i (written by the row pass; >= 8 floats of slack after)
  const float* S;                   // k x k8  C C^T, ld k8 = round_up(k, 8), zero columns k..k8-1
  const float* W1; int64_t ldw;
  const float* A; int64_t lda;      // A1 = A(:, 0:k) for f_w
  const float* Xold; float* Xnew; float* Dnew;   // m x kp
  double* fw_part;                  // gridDim.x partials of f_w
  int* flags;
  int64_t m; int k, kp;
  const int* stop;                  // eps mode: the iteration's latched stop flag, or nullptr
  int e_lin;                        // 1: E holds only the linear part [A | X1_p] W'' (the tensor-core row
                                    //    pass); the solver adds A1 . W1^2 (it reads both rows anyway)
};
bool row_solve_ok(int k);
size_t row_solve_smem(int k);
int row_solve_grid(int k, int nsm);
cudaError_t launch_row_solve(const RowSolveArgs& a, int grid, cudaStream_t st);

// tensor-core increments (incr_tc.cu): fp32, kp <= 32; partial layout nz' = nA32 + 64 columns
struct IncrTcArgs {
  CUtensorMap tmA, tmX, tmD;        // boxes 32 columns x 32 rows (SWIZZLE_128B): A, X1_p, Delta
  double* part;                     // nsplit x k x nz' (cs == 1) or (nsplit / cs) x k x nz' (clusters)
  int64_t m, rows_per_split;
  int cs;                           // row splits per thread-block cluster (DSMEM pre-reduction)
  int k, k0, nA32, nz;              // nz = nA32 + 2 kpd
  int kpd;                          // Delta / X1_p width in the layout: kp rounded up to 32 (<= 128)
  const int* gate;                  // runs only when *gate != 0 (set by the small step)
  unsigned long long* tstamp;       // diagnostics (WLR_TC_DBG bit 32): 8 stamps per CTA, or nullptr
};
cudaError_t launch_incr_tc(const IncrTcArgs& a, int nsplit, cudaStream_t st);
int incr_tc_kpd(int kp);           // 32 / 64 / 96 / 128, or -1
int incr_bm(int kp);
inline bool incr_cluster_ok() { return true; }   // 8-CTA clusters of 128-512 threads (portable)
int incr_bn(int bm, int elem_bytes);   // columns per CTA
template <typename T> cudaError_t launch_incr(const IncrArgs<T>& a, int bm, cudaStream_t st);
// Partial layouts: (part, nsplit, nz, nA, kp), or -- when gate && *gate -- the tensor-core layout
// (part_t, nsplit_t, nz_t, nA_t, kp_t).
struct ReduceLayout { const double* part; int nsplit, nz, nA, kp; };
void launch_reduce_incr(const double* part, int nsplit, int k, int nk, int nz, int kshift, int nA,
                        int kp, const double* fw_part, int nfw, double* inc, cudaStream_t st,
                        const int* gate = nullptr, ReduceLayout alt = {nullptr, 0, 0, 0, 0},
                        bool pdl = false, int gk = -1);

// ---------------------------------------------------------------- f3 block ALS (als.cu)
struct AlsArgs {
  const double* C; const double* D;     // current C (k x nk), D ((r-k) x nk), fp64
  double* Cout; double* Dout;           // updated C / D
  const double* inc;                    // reduced Grams (layout per kernel, see als.cu)
  double* scal;                         // [f_w, <M', C'>, <C', G' C'>]
  double* Fout;                         // objective of the new state
  void* W; void* Wb; void* Kop;         // X1 row map (KA + KX) x rp, B row map x rpb, C C^T
  float* Sop;                           // fp32 C C^T with ld round_up(k, 8) for the per-row solves (or null)
  double* cct; double* dct;             // C C^T (k x k) and D C^T (t x k) of the current state
  double* part;                         // per-CTA partials of the column-split kernels
  int* flags;
  int k, nk, t, KA, rp, rpb, uniform, c_given;
  double w2, a2sq;
};
// which: 0 = W'' of the X1 row map, 1 = C step + B map, 2 = D step + objective
cudaError_t launch_als(const AlsArgs& a, int which, bool f64, cudaStream_t st);
bool als_ok(int k, int t);
int als_blocks(int nk);
size_t als_part_doubles(int k, int t, int nk);
cudaError_t launch_als_transpose(const double* V, double* D, int nk, int t, cudaStream_t st);

// ---------------------------------------------------------------- small step (small_step.cu)
// Shared-memory plan of the K3 cluster kernel (offsets in doubles; identical in every CTA
// of the cluster so that DSMEM addresses of a peer's buffers equal the local ones).
// Optional regions have offset -1 when they do not fit (then the code reads the global
// originals, or the CTA's slot of the global workspace gws for the Newton-Schulz mats).
struct SSPlan {
  int CL, SL;                       // cluster size, columns per CTA (slice of the n-k index)
  int KS, JS;                       // S-product split: KS reduction chunks x JS column groups
  int PL;                           // DSMEM exchange length (doubles per bank)
  int ccx;                          // C'C'^T partials ride in the DSMEM exchange (else global)
  int64_t oPart, oBuf, oVp, oE, oSE, oWk, oCinE, oSmall, oRed;            // always in smem
  int64_t oCs, oMs, oCin, oXf, oMat3, oGsq, oTail;                         // optional
  int64_t total;                    // doubles of dynamic smem
  int64_t gws_stride;               // doubles of global workspace per CTA (Gsq fallback)
  int64_t flen;                     // final partial length (global reduce-scatter)
};

struct SmallArgs {
  int k, nk, t, b, kp, k0, rp;      // dims; b = eigen block width (t <= b <= 32)
  int pdl;                          // host only: launch as a programmatic dependent (part 1)
  const int* stop;                  // eps mode: the iteration's latched stop flag (skip the step), or nullptr
  const double* GAY;                // G_A Y of the warm block, precomputed (Gram propagation), or nullptr
  const double* dg;                 // Gram propagation: prop2's diagonal terms of f_w (k), or nullptr
  double a1sq;                      //   and ||A1||_F^2: CTA 0 writes f_w for the deferred half
  int KA;                           // row offset of the X1_p block of the row-pass Wt
  void* WtT; int KW;                // fp32 W'^T (RP x KW, K-major) for the tensor-core row pass
  int mode;                         // 0: init (G, M given), 1: iteration (apply increments)
  int dtype;                        // 0 fp32 operands, 1 fp64 operands
  int uniform; double w2;           // uniform weight squared
  const double* GA; double a2sq;    // A2^T A2 ((nk)^2, symmetric), ||A2||_F^2
  const double* inc;                // [N | Gamma | Omega | f_w] (mode 1); f_w at [0] (mode 0)
  const double* G_in; double* G_out;   // k x k
  const double* M_in; double* M_out;   // k x nk
  const double* C_in; double* C_out;   // k x nk
  const double* V_in; double* V_out;     // nk x t  V_p (previous state) / V_{p+1}
  const double* CV_in; double* CV_out;   // k x t   C_p V_p / C_{p+1} V_{p+1}
  const double* th_in; double* th_out;   // b       Ritz values of S_p / S_{p+1}
  double* k3x;                      // small results K3a -> K3b: R (t x t), ZnV (t x t)
  double* Y;                        // nk x b  warm-start Ritz block (updated)
  int* skip;                        // part 2 in a graph: *skip != 0 -> this deferred half already ran
                                    // (flushed by the host or never needed): clear it and return
  double* snapY; double* snapKi;    // part 1: copies of its Y and K^{-1} inputs as read (for the shadow K3a), or nullptr
  const double* Gi_in; double* Gi_out;   // k x k  G^{-1} of the previous / current state
  double* Ki;                       // k x k  (w^2 I + C C^T)^{-1} (uniform W1; updated)
  double* gws;                      // CL x gws_stride global workspace
  double* xchg;                     // CL x flen global partial slots
  double* red;                      // flen reduced partials
  double* scal;                     // persistent scalars (see small_step.cuh)
  double* trace; int trace_cap;     // trace ring (4 doubles per state)
  void* Wt; void* CVop; void* Kop;  // row-pass operands (dtype)
  float* Sop;                       // fp32 C C^T, ld round_up(k, 8), zero padding (per-row solves; or null)
  int* flags;
  double eps, tol; int max_outer, max_deg;
  int cold;                         // 1: Y holds a random block (no Ritz values yet)
  double* tdbg;                     // optional phase timestamps (64 doubles) or nullptr
  SSPlan pl;
};
bool small_step_plan(SmallArgs& a, int CL);       // fills a.pl; false if it cannot fit
int small_step_cluster_size(SmallArgs& a);        // picks CL and fills a.pl (0 = none)
// part 1: critical half (C', eigenpairs, next row-pass operands); part 2: deferred half
// (objective, step norm, trace), which may run concurrently with the next row pass
cudaError_t launch_small_step(const SmallArgs& a, int part, cudaStream_t st);
int small_step_bt(int b);

// ---------------------------------------------------------------- result (result.cu)
template <typename T>
void launch_assemble_x2(const T* X1, int kp, const T* B, int64_t ldb, const double* C,
                        const double* V, int64_t m, int k, int nk, int t, T* X2, int64_t ldx2,
                        cudaStream_t st);
template <typename T>
void launch_copy_x1(const T* X, int kp, int64_t m, int k, T* out, int64_t ldo, cudaStream_t st);

}  // namespace wlr
