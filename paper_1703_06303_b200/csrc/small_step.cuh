// small_step.cuh -- K3: the (C, D) half-step of Algorithm 1
// on the Gram route, plus the objective and the convergence reduction.
//
// ONE thread-block cluster of CL CTAs (<= 16, one per SM).  CTA c owns the columns
// [rs, rs + nl) of the (n-k)-dimensional index ("its slice"); per-slice vectors live in its
// shared memory and every cross-CTA sum is a fixed-order DSMEM reduction behind one hardware
// cluster barrier, so results are bitwise identical on every CTA (and on every rank of a
// row-sharded run).  The kernel is latency-bound: every small dense step is
// written as thread-per-output work or a parallel (round-robin) Jacobi, never as a long
// single-thread chain, and inverses are Newton-Schulz refined from the previous iteration's.
//
//   Gram update   G' = G + Gamma + Gamma^T + Omega,  M' = M + N,  H = G + Gamma
//   C             C' = G'^{-1} M'   (= R^{-1} Q^T A2); G'^{-1} by Newton-Schulz
//                 from G_p^{-1} (fallback and init: symmetric Gauss-Jordan sweep)
//   eigenpairs    top t = r-k of S = G_A - M'^T C' = A2^T P^perp A2 by matrix-free products
//                 S X = G_A X - M'^T (C' X) (G_A streamed from L2): a Rayleigh-Ritz step on the
//                 warm Ritz block and, only while the residual is above tolerance, Chebyshev-
//                 filtered subspace iteration of adaptive degree.  V = right singular vectors of
//                 P^perp A2, lambda = sigma^2, D = U Sigma_{r-k} V^T = (A2 - X1 C) V V^T
//
//   objective     F = f_w + ||A2||^2 - <M', C'> - sum(lambda)
//   step norm     ||X_{p+1} - X_p||_F from small-side products only
//   operands      Wt = [V | C^T], C V and K^{-1} = (w^2 I + C C^T)^{-1} (or C C^T) for the
//                 next row pass, converted to the storage dtype.
//
// scal[] layout: 0 ||X2_p||^2, 1 ||X_p||^2, 2 F_p, 3 step, 4 rel, 5 p, 6 residual ratio
// max_j ||S v_j - lambda_j v_j|| / lambda_1 of the last Rayleigh-Ritz, 7 S-products.
#pragma once
#include <cooperative_groups.h>

#include "kernels.h"
#include "umma.cuh"

namespace cg = cooperative_groups;

namespace wlr {

#define WLR_NOINL static __device__ __noinline__

constexpr int kSST = 512;            // threads per CTA
constexpr int kSSW = kSST / 32;      // warps per CTA
constexpr double kEps = 2.220446049250313e-16;

// Small-region layout (doubles, relative to pl.oSmall)
struct SmallOff {
  int Tb, Ub, Lb, Li, Qb, Wb, Gx, th, dsc, Rt, cs, d0, rb, len;
  __host__ __device__ SmallOff(int b, int t, int k) {
    const int bb = 32 * 32;             // b <= 32; fixed 32 x 32 tiles keep offsets simple
    Tb = 0; Ub = Tb + bb; Lb = Ub + bb; Li = Lb + bb; Qb = Li + bb; Wb = Qb + bb;
    Gx = Wb + bb;                       // reduced Gram exchange: Gyy | Gyz | VpY | VpZ
    th = Gx + 2 * b * b + 2 * t * b + 8;
    dsc = th + 32; Rt = dsc + 32; cs = Rt + t * t + 8; d0 = cs + 64; rb = d0 + k + 8;
    len = rb + 2 * (k + 8);
  }
};

// Final partial layout (global reduce-scatter)
struct FinOff {
  int CnV, CnVn, CVn, MnV, MVn, NV, CE, EE, ESE, CC, len;
  __host__ __device__ FinOff(int k, int t) {
    const int kt = k * t;
    CnV = 5; CnVn = CnV + kt; CVn = CnVn + kt; MnV = CVn + kt; MVn = MnV + kt; NV = MVn + kt;
    CE = NV + kt; EE = CE + kt; ESE = EE + t * t; CC = ESE + t * t; len = CC + k * k;
  }
};

struct SS {
  int c, CL, rs, nl, SL, k, nk, b, t;
  double* sm;
  int bank;
  int nt;                // timestamps recorded (CTA 0, thread 0; a.tdbg != nullptr)
  double* tb;            // cluster-barrier release stamps of the exchanges (a.tdbg + 128)
  int nx;
};

// Phase timestamps for profiling the latency-bound small step: CTA 0 /
// thread 0 writes %globaltimer (ns) into a.tdbg[1..31] and clock64 into a.tdbg[32..].
WLR_DEVI void tmark(SS& s, const SmallArgs& a) {
  if (a.tdbg && s.c == 0 && threadIdx.x == 0 && s.nt < 31) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tdbg[1 + s.nt] = (double)t;
    a.tdbg[32 + s.nt] = (double)clock64();
    a.tdbg[0] = (double)(s.nt + 1);
  }
  s.nt++;
}

WLR_DEVI double* xpart(SS& s, const SSPlan& p) { return s.sm + p.oPart + (int64_t)s.bank * p.PL; }

// Fixed-order cluster sum of the len-long partial every CTA wrote into its exchange bank;
// out is local.  (Arguments by value: this is a shared, non-inlined routine.)
WLR_NOINL void xreduce_impl(const double* mine, int CL, int len, double* out, int len2, double* out2,
                            double* stamp) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (stamp && threadIdx.x == 0) {             // profiling: when the cluster barrier released
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = (double)t;
  }
#pragma unroll 1
  for (int i = threadIdx.x; i < len + len2; i += kSST) {
    double v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = c < CL ? cl.map_shared_rank(mine, c)[i] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) acc += v[c];
    if (i < len) out[i] = acc;
    else out2[i - len] = acc;
  }
  __syncthreads();
}
// The same sum as a reduce-scatter + all-gather: CTA c sums the c-th block of the values over the
// cluster and stores the results into every CTA's out / out2 (remote shared-memory stores), then
// a second cluster barrier.  Each CTA moves ~2 len values through the cluster network instead of
// CL len: the long exchanges are bandwidth-bound.  out / out2 in shared memory.
WLR_NOINL void xreduce_rs_impl(const double* mine, int CL, int c, int len, double* out, int len2, double* out2,
                               double* stamp) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (stamp && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = (double)t;
  }
  const int L = len + len2, chunk = (L + CL - 1) / CL, i1 = min(L, (c + 1) * chunk);
#pragma unroll 1
  for (int i = c * chunk + threadIdx.x; i < i1; i += kSST) {
    double v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = q < CL ? cl.map_shared_rank(mine, q)[i] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += v[q];
    double* dst = i < len ? out + i : out2 + (i - len);
#pragma unroll 1
    for (int d = 0; d < CL; ++d) *cl.map_shared_rank(dst, d) = acc;
  }
  cl.sync();
}
// (a second segment of len2 values, if any, lands in out2)
WLR_DEVI void xreduce(SS& s, const SSPlan& p, int len, double* out, int len2 = 0, double* out2 = nullptr) {
  double* stamp = s.tb && s.c == 0 && s.nx < 32 ? s.tb + s.nx : nullptr;
  if (len + len2 >= 256 && s.CL > 1 && __isShared(out) && (len2 == 0 || __isShared(out2)))
    xreduce_rs_impl(xpart(s, p), s.CL, s.c, len, out, len2, out2, stamp);
  else
    xreduce_impl(xpart(s, p), s.CL, len, out, len2, out2, stamp);
  s.nx++;
  s.bank ^= 1;
}

// block reduction of NV values per thread (sum; result valid on all threads)
template <int NV>
WLR_NOINL void block_sum_n(double (&v)[NV], double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < NV; ++u) v[u] = warp_sum(v[u]);
  if (lane == 0)
#pragma unroll
    for (int u = 0; u < NV; ++u) red[u * kSSW + warp] = v[u];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kSSW; ++w) s += red[u * kSSW + w];
    v[u] = s;
  }
  __syncthreads();
}

// barrier over the nt threads of named barrier `bar` (bar 0 with nt = kSST: __syncthreads)
WLR_DEVI void bar_sync(int bar, int nt) { asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(nt) : "memory"); }

// max over the threads [t0, t0 + nt) (whole warps), valid on all of them
WLR_NOINL double block_max(double v, double* red, int t0 = 0, int nt = kSST, int bar = 0) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = (threadIdx.x - t0) >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  bar_sync(bar, nt);
  double m = 0.0;
  #pragma unroll 1
  for (int w = 0; w < (nt >> 5); ++w) m = fmax(m, red[w]);
  bar_sync(bar, nt);
  return m;
}

// One fp64 tensor-core step (mma.sync m8n8k4, FP64 DMMA): d (8 x 8, two values per lane) +=
// a (8 x 4, one value per lane: row lane / 4, column lane % 4) . b (4 x 8: row lane % 4,
// column lane / 4); d holds row lane / 4, columns 2 (lane % 4) + {0, 1}.
WLR_DEVI void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// This lane's two outputs of the 8 x 8 tile (r0, c0) of sum_q A(r, q) B(q, c), A(r, q) =
// A[r*ars + q*aqs], B(q, c) = B[q*bqs + c*bcs] (m x kk . kk x n): k-steps of 4 on the FP64
// tensor cores, two accumulator chains.  Row r0 + lane / 4, columns c0 + 2 (lane % 4) + {0, 1}.
WLR_DEVI void tc_tile(int m, int n, int kk, const double* A, int ars, int aqs, const double* B, int bqs, int bcs,
                      int r0, int c0, double& v0, double& v1) {
  const int lane = threadIdx.x & 31, ra = lane >> 2, qa = lane & 3;
  const int ar = r0 + ra, bc = c0 + ra;                    // A: row ra, k qa; B: k qa, column ra
  const bool aok = ar < m, bok = bc < n;
  const double* pa = A + (int64_t)ar * ars + (int64_t)qa * aqs;
  const double* pb = B + (int64_t)bc * bcs + (int64_t)qa * bqs;
  const int64_t sa = 4LL * aqs, sb = 4LL * bqs;
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  int q = 0;
  #pragma unroll 1
  for (; q + 8 <= kk; q += 8) {
    const double a0 = aok ? pa[0] : 0.0, b0 = bok ? pb[0] : 0.0;
    const double a1 = aok ? pa[sa] : 0.0, b1 = bok ? pb[sb] : 0.0;
    dmma884(d0, d1, a0, b0);
    dmma884(e0, e1, a1, b1);
    pa += 2 * sa; pb += 2 * sb;
  }
  #pragma unroll 1
  for (; q < kk; q += 4) {
    const bool kin = q + qa < kk;
    const double a0 = aok && kin ? pa[0] : 0.0, b0 = bok && kin ? pb[0] : 0.0;
    dmma884(d0, d1, a0, b0);
    pa += sa; pb += sb;
  }
  v0 = d0 + e0;
  v1 = d1 + e1;
}

// C(r, c) = alpha * sum_q A(r, q) B(q, c) (+ I if addI) with A(r, q) = A[r*ars + q*aqs],
// B(q, c) = B[q*bqs + c*bcs], C(r, c) = C[r*ldc + c]: one 8 x 8 output tile per warp step, on
// the warps of the threads [t0, t0 + nt) (whole warps; no barrier inside).  C must not alias
// A or B.
// Two horizontally adjacent 8 x 8 tiles (c0, c0 + 8) sharing the A fragments: one accumulator
// chain each (used when the tiles outnumber the warps, so that no warp runs two tiles in a row)
WLR_DEVI void tc_tile_pair(int m, int n, int kk, const double* A, int ars, int aqs, const double* B, int bqs,
                           int bcs, int r0, int c0, double (&v)[4]) {
  const int lane = threadIdx.x & 31, ra = lane >> 2, qa = lane & 3;
  const int ar = r0 + ra, bc = c0 + ra;
  const bool aok = ar < m, bok0 = bc < n, bok1 = bc + 8 < n;
  const double* pa = A + (int64_t)ar * ars + (int64_t)qa * aqs;
  const double* pb = B + (int64_t)bc * bcs + (int64_t)qa * bqs;
  const int64_t sa = 4LL * aqs, sb = 4LL * bqs, b8 = 8LL * bcs;
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  #pragma unroll 2
  for (int q = 0; q < kk; q += 4) {
    const bool kin = q + qa < kk;
    const double a0 = aok && kin ? pa[0] : 0.0;
    const double b0 = bok0 && kin ? pb[0] : 0.0, b1 = bok1 && kin ? pb[b8] : 0.0;
    dmma884(d0, d1, a0, b0);
    dmma884(e0, e1, a0, b1);
    pa += sa; pb += sb;
  }
  v[0] = d0; v[1] = d1; v[2] = e0; v[3] = e1;
}

WLR_NOINL void gemm_tc(int m, int n, int kk, const double* A, int ars, int aqs, const double* B, int bqs, int bcs,
                       double* C, int ldc, double alpha, bool addI, int t0 = 0, int nt = kSST) {
  const int lane = threadIdx.x & 31, w = (threadIdx.x - t0) >> 5, nw = nt >> 5;
  const int tn = (n + 7) >> 3, tt = ((m + 7) >> 3) * tn;
  if (tt > nw) {   // more tiles than warps: pairs of column tiles (one round instead of two)
    const int tn2 = (tn + 1) >> 1, tt2 = ((m + 7) >> 3) * tn2;
    #pragma unroll 1
    for (int tile = w; tile < tt2; tile += nw) {
      const int r0 = (tile / tn2) << 3, c0 = (tile - (tile / tn2) * tn2) << 4;
      double v[4];
      tc_tile_pair(m, n, kk, A, ars, aqs, B, bqs, bcs, r0, c0, v);
      const int cr = r0 + (lane >> 2);
      if (cr < m) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c0 + 8 * h + 2 * (lane & 3);
          double v0 = v[2 * h] * alpha, v1 = v[2 * h + 1] * alpha;
          if (addI) { if (cr == cc) v0 += 1.0; if (cr == cc + 1) v1 += 1.0; }
          if (cc < n) C[(int64_t)cr * ldc + cc] = v0;
          if (cc + 1 < n) C[(int64_t)cr * ldc + cc + 1] = v1;
        }
      }
    }
    return;
  }
  #pragma unroll 1
  for (int tile = w; tile < tt; tile += nw) {
    const int r0 = (tile / tn) << 3, c0 = (tile - (tile / tn) * tn) << 3;
    double v0, v1;
    tc_tile(m, n, kk, A, ars, aqs, B, bqs, bcs, r0, c0, v0, v1);
    const int cr = r0 + (lane >> 2), cc = c0 + 2 * (lane & 3);
    if (cr < m) {
      v0 *= alpha; v1 *= alpha;
      if (addI) { if (cr == cc) v0 += 1.0; if (cr == cc + 1) v1 += 1.0; }
      if (cc < n) C[(int64_t)cr * ldc + cc] = v0;
      if (cc + 1 < n) C[(int64_t)cr * ldc + cc + 1] = v1;
    }
  }
}

// C[r][c] = alpha * sum_q A[r*lda + q] B[q*ldb + c] (+ I if addI) on the threads [t0, t0 + nt)
// of the block (no barrier inside)
WLR_DEVI void gemm_nn(int m, int n, int kk, const double* A, int lda, const double* B, int ldb,
                      double* C, int ldc, double alpha, bool addI, int t0 = 0, int nt = kSST) {
  gemm_tc(m, n, kk, A, lda, 1, B, ldb, 1, C, ldc, alpha, addI, t0, nt);
}

// Segments of "transpose-NN" slice contractions: out[r*ncol + c] = sum_{i < nl}
// A[r*ars + i*ais] B[c*bcs + i*bis]  (thread per output, all segments in one pass).
struct TN {
  const double* A; int ars, ais;
  const double* B; int bcs, bis;
  int nrow, ncol;
  double* out;
};
template <int ND>
WLR_DEVI void slice_tn(int nl, const TN (&d)[ND]) {
  // one combined space of 8 x 8 output tiles over the segments, a tile per warp step; the
  // segment loop is unrolled so that every descriptor field is a compile-time access (inlined:
  // the descriptors stay in registers instead of local memory)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base = 0;
#pragma unroll
  for (int u = 0; u < ND; ++u) {
    const int tn = (d[u].ncol + 7) >> 3, nt = ((d[u].nrow + 7) >> 3) * tn;
    int tl = (w - base) % kSSW;
    if (tl < 0) tl += kSSW;
    #pragma unroll 1
    for (; tl < nt; tl += kSSW) {
      const int r0 = (tl / tn) << 3, c0 = (tl - (tl / tn) * tn) << 3;
      double v0, v1;
      tc_tile(d[u].nrow, d[u].ncol, nl, d[u].A, d[u].ars, d[u].ais, d[u].B, d[u].bis, d[u].bcs, r0, c0, v0, v1);
      const int cr = r0 + (lane >> 2), cc = c0 + 2 * (lane & 3);
      if (cr < d[u].nrow) {
        if (cc < d[u].ncol) d[u].out[cr * d[u].ncol + cc] = v0;
        if (cc + 1 < d[u].ncol) d[u].out[cr * d[u].ncol + cc + 1] = v1;
      }
    }
    base += nt;
  }
}

// In-place inverse of the SPD n x n matrix A (row-major) by the sweep operator (symmetric
// Gauss-Jordan), whole CTA.  Returns false (uniformly) if a pivot is not > rel * its
// original diagonal (numerical rank test, reading R6b).  Init / fallback only.
WLR_NOINL bool sweep_inverse(double* A, int n, double rel, double* d0, double* rb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  #pragma unroll 1
  for (int i = threadIdx.x; i < n; i += kSST) d0[i] = A[(int64_t)i * n + i];
  __syncthreads();
  #pragma unroll 1
  for (int j = 0; j < n; ++j) {
    double* rj = rb + (j & 1) * (n + 8);       // double-buffered pivot row
    #pragma unroll 1
    for (int i = threadIdx.x; i < n; i += kSST) rj[i] = A[(int64_t)j * n + i];
    __syncthreads();
    const double p = rj[j];
    if (!(p > rel * d0[j]) || !(p > 0.0) || !isfinite(p)) return false;
    const double pinv = 1.0 / p;
    #pragma unroll 1
    for (int i = warp; i < n; i += kSSW) {
      const double ri = rj[i] * pinv;
      #pragma unroll 1
      for (int l = lane; l < n; l += 32) {
        double v;
        if (i == j) v = (l == j) ? -pinv : rj[l] * pinv;
        else if (l == j) v = ri;
        else v = fma(-ri, rj[l], A[(int64_t)i * n + l]);
        A[(int64_t)i * n + l] = v;
      }
    }
    __syncthreads();
  }
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < n * n; idx += kSST) A[idx] = -A[idx];
  __syncthreads();
  return true;
}

// Newton-Schulz refinement of X ~ G^{-1} (n x n, row-major; R, P scratch n x n):
// R = I - G X, X <- X + X R.  Returns false (uniformly) when max|I - G X| >= 3e-2 (the
// warm start is too far: the caller falls back to the sweep).  The number of steps is
// chosen from the initial residual so that delta^(2^steps) <= 1e-12.
// Runs on the threads [t0, t0 + nt) with named barrier `bar` (defaults: the whole block).
WLR_NOINL bool ns_inverse(const double* G, double* X, double* R, double* P, int n, double* red,
                          int t0 = 0, int nt = kSST, int bar = 0) {
  gemm_nn(n, n, n, G, n, X, n, R, n, -1.0, true, t0, nt);
  bar_sync(bar, nt);
  double dm = 0.0;
  #pragma unroll 1
  for (int idx = threadIdx.x - t0; idx < n * n; idx += nt) dm = fmax(dm, fabs(R[idx]));
  const double delta = block_max(dm, red, t0, nt, bar);
  if (!(delta < 3e-2)) return false;
  const int steps = delta < 1e-6 ? 1 : delta < 1e-3 ? 2 : 3;
  #pragma unroll 1
  for (int st = 0; st < steps; ++st) {
    if (st > 0) {
      gemm_nn(n, n, n, G, n, X, n, R, n, -1.0, true, t0, nt);
      bar_sync(bar, nt);
    }
    gemm_nn(n, n, n, X, n, R, n, P, n, 1.0, false, t0, nt);
    bar_sync(bar, nt);
    #pragma unroll 1
    for (int idx = threadIdx.x - t0; idx < n * n; idx += nt) X[idx] += P[idx];
    bar_sync(bar, nt);
  }
  #pragma unroll 1
  for (int idx = threadIdx.x - t0; idx < n * n; idx += nt) {   // symmetrise
    const int i = idx / n, j = idx - i * n;
    if (i < j) {
      const double v = 0.5 * (X[idx] + X[(int64_t)j * n + i]);
      X[idx] = v;
      X[(int64_t)j * n + i] = v;
    }
  }
  bar_sync(bar, nt);
  return true;
}

// Cholesky of the small n x n SPD matrix A (smem, ld 32) by warp 0 (lower factor in place);
// dinv[j] = 1 / L_jj.  Returns (uniformly, after a block barrier) true iff SPD.
WLR_NOINL bool chol_small(double* A, int n, double* dinv, int* ok_s) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    #pragma unroll 1
    for (int j = 0; j < n; ++j) {
      const double d = A[j * 32 + j];
      ok = ok && (d > 0.0) && isfinite(d);
      const double r = rsqrt(d > 0.0 ? d : 1.0);
      __syncwarp();
      if (lane == 0) { A[j * 32 + j] = d * r; dinv[j] = r; }
      const int i = j + 1 + lane;
      double lij = 0.0;
      if (i < n) { lij = A[i * 32 + j] * r; A[i * 32 + j] = lij; }
      __syncwarp();
      if (i < n)
        #pragma unroll 1
        for (int l = j + 1; l <= i; ++l) A[i * 32 + l] = fma(-lij, A[l * 32 + j], A[i * 32 + l]);
      __syncwarp();
    }
    if (lane == 0) *ok_s = ok ? 1 : 0;
  }
  __syncthreads();
  return *ok_s != 0;
}

// Li = L^{-1} (lower triangular, ld 32), column c by lane c of warp 0.
WLR_NOINL void tri_inverse(const double* L, const double* dinv, int n, double* Li) {
  if (threadIdx.x < 32) {
    const int c = threadIdx.x;
    if (c < n) {
      #pragma unroll 1
      for (int i = 0; i < c; ++i) Li[i * 32 + c] = 0.0;
      Li[c * 32 + c] = dinv[c];
      #pragma unroll 1
      for (int i = c + 1; i < n; ++i) {
        double v = 0.0;
        #pragma unroll 1
        for (int m = c; m < i; ++m) v = fma(L[i * 32 + m], Li[m * 32 + c], v);
        Li[i * 32 + c] = -v * dinv[i];
      }
    }
  }
  __syncthreads();
}

// Parallel (round-robin) cyclic Jacobi on the symmetric b x b matrix T (ld 32), called by warp 0:
// on exit th = eigenvalues in DESCENDING order and U (ld 32) the matching orthonormal
// eigenvectors (columns).  b/2 disjoint rotations per round, b-1 rounds per sweep; stops
// when every off-diagonal is at rounding level.  Deterministic.
// One-warp form (warp 0, beside the K^{-1} refinement): the same round-robin rotations, each round
// applied as ONE update T' = J^T T J, U' = U J from the previous buffers into the other pair
// (T, U) <-> (T2, U2) -- two warp barriers per round instead of three.  pi / pc / ps: for every
// index x its partner in the round and the coefficients of new_row_x = pc x + ps partner.
WLR_NOINL void jacobi_warp(double* T, double* U, double* T2, double* U2, double* th, double* scr, int b) {
  const int lane = threadIdx.x & 31;
  const int nb = (b + 1) & ~1, np = nb / 2;
  double* const Uo = U;                        // (the caller's U: the sorted eigenvectors go here)
  double* pcoef = scr;                         // [32] self coefficient, [32..64) partner coefficient
  int* pidx = reinterpret_cast<int*>(scr + 64);   // [32] partner index (-1: no rotation)
  #pragma unroll 1
  for (int idx = lane; idx < b * b; idx += 32) {
    const int i = idx / b, j = idx - i * b;
    U[i * 32 + j] = (i == j) ? 1.0 : 0.0;
  }
  double dmax = 0.0;
  #pragma unroll 1
  for (int i = 0; i < b; ++i) dmax = fmax(dmax, fabs(T[i * 32 + i]));
  const double tabs = 2e-15 * dmax;
  __syncwarp();
  #pragma unroll 1
  for (int sweep = 0; sweep < 30 && nb > 1; ++sweep) {
    #pragma unroll 1
    for (int rnd = 0; rnd < nb - 1; ++rnd) {
      if (lane < np) {
        int p, q;
        if (lane == 0) { p = rnd; q = nb - 1; }
        else { p = (rnd + lane) % (nb - 1); q = (rnd - lane + nb - 1) % (nb - 1); }
        if (p > q) { const int x = p; p = q; q = x; }
        double c = 1.0, sn = 0.0;
        if (q < b) {
          const double apq = T[p * 32 + q], app = T[p * 32 + p], aqq = T[q * 32 + q];
          if (fabs(apq) > tabs && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq))) {
            // the angle's tangent in fp32 (short-latency MUFU ops; |tau| < 1e15 by the thresholds):
            // c, s from the same fp64 t keep the rotation orthogonal to fp64 rounding, only the
            // angle is fp32-accurate (apq drops to ~1e-7 of itself; the next sweep removes the rest)
            const float tauf = (float)((aqq - app) / (2.0 * apq));
            const double tt = (double)(copysignf(1.0f, tauf) / (fabsf(tauf) + sqrtf(fmaf(tauf, tauf, 1.0f))));
            c = rsqrt(1.0 + tt * tt);
            sn = tt * c;
          }
        }
        const bool rot = q < b && sn != 0.0;
        pcoef[p] = rot ? c : 1.0; pcoef[32 + p] = rot ? -sn : 0.0; pidx[p] = rot ? q : -1;
        if (q < b) { pcoef[q] = rot ? c : 1.0; pcoef[32 + q] = rot ? sn : 0.0; pidx[q] = rot ? p : -1; }
      }
      __syncwarp();
      #pragma unroll 1
      for (int idx = lane; idx < b * b; idx += 32) {
        const int i = idx / b, j = idx - i * b;
        const int pi = pidx[i], pj = pidx[j];
        const double ci = pcoef[i], si = pcoef[32 + i], cj = pcoef[j], sj = pcoef[32 + j];
        // rows first (new row i = ci T_i + si T_pi), then columns (new col j = cj . + sj .pj)
        const double rij = ci * T[i * 32 + j] + (pi >= 0 ? si * T[pi * 32 + j] : 0.0);
        double v = cj * rij;
        if (pj >= 0) v += sj * (ci * T[i * 32 + pj] + (pi >= 0 ? si * T[pi * 32 + pj] : 0.0));
        T2[i * 32 + j] = v;
        U2[i * 32 + j] = cj * U[i * 32 + j] + (pj >= 0 ? sj * U[i * 32 + pj] : 0.0);
      }
      __syncwarp();
      { double* x = T; T = T2; T2 = x; x = U; U = U2; U2 = x; }
    }
    bool big = false;
    #pragma unroll 1
    for (int idx = lane; idx < b * b; idx += 32) {
      const int i = idx / b, j = idx - i * b;
      if (i != j) {
        const double v = fabs(T[i * 32 + j]);
        big = big || (v > tabs && v > 1e-16 * sqrt(fabs(T[i * 32 + i] * T[j * 32 + j])));
      }
    }
    if (!__any_sync(0xffffffffu, big)) break;
  }
  // sort descending (stable by index)
  double wj = lane < b ? T[lane * 32 + lane] : 0.0;
  int rk = 0;
  #pragma unroll 1
  for (int i = 0; i < b; ++i) {
    const double wi = T[i * 32 + i];
    if (wi > wj || (wi == wj && i < lane)) ++rk;
  }
  __syncwarp();
  if (lane < b) th[rk] = wj;
  // U holds the current eigenvectors: permuted into the caller's buffer (through the other one
  // when that is U itself)
  const double* src = U;
  if (U == Uo) {
    #pragma unroll 1
    for (int idx = lane; idx < b * b; idx += 32) {
      const int i = idx / b, j = idx - i * b;
      U2[i * 32 + j] = U[i * 32 + j];
    }
    __syncwarp();
    src = U2;
  }
  if (lane < b)
    #pragma unroll 1
    for (int i = 0; i < b; ++i) Uo[i * 32 + rk] = src[i * 32 + lane];
  __syncwarp();
}

// Threads [0, nt) of the CTA (nt = 32: warp 0 alone, beside the K^{-1} refinement on the other
// warps; nt = kSST: the whole CTA, synchronised by barrier 0).  The arithmetic of every element
// is the same for any nt (bitwise identical results).
WLR_NOINL void jacobi_par(double* T, double* U, double* th, double* cs, int b, int nt, int* flag) {
  {
    const int lane = threadIdx.x;
    auto sync = [&]() { if (nt == 32) __syncwarp(); else __syncthreads(); };
    const int nb = (b + 1) & ~1;
    const int np = nb / 2;
    #pragma unroll 1
    for (int idx = lane; idx < b * b; idx += nt) {
      const int i = idx / b, j = idx - i * b;
      U[i * 32 + j] = (i == j) ? 1.0 : 0.0;
    }
    double dmax = 0.0;
    #pragma unroll 1
    for (int i = 0; i < b; ++i) dmax = fmax(dmax, fabs(T[i * 32 + i]));
    const double tabs = 2e-15 * dmax;
    sync();
    #pragma unroll 1
    for (int sweep = 0; sweep < 30 && nb > 1; ++sweep) {
      #pragma unroll 1
      for (int rnd = 0; rnd < nb - 1; ++rnd) {
        // rotation parameters of pair (lane) from the current T
        if (lane < np) {
          int p, q;
          if (lane == 0) { p = rnd; q = nb - 1; }
          else { p = (rnd + lane) % (nb - 1); q = (rnd - lane + nb - 1) % (nb - 1); }
          if (p > q) { const int x = p; p = q; q = x; }
          double c = 1.0, sn = 0.0;
          if (q < b) {
            const double apq = T[p * 32 + q], app = T[p * 32 + p], aqq = T[q * 32 + q];
            if (fabs(apq) > tabs && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq))) {
              const double tau = (aqq - app) / (2.0 * apq);
              const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
              c = rsqrt(1.0 + tt * tt);
              sn = tt * c;
            }
          }
          cs[4 * lane + 0] = c; cs[4 * lane + 1] = sn;
          cs[4 * lane + 2] = (double)p; cs[4 * lane + 3] = (double)(q < b && sn != 0.0 ? q : -1);
        }
        sync();
        // rows:  T <- J^T T
        #pragma unroll 1
        for (int idx = lane; idx < np * b; idx += nt) {
          const int kq = idx / b, j = idx - kq * b;
          const int q = (int)cs[4 * kq + 3];
          if (q >= 0) {
            const int p = (int)cs[4 * kq + 2];
            const double c = cs[4 * kq], sn = cs[4 * kq + 1];
            const double tp = T[p * 32 + j], tq = T[q * 32 + j];
            T[p * 32 + j] = c * tp - sn * tq;
            T[q * 32 + j] = sn * tp + c * tq;
          }
        }
        sync();
        // columns: T <- T J, U <- U J
        #pragma unroll 1
        for (int idx = lane; idx < np * b; idx += nt) {
          const int kq = idx / b, i = idx - kq * b;
          const int q = (int)cs[4 * kq + 3];
          if (q >= 0) {
            const int p = (int)cs[4 * kq + 2];
            const double c = cs[4 * kq], sn = cs[4 * kq + 1];
            const double tp = T[i * 32 + p], tq = T[i * 32 + q];
            T[i * 32 + p] = c * tp - sn * tq;
            T[i * 32 + q] = sn * tp + c * tq;
            const double up = U[i * 32 + p], uq = U[i * 32 + q];
            U[i * 32 + p] = c * up - sn * uq;
            U[i * 32 + q] = sn * up + c * uq;
          }
        }
        sync();
      }
      // converged when every off-diagonal is at rounding level
      bool big = false;
      #pragma unroll 1
      for (int idx = lane; idx < b * b; idx += nt) {
        const int i = idx / b, j = idx - i * b;
        if (i != j) {
          const double v = fabs(T[i * 32 + j]);
          big = big || (v > tabs && v > 1e-16 * sqrt(fabs(T[i * 32 + i] * T[j * 32 + j])));
        }
      }
      if (nt == 32) {
        if (!__any_sync(0xffffffffu, big)) break;
      } else {
        if (lane == 0) *flag = 0;
        __syncthreads();
        if (__any_sync(0xffffffffu, big) && (lane & 31) == 0) *flag = 1;
        __syncthreads();
        const bool more = *flag != 0;
        __syncthreads();
        if (!more) break;
      }
    }
    if (lane >= 32) return;                   // (nt = kSST: warp 0 sorts; the caller's barrier follows)
    // sort descending (stable by index) and permute U's columns
    double wj = lane < b ? T[lane * 32 + lane] : 0.0;
    int rk = 0;
    #pragma unroll 1
    for (int i = 0; i < b; ++i) {
      const double wi = T[i * 32 + i];
      if (wi > wj || (wi == wj && i < lane)) ++rk;
    }
    __syncwarp();
    if (lane < b) th[rk] = wj;
    #pragma unroll 1
    for (int i = lane; i < b; i += 32)                          // T is free now
      #pragma unroll 1
      for (int j = 0; j < b; ++j) T[i * 32 + j] = U[i * 32 + j];
    __syncwarp();
    if (lane < b)
      #pragma unroll 1
      for (int i = 0; i < b; ++i) U[i * 32 + rk] = T[i * 32 + lane];
  }
}

// Z[slice] = S X[slice] = G_A[slice, :] X - M(:, slice)^T W   with W = C X (reduced, k x w).
// X is distributed: row l lives in CTA l / SL at smem offset xoff (row stride ldx).  It is
// gathered into Xf (local) when planned, else read through DSMEM.  Split: warp = (ks, js);
// ks takes a chunk of the nk + k reduction index, js a group of columns; lanes own output
// rows (i = lane, lane + 32; nl <= 64).  G_A is symmetric, so G_A[rs + i][l] is read as
// G_A[l][rs + i] (coalesced).  Fixed-order sums.
template <int PW>
WLR_DEVI void s_product_impl(double* smb, int rs, int nl, int SL, int k, int nk, int KS, int JS,
                              int64_t oRed, int64_t oXf, const double* GA, int64_t xoff, int ldx,
                              int w, const double* Wk, const double* Mp, int ldm, double* Z,
                              int ldz, SS* ms = nullptr, const SmallArgs* ma = nullptr, bool pre = false,
                              const double* gay = nullptr) {
  struct { int rs, nl, SL, k, nk; double* sm; } s = {rs, nl, SL, k, nk, smb};
  struct { int KS, JS; } p = {KS, JS};
  cg::cluster_group cl = cg::this_cluster();
  double* Red = s.sm + oRed;
  double* Xf = oXf >= 0 ? s.sm + oXf : nullptr;
  if (Xf && !pre) {   // (pre: Xf already holds the whole basis, loaded from global)
    #pragma unroll 1
    for (int idx0 = threadIdx.x; idx0 < s.nk * w; idx0 += 4 * kSST) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = idx0 + u * kSST;
        v[u] = 0.0;
        if (idx < s.nk * w) {
          const int l = idx / w, j = idx - l * w;
          const int owner = l / s.SL;
          v[u] = cl.map_shared_rank(s.sm, owner)[xoff + (int64_t)(l - owner * s.SL) * ldx + j];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (idx0 + u * kSST < s.nk * w) Xf[idx0 + u * kSST] = v[u];
    }
    __syncthreads();
  }
  if (ms) tmark(*ms, *ma);                        // [p3] X gathered
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ks = warp / p.JS, js = warp - ks * p.JS;
  const int cw = (w + p.JS - 1) / p.JS;
  const int j0 = js * cw;
  const int wj = min(w - j0, cw);                 // columns of this warp (may be <= 0)
  // contraction index l over [G_A rows (n-k) | M' rows (k)]; with G_A X given only the M' rows
  // remain, spread over all the k-split warps
  const int KT = s.nk + s.k, LB = gay ? s.nk : 0;
  const int kc = (KT - LB + p.KS - 1) / p.KS;
  const int l0 = LB + ks * kc, l1 = min(KT, l0 + kc);
  const bool has0 = lane < s.nl, has1 = lane + 32 < s.nl;
  double acc0[PW], acc1[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; }
  if (wj > 0 && gay) {   // G_A X precomputed (the propagation kernel, X = the warm block): its slice
    if (ks == 0)
#pragma unroll
      for (int j = 0; j < PW; ++j)
        if (j < wj) {
          acc0[j] = has0 ? gay[(int64_t)(s.rs + lane) * w + j0 + j] : 0.0;
          acc1[j] = has1 ? gay[(int64_t)(s.rs + lane + 32) * w + j0 + j] : 0.0;
        }
  }
  if (wj > 0) {
    const double* gcol = GA + s.rs;
    const int lg = gay ? 0 : min(l1, s.nk);
#ifndef WLR_SP_U
#define WLR_SP_U 8
#endif
    constexpr int U = WLR_SP_U;                   // G_A loads in flight per lane (per row half)
    #pragma unroll 1
    for (int lb = l0; lb < lg; lb += U) {
      double g0[U], g1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = lb + u;
        const double* grow = gcol + (int64_t)l * s.nk;
        g0[u] = (l < lg && has0) ? __ldg(grow + lane) : 0.0;
        g1[u] = (l < lg && has1) ? __ldg(grow + lane + 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = lb + u;
        if (l < lg) {
          const double* xr;
          if (Xf) {
            xr = Xf + (int64_t)l * w + j0;
          } else {
            const int owner = l / s.SL;
            xr = cl.map_shared_rank(s.sm, owner) + xoff + (int64_t)(l - owner * s.SL) * ldx + j0;
          }
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            if (j < wj) {
              const double x = xr[j];
              acc0[j] = fma(g0[u], x, acc0[j]);
              acc1[j] = fma(g1[u], x, acc1[j]);
            }
          }
        }
      }
    }
    #pragma unroll 1
    for (int l = max(l0, s.nk); l < l1; ++l) {
      const int q = l - s.nk;
      const double m0 = has0 ? Mp[(int64_t)q * ldm + lane] : 0.0;
      const double m1 = has1 ? Mp[(int64_t)q * ldm + lane + 32] : 0.0;
#pragma unroll
      for (int j = 0; j < PW; ++j) {
        if (j < wj) {
          const double x = Wk[q * w + j0 + j];
          acc0[j] = fma(-m0, x, acc0[j]);
          acc1[j] = fma(-m1, x, acc1[j]);
        }
      }
    }
  }
  if (ms) tmark(*ms, *ma);                        // [p4] main loop (warp 0's share)
  if (l0 < l1) {
#pragma unroll
    for (int j = 0; j < PW; ++j) {
      if (j < wj) {
        if (has0) Red[((int64_t)ks * s.SL + lane) * w + j0 + j] = acc0[j];
        if (has1) Red[((int64_t)ks * s.SL + lane + 32) * w + j0 + j] = acc1[j];
      }
    }
  }
  __syncthreads();
  const int nks = (KT - LB + kc - 1) / kc;        // chunks that exist (ks >= nks are empty)
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < s.nl * w; idx += kSST) {
    const int i = idx / w, j = idx - i * w;
    double v = 0.0;
    #pragma unroll 1
    for (int q = 0; q < nks; ++q) v += Red[((int64_t)q * s.SL + i) * w + j];
    Z[i * ldz + j] = v;
  }
  __syncthreads();
}

template <int PW>
WLR_DEVI void s_product(SS& s, const SmallArgs& a, int64_t xoff, int ldx, int w,
                        const double* Wk, const double* Mp, int ldm, double* Z, int ldz, bool pre = false,
                        const double* gay = nullptr) {
  s_product_impl<PW>(s.sm, s.rs, s.nl, s.SL, s.k, s.nk, a.pl.KS, a.pl.JS, a.pl.oRed, a.pl.oXf,
                     a.GA, xoff, ldx, w, Wk, Mp, ldm, Z, ldz, &s, &a, pre, gay);
}

// One S-product of the basis X (local slice at offset xoff, width w = row stride):
// exchange of the C' X partials, then the distributed product into Z (local offset).
template <int PW>
WLR_DEVI void s_apply(SS& s, const SmallArgs& a, const double* Cs, int ldc, const double* Ms,
                      int ldm, int64_t xoff, int w, int64_t zoff, int* nprod, bool pre = false,
                      const double* gay = nullptr) {
  const SSPlan& p = a.pl;
  const double* X = s.sm + xoff;
  double* part = xpart(s, p);
  const TN d[1] = {{Cs, ldc, 1, X, 1, w, s.k, w, part}};
  slice_tn<1>(s.nl, d);
  tmark(s, a);                                 // [p1] C X partials
  double* Wk = s.sm + p.oWk;
  xreduce(s, p, s.k * w, Wk);
  tmark(s, a);                                 // [p2] C X exchange
  s_product<PW>(s, a, xoff, w, w, Wk, Ms, ldm, s.sm + zoff, w, pre, gay);
  ++*nprod;
}

// ---------------------------------------------------------------------------------------
// The kernel, in two parts (template PART):
//   PART 1 (K3a, critical path): Gram update, G'^{-1}, C', eigenpairs of S, and the next row
//          pass's operands (Wt, C V, K^{-1} or C C^T).  Writes V_{p+1}, Ritz values, R = V_p^T
//          V_{p+1} and (V_p^T S V_{p+1})^T for PART 2.
//   PART 2 (K3b, deferred): objective F_{p+1}, step norm, trace and stopping flag.  It only
//          reads state that the next iteration's row pass and increment pass do not touch, so
//          the library runs it on a second stream concurrently with them.
template <int BT, int PART>
__global__ void __launch_bounds__(kSST, 1) small_step_kernel(const __grid_constant__ SmallArgs a) {
  if (a.stop && *a.stop) return;               // (eps mode: latched before the iteration; every CTA of the
                                               //  cluster reads the same value, so none waits at a barrier)
  if (PART == 2 && a.skip && *a.skip) {        // (graph node of a deferred half that already ran)
    cg::this_cluster().sync();                 // every CTA has read the flag
    if (cg::this_cluster().block_rank() == 0 && threadIdx.x == 0) *a.skip = 0;
    return;
  }
  if (PART != 1) pdl_wait();                   // (part 1 waits inside its first load round)
  // a programmatic dependent may start now: the only one is the propagation iteration's row pass,
  // which reads W'_p / X1_p (never this kernel's outputs) and never waits on it
  if (PART == 1) pdl_trigger();
  constexpr int PW = BT <= 8 ? BT : (BT <= 16 ? (BT + 1) / 2 : (BT + 3) / 4);
  extern __shared__ __align__(16) double ss_smem[];
  __shared__ double red[8 * kSSW];
  __shared__ int ok_s;
  __shared__ int kok_s;                        // K^{-1} refined during the first Rayleigh-Ritz
  __shared__ int jflag_s;                      // (Jacobi convergence flag, whole-CTA form)
  const SSPlan& p = a.pl;
  SS s;
  s.CL = p.CL;
  s.c = (int)cg::this_cluster().block_rank();
  s.SL = p.SL;
  s.k = a.k; s.nk = a.nk; s.b = a.b; s.t = a.t;
  s.rs = min(a.nk, s.c * s.SL);
  s.nl = min(a.nk, s.rs + s.SL) - s.rs;
  s.sm = ss_smem;
  s.bank = 0;
  s.nt = 0;
  s.tb = a.tdbg ? a.tdbg + 128 : nullptr;
  s.nx = 0;
  tmark(s, a);
  const int k = a.k, nk = a.nk, b = a.b, t = a.t, kt = k * t, kk = k * k;
  const SmallOff so(b, t, k);
  double* sm = s.sm + p.oSmall;
  const int64_t SLb = (int64_t)s.SL * b;
  const int64_t buf[4] = {p.oBuf, p.oBuf + SLb, p.oBuf + 2 * SLb, p.oBuf + 3 * SLb};
  double* Vp = s.sm + p.oVp;                   // nl x t   V_p (previous V)
  double* Es = s.sm + p.oE;                    // nl x t   E = V' - V_p R
  double* SEs = s.sm + p.oSE;                  // nl x t   S_p E
  // C', M', C_in slice accessors: smem (ld SL) or global (ld nk, offset rs)
  double* Cs = p.oCs >= 0 ? s.sm + p.oCs : a.C_out + s.rs;
  const int ldc = p.oCs >= 0 ? (s.SL | 1) : nk;   // odd: conflict-free column walks
  double* Ms = p.oMs >= 0 ? s.sm + p.oMs : a.M_out + s.rs;
  const int ldm = p.oMs >= 0 ? (s.SL | 1) : nk;
  const double* Cin = p.oCin >= 0 ? s.sm + p.oCin : a.C_in + s.rs;
  const int ldci = p.oCin >= 0 ? (s.SL | 1) : nk;
  const double* incN = a.inc;
  const double* incGam = a.inc + (int64_t)k * nk;
  const double* incOm = incGam + (int64_t)kk;
  double* Gq = p.oGsq >= 0 ? s.sm + p.oGsq : a.gws + (int64_t)s.c * p.gws_stride;
  double* Xq = Gq + kk;
  double* Rq = Xq + kk;
  double* Pq = Rq + kk;
  double* Gx = sm + so.Gx;
  double* th = sm + so.th;
  double* Rt = sm + so.Rt;

  if constexpr (PART == 1) {
    int iY = 0, iZ = 1, iA = 2, iB = 3;        // roles of the four slice buffers
    int nprod = 0;
    long long cyc_jac = 0, cyc_cheb = 0;       // (diagnostics, a.tdbg: cycles in the Jacobi / filter products)
    int n_jac = 0;
    // ---------------------------------------------- A: Gram update, G'^{-1}, C', slices
    // G_A Y of the warm block precomputed by the propagation kernel: the first S-product needs no
    // gathered operand at all; otherwise that operand (the whole Y) is loaded with the state
    const bool use_gay = a.mode && a.GAY != nullptr;
    const bool xf_pre = a.mode && p.oXf >= 0 && !use_gay;
    if (a.mode) {
      // rounds of 4 M' elements, 2 G' elements and 2 each of Y, V_p, G^{-1}_p per thread: every
      // load of a round is issued before its stores (the loops one after the other waited one
      // L2 round trip each)
      const int nM = k * s.nl, nY = s.nl * b, nV = s.nl * t;
      if (xf_pre) {   // the whole warm block Y (n-k x b) into the S-product's gathered operand
        double* Xf = s.sm + p.oXf;
        const int nX = nk * b;
        for (int r0 = 0; r0 < nX; r0 += 8 * kSST) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int idx = r0 + threadIdx.x + u * kSST;
            v[u] = idx < nX ? a.Y[idx] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int idx = r0 + threadIdx.x + u * kSST;
            if (idx < nX) Xf[idx] = v[u];
          }
        }
      }
      for (int r0 = 0; r0 < nM || r0 < 2 * kk || r0 < 2 * nY; r0 += 4 * kSST) {
        double mi[4], mn[4], gv[2][5], yv[2], vv[2], xv[2];
        // the previous state first: it does not depend on the reduce kernel, so under programmatic
        // dependent launch these loads overlap the reduce's tail
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = r0 + threadIdx.x + u * kSST;
          const int q = idx / s.nl, i = idx - q * s.nl;
          mi[u] = idx < nM ? a.M_in[(int64_t)q * nk + s.rs + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int idx = r0 / 2 + threadIdx.x + u * kSST;
          const bool in = idx < kk;
          gv[u][0] = in ? a.G_in[idx] : 0.0;
          xv[u] = in ? a.Gi_in[idx] : 0.0;
          yv[u] = idx < nY ? a.Y[(int64_t)s.rs * b + idx] : 0.0;
          vv[u] = idx < nV ? a.V_in[(int64_t)s.rs * t + idx] : 0.0;
        }
        if (a.snapY) {                                       // (each CTA its slice: all of Y once)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int idx = r0 / 2 + threadIdx.x + u * kSST;
            if (idx < nY) a.snapY[(int64_t)s.rs * b + idx] = yv[u];
          }
        }
        pdl_wait();                                          // the increments of the reduce kernel
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = r0 + threadIdx.x + u * kSST;
          const int q = idx / s.nl, i = idx - q * s.nl;
          mn[u] = idx < nM ? incN[(int64_t)q * nk + s.rs + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int idx = r0 / 2 + threadIdx.x + u * kSST;
          const int i = idx / k, j = idx - i * k;
          const bool in = idx < kk;
          gv[u][1] = in ? incGam[i * k + j] : 0.0;
          gv[u][2] = in ? incGam[j * k + i] : 0.0;
          gv[u][3] = in ? incOm[i * k + j] : 0.0;
          gv[u][4] = in ? incOm[j * k + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = r0 + threadIdx.x + u * kSST;
          if (idx < nM) {
            const int q = idx / s.nl, i = idx - q * s.nl;
            const double mv = mi[u] + mn[u];
            if (p.oMs >= 0) Ms[q * ldm + i] = mv;
            a.M_out[(int64_t)q * nk + s.rs + i] = mv;
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int idx = r0 / 2 + threadIdx.x + u * kSST;
          if (idx < kk) {
            const int i = idx / k, j = idx - i * k;
            const double g = gv[u][0] + gv[u][1] + gv[u][2] + 0.5 * (gv[u][3] + gv[u][4]);
            Gq[idx] = g;
            Xq[idx] = xv[u];
            if (s.c == 0) a.G_out[idx] = g;
            if (s.c == 0 && i == j) sm[so.d0 + i] = gv[u][3];      // diag(Omega) for the gate below
          }
          if (idx < nY) s.sm[buf[iY] + idx] = yv[u];
          if (idx < nV) Vp[idx] = vv[u];
        }
      }
    } else {
    pdl_wait();
    for (int idx = threadIdx.x; idx < k * s.nl; idx += kSST) {
      const int q = idx / s.nl, i = idx - q * s.nl;
      const int64_t gi = (int64_t)q * nk + s.rs + i;
      const double mv = a.M_out[gi];
      if (p.oMs >= 0) Ms[q * ldm + i] = mv;
    }
    for (int idx = threadIdx.x; idx < s.nl * b; idx += kSST) s.sm[buf[iY] + idx] = a.Y[(int64_t)s.rs * b + idx];
    for (int idx = threadIdx.x; idx < kk; idx += kSST) {
      const int i = idx / k, j = idx - i * k;
      double g;
      (void)i; (void)j;
      g = a.G_out[idx];
      Gq[idx] = g;
    }
    }
    __syncthreads();
    if (a.mode && s.c == 0 && threadIdx.x >= kSST - 32) {
      // gate of the next increments: tensor cores when ||dX1||^2 = tr(Omega)
      // <= 1e-6 tr(G') (one warp, beside the inverse)
      double tom = 0.0, tg = 0.0;
      for (int q = threadIdx.x & 31; q < k; q += 32) { tom += sm[so.d0 + q]; tg += Gq[q * k + q]; }
      tom = warp_sum(tom);
      tg = warp_sum(tg);
      if ((threadIdx.x & 31) == 0) a.flags[5] = tom <= 1e-6 * tg ? 1 : 0;
      if (a.dg) {   // Gram propagation: f_w = w^2 ||A1 - X1_{p+1}||^2 = w^2 (||A1||^2 + sum_a dg[a]),
                    // dg[a] = (G_{p+1} - 2 A1^T X1_{p+1})[a][a] from prop2 (fixed-order warp sum)
        double sd = 0.0;
        for (int q = threadIdx.x & 31; q < k; q += 32) sd += __ldcg(a.dg + q);
        sd = warp_sum(sd);
        if ((threadIdx.x & 31) == 0) const_cast<double*>(incOm)[(int64_t)kk] = a.w2 * (a.a1sq + sd);
      }
    }
    tmark(s, a);                               // [1a] Gram update loads
    bool okinv = a.mode ? ns_inverse(Gq, Xq, Rq, Pq, k, red) : false;
    if (!okinv) {
      for (int idx = threadIdx.x; idx < kk; idx += kSST) Xq[idx] = Gq[idx];
      __syncthreads();
      if (!sweep_inverse(Xq, k, 256.0 * kEps, sm + so.d0, sm + so.rb)) {   // rank(X1) < k (R6)
        if (s.c == 0 && threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
        return;                                // uniform on every CTA; no barrier issued yet
      }
    }
    if (s.c == 0)
      for (int idx = threadIdx.x; idx < kk; idx += kSST) a.Gi_out[idx] = Xq[idx];
    if (threadIdx.x == 0) kok_s = 0;
    tmark(s, a);                               // [1] Gram update + G'^{-1}
    // K^{-1}_p (read at the first Gram exchange): its loads are issued before the C' product and
    // stored into the free Newton-Schulz scratch after it
    const bool ki_stage = a.mode && a.uniform;
    double kiv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = threadIdx.x + u * kSST;
      kiv[u] = ki_stage && idx < kk ? a.Ki[idx] : 0.0;
      if (ki_stage && a.snapKi && s.c == 0 && idx < kk) a.snapKi[idx] = kiv[u];
    }
    // C'[:, slice] = G'^{-1} M'[:, slice]
    gemm_nn(k, s.nl, k, Xq, k, Ms, ldm, Cs, ldc, 1.0, false);
    if (ki_stage) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = threadIdx.x + u * kSST;
        if (idx < kk) Pq[idx] = kiv[u];
      }
      for (int idx = threadIdx.x + 2 * kSST; idx < kk; idx += kSST) {   // k > 32
        Pq[idx] = a.Ki[idx];
        if (a.snapKi && s.c == 0) a.snapKi[idx] = Pq[idx];
      }
    }
    __syncthreads();
    if (p.oCs >= 0)
      for (int idx = threadIdx.x; idx < k * s.nl; idx += kSST) {
        const int q = idx / s.nl, i = idx - q * s.nl;
        a.C_out[(int64_t)q * nk + s.rs + i] = Cs[q * ldc + i];
      }
    tmark(s, a);                               // [2] C'

    // ---------------------------------------------- B: eigenpairs of S
    const double floor_abs = 4.0 * kEps * sqrt((double)nk) * a.a2sq;   // S-product rounding floor
    bool converged = false, failed = false;
    int outer = 0;
    double rmax = 0.0;
    double* dsc = sm + so.dsc;
    double* rres = s.sm + p.oCinE;             // residuals (t)
    bool ortho = !a.cold;                      // Y expected orthonormal (warm Ritz block)
    while (true) {
      // ---- Rayleigh-Ritz on span(Y):  Z = S Y;  Gyy = Y^T Y, Gyz = Y^T Z (generalised RR)
      s_apply<PW>(s, a, Cs, ldc, Ms, ldm, buf[iY], b, buf[iZ], &nprod, (xf_pre || use_gay) && outer == 0,
                  use_gay && outer == 0 ? a.GAY : nullptr);
      tmark(s, a);                             // product
      {
        const double* Y = s.sm + buf[iY];
        const double* Z = s.sm + buf[iZ];
        double* part = xpart(s, p);
        const int tb = a.mode ? t : 0;
        // first pass: C'C'^T rides along (K = w^2 I + C'C'^T of the next row update) into Gq
        // (through global memory when the exchange bank cannot hold it)
        const int kc = outer == 0 ? k : 0;
        const int lg = 2 * b * b + 2 * tb * b;
        const TN d[5] = {{Y, 1, b, Y, 1, b, b, b, part},
                         {Y, 1, b, Z, 1, b, b, b, part + b * b},
                         {Vp, 1, t, Y, 1, b, tb, b, part + 2 * b * b},
                         {Vp, 1, t, Z, 1, b, tb, b, part + 2 * b * b + t * b},
                         {Cs, ldc, 1, Cs, ldc, 1, kc, k, p.ccx ? part + lg : a.xchg + (int64_t)s.c * p.flen}};
        slice_tn<5>(s.nl, d);
        tmark(s, a);                           // [4a] Gram partials
        xreduce(s, p, lg, Gx, p.ccx ? kc * k : 0, Gq);
        tmark(s, a);                           // [4b] exchange
        if (kc && !p.ccx && !a.uniform) {
          // non-uniform W1: C'C'^T (the row solves' K = C'C'^T + diag(W1^2), next iteration) is only
          // stored: every CTA sums its share of the entries over the cluster's global partials
          // (fixed order), no CTA needs the whole matrix here
          const int e0 = (int)((int64_t)kk * s.c / s.CL), e1 = (int)((int64_t)kk * (s.c + 1) / s.CL);
          #pragma unroll 1
          for (int idx = e0 + threadIdx.x; idx < e1; idx += kSST) {
            const int i = idx / k, j = idx - i * k;
            double v = 0.0;
            for (int c = 0; c < s.CL; ++c)
              v += 0.5 * (__ldcg(a.xchg + (int64_t)c * p.flen + idx) + __ldcg(a.xchg + (int64_t)c * p.flen + j * k + i));
            if (a.dtype) reinterpret_cast<double*>(a.Kop)[idx] = v;
            else reinterpret_cast<float*>(a.Kop)[idx] = (float)v;
            if (a.Sop) a.Sop[i * ((k + 7) & ~7) + j] = (float)v;
          }
        } else if (kc) {
          #pragma unroll 1
          for (int idx = threadIdx.x; idx < kk; idx += kSST) {
            const int i = idx / k, j = idx - i * k;
            double v = 0.0;
            if (p.ccx) {
              v = 0.5 * (Gq[idx] + Gq[j * k + i]);
            } else {
              for (int c = 0; c < s.CL; ++c)
                v += 0.5 * (__ldcg(a.xchg + (int64_t)c * p.flen + idx) + __ldcg(a.xchg + (int64_t)c * p.flen + j * k + i));
            }
            Rq[idx] = v;                       // symmetrised C'C'^T
          }
          __syncthreads();
          #pragma unroll 1
          for (int idx = threadIdx.x; idx < kk; idx += kSST) {
            const int i = idx / k, j = idx - i * k;
            const double v = Rq[idx];
            if (!a.uniform && s.c == 0) {
              if (a.dtype) reinterpret_cast<double*>(a.Kop)[idx] = v;
              else reinterpret_cast<float*>(a.Kop)[idx] = (float)v;
              if (a.Sop) a.Sop[i * ((k + 7) & ~7) + j] = (float)v;
            }
            Gq[idx] = v + (i == j ? a.w2 : 0.0);
            if (a.mode && a.uniform) Xq[idx] = Pq[idx];   // K^{-1}_p (staged after C')
          }
          __syncthreads();
        }
      }
      tmark(s, a);                             // Gram exchange
      // ---- local (every CTA identically): D = diag(Gyy)^-1/2; if D Gyy D = I to rounding
      //      the block is orthonormal: T = D Gyz D, Q = D U.  Otherwise L L^T = D Gyy D,
      //      T = L^-1 (D Gyz D) L^-T, Q = D L^-T U.
      bool gen;
      {
        double* Lb = sm + so.Lb;
        double* Li = sm + so.Li;
        double* Tb = sm + so.Tb;
        double* Ub = sm + so.Ub;
        double* Qb = sm + so.Qb;
        double* Wb = sm + so.Wb;
        if (threadIdx.x < b) {
          const double d = Gx[threadIdx.x * b + threadIdx.x];
          dsc[threadIdx.x] = d > 0.0 ? rsqrt(d) : 1.0;
        }
        __syncthreads();
        double dev = 0.0;
        for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
          const int i = idx / b, j = idx - i * b;
          const double di = dsc[i] * dsc[j];
          const double g = 0.5 * (Gx[i * b + j] + Gx[j * b + i]) * di;
          Lb[i * 32 + j] = g;
          Wb[i * 32 + j] = 0.5 * (Gx[b * b + i * b + j] + Gx[b * b + j * b + i]) * di;
          if (i != j) dev = fmax(dev, fabs(g));
        }
        dev = block_max(dev, red);
        tmark(s, a);                           // (RR: scaled Grams)
        gen = !(ortho && dev < 1e-13);
        if (gen) {
          if (!chol_small(Lb, b, sm + so.rb, &ok_s)) { failed = true; break; }
          tri_inverse(Lb, sm + so.rb, b, Li);
          for (int idx = threadIdx.x; idx < b * b; idx += kSST) {   // Ub = Li Wb
            const int i = idx / b, j = idx - i * b;
            double v = 0.0;
            for (int q = 0; q <= i; ++q) v = fma(Li[i * 32 + q], Wb[q * 32 + j], v);
            Ub[i * 32 + j] = v;
          }
          __syncthreads();
          for (int idx = threadIdx.x; idx < b * b; idx += kSST) {   // Tb = Ub Li^T
            const int i = idx / b, j = idx - i * b;
            double v = 0.0;
            for (int q = 0; q <= j; ++q) v = fma(Ub[i * 32 + q], Li[j * 32 + q], v);
            Tb[i * 32 + j] = v;
          }
          __syncthreads();
          for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
            const int i = idx / b, j = idx - i * b;
            if (i < j) {
              const double v = 0.5 * (Tb[i * 32 + j] + Tb[j * 32 + i]);
              Tb[i * 32 + j] = v;
              Tb[j * 32 + i] = v;
            }
          }
        } else {
          for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
            const int i = idx / b, j = idx - i * b;
            Tb[i * 32 + j] = Wb[i * 32 + j];
          }
        }
        __syncthreads();
        const long long tj0 = a.tdbg ? clock64() : 0;
        // warp 0: Jacobi; warps 1..: K^{-1} by Newton-Schulz from the previous one (first pass);
        // otherwise the whole CTA runs the Jacobi
        const bool ki_side = outer == 0 && a.uniform && a.mode;
        const int jnt = ki_side || b <= 4 ? 32 : kSST;
        if (threadIdx.x < jnt) {
          if (jnt == 32) jacobi_warp(Tb, Ub, Wb, sm + so.Qb, th, sm + so.Lb, b);   // (Wb, Qb, Lb free here)
          else jacobi_par(Tb, Ub, th, sm + so.cs, b, jnt, &jflag_s);
          if (a.tdbg && threadIdx.x == 0 && s.c == 0) a.tdbg[245] = (double)(clock64() - tj0);
        } else if (ki_side) {
          // warps 1..: K^{-1} by Newton-Schulz from the previous one
          const bool okk = ns_inverse(Gq, Xq, Rq, Pq, k, red + 32, 32, kSST - 32, 1);
          if (threadIdx.x == 32) kok_s = okk ? 1 : 0;
          if (a.tdbg && threadIdx.x == 32 && s.c == 0) a.tdbg[246] = (double)(clock64() - tj0);
        }
        __syncthreads();
        if (a.tdbg) { cyc_jac += clock64() - tj0; ++n_jac; }
        tmark(s, a);                           // (RR: Jacobi || K^{-1})
        for (int idx = threadIdx.x; idx < b * b; idx += kSST) {     // Qb = D (Li^T U) or D U
          const int i = idx / b, j = idx - i * b;
          double v;
          if (gen) {
            v = 0.0;
            for (int q = i; q < b; ++q) v = fma(Li[q * 32 + i], Ub[q * 32 + j], v);
          } else {
            v = Ub[i * 32 + j];
          }
          Qb[i * b + j] = v * dsc[i];
        }
        __syncthreads();
      }
      tmark(s, a);                             // local RR
      const double* Qb = sm + so.Qb;
      // ---- rotate: Y' = Y Q, Z' = Z Q  (into the free buffers)
      gemm_nn(s.nl, b, b, s.sm + buf[iY], b, Qb, b, s.sm + buf[iA], b, 1.0, false);
      gemm_nn(s.nl, b, b, s.sm + buf[iZ], b, Qb, b, s.sm + buf[iB], b, 1.0, false);
      {
        const int oy = iY, oz = iZ;
        iY = iA; iZ = iB; iA = oy; iB = oz;
      }
      __syncthreads();
      // ---- residuals of the wanted pairs
      {
        const double* Y = s.sm + buf[iY];
        const double* Z = s.sm + buf[iZ];
        double* part = xpart(s, p);
        {   // one warp per wanted pair (the last warps: the C'V' tiles below start on the first ones)
          const int wq = kSSW - 1 - (threadIdx.x >> 5), ln = threadIdx.x & 31;
          #pragma unroll 1
          for (int j = wq; j < t; j += kSSW) {
            double v = 0.0;
            for (int r = ln; r < s.nl; r += 32) {
              const double d = Z[r * b + j] - th[j] * Y[r * b + j];
              v = fma(d, d, v);
            }
            v = warp_sum(v);
            if (ln == 0) part[j] = v;
          }
        }
        // C'V' (k x t) partials ride along: valid at every exit of this loop (it only leaves
        // right after this exchange), so the operands need no exchange of their own
        const TN d[1] = {{Cs, ldc, 1, Y, 1, b, k, t, part + t}};
        slice_tn<1>(s.nl, d);
        xreduce(s, p, t, rres, kt, rres + t);
      }
      tmark(s, a);                             // residual exchange
      rmax = 0.0;
      for (int j = 0; j < t; ++j) rmax = fmax(rmax, sqrt(fmax(rres[j], 0.0)));
      const double theta0 = th[0];
      const double target = fmax(a.tol * fabs(theta0), floor_abs);
      if (rmax <= target) { converged = true; break; }
      if (++outer > a.max_outer) break;
      // ---- Chebyshev filter of adaptive degree damping [0, theta_{b-1}]
      const double beta = th[b - 1];
      double cc = 0.5 * beta, ee = 0.5 * beta;
      int d = 1;
      if (!(beta > 1e-300 * fabs(theta0)) || beta >= th[t - 1]) {
        cc = 0.0; ee = 1.0; d = 1;              // no gap inside the block: plain power step
      } else {
        const double x0 = (theta0 - cc) / ee, xt = (th[t - 1] - cc) / ee;
        // acosh(x) = log(x + sqrt(x^2 - 1)) for x >= 1
        const double xtc = fmax(xt, 1.0), x0c = fmax(x0, 1.0);
        const double at = log(xtc + sqrt(xtc * xtc - 1.0)), a0 = log(x0c + sqrt(x0c * x0c - 1.0));
        const double need = log(fmax(rmax / target, 1.0)) / fmax(at, 1e-6);
        d = (int)ceil(need) + 1;
        const int dcap = max(1, (int)(9.9 / fmax(a0, 1e-6)));   // amplification <= ~1e4
        d = max(1, min(d, min(a.max_deg, dcap)));
      }
      const double einv = 1.0 / ee;
      int i0 = iY, i1 = iA, iz = iZ, i3 = iB;   // P0 = Y, P1 = (Z - c Y)/e, scratch z, free
      {
        double* P1 = s.sm + buf[i1];
        const double* Y = s.sm + buf[i0];
        const double* Z = s.sm + buf[iz];
        for (int idx = threadIdx.x; idx < s.nl * b; idx += kSST) P1[idx] = (Z[idx] - cc * Y[idx]) * einv;
        __syncthreads();
      }
      for (int j = 2; j <= d; ++j) {
        const long long tc0 = a.tdbg ? clock64() : 0;
        s_apply<PW>(s, a, Cs, ldc, Ms, ldm, buf[i1], b, buf[iz], &nprod);
        if (a.tdbg) cyc_cheb += clock64() - tc0;
        double* pn = s.sm + buf[i0];           // P2 = 2 (S P1 - c P1)/e - P0, in place of P0
        const double* pz = s.sm + buf[iz];
        const double* p1 = s.sm + buf[i1];
        for (int idx = threadIdx.x; idx < s.nl * b; idx += kSST)
          pn[idx] = 2.0 * (pz[idx] - cc * p1[idx]) * einv - pn[idx];
        __syncthreads();
        const int tmp = i0; i0 = i1; i1 = tmp;
      }
      iY = i1; iZ = iz; iA = i0; iB = i3;
      ortho = false;                           // filtered block: generalised Rayleigh-Ritz
    }
    if ((failed || !converged) && s.c == 0 && threadIdx.x == 0) raise_flag(a.flags, DF_EIG);
    if (failed) {          // every CTA took the same decision; keep peers' smem alive
      cg::this_cluster().sync();
      return;
    }
    // ---------------------------------------------- C: operands of the next row pass
    // Linear row update: Wt = [w^2 K^{-1}; U K^{-1}; P K^{-1}] for uniform W1,
    // [0; U; P] otherwise, with U = C'^T - V' (C'V')^T, P = (C'V')(C'V')^T, K = w^2 I + C'C'^T.
    const double* Y = s.sm + buf[iY];          // V' = Y[:, :t]
    double* cvs = rres + t;                    // k x t  C'V', summed with the last residuals
    for (int idx = threadIdx.x; idx < s.nl * t; idx += kSST) {
      const int r = idx / t, j = idx - r * t;
      a.V_out[(int64_t)(s.rs + r) * t + j] = Y[r * b + j];
    }
    for (int idx = threadIdx.x; idx < s.nl * b; idx += kSST) a.Y[(int64_t)s.rs * b + idx] = Y[idx];
    tmark(s, a);                               // operand partials
    tmark(s, a);                               // (C'V' came with the residual exchange)
    if (s.c == 0)
      for (int idx = threadIdx.x; idx < kt; idx += kSST) a.CV_out[idx] = cvs[idx];
    tmark(s, a);                               // [8a] C'V' summed
    if (a.uniform) {
      if (!kok_s) {   // init, or the warm start was too far: sweep K^{-1} from K (still in Gq)
        for (int idx = threadIdx.x; idx < kk; idx += kSST) Xq[idx] = Gq[idx];
        __syncthreads();
        if (!sweep_inverse(Xq, k, 0.0, sm + so.d0, sm + so.rb)) {
          if (s.c == 0 && threadIdx.x == 0) raise_flag(a.flags, DF_ROWSPD);
          cg::this_cluster().sync();
          return;
        }
      }
      if (s.c == 0)
        for (int idx = threadIdx.x; idx < kk; idx += kSST) a.Ki[idx] = Xq[idx];
    }
    tmark(s, a);                               // [8b] K^{-1} (fallback only)
    // U rows of this slice: u[c][q] = C'[q][c] - sum_j V'[c][j] (C'V')[q][j]   (into Red);
    // Qt = (C'V')^T K^{-1} (t x k, uniform) for the X1_p rows, after Us
    double* Us = s.sm + p.oRed;                // nl x k
    double* Qt = Us + (int64_t)s.nl * k;       // t x k
#pragma unroll 1
    for (int idx = threadIdx.x; idx < s.nl * k; idx += kSST) {
      const int c = idx / k, q = idx - c * k;
      double v = Cs[(int64_t)q * ldc + c];
      for (int j = 0; j < t; ++j) v = fma(-Y[c * b + j], cvs[q * t + j], v);
      Us[idx] = v;
    }
    if (a.uniform)
#pragma unroll 1
      for (int idx = threadIdx.x; idx < kt; idx += kSST) {
        const int i = idx / k, l = idx - i * k;
        double v0 = 0.0, v1 = 0.0;
        int q = 0;
        for (; q + 1 < k; q += 2) {
          v0 = fma(cvs[q * t + i], Xq[q * k + l], v0);
          v1 = fma(cvs[(q + 1) * t + i], Xq[(q + 1) * k + l], v1);
        }
        if (q < k) v0 = fma(cvs[q * t + i], Xq[q * k + l], v0);
        Qt[idx] = v0 + v1;
      }
    __syncthreads();
    tmark(s, a);                               // (W': U rows, Qt)
    const int RP = a.rp;
    auto put = [&](int64_t row, int l, double v) {
      const int64_t o = row * RP + l;
      if (a.dtype) reinterpret_cast<double*>(a.Wt)[o] = v;
      else reinterpret_cast<float*>(a.Wt)[o] = (float)v;
      if (a.WtT) {   // K-major fp32 copy W'^T and its 3xTF32 low part (tensor-core row pass)
        float hi, lo;
        tf32_split((float)v, hi, lo);          // 3xTF32 operand pair (umma.cuh)
        float* wt = reinterpret_cast<float*>(a.WtT) + (int64_t)l * a.KW + row;
        wt[0] = hi;
        wt[(int64_t)RP * a.KW] = lo;
      }
    };
    // Wt rows k + rs + c (columns of A2 in this slice): u K^{-1} (FP64 tensor cores, into the free
    // gathered-operand region) or u; then the stores, each array in its coalesced order
    const double* Pw = Us;
    if (a.uniform) {
      double* scr = p.oXf >= 0 && (int64_t)nk * b >= (int64_t)s.nl * k ? s.sm + p.oXf : nullptr;
      if (scr) {
        gemm_tc(s.nl, k, k, Us, k, 1, Xq, k, 1, scr, k, 1.0, false);
        __syncthreads();
        Pw = scr;
      }
    }
#pragma unroll 1
    for (int idx = threadIdx.x; idx < s.nl * k; idx += kSST) {
      const int c = idx / k, l = idx - c * k;
      double v;
      if (a.uniform && Pw == Us) {
        const double* ur = Us + c * k;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int q = 0;
        for (; q + 3 < k; q += 4) {
          v0 = fma(ur[q], Xq[q * k + l], v0);
          v1 = fma(ur[q + 1], Xq[(q + 1) * k + l], v1);
          v2 = fma(ur[q + 2], Xq[(q + 2) * k + l], v2);
          v3 = fma(ur[q + 3], Xq[(q + 3) * k + l], v3);
        }
        for (; q < k; ++q) v0 = fma(ur[q], Xq[q * k + l], v0);
        v = (v0 + v1) + (v2 + v3);
      } else {
        v = Pw[idx];
      }
      const int64_t o = (int64_t)(k + s.rs + c) * RP + l;      // row-major W' (c-major: coalesced)
      if (a.dtype) reinterpret_cast<double*>(a.Wt)[o] = v;
      else reinterpret_cast<float*>(a.Wt)[o] = (float)v;
    }
    if (a.WtT) {
      if (a.uniform && Pw == Us) __syncthreads();
#pragma unroll 1
      for (int idx = threadIdx.x; idx < s.nl * k; idx += kSST) {   // W'^T (l-major: coalesced)
        const int l = idx / s.nl, c = idx - l * s.nl;
        double v;
        if (Pw != Us || !a.uniform) {
          v = Pw[c * k + l];
        } else {   // (no scratch region: recompute u K^{-1})
          const double* ur = Us + c * k;
          v = 0.0;
          for (int q = 0; q < k; ++q) v = fma(ur[q], Xq[q * k + l], v);
        }
        float hi, lo;
        tf32_split((float)v, hi, lo);
        float* wt = reinterpret_cast<float*>(a.WtT) + (int64_t)l * a.KW + k + s.rs + c;
        wt[0] = hi;
        wt[(int64_t)RP * a.KW] = lo;
      }
    }
    tmark(s, a);                               // (W': A2 rows)
    // A1 rows (uniform: w^2 K^{-1}) and X1_p rows (P K^{-1} = (C'V') Qt, or P = (C'V')(C'V')^T),
    // spread over the cluster: output o of [0, 2 k^2) on CTA o mod CL
#pragma unroll 1
    for (int o = s.c + s.CL * threadIdx.x; o < 2 * kk; o += s.CL * kSST) {
      const int blk = o / kk, idx = o - blk * kk, j = idx / k, l = idx - j * k;
      if (blk == 0) {
        if (a.uniform) put(j, l, a.w2 * Xq[idx]);
      } else {
        double v = 0.0;
        for (int i = 0; i < t; ++i) v = fma(cvs[j * t + i], a.uniform ? Qt[i * k + l] : cvs[l * t + i], v);
        put(a.KA + j, l, v);
      }
    }
    tmark(s, a);                               // [8c] Wt rows
    if (s.c != 0) return;
    // ---- CTA 0: small results for the deferred half
    if (a.mode) {
      const double* Qb = sm + so.Qb;
      for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
        const int i = idx / t, j = idx - i * t;
        double r = 0.0, z = 0.0;     // R = (Vp^T Y) Q[:, :t];  ZnV[i][j] = sum_q VpZ[j][q] Q[q][i]
        for (int q = 0; q < b; ++q) {
          r = fma(Gx[2 * b * b + i * b + q], Qb[q * b + j], r);
          z = fma(Gx[2 * b * b + t * b + j * b + q], Qb[q * b + i], z);
        }
        a.k3x[idx] = r;
        a.k3x[t * t + idx] = z;
      }
    }
    for (int j = threadIdx.x; j < b; j += kSST) a.th_out[j] = th[j];
    if (threadIdx.x == 0) {
      if (a.tdbg) {
        a.tdbg[240] = (double)cyc_jac; a.tdbg[241] = (double)n_jac; a.tdbg[242] = (double)cyc_cheb;
        a.tdbg[243] = (double)nprod; a.tdbg[244] = (double)outer;
      }
      a.scal[6] = rmax / fabs(th[0]);
      a.scal[7] = (double)nprod;
      a.flags[3] = outer;
    }
    tmark(s, a);                               // operands
  } else {
    // ================================== PART 2: objective, step norm, trace (deferred)
    const double fw = a.mode ? incOm[(int64_t)kk] : a.inc[0];
    double* Vn = s.sm + p.oBuf;                // nl x t  V_{p+1} (buffer 0)
    const bool ms3 = p.oMat3 >= 0 && a.mode;
    double* mats = s.sm + (p.oMat3 >= 0 ? p.oMat3 : 0);
    if (ms3) {
      for (int idx = threadIdx.x; idx < kk; idx += kSST) {
        mats[idx] = a.G_in[idx];
        mats[kk + idx] = incGam[idx];
        mats[2 * kk + idx] = incOm[idx];
      }
      for (int idx = threadIdx.x; idx < kt; idx += kSST) mats[3 * kk + idx] = a.CV_in[idx];
    }
    const double* Gm = ms3 ? mats : a.G_in;
    const double* Gam = ms3 ? mats + kk : incGam;
    const double* Om = ms3 ? mats + 2 * kk : incOm;
    const double* CVp = ms3 ? mats + 3 * kk : a.CV_in;
    // slices of C', M', C_in and V', V_p in rounds: every load of a round before its stores
    for (int r0 = 0; r0 < k * s.nl; r0 += 4 * kSST) {
      double cv[4], mv[4], ci[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = r0 + threadIdx.x + u * kSST;
        const int q = idx / s.nl, i = idx - q * s.nl;
        const int64_t gi = (int64_t)q * nk + s.rs + i;
        const bool in = idx < k * s.nl;
        cv[u] = in && p.oCs >= 0 ? a.C_out[gi] : 0.0;
        mv[u] = in && p.oMs >= 0 ? a.M_out[gi] : 0.0;
        ci[u] = in && p.oCin >= 0 && a.mode ? a.C_in[gi] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = r0 + threadIdx.x + u * kSST;
        if (idx >= k * s.nl) continue;
        const int q = idx / s.nl, i = idx - q * s.nl;
        if (p.oCs >= 0) Cs[q * ldc + i] = cv[u];
        if (p.oMs >= 0) Ms[q * ldm + i] = mv[u];
        if (p.oCin >= 0 && a.mode) s.sm[p.oCin + q * ldci + i] = ci[u];
      }
    }
    for (int r0 = 0; r0 < s.nl * t; r0 += 2 * kSST) {
      double vn[2], vp[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = r0 + threadIdx.x + u * kSST;
        const bool in = idx < s.nl * t;
        vn[u] = in ? a.V_out[(int64_t)s.rs * t + idx] : 0.0;
        vp[u] = in && a.mode ? a.V_in[(int64_t)s.rs * t + idx] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = r0 + threadIdx.x + u * kSST;
        if (idx >= s.nl * t) continue;
        Vn[idx] = vn[u];
        if (a.mode) Vp[idx] = vp[u];
      }
    }
    if (threadIdx.x < t * t && a.mode) Rt[threadIdx.x] = a.k3x[threadIdx.x];
    __syncthreads();
    if (a.mode) {
      // E = V' - Vp R (slice), C_in E partial -> exchange -> S_p E = G_A E - M_in^T (C_in E)
      for (int idx = threadIdx.x; idx < s.nl * t; idx += kSST) {
        const int r = idx / t, j = idx - r * t;
        double v = Vn[idx];
        for (int q = 0; q < t; ++q) v = fma(-Vp[r * t + q], Rt[q * t + j], v);
        Es[idx] = v;
      }
      __syncthreads();
      double* part = xpart(s, p);
      const TN d[1] = {{Cin, ldci, 1, Es, 1, t, k, t, part}};
      slice_tn<1>(s.nl, d);
      double* CinE = s.sm + p.oCinE;
      xreduce(s, p, kt, CinE);
      s_product<PW>(s, a, p.oE, t, t, CinE, a.M_in + s.rs, nk, SEs, t);
    }
    tmark(s, a);                               // old-S product
    const FinOff fo(k, t);
    double* my = a.xchg + (int64_t)s.c * p.flen;
    {
      // [0] <M',C'> [1] <C', H C_in> [2] <C', Om C'> [3] <C', Gam dC> [4] <dC, G dC>, the last
      // four through k x k slice Grams (FP64 tensor cores): <X, Y Z> over the slice =
      // sum_{l,q} Y[l][q] (X Z^T)[l][q] with X Z^T = C' C_in^T, C' C'^T, C' dC^T, dC dC^T
      double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int idx = threadIdx.x; idx < k * s.nl; idx += kSST) {
        const int l = idx / s.nl, i = idx - l * s.nl;
        v[0] = fma(Ms[(int64_t)l * ldm + i], Cs[(int64_t)l * ldc + i], v[0]);
      }
      if (a.mode && 4 * kk <= 6 * 1024) {
        double* dC = s.sm + p.oRed;              // k x nl (the S-product's partials are consumed)
        for (int idx = threadIdx.x; idx < k * s.nl; idx += kSST) {
          const int l = idx / s.nl, i = idx - l * s.nl;
          dC[idx] = Cs[(int64_t)l * ldc + i] - Cin[(int64_t)l * ldci + i];
        }
        __syncthreads();
        double* gr = sm + so.Tb;                  // 4 x k x k (the local RR blocks are free here)
        const TN d[4] = {{Cs, ldc, 1, Cin, ldci, 1, k, k, gr},
                         {Cs, ldc, 1, Cs, ldc, 1, k, k, gr + kk},
                         {Cs, ldc, 1, dC, s.nl, 1, k, k, gr + 2 * kk},
                         {dC, s.nl, 1, dC, s.nl, 1, k, k, gr + 3 * kk}};
        slice_tn<4>(s.nl, d);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kk; idx += kSST) {
          const int l = idx / k, q = idx - l * k;
          const double gm = Gm[idx], gam = Gam[idx];
          v[1] = fma(gm + gam, gr[idx], v[1]);
          v[2] = fma(0.5 * (Om[idx] + Om[q * k + l]), gr[kk + idx], v[2]);
          v[3] = fma(gam, gr[2 * kk + idx], v[3]);
          v[4] = fma(gm, gr[3 * kk + idx], v[4]);
        }
      } else if (a.mode) {   // k > 39: the k x k Grams do not fit the scratch; per-element sums
        for (int idx = threadIdx.x; idx < k * s.nl; idx += kSST) {
          const int l = idx / s.nl, i = idx - l * s.nl;
          const double cn = Cs[(int64_t)l * ldc + i];
          double hc = 0.0, omc = 0.0, gdc = 0.0, ggdc = 0.0;
          for (int q = 0; q < k; ++q) {
            const double co = Cin[(int64_t)q * ldci + i], cq = Cs[(int64_t)q * ldc + i];
            const double dq = cq - co;
            const double gam = Gam[l * k + q], gm = Gm[l * k + q];
            hc = fma(gm + gam, co, hc);
            omc = fma(0.5 * (Om[l * k + q] + Om[q * k + l]), cq, omc);
            gdc = fma(gam, dq, gdc);
            ggdc = fma(gm, dq, ggdc);
          }
          const double dl = cn - Cin[(int64_t)l * ldci + i];
          v[1] = fma(cn, hc, v[1]);
          v[2] = fma(cn, omc, v[2]);
          v[3] = fma(cn, gdc, v[3]);
          v[4] = fma(dl, ggdc, v[4]);
        }
      }
      block_sum_n<5>(v, red);
      if (threadIdx.x == 0)
        for (int u = 0; u < 5; ++u) my[u] = v[u];
    }
    {
      const int km = a.mode ? k : 0, tm = a.mode ? t : 0;
      const TN d[9] = {{Cs, ldc, 1, Vp, 1, t, km, t, my + fo.CnV},
                       {Cs, ldc, 1, Vn, 1, t, k, t, my + fo.CnVn},
                       {Cin, ldci, 1, Vn, 1, t, km, t, my + fo.CVn},
                       {Ms, ldm, 1, Vp, 1, t, km, t, my + fo.MnV},
                       {a.M_in + s.rs, nk, 1, Vn, 1, t, km, t, my + fo.MVn},
                       {incN + s.rs, nk, 1, Vp, 1, t, km, t, my + fo.NV},
                       {Cs, ldc, 1, Es, 1, t, km, t, my + fo.CE},
                       {Es, 1, t, Es, 1, t, tm, t, my + fo.EE},
                       {Es, 1, t, SEs, 1, t, tm, t, my + fo.ESE}};
      slice_tn<9>(s.nl, d);
      if (!a.mode)
        for (int idx = threadIdx.x; idx < fo.CC; idx += kSST)
          if (idx >= fo.CnV && (idx < fo.CnVn || idx >= fo.CnVn + kt)) my[idx] = 0.0;
    }
    tmark(s, a);                               // final partials
    cg::this_cluster().sync();
    {   // reduce-scatter of the 5 + 7kt + 2t^2 partials
      const int flen = fo.CC;
      const int fc = (flen + s.CL - 1) / s.CL;
      const int f0 = s.c * fc, f1 = min(flen, f0 + fc);
      for (int i = f0 + threadIdx.x; i < f1; i += kSST) {
        double v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = c < s.CL ? __ldcg(a.xchg + (int64_t)c * p.flen + i) : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) acc += v[c];
        a.red[i] = acc;
      }
    }
    cg::this_cluster().sync();
    tmark(s, a);                               // reduce-scatter
    if (s.c != 0) return;
    // ---- CTA 0: F, step norm, trace
    const bool rsm = p.oTail >= 0;
    double* R = rsm ? s.sm + p.oTail : a.red;
    if (rsm)
      for (int i = threadIdx.x; i < fo.CC; i += kSST) R[i] = __ldcg(a.red + i);
    double* HCV = R + p.flen;                  // k x t
    double* HCVn = HCV + kt;                   // k x t
    double* Wm = HCVn + kt;                    // k x t
    double* ZnV = sm + so.Tb;                  // t x t
    if (threadIdx.x < t * t && a.mode) ZnV[threadIdx.x] = a.k3x[t * t + threadIdx.x];
    __syncthreads();
    // sum of the Ritz values, tr(G'), tr(Omega): one warp, lanes over the index (a serial loop
    // of dependent global loads per thread cost several microseconds here)
    __shared__ double tr3[3];
    if (threadIdx.x < 32) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int j = threadIdx.x; j < t; j += 32) s0 += a.th_out[j];
      for (int i = threadIdx.x; i < k; i += 32) {
        s1 += a.G_out[i * k + i];
        if (a.mode) s2 += Om[i * k + i];
      }
      s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
      if (threadIdx.x == 0) { tr3[0] = s0; tr3[1] = s1; tr3[2] = s2; }
    }
    __syncthreads();
    const double sum_theta = tr3[0], trG = tr3[1];
    const double x2sq_new = R[0] + sum_theta;
    const double F = fw + a.a2sq - R[0] - sum_theta;
    double step = -1.0, rel = -1.0;
    if (a.mode) {
      for (int idx = threadIdx.x; idx < kt; idx += kSST) {
        const int l = idx / t, j = idx - l * t;
        double h1 = 0.0, h2 = 0.0;
        for (int q = 0; q < k; ++q) {
          const double hq = Gm[l * k + q] + Gam[l * k + q];
          h1 = fma(hq, CVp[q * t + j], h1);
          h2 = fma(hq, R[fo.CVn + q * t + j], h2);
        }
        HCV[idx] = h1;
        HCVn[idx] = h2;
      }
      __syncthreads();
      // (a) exact Gram identity   (b) first-order expansion (small steps; no cancellation)
      double v[2] = {0.0, 0.0};
      for (int idx = threadIdx.x; idx < kt; idx += kSST) {
        v[0] -= R[fo.CnV + idx] * HCV[idx] + R[fo.CnVn + idx] * HCVn[idx];
        v[0] += R[fo.MVn + idx] * R[fo.CVn + idx] + R[fo.MnV + idx] * R[fo.CnV + idx];
        const int l = idx / t, j = idx - l * t;
        double om = 0.0, gd = 0.0, gg = 0.0, gcv = 0.0;
        for (int q = 0; q < k; ++q) {
          const double cvq = R[fo.CnVn + q * t + j];
          const double dq = cvq - R[fo.CVn + q * t + j];
          om = fma(0.5 * (Om[l * k + q] + Om[q * k + l]), cvq, om);
          gd = fma(Gam[l * k + q], dq, gd);
          gg = fma(Gm[l * k + q], dq, gg);
          gcv = fma(Gam[l * k + q], CVp[q * t + j], gcv);
        }
        const double cvl = R[fo.CnVn + idx], dl = cvl - R[fo.CVn + idx];
        v[1] -= cvl * om + 2.0 * cvl * gd + dl * gg;
        Wm[idx] = R[fo.NV + idx] - gcv;
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
        const int aa = idx / t, bb = idx - aa * t;
        const double vnv = Rt[bb * t + aa];    // (V'^T Vp)[aa][bb]
        double x1 = 0.0, x3 = 0.0;
        for (int l = 0; l < k; ++l) {
          x1 = fma(R[fo.CnVn + l * t + aa], HCV[l * t + bb], x1);
          x3 = fma(CVp[l * t + bb], R[fo.MVn + l * t + aa], x3);
        }
        v[0] += vnv * (x1 + ZnV[idx]) - vnv * x3;
        const int i = aa, j = bb;
        double rlr = 0.0, rr = 0.0, xw = 0.0;
        for (int q = 0; q < t; ++q) {
          rlr = fma(Rt[q * t + i] * a.th_in[q], Rt[q * t + j], rlr);   // previous Ritz values
          rr = fma(Rt[q * t + i], Rt[q * t + j], rr);
        }
        for (int l = 0; l < k; ++l) xw = fma(R[fo.CE + l * t + i], Wm[l * t + j], xw);
        v[1] += rlr * R[fo.EE + j * t + i] + rr * R[fo.ESE + j * t + i] + 2.0 * xw * Rt[j * t + i];
      }
      block_sum_n<2>(v, red);
      const double cross = R[1] + v[0];
      const double trOm = tr3[2];
      const double x2sq_old = a.scal[0], xn2_old = a.scal[1];
      const double st2_big = trOm + x2sq_new + x2sq_old - 2.0 * cross;
      const double st2_small = trOm + R[2] + 2.0 * R[3] + R[4] + v[1];
      const double st2 = st2_big > 1e-8 * xn2_old ? st2_big : st2_small;
      step = sqrt(fmax(st2, 0.0));
      rel = step / sqrt(xn2_old);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t pnew = a.mode ? (int64_t)llround(a.scal[5]) + 1 : 0;   // canonical state index
      a.scal[0] = x2sq_new;
      a.scal[1] = trG + x2sq_new;
      a.scal[2] = F;
      a.scal[3] = step;
      a.scal[4] = rel;
      a.scal[5] = (double)pnew;
      const int64_t slotp = pnew % a.trace_cap;
      a.trace[slotp * 4 + 0] = F;
      a.trace[slotp * 4 + 1] = step;
      a.trace[slotp * 4 + 2] = rel;
      a.trace[slotp * 4 + 3] = (double)pnew;
      if (!isfinite(F)) raise_flag(a.flags, DF_NONFINITE);
      if (a.mode && a.eps > 0.0 && (step < a.eps || rel < a.eps)) a.flags[2] = 1;   // converged
    }
    tmark(s, a);                               // objective + step norm
  }
}

template <int BT, int PART>
cudaError_t ss_configure(int CL, size_t smem) {
  static size_t done_smem = 0;
  static int done_cl = 0;
  if (smem <= done_smem && (CL <= 8 || done_cl > 8)) return cudaSuccess;
  auto kern = small_step_kernel<BT, PART>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (CL > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) {
    done_smem = std::max(done_smem, smem);
    done_cl = std::max(done_cl, CL);
  }
  return e;
}

template <int BT>
int ss_max_clusters(int CL, size_t smem) {
  if (ss_configure<BT, 1>(CL, smem) != cudaSuccess || ss_configure<BT, 2>(CL, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kSST);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n1 = 0, n2 = 0;
  if (cudaOccupancyMaxActiveClusters(&n1, small_step_kernel<BT, 1>, &cfg) != cudaSuccess ||
      cudaOccupancyMaxActiveClusters(&n2, small_step_kernel<BT, 2>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(n1, n2);
}

template <int BT>
cudaError_t launch_ss(const SmallArgs& a, int part, cudaStream_t st) {
  const size_t smem = (size_t)a.pl.total * sizeof(double);
  cudaError_t e = part == 1 ? ss_configure<BT, 1>(a.pl.CL, smem) : ss_configure<BT, 2>(a.pl.CL, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.pl.CL);
  cfg.blockDim = dim3(kSST);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.pl.CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (part == 1 && a.pdl) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  if (part == 2) {
    // the deferred half runs beside the next critical half: schedule its cluster first
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = hi;
    cfg.numAttrs = 2;
  }
  if (part == 1) return cudaLaunchKernelEx(&cfg, small_step_kernel<BT, 1>, a);
  return cudaLaunchKernelEx(&cfg, small_step_kernel<BT, 2>, a);
}

}  // namespace wlr
