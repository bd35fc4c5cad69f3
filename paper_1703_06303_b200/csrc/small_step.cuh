// small_step.cu -- K3: the (C, D) half-step of Algorithm 1
// on the Gram route, plus the objective and the convergence reduction.
//
// Runs as ONE thread-block cluster (CL CTAs, up to 16, one per SM) so that every
// cross-CTA exchange is a hardware cluster barrier instead of a grid barrier.  Each CTA
// owns a contiguous slice of the (n-k)-dimensional column index space and keeps its
// rows of G_A = A2^T A2 resident in shared memory when they fit.
//
//   Gram update   G' = G + Gamma + Gamma^T + Omega,  M' = M + N,  H = G + Gamma
//   C             C' = G'^{-1} M'          (= R^{-1} Q^T A2 with X1 = QR)
//   eigenpairs    top r-k of  S = G_A - M'^T C' = A2^T P^perp A2   (matrix-free S.Y)
//                 -> V (right singular vectors of P^perp A2), lambda = sigma^2
//                 so D = U Sigma_{r-k} V^T = (A2 - X1 C) V V^T
//                 Chebyshev-filtered subspace iteration with Rayleigh-Ritz, warm-started
//                 from the previous iteration's Ritz block.
//   objective     F = f_w + ||A2||^2 - <M', C'> - sum(lambda)
//   step norm     ||X_{p+1} - X_p||_F from small-side products only
//   operands      Wt = [V | C^T], C V and K^{-1} = (w^2 I + C C^T)^{-1} (or C C^T) for
//                 the next row pass, converted to the storage dtype.
#pragma once
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace wlr {


constexpr int kSST = 512;            // threads per CTA
constexpr int kSSW = kSST / 32;

struct SSCtx {
  SmallArgs a;
  int c, CL, rs, re, nloc;
  double* GAs;         // nloc x nk (smem) or nullptr
  double* Ls;          // k x k
  double* Hs;          // k x k
  double* Wk;          // k x b
  double* Tb;          // b x b (Gram / T)
  double* Ub;          // b x b
  double* vb;          // b (theta / scale)
  double* Yst;         // nk x b staged transposed (smem) or nullptr
  double* Xw;          // per-warp solve scratch (kSSW x k)
  double* red;         // smem reduction scratch (kSSW)
  int* bank;           // exchange bank parity (per-CTA, uniform)
};

WLR_DEVI void cl_sync() {
  __threadfence();
  cg::this_cluster().sync();
}

WLR_DEVI double* slot(SSCtx& s, int cta) {
  return s.a.xchg + ((int64_t)(*s.bank) * s.CL + cta) * s.a.xchg_stride;
}

// one exchange round: every CTA wrote its partial of length len into slot(c); after the
// barrier, out[i] = sum_c slot(c)[i] in fixed CTA order (identical on every CTA).
WLR_DEVI void xchg_reduce(SSCtx& s, int len, double* out) {
  cl_sync();
  for (int i = threadIdx.x; i < len; i += kSST) {
    double v = 0.0;
    for (int c = 0; c < s.CL; ++c) v += __ldcg(s.a.xchg + ((int64_t)(*s.bank) * s.CL + c) * s.a.xchg_stride + i);
    out[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) *s.bank ^= 1;
  __syncthreads();
}

// Cholesky of the n x n symmetric matrix in smem (row-major, lower result in place) by
// warp 0.  Returns true iff every pivot d_j > rel * A_jj (the original diagonal, after the
// shift); result broadcast to the block.  rel > 0 is the numerical-rank test of the Gram
// route (reading R6b): a pivot at rounding level of its column's squared norm
// means that column lies in the span of the previous ones.
WLR_DEVI bool chol_warp0(double* A, int n, int ld, double shift, double rel = 0.0) {
  __shared__ int ok_s;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    if (shift != 0.0)
      for (int i = lane; i < n; i += 32) A[i * ld + i] += shift;
    __syncwarp();
    double od[4];                            // original diagonal, lane + 32q (n <= 128)
#pragma unroll
    for (int q = 0; q < 4; ++q) od[q] = (lane + 32 * q < n) ? A[(lane + 32 * q) * (ld + 1)] : 0.0;
    __syncwarp();
    for (int j = 0; j < n; ++j) {
      const double d = A[j * ld + j];
      const int q = j >> 5;
      const double oq = q == 0 ? od[0] : q == 1 ? od[1] : q == 2 ? od[2] : od[3];
      const double d0 = __shfl_sync(0xffffffffu, oq, j & 31);
      ok = ok && (d > rel * d0) && (d > 0.0) && isfinite(d);
      const double r = sqrt(d > 0.0 ? d : 1.0);
      const double inv = 1.0 / r;
      __syncwarp();
      if (lane == 0) A[j * ld + j] = r;
      for (int i = j + 1 + lane; i < n; i += 32) A[i * ld + j] *= inv;
      __syncwarp();
      for (int i = j + 1 + lane; i < n; i += 32) {
        const double lij = A[i * ld + j];
        for (int l = j + 1; l <= i; ++l) A[i * ld + l] = fma(-lij, A[l * ld + j], A[i * ld + l]);
      }
      __syncwarp();
    }
    if (lane == 0) ok_s = ok ? 1 : 0;
  }
  __syncthreads();
  return ok_s != 0;
}

// x := L^{-T} L^{-1} x for one vector x in smem/global (stride sx), by one warp
WLR_DEVI void chol_solve_warp(const double* L, int n, int ld, double* x, int sx, int lane) {
  for (int j = 0; j < n; ++j) {
    const double zj = x[j * sx] / L[j * ld + j];
    for (int i = j + 1 + lane; i < n; i += 32) x[i * sx] = fma(-L[i * ld + j], zj, x[i * sx]);
    __syncwarp();
    if (lane == 0) x[j * sx] = zj;
    __syncwarp();
  }
  for (int j = n - 1; j >= 0; --j) {
    const double xj = x[j * sx] / L[j * ld + j];
    for (int i = lane; i < j; i += 32) x[i * sx] = fma(-L[j * ld + i], xj, x[i * sx]);
    __syncwarp();
    if (lane == 0) x[j * sx] = xj;
    __syncwarp();
  }
}

// Cyclic Jacobi eigen-decomposition of the symmetric b x b matrix T (smem), by warp 0:
// on exit theta = eigenvalues in DESCENDING order and U (b x b, columns) the matching
// orthonormal eigenvectors.  Deterministic, so every CTA obtains identical results.
WLR_DEVI void jacobi_warp0(double* T, double* U, double* theta, int b) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = lane; i < b * b; i += 32) U[i] = (i / b == i % b) ? 1.0 : 0.0;
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
      for (int p = 0; p < b - 1; ++p) {
        for (int q = p + 1; q < b; ++q) {
          const double apq = T[p * b + q];
          const double app = T[p * b + p], aqq = T[q * b + q];
          if (!(fabs(apq) > 1e-300) || fabs(apq) <= 1e-17 * sqrt(fabs(app * aqq))) continue;
          rotated = true;
          const double tau = (aqq - app) / (2.0 * apq);
          const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          const double c = 1.0 / sqrt(1.0 + tt * tt), s = tt * c;
          __syncwarp();
          if (lane < b && lane != p && lane != q) {
            const double tip = T[lane * b + p], tiq = T[lane * b + q];
            const double nip = c * tip - s * tiq, niq = s * tip + c * tiq;
            T[lane * b + p] = nip; T[p * b + lane] = nip;
            T[lane * b + q] = niq; T[q * b + lane] = niq;
          }
          if (lane < b) {
            const double uip = U[lane * b + p], uiq = U[lane * b + q];
            U[lane * b + p] = c * uip - s * uiq;
            U[lane * b + q] = s * uip + c * uiq;
          }
          if (lane == 0) {
            T[p * b + p] = app - tt * apq;
            T[q * b + q] = aqq + tt * apq;
            T[p * b + q] = 0.0;
            T[q * b + p] = 0.0;
          }
          __syncwarp();
        }
      }
      if (!rotated) break;
    }
    // sort descending (stable by index) and permute U's columns
    double wj = lane < b ? T[lane * b + lane] : 0.0;
    int rk = 0;
    for (int i = 0; i < b; ++i) {
      const double wi = T[i * b + i];
      if (wi > wj || (wi == wj && i < lane)) ++rk;
    }
    double ucol[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) ucol[i] = (i < b && lane < b) ? U[i * b + lane] : 0.0;
    __syncwarp();
    if (lane < b) {
      theta[rk] = wj;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < b) U[i * b + rk] = ucol[i];
    }
    __syncwarp();
  }
  __syncthreads();
}

// block reduction of one double per thread (result valid on all threads)
WLR_DEVI double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kSSW; ++w) s += red[w];
  __syncthreads();
  return s;
}

// Z[slice] = S . Yin[slice] = G_A[slice,:] Yin - M'[:,slice]^T (C' Yin)    (one product)
template <int BT>
WLR_DEVI void s_product(SSCtx& s, const double* Yin, double* Zout, const double* Mx = nullptr,
                        const double* Cx = nullptr) {
  constexpr int RG = BT <= 12 ? 4 : 2;       // rows per warp pass (register blocking)
  const SmallArgs& a = s.a;
  const int k = a.k, nk = a.nk, b = a.b;
  if (!Mx) Mx = a.M_out;
  if (!Cx) Cx = a.C_out;
  // (1) partial W_c = C'[:, slice] . Yin[slice, :]
  double* my = slot(s, s.c);
  for (int idx = threadIdx.x; idx < k * b; idx += kSST) {
    const int l = idx / b, j = idx % b;
    double v = 0.0;
    for (int i = s.rs; i < s.re; ++i) v = fma(Cx[(int64_t)l * nk + i], Yin[(int64_t)i * b + j], v);
    my[idx] = v;
  }
  xchg_reduce(s, k * b, s.Wk);               // includes the cluster barrier (Yin complete)
  if (s.Yst) {                               // stage Yin transposed: Yst[j][l]
    for (int idx = threadIdx.x; idx < nk * b; idx += kSST) {
      const int l = idx / b, j = idx % b;
      s.Yst[(int64_t)j * nk + l] = Yin[idx];
    }
    __syncthreads();
  }
  // (2) rows of the slice, RG rows per warp pass, lanes over the reduction index
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g0 = warp * RG; g0 < s.nloc; g0 += kSSW * RG) {
    double acc[RG][BT];
#pragma unroll
    for (int r = 0; r < RG; ++r)
#pragma unroll
      for (int j = 0; j < BT; ++j) acc[r][j] = 0.0;
    const double* grow[RG];
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const int il = g0 + r < s.nloc ? g0 + r : g0;
      grow[r] = s.GAs ? s.GAs + (int64_t)il * nk : a.GA + (int64_t)(s.rs + il) * nk;
    }
    for (int l = lane; l < nk; l += 32) {
      double yv[BT];
#pragma unroll
      for (int j = 0; j < BT; ++j)
        yv[j] = j < b ? (s.Yst ? s.Yst[(int64_t)j * nk + l] : Yin[(int64_t)l * b + j]) : 0.0;
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const double gv = grow[r][l];
#pragma unroll
        for (int j = 0; j < BT; ++j) acc[r][j] = fma(gv, yv[j], acc[r][j]);
      }
    }
    for (int l = lane; l < k; l += 32) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const int i = s.rs + (g0 + r < s.nloc ? g0 + r : g0);
        const double mli = Mx[(int64_t)l * nk + i];
#pragma unroll
        for (int j = 0; j < BT; ++j)
          if (j < b) acc[r][j] = fma(-mli, s.Wk[l * b + j], acc[r][j]);
      }
    }
#pragma unroll
    for (int r = 0; r < RG; ++r)
#pragma unroll
      for (int j = 0; j < BT; ++j) acc[r][j] = warp_sum(acc[r][j]);
#pragma unroll
    for (int r = 0; r < RG; ++r)
#pragma unroll
      for (int j = 0; j < BT; ++j)
        if (j < b && lane == j && g0 + r < s.nloc) Zout[(int64_t)(s.rs + g0 + r) * b + j] = acc[r][j];
  }
  __syncthreads();
}

// Y[slice] := Y[slice] R^{-1} with Gram = R^T R (CholQR pass).  scaled: Jacobi-scaled and
// shifted first pass.  Returns false if the Gram is not numerically positive definite.
template <int BT>
WLR_DEVI bool cholqr_pass(SSCtx& s, double* Y, bool scaled) {
  const SmallArgs& a = s.a;
  const int b = a.b;
  double* my = slot(s, s.c);
  for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
    const int p = idx / b, q = idx % b;
    double v = 0.0;
    for (int i = s.rs; i < s.re; ++i) v = fma(Y[(int64_t)i * b + p], Y[(int64_t)i * b + q], v);
    my[idx] = v;
  }
  xchg_reduce(s, b * b, s.Tb);
  if (scaled) {
    if (threadIdx.x < b) {
      const double d = s.Tb[threadIdx.x * b + threadIdx.x];
      s.vb[threadIdx.x] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < b * b; idx += kSST) s.Tb[idx] *= s.vb[idx / b] * s.vb[idx % b];
    __syncthreads();
  }
  const bool ok = chol_warp0(s.Tb, b, b, scaled ? 1e-13 * b : 0.0);
  if (!ok) return false;
  // rows: y := (y .* scale) L^{-T}   i.e. solve x L^T = y'
  for (int i = s.rs + threadIdx.x; i < s.re; i += kSST) {
    double y[BT];
#pragma unroll
    for (int j = 0; j < BT; ++j) y[j] = j < b ? Y[(int64_t)i * b + j] * (scaled ? s.vb[j] : 1.0) : 0.0;
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      if (j < b) {
        double v = y[j];
#pragma unroll
        for (int p = 0; p < BT; ++p)
          if (p < j) v = fma(-s.Tb[j * b + p], y[p], v);
        y[j] = v / s.Tb[j * b + j];
      }
    }
#pragma unroll
    for (int j = 0; j < BT; ++j)
      if (j < b) Y[(int64_t)i * b + j] = y[j];
  }
  __syncthreads();
  return true;
}

// rows of M := M U  (b x b rotation) on the slice
template <int BT>
WLR_DEVI void rotate_rows(SSCtx& s, double* Mx) {
  const int b = s.a.b;
  for (int i = s.rs + threadIdx.x; i < s.re; i += kSST) {
    double y[BT], o[BT];
#pragma unroll
    for (int j = 0; j < BT; ++j) { y[j] = j < b ? Mx[(int64_t)i * b + j] : 0.0; o[j] = 0.0; }
#pragma unroll
    for (int p = 0; p < BT; ++p)
#pragma unroll
      for (int j = 0; j < BT; ++j)
        if (p < b && j < b) o[j] = fma(y[p], s.Ub[p * b + j], o[j]);
#pragma unroll
    for (int j = 0; j < BT; ++j)
      if (j < b) Mx[(int64_t)i * b + j] = o[j];
  }
  __syncthreads();
}

template <int BT>
__global__ void __launch_bounds__(kSST, 1) small_step_kernel(SmallArgs a, int smem_flags) {
  extern __shared__ __align__(16) double ss_smem[];
  __shared__ int bank_s;
  __shared__ double red_s[kSSW];
  __shared__ int flag_s;
  SSCtx s;
  s.a = a;
  s.CL = gridDim.x;
  s.c = blockIdx.x;
  const int k = a.k, nk = a.nk, b = a.b, t = a.t;
  const int SL = (int)ceil_div(nk, s.CL);
  s.rs = std::min(nk, s.c * SL);
  s.re = std::min(nk, s.rs + SL);
  s.nloc = s.re - s.rs;
  double* p = ss_smem;
  s.GAs = nullptr;
  s.Yst = nullptr;
  if (smem_flags & 1) { s.GAs = p; p += (int64_t)SL * nk; }
  if (smem_flags & 2) { s.Yst = p; p += (int64_t)nk * b; }
  s.Ls = p; p += k * k;
  s.Hs = p; p += k * k;
  s.Wk = p; p += k * b;
  s.Tb = p; p += b * b;
  s.Ub = p; p += b * b;
  s.vb = p; p += 32;
  s.Xw = p; p += kSSW * k;
  s.red = red_s;
  s.bank = &bank_s;
  if (threadIdx.x == 0) bank_s = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ------------------------------------------------ stage G_A rows of the slice
  if (s.GAs)
    for (int64_t idx = threadIdx.x; idx < (int64_t)s.nloc * nk; idx += kSST)
      s.GAs[idx] = a.GA[(int64_t)s.rs * nk + idx];

  // ------------------------------------------------ A: Gram update, Cholesky, C
  const double* incN = a.inc;
  const double* incGam = a.inc + (int64_t)k * nk;
  const double* incOm = incGam + (int64_t)k * k;
  const double fw = a.mode ? incOm[(int64_t)k * k] : a.inc[0];
  for (int idx = threadIdx.x; idx < k * k; idx += kSST) {
    const int i = idx / k, j = idx % k;
    if (a.mode) {
      const double g = a.G_in[idx];
      const double om = 0.5 * (incOm[i * k + j] + incOm[j * k + i]);
      s.Ls[idx] = g + incGam[i * k + j] + incGam[j * k + i] + om;
      s.Hs[idx] = g + incGam[i * k + j];
    } else {
      s.Ls[idx] = a.G_out[idx];
      s.Hs[idx] = 0.0;
    }
  }
  if (a.mode) {
    for (int64_t idx = threadIdx.x; idx < (int64_t)k * s.nloc; idx += kSST) {
      const int l = (int)(idx / s.nloc), c = s.rs + (int)(idx % s.nloc);
      a.M_out[(int64_t)l * nk + c] = a.M_in[(int64_t)l * nk + c] + incN[(int64_t)l * nk + c];
    }
  }
  __syncthreads();
  double trG = 0.0;
  for (int i = 0; i < k; ++i) trG += s.Ls[i * k + i];
  if (s.c == 0 && a.mode)
    for (int idx = threadIdx.x; idx < k * k; idx += kSST) a.G_out[idx] = s.Ls[idx];
  __syncthreads();
  if (!chol_warp0(s.Ls, k, k, 0.0, 256.0 * 2.220446049250313e-16)) {   // rank(X1) < k (R6)
    if (s.c == 0 && threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;                                  // every CTA takes this branch identically
  }
  // C'[:, c] = G'^{-1} M'[:, c] for the slice columns (warp per column)
  for (int cl = warp; cl < s.nloc; cl += kSSW) {
    const int c = s.rs + cl;
    double* xw = s.Xw + warp * k;
    for (int l = lane; l < k; l += 32) xw[l] = a.M_out[(int64_t)l * nk + c];
    __syncwarp();
    chol_solve_warp(s.Ls, k, k, xw, 1, lane);
    for (int l = lane; l < k; l += 32) a.C_out[(int64_t)l * nk + c] = xw[l];
    __syncwarp();
  }
  __syncthreads();
  cl_sync();                                  // C', M' complete on every slice

  // ------------------------------------------------ B: eigenpairs of S (ChFSI + RR)
  const double floor_abs = 8.0 * 2.220446049250313e-16 * a.a2sq;
  double* Yb[3] = {a.Y, a.Y1, a.Y2};
  int outer = 0;
  const int max_outer = a.max_outer;
  bool converged = false, failed = false;
  while (true) {
    // Rayleigh-Ritz on span(Y)
    if (!cholqr_pass<BT>(s, a.Y, true) || !cholqr_pass<BT>(s, a.Y, false)) { failed = true; break; }
    s_product<BT>(s, a.Y, a.Z);
    {
      double* my = slot(s, s.c);
      for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
        const int pp = idx / b, q = idx % b;
        double v = 0.0;
        for (int i = s.rs; i < s.re; ++i) v = fma(a.Y[(int64_t)i * b + pp], a.Z[(int64_t)i * b + q], v);
        my[idx] = v;
      }
      xchg_reduce(s, b * b, s.Tb);
      for (int idx = threadIdx.x; idx < b * b; idx += kSST) {
        const int pp = idx / b, q = idx % b;
        if (pp < q) {
          const double v = 0.5 * (s.Tb[pp * b + q] + s.Tb[q * b + pp]);
          s.Tb[pp * b + q] = v;
          s.Tb[q * b + pp] = v;
        }
      }
      __syncthreads();
      jacobi_warp0(s.Tb, s.Ub, s.vb, b);
    }
    rotate_rows<BT>(s, a.Y);
    rotate_rows<BT>(s, a.Z);
    {   // residual norms of the wanted pairs
      double* my = slot(s, s.c);
      for (int j = threadIdx.x; j < b; j += kSST) {
        double v = 0.0;
        for (int i = s.rs; i < s.re; ++i) {
          const double r = a.Z[(int64_t)i * b + j] - s.vb[j] * a.Y[(int64_t)i * b + j];
          v = fma(r, r, v);
        }
        my[j] = v;
      }
      xchg_reduce(s, b, s.Tb);    // Tb[j] = ||S y_j - theta_j y_j||^2
    }
    double rmax = 0.0;
    for (int j = 0; j < t; ++j) rmax = fmax(rmax, sqrt(fmax(s.Tb[j], 0.0)));
    const double theta0 = s.vb[0];
    if (rmax <= a.tol * fabs(theta0) + floor_abs) { converged = true; break; }
    if (++outer > max_outer) break;
    // Chebyshev filter of degree d damping [0, theta_{b-1}]
    const double beta = s.vb[b - 1];
    int d = a.max_deg;
    double cc = 0.5 * beta, ee = 0.5 * beta;
    if (!(beta > 1e-300 * fabs(theta0)) || beta >= theta0) {
      cc = 0.0; ee = 1.0; d = 1;                // plain power step
    } else {
      const double x0 = (theta0 - cc) / ee, xt = (s.vb[t - 1] - cc) / ee;
      const double gap = acosh(fmax(x0, 1.0)) - acosh(fmax(xt, 1.0));
      if (gap > 0.0) d = std::max(1, std::min(d, (int)(11.5 / gap)));   // amplification <= 1e5
    }
    // Y1 = (Z - c Y)/e
    double* Yp = Yb[0];
    double* Yc = Yb[1];
    double* Yn = Yb[2];
    for (int64_t idx = (int64_t)s.rs * b + threadIdx.x; idx < (int64_t)s.re * b; idx += kSST)
      Yc[idx] = (a.Z[idx] - cc * Yp[idx]) / ee;
    __syncthreads();
    for (int j = 2; j <= d; ++j) {
      s_product<BT>(s, Yc, a.Z);
      for (int64_t idx = (int64_t)s.rs * b + threadIdx.x; idx < (int64_t)s.re * b; idx += kSST)
        Yn[idx] = 2.0 * (a.Z[idx] - cc * Yc[idx]) / ee - Yp[idx];
      __syncthreads();
      double* tmp = Yp; Yp = Yc; Yc = Yn; Yn = tmp;
    }
    if (Yc != a.Y) {
      for (int64_t idx = (int64_t)s.rs * b + threadIdx.x; idx < (int64_t)s.re * b; idx += kSST)
        a.Y[idx] = Yc[idx];
      __syncthreads();
    }
  }
  if (failed || !converged) {
    if (s.c == 0 && threadIdx.x == 0) raise_flag(a.flags, DF_EIG);
  }
  if (failed) return;

  // ------------------------------------------------ C: objective, step norm, operands
  // Step norm: ||X_{p+1}-X_p||^2 = tr(Omega) + ||X2'-X2||^2.  Two
  // evaluations: the exact Gram identity (accurate while the relative step is >= 1e-4)
  // and, below that, the first-order expansion ||T1||^2 + ||T2||^2 + 2<T1,T2> with
  //   T1 = (X1'C' - X1 C)(I - Q'),  T2 = P^perp A2 (Q' - Q),  Q = V V^T,
  //   V' = V R + E (R = V^T V', E orthogonal to V): every term is a product of O(step)
  //   factors, so no second-order cancellation.
  const int kt = k * t;
  double* Rt = s.Tb;                               // R = V^T V' (t x t), all CTAs
  if (a.mode) {
    double* my = slot(s, s.c);
    for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
      const int i = idx / t, j = idx % t;
      double v = 0.0;
      for (int c = s.rs; c < s.re; ++c) v = fma(a.Vprev[(int64_t)c * t + i], a.Y[(int64_t)c * b + j], v);
      my[idx] = v;
    }
    xchg_reduce(s, t * t, Rt);
    // E = V' - V R into Y1 (first t columns, stride b; other columns zero)
    for (int64_t idx = threadIdx.x; idx < (int64_t)s.nloc * b; idx += kSST) {
      const int c = s.rs + (int)(idx / b), j = (int)(idx % b);
      double v = 0.0;
      if (j < t) {
        v = a.Y[(int64_t)c * b + j];
        for (int q = 0; q < t; ++q) v = fma(-a.Vprev[(int64_t)c * t + q], Rt[q * t + j], v);
      }
      a.Y1[(int64_t)c * b + j] = v;
    }
    __syncthreads();
    s_product<BT>(s, a.Y1, a.Y2, a.M_in, a.C_in);   // S_p E  (old S)
  }
  // partial layout of the final round:
  //   [0] <M',C'> [1] <C',H C> [2] <C',Om C'> [3] <C',Gam dC> [4] <dC, G dC>
  //   | CnV | CnVn | CVn | MnV | MVn | NV | CE  (k x t each)
  //   | VnV | ZnV | EE | ESE (t x t each) | C'C'^T (k x k)
  const int oCnV = 5, oCnVn = oCnV + kt, oCVn = oCnVn + kt, oMnV = oCVn + kt, oMVn = oMnV + kt;
  const int oNV = oMVn + kt, oCE = oNV + kt;
  const int oVnV = oCE + kt, oZnV = oVnV + t * t, oEE = oZnV + t * t, oESE = oEE + t * t;
  const int oCC = oESE + t * t, flen = oCC + k * k;
  {
    double* my = slot(s, s.c);
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;
    for (int64_t idx = threadIdx.x; idx < (int64_t)k * s.nloc; idx += kSST) {
      const int l = (int)(idx / s.nloc), c = s.rs + (int)(idx % s.nloc);
      const double cn = a.C_out[(int64_t)l * nk + c];
      v0 = fma(a.M_out[(int64_t)l * nk + c], cn, v0);
      if (a.mode) {
        double hc = 0.0, omc = 0.0, gdc = 0.0, ggdc = 0.0;
        for (int q = 0; q < k; ++q) {
          const double co = a.C_in[(int64_t)q * nk + c], cq = a.C_out[(int64_t)q * nk + c];
          const double dq = cq - co;
          hc = fma(s.Hs[l * k + q], co, hc);
          omc = fma(0.5 * (incOm[l * k + q] + incOm[q * k + l]), cq, omc);
          gdc = fma(incGam[l * k + q], dq, gdc);
          ggdc = fma(a.G_in[l * k + q], dq, ggdc);
        }
        const double dl = cn - a.C_in[(int64_t)l * nk + c];
        v1 = fma(cn, hc, v1);
        v2 = fma(cn, omc, v2);
        v3 = fma(cn, gdc, v3);
        v4 = fma(dl, ggdc, v4);
      }
    }
    v0 = block_sum(v0, s.red);
    v1 = block_sum(v1, s.red);
    v2 = block_sum(v2, s.red);
    v3 = block_sum(v3, s.red);
    v4 = block_sum(v4, s.red);
    if (threadIdx.x == 0) { my[0] = v0; my[1] = v1; my[2] = v2; my[3] = v3; my[4] = v4; }
    for (int idx = threadIdx.x; idx < kt; idx += kSST) {
      const int l = idx / t, j = idx % t;
      double cnv = 0.0, cnvn = 0.0, cvn = 0.0, mnv = 0.0, mvn = 0.0, nv = 0.0, ce = 0.0;
      for (int c = s.rs; c < s.re; ++c) {
        const double cn = a.C_out[(int64_t)l * nk + c], mn = a.M_out[(int64_t)l * nk + c];
        const double vn = a.Y[(int64_t)c * b + j];
        cnvn = fma(cn, vn, cnvn);
        if (a.mode) {
          const double vp = a.Vprev[(int64_t)c * t + j];
          cnv = fma(cn, vp, cnv);
          cvn = fma(a.C_in[(int64_t)l * nk + c], vn, cvn);
          mnv = fma(mn, vp, mnv);
          mvn = fma(a.M_in[(int64_t)l * nk + c], vn, mvn);
          nv = fma(incN[(int64_t)l * nk + c], vp, nv);
          ce = fma(cn, a.Y1[(int64_t)c * b + j], ce);
        }
      }
      my[oCnV + idx] = cnv; my[oCnVn + idx] = cnvn; my[oCVn + idx] = cvn;
      my[oMnV + idx] = mnv; my[oMVn + idx] = mvn; my[oNV + idx] = nv; my[oCE + idx] = ce;
    }
    for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
      const int i = idx / t, j = idx % t;
      double vv = 0.0, zv = 0.0, ee = 0.0, ese = 0.0;
      if (a.mode)
        for (int c = s.rs; c < s.re; ++c) {
          const double vp = a.Vprev[(int64_t)c * t + j];
          vv = fma(a.Y[(int64_t)c * b + i], vp, vv);
          zv = fma(a.Z[(int64_t)c * b + i], vp, zv);
          const double ei = a.Y1[(int64_t)c * b + i];
          ee = fma(ei, a.Y1[(int64_t)c * b + j], ee);
          ese = fma(ei, a.Y2[(int64_t)c * b + j], ese);
        }
      my[oVnV + idx] = vv; my[oZnV + idx] = zv; my[oEE + idx] = ee; my[oESE + idx] = ese;
    }
    for (int idx = threadIdx.x; idx < k * k; idx += kSST) {
      const int i = idx / k, j = idx % k;
      double v = 0.0;
      for (int c = s.rs; c < s.re; ++c) v = fma(a.C_out[(int64_t)i * nk + c], a.C_out[(int64_t)j * nk + c], v);
      my[oCC + idx] = v;
    }
    __syncthreads();
    // slice-local outputs: Wt rows, Vprev <- Vn (own slice only; read above by this CTA only)
    const int RP = a.rp;
    for (int64_t idx = threadIdx.x; idx < (int64_t)s.nloc * RP; idx += kSST) {
      const int cl = (int)(idx / RP), j = (int)(idx % RP);
      const int c = s.rs + cl;
      double v = 0.0;
      if (j < t) v = a.Y[(int64_t)c * b + j];
      else if (j < t + k) v = a.C_out[(int64_t)(j - t) * nk + c];
      const int64_t o = (int64_t)(k + c - a.k0) * RP + j;
      if (a.dtype) reinterpret_cast<double*>(a.Wt)[o] = v;
      else reinterpret_cast<float*>(a.Wt)[o] = (float)v;
    }
    for (int64_t idx = threadIdx.x; idx < (int64_t)s.nloc * t; idx += kSST) {
      const int cl = (int)(idx / t), j = (int)(idx % t);
      const int c = s.rs + cl;
      a.Vprev[(int64_t)c * t + j] = a.Y[(int64_t)c * b + j];
    }
  }
  cl_sync();
  if (s.c != 0) return;

  // ---- CTA 0: reduce the final partials (fixed order) and finish
  double* R = a.red;
  for (int i = threadIdx.x; i < flen; i += kSST) {
    double v = 0.0;
    for (int c = 0; c < s.CL; ++c) v += __ldcg(a.xchg + ((int64_t)bank_s * s.CL + c) * a.xchg_stride + i);
    R[i] = v;
  }
  __syncthreads();
  double sum_theta = 0.0;
  for (int j = 0; j < t; ++j) sum_theta += s.vb[j];
  const double x2sq_new = R[0] + sum_theta;
  const double F = fw + a.a2sq - R[0] - sum_theta;
  double step = -1.0, rel = -1.0;
  if (a.mode) {
    double* HCV = R + flen + (int64_t)k * k;     // global scratch after Kinv
    double* HCVn = HCV + kt;
    for (int idx = threadIdx.x; idx < kt; idx += kSST) {
      const int l = idx / t, j = idx % t;
      double h1 = 0.0, h2 = 0.0;
      for (int q = 0; q < k; ++q) {
        h1 = fma(s.Hs[l * k + q], a.CVprev[q * t + j], h1);
        h2 = fma(s.Hs[l * k + q], R[oCVn + q * t + j], h2);
      }
      HCV[idx] = h1;
      HCVn[idx] = h2;
    }
    __syncthreads();
    // (a) exact Gram identity
    double v = 0.0;
    for (int idx = threadIdx.x; idx < kt; idx += kSST) {
      // t1: - <CnV, HCV> - <CnVn, HCVn>;  t3: + <MVn, CVn>;  t2+t4: + <MnV, CnV>
      v -= R[oCnV + idx] * HCV[idx] + R[oCnVn + idx] * HCVn[idx];
      v += R[oMVn + idx] * R[oCVn + idx] + R[oMnV + idx] * R[oCnV + idx];
    }
    for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
      const int aa = idx / t, bb = idx % t;     // VnV[aa][bb] = (Vn^T V)[aa][bb]
      double x1 = 0.0, x3 = 0.0;
      for (int l = 0; l < k; ++l) {
        x1 = fma(R[oCnVn + l * t + aa], HCV[l * t + bb], x1);             // (CnVn^T HCV)[aa][bb]
        x3 = fma(a.CVprev[l * t + bb], R[oMVn + l * t + aa], x3);         // (CVprev^T MVn)[bb][aa]
      }
      v += R[oVnV + idx] * (x1 + R[oZnV + idx]) - R[oVnV + idx] * x3;
    }
    v = block_sum(v, s.red);
    const double cross = R[1] + v;
    double trOm = 0.0;
    for (int i = 0; i < k; ++i) trOm += incOm[i * k + i];
    const double x2sq_old = a.scal[0], xn2_old = a.scal[1];
    const double st2_big = trOm + x2sq_new + x2sq_old - 2.0 * cross;
    // (b) first-order expansion (small steps)
    double u = 0.0;
    for (int idx = threadIdx.x; idx < kt; idx += kSST) {
      const int l = idx / t, j = idx % t;
      double om = 0.0, gd = 0.0, gg = 0.0, gcv = 0.0;
      for (int q = 0; q < k; ++q) {
        const double cvq = R[oCnVn + q * t + j];
        const double dq = cvq - R[oCVn + q * t + j];                      // (dC V')[q][j]
        om = fma(0.5 * (incOm[l * k + q] + incOm[q * k + l]), cvq, om);
        gd = fma(incGam[l * k + q], dq, gd);
        gg = fma(a.G_in[l * k + q], dq, gg);
        gcv = fma(incGam[l * k + q], a.CVprev[q * t + j], gcv);
      }
      const double cvl = R[oCnVn + idx], dl = cvl - R[oCVn + idx];
      u -= cvl * om + 2.0 * cvl * gd + dl * gg;                          // -||Z V'||^2
      HCV[idx] = R[oNV + idx] - gcv;                                     // W = N V - Gam C V
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < t * t; idx += kSST) {
      const int i = idx / t, j = idx % t;
      double rlr = 0.0, rr = 0.0, xw = 0.0;
      for (int q = 0; q < t; ++q) {
        rlr = fma(Rt[q * t + i] * a.theta[q], Rt[q * t + j], rlr);       // (R^T Lam R)[i][j]
        rr = fma(Rt[q * t + i], Rt[q * t + j], rr);                       // (R^T R)[i][j]
      }
      for (int l = 0; l < k; ++l) xw = fma(R[oCE + l * t + i], HCV[l * t + j], xw);   // ((CE)^T W)[i][j]
      u += rlr * R[oEE + j * t + i] + rr * R[oESE + j * t + i] + 2.0 * xw * Rt[j * t + i];
    }
    u = block_sum(u, s.red);
    const double st2_small = trOm + R[2] + 2.0 * R[3] + R[4] + u;
    const double st2 = st2_big > 1e-8 * xn2_old ? st2_big : st2_small;
    step = sqrt(fmax(st2, 0.0));
    rel = step / sqrt(xn2_old);
  }
  for (int j = threadIdx.x; j < b; j += kSST) a.theta[j] = s.vb[j];
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
    a.flags[3] = outer;
  }
  // operands: CV (k x t), K (k x k)
  for (int idx = threadIdx.x; idx < kt; idx += kSST) {
    const double v = R[oCnVn + idx];
    a.CVprev[idx] = v;
    if (a.dtype) reinterpret_cast<double*>(a.CVop)[idx] = v;
    else reinterpret_cast<float*>(a.CVop)[idx] = (float)v;
  }
  if (!a.uniform) {
    for (int idx = threadIdx.x; idx < k * k; idx += kSST) {
      const double v = R[oCC + idx];
      if (a.dtype) reinterpret_cast<double*>(a.Kop)[idx] = v;
      else reinterpret_cast<float*>(a.Kop)[idx] = (float)v;
    }
    return;
  }
  // uniform W1: K = w^2 I + C'C'^T, K^{-1} by Cholesky + k column solves (Ls as scratch)
  double* Kf = s.Ls;
  for (int idx = threadIdx.x; idx < k * k; idx += kSST)
    Kf[idx] = R[oCC + idx] + ((idx / k == idx % k) ? a.w2 : 0.0);
  __syncthreads();
  if (!chol_warp0(Kf, k, k, 0.0)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_ROWSPD);
    return;
  }
  double* Kinv = R + flen;             // scratch after the reduced partials (k x k)
  for (int col = warp; col < k; col += kSSW) {
    double* xw = s.Xw + warp * k;
    for (int i = lane; i < k; i += 32) xw[i] = (i == col) ? 1.0 : 0.0;
    __syncwarp();
    chol_solve_warp(Kf, k, k, xw, 1, lane);
    for (int i = lane; i < k; i += 32) Kinv[(int64_t)i * k + col] = xw[i];
    __syncwarp();
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < k * k; idx += kSST) {
    const int i = idx / k, j = idx % k;
    const double v = 0.5 * (Kinv[i * k + j] + Kinv[j * k + i]);
    if (a.dtype) reinterpret_cast<double*>(a.Kop)[idx] = v;
    else reinterpret_cast<float*>(a.Kop)[idx] = (float)v;
  }
}

inline size_t ss_smem_bytes(const SmallArgs& a, int CL, int flags) {
  const int SL = (int)ceil_div(a.nk, CL);
  size_t d = (size_t)2 * a.k * a.k + (size_t)a.k * a.b + 2 * (size_t)a.b * a.b + 32 +
             (size_t)kSSW * a.k;
  if (flags & 1) d += (size_t)SL * a.nk;
  if (flags & 2) d += (size_t)a.nk * a.b;
  return d * sizeof(double);
}

template <int BT>
cudaError_t ss_configure(int CL, size_t smem) {
  static size_t done_smem = 0;
  static int done_cl = 0;
  if (smem <= done_smem && (CL <= 8 || done_cl > 8)) return cudaSuccess;
  auto kern = small_step_kernel<BT>;
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
  if (ss_configure<BT>(CL, smem) != cudaSuccess) { cudaGetLastError(); return 0; }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kSST);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, small_step_kernel<BT>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <int BT>
cudaError_t launch_ss(const SmallArgs& a, int CL, size_t smem, int fl, cudaStream_t st) {
  cudaError_t e = ss_configure<BT>(CL, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kSST);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, small_step_kernel<BT>, a, fl);
}


}  // namespace wlr
