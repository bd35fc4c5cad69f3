// als.cu -- SURVEY.md §8(f3): the factorised WLR as a one-sweep block ALS on (X1, C, B, D),
// X2 = X1 C + B D (reading R21).  The m-scaled work reuses the sWLR kernels (the linear
// row map with Z = [A | B], the row Grams, the fixed-order reduce, the result-mode row map for
// B); this file holds the three fp64 small steps, one CTA each (k, r - k and n - k are small):
//
//   als_w_kernel : W'' = [w^2 K^{-1}; C^T K^{-1}; -(D C^T) K^{-1}] (uniform W1) or
//                  [0; C^T; -(D C^T)] with Kop = C C^T (per-row solves), K = w^2 I + C C^T
//                  (the X1 update of PAPER.md:184-196 with D_p := B_p D_p)
//   als_c_kernel : C' = G'^{-1} (M' - H' D_p) with G' = X1'^T X1', M' = X1'^T A2, H' = X1'^T B_p
//                  (least squares in C), then the B map Wb = [0; D^T S^{-1}; -C' D^T S^{-1}],
//                  S = D D^T (least squares in B)
//   als_d_kernel : D' = (B'^T B')^{-1} (B'^T A2 - (B'^T X1') C') (least squares in D) and the
//                  objective F from the Grams
#include "kernels.h"

namespace wlr {

constexpr int kAlsT = 512;

// In-place Gauss-Jordan inverse of the SPD n x n matrix A (row-major, ld n) into Ai; whole CTA.
// (SPD: no pivoting; returns false uniformly if a pivot is not > 0.)
__device__ bool als_gj_inverse(double* A, double* Ai, double* fac, int n) {
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Ai[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();
  for (int p = 0; p < n; ++p) {
    const double piv = A[p * n + p];
    if (!(piv > 0.0)) return false;
    const double inv = 1.0 / piv;
    __syncthreads();
    for (int j = threadIdx.x; j < 2 * n; j += blockDim.x) {
      if (j < n) A[p * n + j] *= inv;
      else Ai[p * n + j - n] *= inv;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) fac[i] = A[i * n + p];
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * 2 * n; idx += blockDim.x) {
      const int i = idx / (2 * n), j = idx - i * 2 * n;
      if (i == p) continue;
      if (j < n) A[i * n + j] -= fac[i] * A[p * n + j];
      else Ai[i * n + j - n] -= fac[i] * Ai[p * n + j - n];
    }
    __syncthreads();
  }
  return true;
}

template <typename T>
__device__ void als_store(void* W, int64_t o, double v) { reinterpret_cast<T*>(W)[o] = (T)v; }

// ------------------------------------------------------------------ W'' of the X1 row map
template <typename T>
__global__ void __launch_bounds__(kAlsT) als_w_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  double* cct = sm;                 // k x k
  double* ki = cct + k * k;         // k x k   K^{-1}
  double* dct = ki + k * k;         // t x k   D C^T
  double* fac = dct + t * k;        // k
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int i = idx / k, j = idx - i * k;
    double v = 0.0;
    for (int c = 0; c < nk; ++c) v = fma(a.C[(int64_t)i * nk + c], a.C[(int64_t)j * nk + c], v);
    cct[idx] = v;
  }
  for (int idx = threadIdx.x; idx < t * k; idx += blockDim.x) {
    const int j = idx / k, q = idx - j * k;
    double v = 0.0;
    for (int c = 0; c < nk; ++c) v = fma(a.D[(int64_t)j * nk + c], a.C[(int64_t)q * nk + c], v);
    dct[idx] = v;
  }
  __syncthreads();
  if (!a.uniform) {   // Kop = C C^T for the per-row solves (diag(W1(i,:)^2) added per row)
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) als_store<T>(a.Kop, idx, cct[idx]);
  } else {
    double* kk = cct;   // K = w^2 I + C C^T (in place), inverse into ki
    for (int i = threadIdx.x; i < k; i += blockDim.x) kk[i * k + i] += a.w2;
    __syncthreads();
    if (!als_gj_inverse(kk, ki, fac, k)) {
      if (threadIdx.x == 0) raise_flag(a.flags, DF_ROWSPD);
      return;
    }
  }
  const int RP = a.rp;
  // A1 rows j < k: w^2 K^{-1} (uniform; 0 otherwise -- the epilogue adds a1 w^2 before the solve)
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int j = idx / k, l = idx - j * k;
    als_store<T>(a.W, (int64_t)j * RP + l, a.uniform ? a.w2 * ki[idx] : 0.0);
  }
  // A2 rows k + c: C[:, c]^T K^{-1} (or C[:, c]^T)
  for (int idx = threadIdx.x; idx < nk * k; idx += blockDim.x) {
    const int c = idx / k, l = idx - c * k;
    double v;
    if (a.uniform) {
      v = 0.0;
      for (int q = 0; q < k; ++q) v = fma(a.C[(int64_t)q * nk + c], ki[q * k + l], v);
    } else {
      v = a.C[(int64_t)l * nk + c];
    }
    als_store<T>(a.W, (int64_t)(k + c) * RP + l, v);
  }
  // B rows KA + j: -(D C^T)[j, :] K^{-1} (or -(D C^T)[j, :])
  for (int idx = threadIdx.x; idx < t * k; idx += blockDim.x) {
    const int j = idx / k, l = idx - j * k;
    double v;
    if (a.uniform) {
      v = 0.0;
      for (int q = 0; q < k; ++q) v = fma(dct[j * k + q], ki[q * k + l], v);
    } else {
      v = dct[idx];
    }
    als_store<T>(a.W, (int64_t)(a.KA + j) * RP + l, -v);
  }
}

// ------------------------------------------------------------------ C step + the B map
template <typename T>
__global__ void __launch_bounds__(kAlsT) als_c_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  const int64_t kn = (int64_t)k * nk;
  double* g = sm;                   // k x k  G'
  double* gi = g + k * k;           // k x k  G'^{-1}
  double* s = gi + k * k;           // t x t  D D^T
  double* si = s + t * t;           // t x t
  double* cds = si + t * t;         // k x t  C' D^T S^{-1}
  double* dtc = cds + k * t;        // k x t  C' D^T
  double* fac = dtc + k * t;        // max(k, t)
  double* red = fac + (k > t ? k : t);   // kAlsT / 32 x 2
  if (a.c_given) {   // initial state: C given, D given (D D^T = I for D = V^T)
    for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
      const int i = idx / t, j = idx - i * t;
      double v = 0.0;
      for (int c = 0; c < nk; ++c) v = fma(a.D[(int64_t)i * nk + c], a.D[(int64_t)j * nk + c], v);
      s[idx] = v;
    }
  } else {
    const double* M = a.inc;                          // k x nk   X1'^T A2
    const double* H = a.inc + kn;                     // k x k    X1'^T B_p (first t columns)
    const double* G = H + (int64_t)k * k;             // k x k    X1'^T X1'
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      const int i = idx / k, j = idx - i * k;
      g[idx] = 0.5 * (G[i * k + j] + G[j * k + i]);
    }
    for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
      const int i = idx / t, j = idx - i * t;
      double v = 0.0;
      for (int c = 0; c < nk; ++c) v = fma(a.D[(int64_t)i * nk + c], a.D[(int64_t)j * nk + c], v);
      s[idx] = v;
    }
    __syncthreads();
    if (!als_gj_inverse(g, gi, fac, k)) {
      if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
      return;
    }
    // reload G' (the inverse destroyed it) for the objective terms
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      const int i = idx / k, j = idx - i * k;
      g[idx] = 0.5 * (G[i * k + j] + G[j * k + i]);
    }
    __syncthreads();
    // C' = G'^{-1} (M' - H' D_p), column by column of the n-k index; <M', C'> accumulated
    double mc = 0.0;
    for (int64_t idx = threadIdx.x; idx < kn; idx += blockDim.x) {
      const int q = (int)(idx / nk), c = (int)(idx - (int64_t)q * nk);
      double v = 0.0;
      for (int l = 0; l < k; ++l) {
        double r = M[(int64_t)l * nk + c];
        for (int j = 0; j < t; ++j) r = fma(-H[(int64_t)l * k + j], a.D[(int64_t)j * nk + c], r);
        v = fma(gi[q * k + l], r, v);
      }
      a.Cout[idx] = v;
      mc = fma(M[idx], v, mc);
    }
    mc = warp_sum(mc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
      a.scal[1] = v;                                  // <M', C'>
      a.scal[0] = a.inc[kn + 2LL * k * k];            // f_w of X1'
    }
  }
  __syncthreads();
  const double* Cn = a.c_given ? a.C : a.Cout;
  // S^{-1}
  if (!als_gj_inverse(s, si, fac, t)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;
  }
  // C' D^T (k x t)
  for (int idx = threadIdx.x; idx < k * t; idx += blockDim.x) {
    const int q = idx / t, j = idx - q * t;
    double v = 0.0;
    for (int c = 0; c < nk; ++c) v = fma(Cn[(int64_t)q * nk + c], a.D[(int64_t)j * nk + c], v);
    dtc[idx] = v;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < k * t; idx += blockDim.x) {
    const int q = idx / t, j = idx - q * t;
    double v = 0.0;
    for (int i = 0; i < t; ++i) v = fma(dtc[q * t + i], si[i * t + j], v);
    cds[idx] = v;
  }
  __syncthreads();
  if (!a.c_given) {   // <C', G' C'> for the objective
    double cgc = 0.0;
    for (int64_t idx = threadIdx.x; idx < kn; idx += blockDim.x) {
      const int q = (int)(idx / nk), c = (int)(idx - (int64_t)q * nk);
      double v = 0.0;
      for (int l = 0; l < k; ++l) v = fma(g[q * k + l], Cn[(int64_t)l * nk + c], v);
      cgc = fma(Cn[idx], v, cgc);
    }
    cgc = warp_sum(cgc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cgc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
      a.scal[2] = v;
    }
  }
  // Wb: A2 rows k + c: (D^T S^{-1})[c, :]; X1 rows KA + q: -(C' D^T S^{-1})[q, :]
  const int RB = a.rpb;
  for (int idx = threadIdx.x; idx < nk * t; idx += blockDim.x) {
    const int c = idx / t, j = idx - c * t;
    double v = 0.0;
    for (int i = 0; i < t; ++i) v = fma(a.D[(int64_t)i * nk + c], si[i * t + j], v);
    als_store<T>(a.Wb, (int64_t)(k + c) * RB + j, v);
  }
  for (int idx = threadIdx.x; idx < k * t; idx += blockDim.x) {
    const int q = idx / t, j = idx - q * t;
    als_store<T>(a.Wb, (int64_t)(a.KA + q) * RB + j, -cds[idx]);
  }
}

// ------------------------------------------------------------------ D step + objective
__global__ void __launch_bounds__(kAlsT) als_d_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  const double* BA = a.inc;                          // t x nk   B'^T A2
  const double* BX = a.inc + (int64_t)t * nk;        // t x k    B'^T X1'
  const double* BB = BX + (int64_t)t * k;            // t x t    B'^T B'
  double* bb = sm;                   // t x t
  double* bbi = bb + t * t;          // t x t
  double* fac = bbi + t * t;         // t
  double* red = fac + t;             // 2 x warps
  for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
    const int i = idx / t, j = idx - i * t;
    bb[idx] = 0.5 * (BB[i * t + j] + BB[j * t + i]);
  }
  __syncthreads();
  if (!als_gj_inverse(bb, bbi, fac, t)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;
  }
  // D' = (B'^T B')^{-1} (B'^T A2 - (B'^T X1') C'); objective terms <B'^T A2, D'>,
  // <D', (B'^T X1') C'>, <D', (B'^T B') D'>  (the last one from the symmetric BB)
  double v1 = 0.0, v2 = 0.0;
  for (int64_t idx = threadIdx.x; idx < (int64_t)t * nk; idx += blockDim.x) {
    const int j = (int)(idx / nk), c = (int)(idx - (int64_t)j * nk);
    double d = 0.0;
    for (int i = 0; i < t; ++i) {
      double r = BA[(int64_t)i * nk + c];
      for (int q = 0; q < k; ++q) r = fma(-BX[(int64_t)i * k + q], a.C[(int64_t)q * nk + c], r);
      d = fma(bbi[j * t + i], r, d);
    }
    a.Dout[idx] = d;
    double xc = 0.0;
    for (int q = 0; q < k; ++q) xc = fma(BX[(int64_t)j * k + q], a.C[(int64_t)q * nk + c], xc);
    v1 = fma(BA[idx], d, v1);
    v2 = fma(xc, d, v2);
  }
  __syncthreads();   // every D' entry written before the quadratic term reads it
  double v3 = 0.0;
  for (int64_t idx = threadIdx.x; idx < (int64_t)t * nk; idx += blockDim.x) {
    const int j = (int)(idx / nk), c = (int)(idx - (int64_t)j * nk);
    double u = 0.0;
    for (int i = 0; i < t; ++i) u = fma(0.5 * (BB[j * t + i] + BB[i * t + j]), a.Dout[(int64_t)i * nk + c], u);
    v3 = fma(a.Dout[idx], u, v3);
  }
  v1 = warp_sum(v1); v2 = warp_sum(v2); v3 = warp_sum(v3);
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[w] = v1; red[nw + w] = v2; red[2 * nw + w] = v3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int i = 0; i < nw; ++i) { s1 += red[i]; s2 += red[nw + i]; s3 += red[2 * nw + i]; }
    // F = f_w + ||A2||^2 - 2 <M', C'> - 2 <B'^T A2, D'> + <C', G' C'> + 2 <D', (B'^T X1') C'>
    //     + <D', (B'^T B') D'>   (||A2 - X1 C - B D||^2 expanded through the Grams)
    const double F = a.scal[0] + a.a2sq - 2.0 * a.scal[1] - 2.0 * s1 + a.scal[2] + 2.0 * s2 + s3;
    a.Fout[0] = F;
  }
}

size_t als_smem_w(int k, int t) { return sizeof(double) * (size_t)(2 * k * k + t * k + k + 8); }
size_t als_smem_c(int k, int t) {
  return sizeof(double) * (size_t)(2 * k * k + 2 * t * t + 2 * k * t + (k > t ? k : t) + 2 * (kAlsT / 32) + 8);
}
size_t als_smem_d(int t) { return sizeof(double) * (size_t)(2 * t * t + t + 3 * (kAlsT / 32) + 8); }

template <typename T>
static cudaError_t launch_als_t(const AlsArgs& a, int which, cudaStream_t st) {
  size_t smem;
  switch (which) {
    case 0:
      smem = als_smem_w(a.k, a.t);
      cudaFuncSetAttribute(als_w_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      als_w_kernel<T><<<1, kAlsT, smem, st>>>(a);
      break;
    case 1:
      smem = als_smem_c(a.k, a.t);
      cudaFuncSetAttribute(als_c_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      als_c_kernel<T><<<1, kAlsT, smem, st>>>(a);
      break;
    default:
      smem = als_smem_d(a.t);
      als_d_kernel<<<1, kAlsT, smem, st>>>(a);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_als(const AlsArgs& a, int which, bool f64, cudaStream_t st) {
  return f64 ? launch_als_t<double>(a, which, st) : launch_als_t<float>(a, which, st);
}

bool als_ok(int k, int t) { return als_smem_c(k, t) <= 200 * 1024 && als_smem_w(k, t) <= 200 * 1024; }

}  // namespace wlr

namespace wlr {
// D_0 = V_0^T  (V: nk x t row-major -> D: t x nk)
__global__ void als_transpose_kernel(const double* V, double* D, int nk, int t) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nk * t; idx += gridDim.x * blockDim.x) {
    const int c = idx / t, j = idx - c * t;
    D[(int64_t)j * nk + c] = V[idx];
  }
}
cudaError_t launch_als_transpose(const double* V, double* D, int nk, int t, cudaStream_t st) {
  als_transpose_kernel<<<(nk * t + 255) / 256, 256, 0, st>>>(V, D, nk, t);
  return cudaGetLastError();
}
}  // namespace wlr
