// als.cu -- SURVEY.md §8(f3): the factorised WLR as a one-sweep block ALS on (X1, C, B, D),
// X2 = X1 C + B D (reading R21).  The m-scaled work reuses the sWLR kernels (the linear
// row map with Z = [A | B], the row Grams, the fixed-order reduce, the result-mode row map for
// B); this file holds the fp64 small steps.  The (n-k)-indexed work is split over CTAs by column
// blocks of CW columns (each CTA redoes the k x k / t x t inverses it needs), and the cross-column
// sums go through per-CTA partials summed in fixed order by a one-CTA finishing kernel:
//
//   als_w   : W'' = [w^2 K^{-1}; C^T K^{-1}; -(D C^T) K^{-1}] (uniform W1) or [0; C^T; -(D C^T)]
//             with Kop = C C^T (per-row solves), K = w^2 I + C C^T: the X1 update of
//             PAPER.md:184-196 with D_p := B_p D_p.  Needs C C^T and D C^T (from cx / dx).
//   als_c   : C' = G'^{-1} (M' - H' D) per column (G' = X1'^T X1', M' = X1'^T A2, H' = X1'^T B),
//             the B map's A2 rows D^T S^{-1} (S = D D^T); partials C' D^T, C' C'^T, <M', C'>,
//             <C', G' C'>
//   als_cx  : sums them; the B map's X1 rows -C' D^T S^{-1}; C C^T for the next als_w
//   als_d   : D' = (B'^T B')^{-1} (B'^T A2 - (B'^T X1') C') per column; partials of the objective
//             terms and of D' C'^T
//   als_dx  : sums them: F, and D C^T for the next als_w
#include "kernels.h"

namespace wlr {

constexpr int kAlsT = 512;
constexpr int kAlsCW = 16;         // columns of the (n-k) index per CTA

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

// block sum of NV values per thread into out[0..NV) (thread 0)
template <int NV>
__device__ void als_block_sum(double (&v)[NV], double* red, double* out) {
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    v[u] = warp_sum(v[u]);
    if ((threadIdx.x & 31) == 0) red[u * 32 + w] = v[u];
  }
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      double s = 0.0;
      for (int i = 0; i < nw; ++i) s += red[u * 32 + i];
      out[u] = s;
    }
  __syncthreads();
}

// ------------------------------------------------------------------ W'' of the X1 row map
template <typename T>
__global__ void __launch_bounds__(kAlsT) als_w_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  double* kk = sm;                  // k x k   K (destroyed)
  double* ki = kk + k * k;          // k x k   K^{-1}
  double* fac = ki + k * k;         // k
  const int c0 = blockIdx.x * kAlsCW, c1 = min(nk, c0 + kAlsCW);
  if (a.uniform) {
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x)
      kk[idx] = a.cct[idx] + ((idx / k == idx % k) ? a.w2 : 0.0);
    __syncthreads();
    if (!als_gj_inverse(kk, ki, fac, k)) {
      if (threadIdx.x == 0) raise_flag(a.flags, DF_ROWSPD);
      return;
    }
  } else if (blockIdx.x == 0) {   // Kop = C C^T for the per-row solves (diag(W1(i,:)^2) per row)
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      als_store<T>(a.Kop, idx, a.cct[idx]);
      if (a.Sop) a.Sop[(idx / k) * ((k + 7) & ~7) + idx % k] = (float)a.cct[idx];
    }
  }
  const int RP = a.rp;
  if (blockIdx.x == 0) {
    // A1 rows j < k: w^2 K^{-1} (uniform; 0 otherwise -- the epilogue adds a1 w^2 before the solve)
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      const int j = idx / k, l = idx - j * k;
      als_store<T>(a.W, (int64_t)j * RP + l, a.uniform ? a.w2 * ki[idx] : 0.0);
    }
    // B rows KA + j: -(D C^T)[j, :] K^{-1} (or -(D C^T)[j, :])
    for (int idx = threadIdx.x; idx < t * k; idx += blockDim.x) {
      const int j = idx / k, l = idx - j * k;
      double v;
      if (a.uniform) {
        v = 0.0;
        for (int q = 0; q < k; ++q) v = fma(a.dct[j * k + q], ki[q * k + l], v);
      } else {
        v = a.dct[idx];
      }
      als_store<T>(a.W, (int64_t)(a.KA + j) * RP + l, -v);
    }
  }
  // A2 rows k + c of this CTA's columns: C[:, c]^T K^{-1} (or C[:, c]^T)
  for (int idx = threadIdx.x; idx < (c1 - c0) * k; idx += blockDim.x) {
    const int c = c0 + idx / k, l = idx % k;
    double v;
    if (a.uniform) {
      v = 0.0;
      for (int q = 0; q < k; ++q) v = fma(a.C[(int64_t)q * nk + c], ki[q * k + l], v);
    } else {
      v = a.C[(int64_t)l * nk + c];
    }
    als_store<T>(a.W, (int64_t)(k + c) * RP + l, v);
  }
}

// partial block of one CTA of als_c: [C D^T (k x t) | C C^T (k x k) | <M',C'> | <C',G'C'>]
__host__ __device__ inline int als_pc(int k, int t) { return k * t + k * k + 2; }
// partial block of one CTA of als_d: [D C^T (t x k) | v1 | v2 | v3]
__host__ __device__ inline int als_pd(int k, int t) { return t * k + 3; }

// ------------------------------------------------------------------ C step + the B map's A2 rows
template <typename T>
__global__ void __launch_bounds__(kAlsT) als_c_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  const int64_t kn = (int64_t)k * nk;
  const int c0 = blockIdx.x * kAlsCW, c1 = min(nk, c0 + kAlsCW), nc = c1 - c0;
  double* g = sm;                   // k x k  G' (symmetrised), then kept for <C', G' C'>
  double* gi = g + k * k;           // k x k  G'^{-1}
  double* s = gi + k * k;           // t x t  D D^T
  double* si = s + t * t;           // t x t
  double* cb = si + t * t;          // k x CW  C' of this CTA's columns
  double* fac = cb + k * kAlsCW;    // max(k, t)
  double* red = fac + (k > t ? k : t);   // 32 x 2
  double* gw = red + 64;            // k x k  work copy for the inverse
  double* rb = gw + k * k;          // k x CW  M' - H' D of this CTA's columns
  const double* M = a.inc;                          // k x nk   X1'^T A2
  const double* H = a.inc + kn;                     // k x k    X1'^T B (first t columns)
  const double* G = H + (int64_t)k * k;             // k x k    X1'^T X1'
  for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
    const int i = idx / t, j = idx - i * t;
    double v = 0.0;
    for (int c = 0; c < nk; ++c) v = fma(a.D[(int64_t)i * nk + c], a.D[(int64_t)j * nk + c], v);
    s[idx] = v;
  }
  if (!a.c_given) {
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
      const int i = idx / k, j = idx - i * k;
      g[idx] = 0.5 * (G[i * k + j] + G[j * k + i]);
      gw[idx] = g[idx];
    }
    __syncthreads();
    if (!als_gj_inverse(gw, gi, fac, k)) {
      if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
      return;
    }
    // C'[:, c] = G'^{-1} (M'[:, c] - H' D[:, c]) for this CTA's columns
    for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {   // R into cb first
      const int l = idx / nc, cc = idx - l * nc, c = c0 + cc;
      double r = M[(int64_t)l * nk + c];
      for (int j = 0; j < t; ++j) r = fma(-H[(int64_t)l * k + j], a.D[(int64_t)j * nk + c], r);
      rb[l * kAlsCW + cc] = r;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {
      const int q = idx / nc, cc = idx - q * nc;
      double v = 0.0;
      for (int l = 0; l < k; ++l) v = fma(gi[q * k + l], rb[l * kAlsCW + cc], v);
      cb[q * kAlsCW + cc] = v;
      a.Cout[(int64_t)q * nk + c0 + cc] = v;
    }
  } else {
    for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {
      const int q = idx / nc, cc = idx - q * nc;
      cb[q * kAlsCW + cc] = a.C[(int64_t)q * nk + c0 + cc];
    }
  }
  __syncthreads();
  if (!als_gj_inverse(s, si, fac, t)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;
  }
  // partials over this CTA's columns
  double* out = a.part + (int64_t)blockIdx.x * als_pc(k, t);
  for (int idx = threadIdx.x; idx < k * t; idx += blockDim.x) {     // C D^T
    const int q = idx / t, j = idx - q * t;
    double v = 0.0;
    for (int cc = 0; cc < nc; ++cc) v = fma(cb[q * kAlsCW + cc], a.D[(int64_t)j * nk + c0 + cc], v);
    out[idx] = v;
  }
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {     // C C^T
    const int i = idx / k, j = idx - i * k;
    double v = 0.0;
    for (int cc = 0; cc < nc; ++cc) v = fma(cb[i * kAlsCW + cc], cb[j * kAlsCW + cc], v);
    out[k * t + idx] = v;
  }
  double v[2] = {0.0, 0.0};
  if (!a.c_given)
    for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {  // <M', C'>, <C', G' C'>
      const int q = idx / nc, cc = idx - q * nc;
      double gc = 0.0;
      for (int l = 0; l < k; ++l) gc = fma(g[q * k + l], cb[l * kAlsCW + cc], gc);
      v[0] = fma(M[(int64_t)q * nk + c0 + cc], cb[q * kAlsCW + cc], v[0]);
      v[1] = fma(cb[q * kAlsCW + cc], gc, v[1]);
    }
  als_block_sum<2>(v, red, out + k * t + k * k);
  // the B map's A2 rows k + c: (D^T S^{-1})[c, :]
  const int RB = a.rpb;
  for (int idx = threadIdx.x; idx < nc * t; idx += blockDim.x) {
    const int c = c0 + idx / t, j = idx % t;
    double w = 0.0;
    for (int i = 0; i < t; ++i) w = fma(a.D[(int64_t)i * nk + c], si[i * t + j], w);
    als_store<T>(a.Wb, (int64_t)(k + c) * RB + j, w);
  }
}

// ------------------------------------------------------------------ sums of als_c's partials
template <typename T>
__global__ void __launch_bounds__(kAlsT) als_cx_kernel(AlsArgs a, int nblk) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t, pc = als_pc(k, t);
  double* cd = sm;                  // k x t  C' D^T
  double* s = cd + k * t;           // t x t
  double* si = s + t * t;
  double* fac = si + t * t;         // t
  for (int i = threadIdx.x; i < pc; i += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < nblk; ++b) v += a.part[(int64_t)b * pc + i];
    if (i < k * t) cd[i] = v;
    else if (i < k * t + k * k) a.cct[i - k * t] = v;
    else if (i == k * t + k * k && !a.c_given) a.scal[1] = v;   // <M', C'>
    else if (!a.c_given) a.scal[2] = v;                          // <C', G' C'>
  }
  if (threadIdx.x == 0 && !a.c_given) a.scal[0] = a.inc[(int64_t)k * nk + 2LL * k * k];   // f_w of X1'
  for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
    const int i = idx / t, j = idx - i * t;
    double v = 0.0;
    for (int c = 0; c < nk; ++c) v = fma(a.D[(int64_t)i * nk + c], a.D[(int64_t)j * nk + c], v);
    s[idx] = v;
  }
  __syncthreads();
  if (a.c_given)   // the GHS start: D C^T of (C_0, D_0) for the first als_w
    for (int idx = threadIdx.x; idx < t * k; idx += blockDim.x) {
      const int j = idx / k, q = idx - j * k;
      a.dct[idx] = cd[q * t + j];
    }
  if (!als_gj_inverse(s, si, fac, t)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;
  }
  const int RB = a.rpb;
  for (int idx = threadIdx.x; idx < k * t; idx += blockDim.x) {   // X1 rows: -(C' D^T S^{-1})
    const int q = idx / t, j = idx - q * t;
    double v = 0.0;
    for (int i = 0; i < t; ++i) v = fma(cd[q * t + i], si[i * t + j], v);
    als_store<T>(a.Wb, (int64_t)(a.KA + q) * RB + j, -v);
  }
}

// ------------------------------------------------------------------ D step
__global__ void __launch_bounds__(kAlsT) als_d_kernel(AlsArgs a) {
  extern __shared__ double sm[];
  const int k = a.k, nk = a.nk, t = a.t;
  const int c0 = blockIdx.x * kAlsCW, c1 = min(nk, c0 + kAlsCW), nc = c1 - c0;
  const double* BA = a.inc;                          // t x nk   B'^T A2
  const double* BX = a.inc + (int64_t)t * nk;        // t x k    B'^T X1'
  const double* BB = BX + (int64_t)t * k;            // t x t    B'^T B'
  double* bb = sm;                   // t x t
  double* bbi = bb + t * t;          // t x t
  double* bs = bbi + t * t;          // t x t  symmetrised B'^T B'
  double* db = bs + t * t;           // t x CW  D' of this CTA's columns
  double* xc = db + t * kAlsCW;      // t x CW  (B'^T X1') C'
  double* fac = xc + t * kAlsCW;     // t
  double* red = fac + t;             // 3 x 32
  for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
    const int i = idx / t, j = idx - i * t;
    bb[idx] = 0.5 * (BB[i * t + j] + BB[j * t + i]);
    bs[idx] = bb[idx];
  }
  for (int idx = threadIdx.x; idx < t * nc; idx += blockDim.x) {
    const int j = idx / nc, cc = idx - j * nc;
    double v = 0.0;
    for (int q = 0; q < k; ++q) v = fma(BX[(int64_t)j * k + q], a.C[(int64_t)q * nk + c0 + cc], v);
    xc[j * kAlsCW + cc] = v;
  }
  __syncthreads();
  if (!als_gj_inverse(bb, bbi, fac, t)) {
    if (threadIdx.x == 0) raise_flag(a.flags, DF_RANK);
    return;
  }
  for (int idx = threadIdx.x; idx < t * nc; idx += blockDim.x) {
    const int j = idx / nc, cc = idx - j * nc;
    double d = 0.0;
    for (int i = 0; i < t; ++i) d = fma(bbi[j * t + i], BA[(int64_t)i * nk + c0 + cc] - xc[i * kAlsCW + cc], d);
    db[j * kAlsCW + cc] = d;
    a.Dout[(int64_t)j * nk + c0 + cc] = d;
  }
  __syncthreads();
  double* out = a.part + (int64_t)blockIdx.x * als_pd(k, t);
  for (int idx = threadIdx.x; idx < t * k; idx += blockDim.x) {   // D' C'^T over this CTA's columns
    const int j = idx / k, q = idx - j * k;
    double v = 0.0;
    for (int cc = 0; cc < nc; ++cc) v = fma(db[j * kAlsCW + cc], a.C[(int64_t)q * nk + c0 + cc], v);
    out[idx] = v;
  }
  // objective terms <B'^T A2, D'>, <D', (B'^T X1') C'>, <D', (B'^T B') D'>
  double v[3] = {0.0, 0.0, 0.0};
  for (int idx = threadIdx.x; idx < t * nc; idx += blockDim.x) {
    const int j = idx / nc, cc = idx - j * nc;
    const double d = db[j * kAlsCW + cc];
    double u = 0.0;
    for (int i = 0; i < t; ++i) u = fma(bs[j * t + i], db[i * kAlsCW + cc], u);
    v[0] = fma(BA[(int64_t)j * nk + c0 + cc], d, v[0]);
    v[1] = fma(xc[j * kAlsCW + cc], d, v[1]);
    v[2] = fma(d, u, v[2]);
  }
  als_block_sum<3>(v, red, out + t * k);
}

// ------------------------------------------------------------------ sums of als_d's partials, F
__global__ void __launch_bounds__(kAlsT) als_dx_kernel(AlsArgs a, int nblk) {
  const int k = a.k, t = a.t, pd = als_pd(k, t);
  __shared__ double tr[3];
  for (int i = threadIdx.x; i < pd; i += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < nblk; ++b) v += a.part[(int64_t)b * pd + i];
    if (i < t * k) a.dct[i] = v;
    else tr[i - t * k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // F = f_w + ||A2||^2 - 2 <M', C'> - 2 <B'^T A2, D'> + <C', G' C'> + 2 <D', (B'^T X1') C'>
    //     + <D', (B'^T B') D'>   (||A2 - X1 C - B D||^2 expanded through the Grams)
    a.Fout[0] = a.scal[0] + a.a2sq - 2.0 * a.scal[1] - 2.0 * tr[0] + a.scal[2] + 2.0 * tr[1] + tr[2];
  }
}

static size_t als_smem_w(int k) { return sizeof(double) * (size_t)(2 * k * k + k + 8); }
static size_t als_smem_c(int k, int t) {
  return sizeof(double) * (size_t)(3 * k * k + 2 * t * t + 2 * k * kAlsCW + (k > t ? k : t) + 64 + 8);
}
static size_t als_smem_cx(int k, int t) { return sizeof(double) * (size_t)(k * t + 2 * t * t + t + 8); }
static size_t als_smem_d(int t) { return sizeof(double) * (size_t)(3 * t * t + 2 * t * kAlsCW + t + 96 + 8); }

int als_blocks(int nk) { return (nk + kAlsCW - 1) / kAlsCW; }
size_t als_part_doubles(int k, int t, int nk) {
  return (size_t)als_blocks(nk) * (size_t)std::max(als_pc(k, t), als_pd(k, t));
}

template <typename T>
static cudaError_t launch_als_t(const AlsArgs& a, int which, cudaStream_t st) {
  const int nb = als_blocks(a.nk);
  size_t smem;
  switch (which) {
    case 0:
      smem = als_smem_w(a.k);
      cudaFuncSetAttribute(als_w_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      als_w_kernel<T><<<nb, kAlsT, smem, st>>>(a);
      break;
    case 1:
      smem = als_smem_c(a.k, a.t);
      cudaFuncSetAttribute(als_c_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      als_c_kernel<T><<<nb, kAlsT, smem, st>>>(a);
      if (cudaGetLastError() != cudaSuccess) break;
      smem = als_smem_cx(a.k, a.t);
      als_cx_kernel<T><<<1, kAlsT, smem, st>>>(a, nb);
      break;
    default:
      smem = als_smem_d(a.t);
      als_d_kernel<<<nb, kAlsT, smem, st>>>(a);
      if (cudaGetLastError() != cudaSuccess) break;
      als_dx_kernel<<<1, kAlsT, 0, st>>>(a, nb);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_als(const AlsArgs& a, int which, bool f64, cudaStream_t st) {
  return f64 ? launch_als_t<double>(a, which, st) : launch_als_t<float>(a, which, st);
}

bool als_ok(int k, int t) { return als_smem_c(k, t) <= 200 * 1024 && als_smem_w(k) <= 200 * 1024; }

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
