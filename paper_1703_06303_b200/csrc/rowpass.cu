// rowpass.cu -- the m-scaled part of one sWLR iteration.
//
// K2a  row_pass_kernel : for every pixel row i (Algorithm 1 lines 7-9)
//        y   = A2(i,:) [V_p | C_p^T]                      (tall-skinny GEMM, CUDA-core FP32)
//        b   = y_V - X1_p(i,:) (C_p V_p)                   (= B_p(i,:), D_p = B_p V_p^T)
//        e   = A1(i,:) . W1(i,:)^2 + y_C - b (C_p V_p)^T   (= E_p(i,:) = [A1.W1.W1 + (A2-D_p)C_p^T](i,:))
//        x'  = e (diag(W1(i,:)^2) + C_p C_p^T)^{-1}        (uniform W1: one shared inverse;
//                                                           otherwise warp-per-row Cholesky)
//      writes X1_{p+1}(i,:) and an fp64 partial of f_w = sum W1^2 (A1 - X1_{p+1})^2.
//      MODE_RESULT writes b (row of B) instead of solving (wlr_result).
// K2b  incr_kernel : Gram increments with Delta = X1_{p+1} - X1_p (fp32, from the stored
//        values):  N = Delta^T A2,  Gamma = Delta^T X1_p,  Omega = Delta^T Delta.
//        fp32 inside 256-row super-chunks, fp64 across them and across CTAs.
// K2c  reduce_incr_kernel : fixed-order fp64 sum of the K2b/K2a partials into the packed
//        increment vector [N | Gamma | Omega | f_w] that is all-reduced across ranks.
#include "kernels.h"

namespace wlr {

// ------------------------------------------------------------------------------ K2a
template <int RP> struct RowPassShape;
template <> struct RowPassShape<16>  { static constexpr int TM = 128, TR = 4, TC = 2; };
template <> struct RowPassShape<32>  { static constexpr int TM = 128, TR = 4, TC = 4; };
template <> struct RowPassShape<64>  { static constexpr int TM = 128, TR = 8, TC = 4; };
template <> struct RowPassShape<128> { static constexpr int TM = 64,  TR = 4, TC = 8; };

constexpr int kRowKC = 32;        // reduction chunk (columns of A2)
constexpr int kRowThreads = 256;

template <typename T, int RP>
struct RowPassSmem {
  using S = RowPassShape<RP>;
  static constexpr int TMP = S::TM + 4;                         // padded row count (As)
  static constexpr int kAsBs = kRowKC * TMP + kRowKC * RP;      // GEMM phase
  static constexpr int kYs = S::TM * (RP + 1);                  // epilogue y tile
  static constexpr int kUnion = kAsBs > kYs ? kAsBs : kYs;
};

// Per-warp scratch for the epilogue: b (t values), e / solution (kp values), and for
// non-uniform W1 the packed lower triangle of the row matrix.
__host__ __device__ inline int chol_packed(int kp) { return kp * (kp + 1) / 2; }

template <typename T>
WLR_DEVI void load_vec4_or_scalar(const T* p, bool vec, T out[4], int valid) {
  if (vec && valid == 4) {
    auto v = ldg4<T>(p);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = q < valid ? __ldg(p + q) : T(0);
  }
}

template <typename T, int RP, bool UNIFORM, int MODE>
__global__ void __launch_bounds__(kRowThreads)
row_pass_kernel(RowPassArgs<T> a) {
  using S = RowPassShape<RP>;
  constexpr int TM = S::TM, TR = S::TR, TC = S::TC;
  constexpr int TMP = RowPassSmem<T, RP>::TMP;
  constexpr int THC = RP / TC;                 // threads along columns
  static_assert((TM / TR) * THC == kRowThreads, "thread tile");
  constexpr int AV = TM * kRowKC / 4 / kRowThreads;     // vec4 loads of A per thread
  constexpr int BVN = kRowKC * RP / 4;                  // vec4 of one Wt chunk
  constexpr int BV = (BVN + kRowThreads - 1) / kRowThreads;   // per thread (guarded)
  constexpr int BVc = BV;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* As = sm;                                   // [KC][TMP]
  T* Bs = sm + kRowKC * TMP;                    // [KC][RP]
  T* Ys = sm;                                   // [TM][RP+1] (aliases As/Bs after the GEMM)
  T* sK = sm + RowPassSmem<T, RP>::kUnion;      // uniform: K^{-1} (k x k); else C C^T (k x k)
  T* sCV = sK + (UNIFORM ? a.k * a.k : 0);      // C V (k x t)
  T* sW = sCV + a.k * a.t;                      // per-warp scratch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kp = a.kp, k = a.k, t = a.t;
  const int wstride = 32 + kp + (UNIFORM ? 0 : chol_packed(kp));
  T* wb = sW + warp * wstride;                  // b   [32]
  T* we = wb + 32;                              // e   [kp]
  T* wL = we + kp;                              // packed L (non-uniform)

  for (int i = threadIdx.x; i < (UNIFORM ? k * k : 0); i += kRowThreads) sK[i] = a.Kmat[i];
  for (int i = threadIdx.x; i < k * t; i += kRowThreads) sCV[i] = a.CV[i];

  const int ty = threadIdx.x / THC, tx = threadIdx.x % THC;
  const int nch = (int)ceil_div(a.n - a.k0, kRowKC);
  double fw = 0.0;
  const int64_t ntiles = ceil_div(a.m, TM);

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TM;
    // ---------------- GEMM  Y[TM x RP] = A2_tile . Wt  (register-prefetched chunks)
    T acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = T(0);
    T ra[AV][4];
    T rb[BVc][4];
    auto gload = [&](int ch) {
      const int cb = a.k0 + ch * kRowKC;       // absolute first column of the chunk
#pragma unroll
      for (int e = 0; e < AV; ++e) {
        const int idx = threadIdx.x + e * kRowThreads;
        const int rr = idx / (kRowKC / 4), c4 = (idx % (kRowKC / 4)) * 4;
        const int64_t row = r0 + rr;
        const int col = cb + c4;
        int valid = a.n - col;
        valid = valid > 4 ? 4 : (valid < 0 ? 0 : valid);
        if (row >= a.m) valid = 0;
        load_vec4_or_scalar<T>(a.A + row * a.lda + col, a.vec_ok, ra[e], row < a.m ? valid : 0);
      }
#pragma unroll
      for (int e = 0; e < BV; ++e) {
        const int idx = threadIdx.x + e * kRowThreads;
        if (idx < BVN) {
          const int rr = idx / (RP / 4), c4 = (idx % (RP / 4)) * 4;
          const T* p = a.Wt + (int64_t)(ch * kRowKC + rr) * RP + c4;   // Wt padded: no bounds
          auto v = ldg4<T>(p);
          rb[e][0] = v.x; rb[e][1] = v.y; rb[e][2] = v.z; rb[e][3] = v.w;
        }
      }
    };
    auto sstore = [&]() {
#pragma unroll
      for (int e = 0; e < AV; ++e) {
        const int idx = threadIdx.x + e * kRowThreads;
        const int rr = idx / (kRowKC / 4), c4 = (idx % (kRowKC / 4)) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) As[(c4 + q) * TMP + rr] = ra[e][q];
      }
#pragma unroll
      for (int e = 0; e < BV; ++e) {
        const int idx = threadIdx.x + e * kRowThreads;
        if (idx < BVN) {
          const int rr = idx / (RP / 4), c4 = (idx % (RP / 4)) * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q) Bs[rr * RP + c4 + q] = rb[e][q];
        }
      }
    };
    gload(0);
    __syncthreads();            // previous tile's epilogue finished with Ys (aliases As)
    sstore();
    __syncthreads();
    for (int ch = 0; ch < nch; ++ch) {
      if (ch + 1 < nch) gload(ch + 1);
#pragma unroll 8
      for (int kk = 0; kk < kRowKC; ++kk) {
        T av[TR], bv[TC];
#pragma unroll
        for (int i = 0; i < TR; ++i) av[i] = As[kk * TMP + ty * TR + i];
#pragma unroll
        for (int j = 0; j < TC; ++j) bv[j] = Bs[kk * RP + tx * TC + j];
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
      if (ch + 1 < nch) {
        sstore();
        __syncthreads();
      }
    }
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) Ys[(ty * TR + i) * (RP + 1) + tx * TC + j] = acc[i][j];
    __syncthreads();

    // ---------------- epilogue: warp per row
    for (int rl = warp; rl < TM; rl += kRowThreads / 32) {
      const int64_t g = r0 + rl;
      if (g >= a.m) break;
      const T* yr = Ys + rl * (RP + 1);
      const T* xo = a.Xold + g * kp;
      // b_j = y_V[j] - sum_l x_l (CV)_{lj}
      for (int j = 0; j < t; ++j) {
        T part = T(0);
        for (int l = lane; l < k; l += 32) part = fma(xo[l], sCV[l * t + j], part);
        part = warp_sum(part);
        if (lane == 0) wb[j] = yr[j] - part;
      }
      __syncwarp();
      if (MODE == 1) {                       // wlr_result: B(i,:) = b
        for (int j = lane; j < t; j += 32) a.Bout[g * a.ldb + j] = wb[j];
        __syncwarp();
        continue;
      }
      // e_l = a1_l w_l^2 + y_C[l] - sum_j b_j (CV)_{lj}
      for (int l = lane; l < kp; l += 32) {
        T e = T(0);
        if (l < k) {
          const T a1 = a.A[g * a.lda + l];
          const T w2 = UNIFORM ? a.w2s : a.W1[g * a.ldw + l] * a.W1[g * a.ldw + l];
          e = fma(a1, w2, yr[t + l]);
          for (int j = 0; j < t; ++j) e = fma(-wb[j], sCV[l * t + j], e);
        }
        we[l] = e;
      }
      __syncwarp();
      if (UNIFORM) {
        // x'_l = sum_m e_m (K^{-1})_{ml}
        for (int l = lane; l < kp; l += 32) {
          T x = T(0);
          if (l < k)
            for (int mm = 0; mm < k; ++mm) x = fma(we[mm], sK[mm * k + l], x);
          a.Xnew[g * kp + l] = x;
          if (l < k) {
            const double d = (double)a.A[g * a.lda + l] - (double)x;
            fw += (double)a.w2s * d * d;
          }
        }
      } else {
        // K = C C^T + diag(w^2), packed lower triangle P(i,j) = i(i+1)/2 + j
        for (int idx = lane; idx < chol_packed(k); idx += 32) {
          int i = (int)((sqrtf(8.f * idx + 1.f) - 1.f) * 0.5f);
          while ((i + 1) * (i + 2) / 2 <= idx) ++i;
          while (i * (i + 1) / 2 > idx) --i;
          const int j = idx - i * (i + 1) / 2;
          T v = a.Kmat[i * k + j];
          if (i == j) v += a.W1[g * a.ldw + i] * a.W1[g * a.ldw + i];
          wL[idx] = v;
        }
        __syncwarp();
        bool spd = true;
        for (int j = 0; j < k; ++j) {
          const T djj = wL[j * (j + 1) / 2 + j];
          spd = spd && (djj > T(0));
          const T d = sqrt(djj > T(0) ? djj : T(1));
          const T inv = T(1) / d;
          __syncwarp();
          if (lane == 0) wL[j * (j + 1) / 2 + j] = d;
          for (int i = j + 1 + lane; i < k; i += 32) wL[i * (i + 1) / 2 + j] *= inv;
          __syncwarp();
          for (int i = j + 1 + lane; i < k; i += 32) {
            const T lij = wL[i * (i + 1) / 2 + j];
            T* rowi = wL + i * (i + 1) / 2;
            for (int l = j + 1; l <= i; ++l) rowi[l] = fma(-lij, wL[l * (l + 1) / 2 + j], rowi[l]);
          }
          __syncwarp();
        }
        if (!spd && lane == 0) raise_flag(a.flags, DF_ROWSPD);
        // forward: L z = e
        for (int j = 0; j < k; ++j) {
          const T zj = we[j] / wL[j * (j + 1) / 2 + j];
          for (int i = j + 1 + lane; i < k; i += 32) we[i] = fma(-wL[i * (i + 1) / 2 + j], zj, we[i]);
          __syncwarp();
          if (lane == 0) we[j] = zj;
          __syncwarp();
        }
        // backward: L^T x = z
        for (int j = k - 1; j >= 0; --j) {
          const T xj = we[j] / wL[j * (j + 1) / 2 + j];
          const T* rowj = wL + j * (j + 1) / 2;
          for (int i = lane; i < j; i += 32) we[i] = fma(-rowj[i], xj, we[i]);
          __syncwarp();
          if (lane == 0) we[j] = xj;
          __syncwarp();
        }
        for (int l = lane; l < kp; l += 32) {
          const T x = l < k ? we[l] : T(0);
          a.Xnew[g * kp + l] = x;
          if (l < k) {
            const double w = (double)a.W1[g * a.ldw + l];
            const double d = (double)a.A[g * a.lda + l] - (double)x;
            fw += w * w * d * d;
          }
        }
      }
      __syncwarp();
    }
  }
  if (MODE == 0) {
    fw = warp_sum(fw);
    __shared__ double wsum[kRowThreads / 32];
    if (lane == 0) wsum[warp] = fw;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kRowThreads / 32; ++w) s += wsum[w];
      a.fw_part[blockIdx.x] = s;
    }
  }
}

template <typename T, int RP, bool UNIFORM>
size_t row_pass_smem_bytes(int k, int t, int kp) {
  const int wstride = 32 + kp + (UNIFORM ? 0 : chol_packed(kp));
  return sizeof(T) * ((size_t)RowPassSmem<T, RP>::kUnion + (UNIFORM ? (size_t)k * k : 0) +
                      (size_t)k * t + (size_t)(kRowThreads / 32) * wstride);
}

template <typename T, int RP, bool UNIFORM, int MODE>
static cudaError_t launch_rp(const RowPassArgs<T>& a, int grid, cudaStream_t st) {
  auto kern = row_pass_kernel<T, RP, UNIFORM, MODE>;
  const size_t smem = row_pass_smem_bytes<T, RP, UNIFORM>(a.k, a.t, a.kp);
  static size_t configured = 0;            // cudaFuncSetAttribute once per size increase
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  kern<<<grid, kRowThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int RP>
static cudaError_t dispatch_rp(const RowPassArgs<T>& a, bool uniform, int mode, int grid,
                               cudaStream_t st) {
  if (uniform) return mode ? launch_rp<T, RP, true, 1>(a, grid, st) : launch_rp<T, RP, true, 0>(a, grid, st);
  return mode ? launch_rp<T, RP, false, 1>(a, grid, st) : launch_rp<T, RP, false, 0>(a, grid, st);
}

int row_pass_rp(int r) { return r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : r <= 128 ? 128 : -1; }
int row_pass_tm(int rp) { return rp == 128 ? RowPassShape<128>::TM : 128; }

template <typename T>
size_t row_pass_smem(int rp, bool uniform, int k, int t, int kp) {
  switch (rp) {
    case 16: return uniform ? row_pass_smem_bytes<T, 16, true>(k, t, kp) : row_pass_smem_bytes<T, 16, false>(k, t, kp);
    case 32: return uniform ? row_pass_smem_bytes<T, 32, true>(k, t, kp) : row_pass_smem_bytes<T, 32, false>(k, t, kp);
    case 64: return uniform ? row_pass_smem_bytes<T, 64, true>(k, t, kp) : row_pass_smem_bytes<T, 64, false>(k, t, kp);
    default: return uniform ? row_pass_smem_bytes<T, 128, true>(k, t, kp) : row_pass_smem_bytes<T, 128, false>(k, t, kp);
  }
}
template size_t row_pass_smem<float>(int, bool, int, int, int);
template size_t row_pass_smem<double>(int, bool, int, int, int);

template <typename T>
cudaError_t launch_row_pass(const RowPassArgs<T>& a, int rp, bool uniform, int mode, int grid,
                            cudaStream_t st) {
  switch (rp) {
    case 16: return dispatch_rp<T, 16>(a, uniform, mode, grid, st);
    case 32: return dispatch_rp<T, 32>(a, uniform, mode, grid, st);
    case 64: return dispatch_rp<T, 64>(a, uniform, mode, grid, st);
    case 128: return dispatch_rp<T, 128>(a, uniform, mode, grid, st);
  }
  return cudaErrorInvalidValue;
}
template cudaError_t launch_row_pass<float>(const RowPassArgs<float>&, int, bool, int, int, cudaStream_t);
template cudaError_t launch_row_pass<double>(const RowPassArgs<double>&, int, bool, int, int, cudaStream_t);

// ------------------------------------------------------------------------------ K2b
template <int BM> struct IncrShape;
template <> struct IncrShape<16>  { static constexpr int BN = 128, TR = 2, TC = 4; };
template <> struct IncrShape<32>  { static constexpr int BN = 128, TR = 4, TC = 4; };
template <> struct IncrShape<64>  { static constexpr int BN = 64,  TR = 4, TC = 4; };
template <> struct IncrShape<128> { static constexpr int BN = 64,  TR = 8, TC = 4; };
constexpr int kIncRC = 32;          // rows per smem stage
constexpr int kIncSuper = 8;        // stages per fp32 super-chunk (256 rows)

int incr_bm(int kp) { return kp <= 16 ? 16 : kp <= 32 ? 32 : kp <= 64 ? 64 : kp <= 128 ? 128 : -1; }
int incr_bn(int bm) { return bm <= 32 ? 128 : 64; }

template <typename T, int BM>
__global__ void __launch_bounds__(256) incr_kernel(IncrArgs<T> a) {
  using S = IncrShape<BM>;
  constexpr int BN = S::BN, TR = S::TR, TC = S::TC;
  constexpr int THC = BN / TC;
  static_assert((BM / TR) * THC == 256, "thread tile");
  __shared__ __align__(16) T Ds[kIncRC][BM];
  __shared__ __align__(16) T Zs[kIncRC][BN];
  const int ty = threadIdx.x / THC, tx = threadIdx.x % THC;
  const int j0 = blockIdx.x * BN;
  const int64_t rb0 = (int64_t)blockIdx.y * a.rows_per_split;
  const int64_t re = rb0 + a.rows_per_split < a.m ? rb0 + a.rows_per_split : a.m;
  const int kp = a.kp;
  const int nA = a.n - a.k0;
  float acc32[TR][TC];
  double acc64[TR][TC];
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) { acc32[i][j] = 0.f; acc64[i][j] = 0.0; }
  int stage = 0;
  for (int64_t rb = rb0; rb < re; rb += kIncRC) {
    // Delta rows (BM wide; columns >= kp are zero)
    for (int idx = threadIdx.x; idx < kIncRC * BM; idx += 256) {
      const int rr = idx / BM, l = idx % BM;
      const int64_t row = rb + rr;
      T d = T(0);
      if (row < re && l < kp) d = a.Xnew[row * kp + l] - a.Xold[row * kp + l];
      Ds[rr][l] = d;
    }
    // Z = [A(:, k0:n) | X1_p | Delta] columns j0 .. j0+BN
    for (int idx = threadIdx.x; idx < kIncRC * (BN / 4); idx += 256) {
      const int rr = idx / (BN / 4), c4 = (idx % (BN / 4)) * 4;
      const int64_t row = rb + rr;
      const int zc = j0 + c4;
      T v[4] = {T(0), T(0), T(0), T(0)};
      if (row < re) {
        if (a.vec_ok && zc + 4 <= nA) {
          load_vec4_or_scalar<T>(a.A + row * a.lda + a.k0 + zc, true, v, 4);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = zc + q;
            if (c < nA) v[q] = a.A[row * a.lda + a.k0 + c];
            else if (c < nA + kp) v[q] = a.Xold[row * kp + (c - nA)];
            else if (c < nA + 2 * kp) v[q] = a.Xnew[row * kp + (c - nA - kp)] - a.Xold[row * kp + (c - nA - kp)];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) Zs[rr][c4 + q] = v[q];
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < kIncRC; ++rr) {
      T dv[TR], zv[TC];
#pragma unroll
      for (int i = 0; i < TR; ++i) dv[i] = Ds[rr][ty * TR + i];
#pragma unroll
      for (int j = 0; j < TC; ++j) zv[j] = Zs[rr][tx * TC + j];
      if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc64[i][j] = fma((double)dv[i], (double)zv[j], acc64[i][j]);
      } else {
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc32[i][j] = fmaf((float)dv[i], (float)zv[j], acc32[i][j]);
      }
    }
    __syncthreads();
    if (++stage == kIncSuper) {
      stage = 0;
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) { acc64[i][j] += (double)acc32[i][j]; acc32[i][j] = 0.f; }
    }
  }
  double* out = a.part + (int64_t)blockIdx.y * a.k * a.nz;
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    const int l = ty * TR + i;
    if (l >= a.k) continue;
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      const int zc = j0 + tx * TC + j;
      if (zc < a.nz) out[(int64_t)l * a.nz + zc] = acc64[i][j] + (double)acc32[i][j];
    }
  }
}

template <typename T>
cudaError_t launch_incr(const IncrArgs<T>& a, int bm, cudaStream_t st) {
  const int bn = incr_bn(bm);
  dim3 grid((unsigned)ceil_div(a.nz, bn), (unsigned)a.nsplit);
  switch (bm) {
    case 16: incr_kernel<T, 16><<<grid, 256, 0, st>>>(a); break;
    case 32: incr_kernel<T, 32><<<grid, 256, 0, st>>>(a); break;
    case 64: incr_kernel<T, 64><<<grid, 256, 0, st>>>(a); break;
    case 128: incr_kernel<T, 128><<<grid, 256, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template cudaError_t launch_incr<float>(const IncrArgs<float>&, int, cudaStream_t);
template cudaError_t launch_incr<double>(const IncrArgs<double>&, int, cudaStream_t);

// ------------------------------------------------------------------------------ K2c
// inc = [N (k x nk) | Gamma (k x k) | Omega (k x k) | f_w]
__global__ void reduce_incr_kernel(const double* __restrict__ part, int nsplit, int k, int nk,
                                   int nz, int kshift, int nA, int kp,
                                   const double* __restrict__ fw_part, int nfw,
                                   double* __restrict__ inc) {
  const int64_t nN = (int64_t)k * nk, nG = (int64_t)k * k;
  const int64_t tot = nN + 2 * nG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    int l, zc;
    if (i < nN) { l = (int)(i / nk); zc = (int)(i % nk) + kshift; }
    else if (i < nN + nG) { const int64_t q = i - nN; l = (int)(q / k); zc = nA + (int)(q % k); }
    else { const int64_t q = i - nN - nG; l = (int)(q / k); zc = nA + kp + (int)(q % k); }
    double s = 0.0;
    for (int p = 0; p < nsplit; ++p) s += part[((int64_t)p * k + l) * nz + zc];
    inc[i] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int p = 0; p < nfw; ++p) s += fw_part[p];
    inc[tot] = s;
  }
}

void launch_reduce_incr(const double* part, int nsplit, int k, int nk, int nz, int kshift, int nA,
                        int kp, const double* fw_part, int nfw, double* inc, cudaStream_t st) {
  const int64_t tot = (int64_t)k * nk + 2LL * k * k;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tot, 256), 1184));
  reduce_incr_kernel<<<blocks, 256, 0, st>>>(part, nsplit, k, nk, nz, kshift, nA, kp, fw_part, nfw, inc);
}

}  // namespace wlr
