// rowpass.cu -- the m-scaled part of one sWLR iteration.
//
// K2a  row_pass_kernel : for every pixel row i (Algorithm 1 lines 7-9)
//        y   = A2(i,:) [V_p | C_p^T]                      (tall-skinny GEMM, CUDA-core FP32)
//        b   = y_V - X1_p(i,:) (C_p V_p)                   (= B_p(i,:), D_p = B_p V_p^T)
//        e   = A1(i,:) . W1(i,:)^2 + y_C - b (C_p V_p)^T   (= E_p(i,:) = [A1.W1.W1 + (A2-D_p)C_p^T](i,:))
//        x'  = e (diag(W1(i,:)^2) + C_p C_p^T)^{-1}        (uniform W1: one shared inverse;
//                                                           otherwise warp-per-row Cholesky)
//      writes X1_{p+1}(i,:), Delta(i,:) = X1_{p+1}(i,:) - X1_p(i,:) (from the stored values) and
//      an fp64 partial of f_w = sum W1^2 (A1 - X1_{p+1})^2.
//      MODE_RESULT writes b (row of B) instead of solving (wlr_result).
// K2b  incr_kernel : Gram increments  N = Delta^T A2,  Gamma = Delta^T X1_p,  Omega = Delta^T Delta.
//        fp32 inside <= 256-row chunks, fp64 across them and across CTAs.
// K2c  reduce_incr_kernel : fixed-order fp64 sum of the K2b/K2a partials into the packed
//        increment vector [N | Gamma | Omega | f_w] that is all-reduced across ranks.
//
// Mainloops: operands stream global -> shared with cp.async (LDGSTS) into
// double-buffered stages, so no registers hold in-flight tiles; each thread owns an
// 8 x TC register tile fed by 128-bit shared loads (row pass: A rows read 4 k at a time, rows
// interleaved by 8 so a warp's A loads hit distinct banks).  The row pass splits the
// reduction over KG = 4 thread groups (in-CTA split-K, fixed-order sum).  Its epilogue runs
// from shared memory (X1_p and A1 of the tile are staged with the first chunk), as
// thread-per-output small products.  A is streamed once from HBM by the row pass; the
// increment pass re-reads it from L2 (46 MB at the metric's config fits the 126 MB L2).
#include "kernels.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace wlr {

// ------------------------------------------------------------------------- cp.async
WLR_DEVI void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
WLR_DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
WLR_DEVI void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

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

// N consecutive T from shared memory with 128-bit loads where possible
template <typename T, int N>
WLR_DEVI void lds_vec(const T* p, T (&o)[N]) {
  if constexpr (sizeof(T) == 4 && N % 4 == 0) {
#pragma unroll
    for (int q = 0; q < N; q += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + q);
      o[q] = v.x; o[q + 1] = v.y; o[q + 2] = v.z; o[q + 3] = v.w;
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      if constexpr (sizeof(T) == 4) {
        const float2 v = *reinterpret_cast<const float2*>(p + q);
        o[q] = v.x; o[q + 1] = v.y;
      } else {
        const double2 v = *reinterpret_cast<const double2*>(p + q);
        o[q] = v.x; o[q + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) o[q] = p[q];
  }
}

// ------------------------------------------------------------------------------ K2a
template <int RP> struct RowPassShape;   // TC columns per thread, RS row groups (BM = RS * TR)
template <> struct RowPassShape<16>  { static constexpr int TC = 2, RS = 8; };
template <> struct RowPassShape<32>  { static constexpr int TC = 4, RS = 8; };
template <> struct RowPassShape<64>  { static constexpr int TC = 8, RS = 8; };
template <> struct RowPassShape<128> { static constexpr int TC = 8, RS = 4; };

constexpr int kRowKC = 32;        // reduction chunk (columns of [A | X1_p])
constexpr int kRowKG = 4;         // k-groups (in-CTA split-K); each takes 8 k of a chunk
// TR (rows per thread, interleaved by RS) is a template parameter: the host picks the tile
// height BM = RS * TR that balances the tiles over the SMs (row_pass_pick_tr)
constexpr int kRowThreads = 256;

// Per-warp scratch for the non-uniform epilogue: the packed lower triangle of the row matrix.
__host__ __device__ inline int chol_packed(int kp) { return kp * (kp + 1) / 2; }

template <typename T, int RP, int TR>
struct RowPassLayout {            // shared memory layout (elements of T; base 1024-byte aligned)
  using S = RowPassShape<RP>;
  static constexpr int BM = S::RS * TR;
  static constexpr int PE = 128 / (int)sizeof(T);               // elements per 128-byte panel row
  static constexpr int NP = kRowKC / PE;                        // panels per A chunk (1 fp32, 2 fp64)
  static constexpr int kA = NP * BM * PE;                       // one A stage (SWIZZLE_128B panels)
  static constexpr int kB = kRowKC * RP;                        // one Wt stage
  static constexpr int YLD = RP + 1;
  static constexpr int NST = 4;                                 // TMA pipeline stages
  static constexpr int oA = 0, oB = NST * kA, oStEnd = oB + NST * kB;
  // epilogue buffers alias the stages (free once the mainloop is done): Ys [BM][RP+1] at 0,
  // then the e tile [BM][kp] (non-uniform)
  static constexpr int oY = 0, oE = BM * YLD;
  static constexpr int ALIGN = 1024 / (int)sizeof(T);           // SWIZZLE_128B destinations
};

__host__ __device__ inline int64_t align_up_i(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// offsets (elements) of the X1_p / A1 staging panels and of the tail buffers
template <typename T, int RP, int TR>
struct RowPassTail {
  int64_t oXs, oA1s, oK, oL, end;
  __host__ __device__ RowPassTail(bool uniform, int k, int kp, int nwc) {
    using L = RowPassLayout<T, RP, TR>;
    const int npk = (kp + L::PE - 1) / L::PE;
    const int64_t alias = (int64_t)L::oE + (uniform ? 0 : (int64_t)L::BM * kp);
    oXs = align_up_i(alias > L::oStEnd ? alias : L::oStEnd, L::ALIGN);
    oA1s = oXs + (int64_t)npk * L::BM * L::PE;
    oK = oA1s + (int64_t)npk * L::BM * L::PE;
    oL = oK + (uniform ? 0 : (int64_t)k * k);
    end = oL + (uniform ? 0 : (int64_t)nwc * chol_packed(kp));
  }
};

template <typename T, int RP, int TR>
size_t row_pass_smem_elems(bool uniform, int k, int kp, int nwc) {
  return (size_t)RowPassTail<T, RP, TR>(uniform, k, kp, nwc).end + RowPassLayout<T, RP, TR>::ALIGN;
}

// warps that can hold a packed k x k factor in the remaining shared memory (<= 8)
template <typename T, int RP, int TR>
int row_pass_nwc(bool uniform, int k, int kp) {
  if (uniform) return 8;
  const size_t base = row_pass_smem_elems<T, RP, TR>(false, k, kp, 0);
  const size_t cap = 227 * 1024 / sizeof(T);
  if (base >= cap) return 0;
  return (int)std::min<size_t>(8, (cap - base) / chol_packed(kp));
}

template <typename T, int RP, int TR, bool UNIFORM, int MODE>
__global__ void __launch_bounds__(kRowThreads, RP <= 32 ? 3 : 1)
row_pass_kernel(const __grid_constant__ RowPassArgs<T> a) {
  if (a.stop && *a.stop) return;               // (eps mode: converged before this iteration)
  pdl_trigger();                               // the increments may be scheduled (they wait)
  using S = RowPassShape<RP>;
  using L = RowPassLayout<T, RP, TR>;
  constexpr int BM = L::BM, TC = S::TC, KG = kRowKG, PE = L::PE, NST = L::NST;
  constexpr int THC = RP / TC;                 // threads along columns (per k-group)
  constexpr int GT = (BM / TR) * THC;          // threads per k-group
  static_assert(GT * KG == kRowThreads, "thread tile");
  constexpr int KPG = kRowKC / KG;             // k per group per chunk (8)
  constexpr int VE = 16 / (int)sizeof(T);      // elements per 16-byte chunk
  constexpr int RS = BM / TR;                  // row interleave stride

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full[NST];    // stage filled (TMA bytes landed)
  __shared__ __align__(8) uint64_t empty[NST];   // stage drained (one arrival per warp)
  __shared__ __align__(8) uint64_t epb;
  const int kp = a.kp, k = a.k;
  const RowPassTail<T, RP, TR> tl(UNIFORM || MODE == 1, k, kp, a.nwc);
  T* As = sm + L::oA;                          // [NST][NP][BM][PE]  (swizzled panels)
  T* Bs = sm + L::oB;                          // [NST][KC][RP]
  T* Ys = sm + L::oY;                          // [BM][RP+1]   (aliases the stages)
  T* Es = sm + L::oE;                          // [BM][kp]     (aliases; non-uniform)
  T* Xs = sm + tl.oXs;                         // [npk][BM][PE] X1_p rows (swizzled)
  T* A1s = sm + tl.oA1s;                       // [npk][BM][PE] A1 columns (swizzled)
  T* sK = sm + tl.oK;                          // [k][k]    C C^T (non-uniform)
  T* sL = sm + tl.oL;                          // per-warp packed L (non-uniform)
  const int npk = (kp + PE - 1) / PE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto pan = [&](const T* base, int r, int c) -> T {   // staged X1_p / A1 element (r, c)
    return base[(c / PE) * (BM * PE) + swz128<T>(r, c % PE)];
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRowThreads / 32);
    }
    mbar_init(&epb, 1);
    mbar_init_fence();
  }
  if (!UNIFORM && MODE == 0)
    for (int i = threadIdx.x; i < k * k; i += kRowThreads) sK[i] = a.Kmat[i];
  // The small step that follows is latency-bound and reads G_A and its previous state:
  // pull them into L2 while this pass streams A (bulk L2 prefetch, 64 KB per request).
  if (MODE == 0 && threadIdx.x < 32) {
    for (int r = 0; r < kPf; ++r) {
      const char* base = reinterpret_cast<const char*>(a.pf_ptr[r]);
      const int64_t nb = a.pf_bytes[r] & ~(int64_t)15;
      if (!base || nb <= 0) continue;
      const int64_t chunk = 65536;
      const int64_t nchunk = ceil_div(nb, chunk);
      for (int64_t c = blockIdx.x * 32 + threadIdx.x; c < nchunk; c += (int64_t)gridDim.x * 32) {
        const int64_t off = c * chunk;
        const unsigned sz = (unsigned)(nb - off < chunk ? nb - off : chunk);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base + off), "r"(sz) : "memory");
      }
    }
  }
  __syncthreads();

  const int kg = threadIdx.x / GT, gt = threadIdx.x - kg * GT;
  const int ty = gt / THC, tx = gt - ty * THC;
  const int nchA = a.KA / kRowKC;              // chunks over the columns of A
  const int nch = nchA + (kp + kRowKC - 1) / kRowKC;   // + chunks over X1_p
  double fw = 0.0;
  const int64_t ntiles = ceil_div(a.m, BM);
  constexpr uint32_t kStageBytes = (uint32_t)((L::kA + L::kB) * sizeof(T));

  // thread 0: TMA loads of chunk c of the tile at row r0 into stage st
  auto load_chunk = [&](int64_t r0, int c, int st) {
    const bool isA = c < nchA;
    const int cb = (isA ? c : c - nchA) * kRowKC;
    mbar_expect_tx(&full[st], kStageBytes);
#pragma unroll
    for (int p = 0; p < L::NP; ++p)
      tma_load_2d(As + st * L::kA + p * BM * PE, isA ? &a.tmA : &a.tmX, &full[st], cb + p * PE, (int)r0);
    tma_load_2d(Bs + st * L::kB, &a.tmW, &full[st], 0, isA ? cb : a.KA + cb);
  };

  int64_t G = 0;                               // chunks consumed so far (stage / parity)
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t r0 = tile * BM;
    __syncthreads();                           // previous tile's epilogue done with the smem
    if (threadIdx.x == 0) {
      fence_proxy_async();
      if (MODE == 0) {   // epilogue operands of this tile: X1_p rows and A1 columns
        mbar_expect_tx(&epb, (uint32_t)(2 * npk * BM * PE * sizeof(T)));
        for (int pp = 0; pp < npk; ++pp) {
          tma_load_2d(Xs + pp * BM * PE, &a.tmX, &epb, pp * PE, (int)r0);
          tma_load_2d(A1s + pp * BM * PE, &a.tmA, &epb, pp * PE, (int)r0);
        }
      }
      for (int q = 0; q < NST - 1 && q < nch; ++q) load_chunk(r0, q, (int)((G + q) % NST));
    }

    T acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = T(0);

    for (int ch = 0; ch < nch; ++ch) {
      const int64_t g = G + ch;
      const int st = (int)(g % NST);
      if (threadIdx.x == 0 && ch + NST - 1 < nch) {   // refill the stage chunk g-1 used
        if (ch > 0) mbar_wait(&empty[(g - 1) % NST], (uint32_t)(((g - 1) / NST) & 1));
        fence_proxy_async();
        load_chunk(r0, ch + NST - 1, (int)((g + NST - 1) % NST));
      }
      mbar_wait(&full[st], (uint32_t)((g / NST) & 1));
      const T* as = As + st * L::kA;
      const T* bs = Bs + st * L::kB;
#pragma unroll
      for (int k4 = 0; k4 < KPG; k4 += VE) {
        const int kk0 = kg * KPG + k4;
        const T* ap = as + (kk0 / PE) * (BM * PE);
        T av[TR][VE];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
          T tmp[VE];
          lds_vec<T, VE>(ap + swz128<T>(ty + i * RS, kk0 % PE), tmp);
#pragma unroll
          for (int q = 0; q < VE; ++q) av[i][q] = tmp[q];
        }
#pragma unroll
        for (int q = 0; q < VE; ++q) {
          T bv[TC];
          lds_vec<T, TC>(bs + (kk0 + q) * RP + tx * TC, bv);
#pragma unroll
          for (int i = 0; i < TR; ++i)
#pragma unroll
            for (int j = 0; j < TC; ++j) acc[i][j] = fma(av[i][q], bv[j], acc[i][j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with stage st
    }
    G += nch;
    __syncthreads();                           // every warp is out of the stages (Ys aliases them)
    // fixed-order sum of the KG partial tiles into Ys
#pragma unroll 1
    for (int gg = 0; gg < KG; ++gg) {
      if (kg == gg) {
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) {
            T* y = Ys + (ty + i * RS) * L::YLD + tx * TC + j;
            *y = gg == 0 ? acc[i][j] : *y + acc[i][j];
          }
      }
      __syncthreads();
    }
    const int nrow = (int)((a.m - r0) < BM ? (a.m - r0) : BM);

    // ---------------- epilogue (shared memory; thread per output)
    if (MODE == 1) {                           // wlr_result: B rows
      for (int o = threadIdx.x; o < nrow * a.no; o += kRowThreads) {
        const int r = o / a.no, j = o - r * a.no;
        a.Bout[(r0 + r) * a.ldb + j] = Ys[r * L::YLD + j];
      }
      continue;
    }
    mbar_wait(&epb, (uint32_t)(it & 1));
    if (UNIFORM) {                             // out = X1_{p+1} rows; Delta; f_w
      for (int o = threadIdx.x; o < nrow * kp; o += kRowThreads) {
        const int r = o / kp, l = o - r * kp;
        const T x = l < k ? Ys[r * L::YLD + l] : T(0);
        const int64_t gi = (r0 + r) * kp + l;
        a.Xnew[gi] = x;
        a.Dnew[gi] = x - pan(Xs, r, l);
        if (l < k) {
          const double d = (double)pan(A1s, r, l) - (double)x;
          fw += (double)a.w2s * d * d;
        }
      }
    } else {
      // e = out + A1 . W1^2, then x' = e (diag(W1^2) + C C^T)^{-1}: warp per row, packed
      // lower triangle P(i,j) = i(i+1)/2 + j
      for (int o = threadIdx.x; o < nrow * kp; o += kRowThreads) {
        const int r = o / kp, l = o - r * kp;
        T e = T(0);
        if (l < k) {
          const T w = a.W1[(r0 + r) * a.ldw + l];
          e = fma(pan(A1s, r, l), w * w, Ys[r * L::YLD + l]);
        }
        Es[r * kp + l] = e;
        if (a.Ebuf) a.Ebuf[(r0 + r) * kp + l] = e;    // the warp-per-row solver takes over
      }
      __syncthreads();
      if (a.Ebuf) continue;
      T* wL = sL + warp * chol_packed(kp);
      for (int rl = warp; rl < (warp < a.nwc ? nrow : 0); rl += a.nwc) {
        const int64_t g = r0 + rl;
        T* we = Es + rl * kp;
        for (int idx = lane; idx < chol_packed(k); idx += 32) {
          int i = (int)((sqrtf(8.f * idx + 1.f) - 1.f) * 0.5f);
          while ((i + 1) * (i + 2) / 2 <= idx) ++i;
          while (i * (i + 1) / 2 > idx) --i;
          const int j = idx - i * (i + 1) / 2;
          T v = sK[i * k + j];
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
            int l = j + 1;
            for (; l + 3 <= i; l += 4) {           // 4 independent element updates in flight
              const T c0 = wL[l * (l + 1) / 2 + j], c1 = wL[(l + 1) * (l + 2) / 2 + j];
              const T c2 = wL[(l + 2) * (l + 3) / 2 + j], c3 = wL[(l + 3) * (l + 4) / 2 + j];
              const T r0 = rowi[l], r1 = rowi[l + 1], r2 = rowi[l + 2], r3 = rowi[l + 3];
              rowi[l] = fma(-lij, c0, r0);
              rowi[l + 1] = fma(-lij, c1, r1);
              rowi[l + 2] = fma(-lij, c2, r2);
              rowi[l + 3] = fma(-lij, c3, r3);
            }
            for (; l <= i; ++l) rowi[l] = fma(-lij, wL[l * (l + 1) / 2 + j], rowi[l]);
          }
          __syncwarp();
        }
        if (!spd && lane == 0) raise_flag(a.flags, DF_ROWSPD);
        for (int j = 0; j < k; ++j) {          // forward: L z = e
          const T zj = we[j] / wL[j * (j + 1) / 2 + j];
          for (int i = j + 1 + lane; i < k; i += 32) we[i] = fma(-wL[i * (i + 1) / 2 + j], zj, we[i]);
          __syncwarp();
          if (lane == 0) we[j] = zj;
          __syncwarp();
        }
        for (int j = k - 1; j >= 0; --j) {     // backward: L^T x = z
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
          a.Dnew[g * kp + l] = x - pan(Xs, rl, l);
          if (l < k) {
            const double w = (double)a.W1[g * a.ldw + l];
            const double d = (double)pan(A1s, rl, l) - (double)x;
            fw += w * w * d * d;
          }
        }
        __syncwarp();
      }
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

template <typename T, int RP, int TR, bool UNIFORM, int MODE>
static cudaError_t launch_rp(const RowPassArgs<T>& a, int grid, cudaStream_t st, int* occ, bool pdl) {
  auto kern = row_pass_kernel<T, RP, TR, UNIFORM, MODE>;
  const size_t smem = sizeof(T) * row_pass_smem_elems<T, RP, TR>(UNIFORM || MODE == 1, a.k, a.kp, a.nwc);
  static size_t configured = 0;            // cudaFuncSetAttribute once per size increase
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // all of the unified L1/shared storage as shared memory, so 3 CTAs/SM fit
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, kRowThreads, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRowThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

int row_pass_rp(int r) { return r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : r <= 128 ? 128 : -1; }
bool row_pass_tr_ok(int rp, int tr) { return rp == 128 ? tr == 8 : (tr == 4 || tr == 6 || tr == 8); }
int row_pass_bm(int rp, int tr) { return (rp == 128 ? RowPassShape<128>::RS : RowPassShape<32>::RS) * tr; }

#define WLR_RP_SWITCH(RPV, TRV, CALL)                                                    \
  switch (RPV) {                                                                         \
    case 16: switch (TRV) { case 4: CALL(16, 4); case 6: CALL(16, 6); default: CALL(16, 8); } \
    case 32: switch (TRV) { case 4: CALL(32, 4); case 6: CALL(32, 6); default: CALL(32, 8); } \
    case 64: switch (TRV) { case 4: CALL(64, 4); case 6: CALL(64, 6); default: CALL(64, 8); } \
    default: CALL(128, 8);                                                               \
  }

template <typename T>
size_t row_pass_smem(int rp, int tr, bool uniform, int k, int kp) {
#define WLR_SMEM(R, TT) \
  return sizeof(T) * row_pass_smem_elems<T, R, TT>(uniform, k, kp, row_pass_nwc<T, R, TT>(uniform, k, kp))
  WLR_RP_SWITCH(rp, tr, WLR_SMEM)
#undef WLR_SMEM
}
template size_t row_pass_smem<float>(int, int, bool, int, int);
template size_t row_pass_smem<double>(int, int, bool, int, int);
template <typename T>
int row_pass_chol_warps(int rp, int tr, bool uniform, int k, int kp) {
#define WLR_NWC(R, TT) return row_pass_nwc<T, R, TT>(uniform, k, kp)
  WLR_RP_SWITCH(rp, tr, WLR_NWC)
#undef WLR_NWC
}
template int row_pass_chol_warps<float>(int, int, bool, int, int);
template int row_pass_chol_warps<double>(int, int, bool, int, int);

// The result pass (mode 1) exists for TR = 8 only.
template <typename T>
cudaError_t launch_row_pass(const RowPassArgs<T>& a, int rp, int tr, bool uniform, int mode, int grid,
                            cudaStream_t st, int* occ, bool pdl) {
  if (rp != 16 && rp != 32 && rp != 64 && rp != 128) return cudaErrorInvalidValue;
  if (!row_pass_tr_ok(rp, tr) || (mode && tr != 8)) return cudaErrorInvalidValue;
  if (mode) {
#define WLR_RES(R, TT) return launch_rp<T, R, 8, true, 1>(a, grid, st, occ, pdl)
    WLR_RP_SWITCH(rp, 8, WLR_RES)
#undef WLR_RES
  }
#define WLR_RUN(R, TT) \
  return uniform ? launch_rp<T, R, TT, true, 0>(a, grid, st, occ, pdl) : launch_rp<T, R, TT, false, 0>(a, grid, st, occ, pdl)
  WLR_RP_SWITCH(rp, tr, WLR_RUN)
#undef WLR_RUN
}
template cudaError_t launch_row_pass<float>(const RowPassArgs<float>&, int, int, bool, int, int, cudaStream_t, int*, bool);
template cudaError_t launch_row_pass<double>(const RowPassArgs<double>&, int, int, bool, int, int, cudaStream_t, int*, bool);

// ------------------------------------------------------------------------------ K2b
// Thread tile 8 (q) x TW (columns); warp w owns q in [8w, 8w+8) and lane l the columns
// [l TW, l TW + TW) of the CTA's BN-wide block (BN = 32 TW), so the Delta operand is a warp
// broadcast and the Z operand TW/4 LDS.128 per lane.  Z = [A(:, k0:n) | X1_p | Delta] arrives by
// cp.async (4-stage ring of 16-row stages); every thread copies ONE fixed 16-byte column of Z
// (its source pointer and row stride are set once).  fp32 inside 256-row chunks, then fp64.
// BN = 128 (8 x 4 tiles).  A BN = 256 variant (8 x 8 tiles, 64 FFMA per 4 LDS.128) needed 168
// registers and ran 1.7x slower at config 3 (3 CTAs/SM, a second wave).
constexpr int kIncRC = 16;          // rows per stage
constexpr int kIncNST = 4;          // cp.async pipeline stages
constexpr int kIncFlush = 16;       // stages per fp32 chunk (256 rows), then fp64

int incr_bm(int kp) { return kp <= 32 ? 32 : kp <= 64 ? 64 : kp <= 128 ? 128 : -1; }
int incr_bn(int, int) { return 128; }   // (BN = 256 with 8 x 8 tiles measured slower: 168 regs)

template <typename T, int BM, int BN>
size_t incr_smem_bytes() {   // stages; after the mainloop the fp64 BM x BN tile of the cluster sum
  return std::max(sizeof(T) * kIncNST * (size_t)kIncRC * (BM + BN), sizeof(double) * BM * BN);
}

template <typename T, int BM, int BN>
__global__ void __launch_bounds__(BM * 4, BM == 32 ? 5 : 1) incr_kernel(IncrArgs<T> a) {
  pdl_wait();                                   // Delta / X1_{p+1} of the row pass
  pdl_trigger();
  if (a.gate && *a.gate) return;                // the tensor-core kernel computes this iteration
  constexpr int NT = BM * 4;                    // threads: BM/8 warps
  constexpr int TW = BN / 32;                   // columns per lane
  constexpr int VE = 16 / (int)sizeof(T);
  constexpr int CPR = BN / VE;                  // 16-byte copies per Z row
  static_assert(NT % CPR == 0 || CPR % NT == 0, "copy mapping");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ds = reinterpret_cast<T*>(smem_raw);       // [NST][RC][BM]
  T* Zs = Ds + kIncNST * kIncRC * BM;           // [NST][RC][BN]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = warp * 8, c0 = lane * TW;
  const int j0 = blockIdx.x * BN;
  const int64_t rb0 = (int64_t)blockIdx.y * a.rows_per_split;
  const int64_t re = rb0 + a.rows_per_split < a.m ? rb0 + a.rows_per_split : (rb0 < a.m ? a.m : rb0);
  const int kp = a.kp;
  const int nA = a.n - a.k0;
  const bool vec = a.vec_ok;

  // Z copy slot of this thread: column cv (fixed), rows rr0, rr0 + RS, ...
  constexpr int RS = NT >= CPR ? NT / CPR : 1;  // rows per pass of all threads
  const int cv = (threadIdx.x % CPR) * VE, rr0 = threadIdx.x / CPR;
  const int zc = j0 + cv;
  const T* zsrc = nullptr;
  int64_t zld = 0;
  if (zc < nA) { zsrc = a.A + a.k0 + zc; zld = a.lda; }
  else if (zc < nA + kp) { zsrc = a.Xold + (zc - nA); zld = kp; }
  else if (zc < nA + 2 * kp) { zsrc = a.Dnew + (zc - nA - kp); zld = kp; }
  auto issue = [&](int64_t rb, int st) {
    T* ds = Ds + st * kIncRC * BM;
    for (int idx = threadIdx.x; idx < kIncRC * (BM / VE); idx += NT) {
      const int rr = idx / (BM / VE), lv = (idx % (BM / VE)) * VE;
      const int64_t row = rb + rr;
      const bool in = row < re && lv < kp;
      cp_async16(ds + rr * BM + lv, in ? a.Dnew + row * kp + lv : a.Dnew, in ? 16 : 0);
    }
    T* zs = Zs + st * kIncRC * BN;
    if (vec) {
#pragma unroll
      for (int rr = rr0; rr < kIncRC; rr += RS) {
        const int64_t row = rb + rr;
        const bool in = zsrc != nullptr && row < re;
        cp_async16(zs + rr * BN + cv, in ? zsrc + row * zld : a.A, in ? 16 : 0);
      }
    } else {
      for (int idx = threadIdx.x; idx < kIncRC * CPR; idx += NT) {
        const int rr = idx / CPR, cc = (idx % CPR) * VE;
        const int64_t row = rb + rr;
        const int zcc = j0 + cc;
        T* dst = zs + rr * BN + cc;
#pragma unroll
        for (int q = 0; q < VE; ++q) {
          const int c = zcc + q;
          T v = T(0);
          if (row < re) {
            if (c < nA) v = a.A[row * a.lda + a.k0 + c];
            else if (c < nA + kp) v = a.Xold[row * kp + (c - nA)];
            else if (c < nA + 2 * kp) v = a.Dnew[row * kp + (c - nA - kp)];
          }
          dst[q] = v;
        }
      }
    }
  };

  T acc[8][TW];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TW; ++j) acc[i][j] = T(0);
  double* out = a.part + (int64_t)blockIdx.y * a.k * a.nz;
  bool first = true;
  // fp32 chunk sums are added into this CTA's fp64 partial (fixed order)
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = q0 + i;
#pragma unroll
      for (int j = 0; j < TW; ++j) {
        const int zcol = j0 + c0 + j;
        if (l < a.k && zcol < a.nz) {
          double* o = out + (int64_t)l * a.nz + zcol;
          *o = first ? (double)acc[i][j] : *o + (double)acc[i][j];
        }
        acc[i][j] = T(0);
      }
    }
    first = false;
  };
  const int nst = (int)ceil_div(re - rb0, (int64_t)kIncRC);   // 0 for padding CTAs of a cluster
#pragma unroll
  for (int q = 0; q < kIncNST - 1; ++q) {
    if (q < nst) issue(rb0 + (int64_t)q * kIncRC, q);
    cp_async_commit();
  }
  int stage = 0;
  for (int s = 0; s < nst; ++s) {
    const int st = s % kIncNST;
    if (s + kIncNST - 1 < nst) issue(rb0 + (int64_t)(s + kIncNST - 1) * kIncRC, (s + kIncNST - 1) % kIncNST);
    cp_async_commit();
    cp_async_wait<kIncNST - 1>();
    __syncthreads();
    const T* ds = Ds + st * kIncRC * BM;
    const T* zs = Zs + st * kIncRC * BN;
#pragma unroll 4
    for (int rr = 0; rr < kIncRC; ++rr) {
      T dv[8], zv[TW];
      lds_vec<T, 8>(ds + rr * BM + q0, dv);
      lds_vec<T, TW>(zs + rr * BN + c0, zv);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TW; ++j) acc[i][j] = fma(dv[i], zv[j], acc[i][j]);
    }
    if (sizeof(T) == 4 && ++stage == kIncFlush && s + 1 < nst) {
      stage = 0;
      flush();
    }
    __syncthreads();
  }
  if (a.cs <= 1) {
    flush();
    return;
  }
  // cluster pre-reduction: the cs row splits of this cluster sum their fp64 tiles through DSMEM
  // in rank order; rank r writes rows [r BM / cs, (r+1) BM / cs) of the cluster's partial
  double* tile = reinterpret_cast<double*>(smem_raw);         // BM x BN (the stages are free)
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TW; ++j) {
      const int l = q0 + i, zcol = j0 + c0 + j;
      double v = (double)acc[i][j];
      if (!first && l < a.k && zcol < a.nz) v += out[(int64_t)l * a.nz + zcol];
      tile[l * BN + c0 + j] = v;
    }
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const int rk = (int)cl.block_rank(), rows = BM / a.cs;
  double* o2 = a.part2 + (int64_t)(blockIdx.y / a.cs) * a.k * a.nz;
  for (int idx = threadIdx.x; idx < rows * BN; idx += NT) {
    const int q = rk * rows + idx / BN, c = idx % BN;
    double v = 0.0;
    for (int r = 0; r < a.cs; ++r) v += cl.map_shared_rank(tile, r)[q * BN + c];
    if (q < a.k && j0 + c < a.nz) o2[(int64_t)q * a.nz + j0 + c] = v;
  }
  cl.sync();                                                  // peers' tiles stay alive until read
}

template <typename T, int BM, int BN>
static cudaError_t launch_incr_bm(const IncrArgs<T>& a, cudaStream_t st) {
  auto kern = incr_kernel<T, BM, BN>;
  const size_t smem = incr_smem_bytes<T, BM, BN>();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int cs = a.cs > 1 ? a.cs : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ceil_div(a.nz, BN), (unsigned)(ceil_div(a.nsplit, cs) * cs));
  cfg.blockDim = dim3(BM * 4);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = cs; at[0].val.clusterDim.z = 1;
  cudaLaunchAttribute atp[2] = {at[0], {}};
  int na = cs > 1 ? 1 : 0;
  if (a.pdl) {
    atp[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    atp[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = atp;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename T>
cudaError_t launch_incr(const IncrArgs<T>& a, int bm, cudaStream_t st) {
  switch (bm) {
    case 32:
      return launch_incr_bm<T, 32, 128>(a, st);
    case 64: return launch_incr_bm<T, 64, 128>(a, st);
    case 128: return launch_incr_bm<T, 128, 128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}
template cudaError_t launch_incr<float>(const IncrArgs<float>&, int, cudaStream_t);
template cudaError_t launch_incr<double>(const IncrArgs<double>&, int, cudaStream_t);

// ------------------------------------------------------------------------------ K2c
// inc = [N (k x nk) | Gamma (k x k) | Omega (k x k) | f_w]; thread per output, the split
// partials summed in fixed order with 8 independent loads in flight.
__global__ void reduce_incr_kernel(const double* __restrict__ part, int nsplit, int k, int nk,
                                   int nz, int kshift, int nA, int kp,
                                   const double* __restrict__ fw_part, int nfw,
                                   double* __restrict__ inc, const int* gate, ReduceLayout alt, int gk) {
  pdl_wait();
  pdl_trigger();
  if (gate && *gate) {   // tensor-core partial layout this iteration
    part = alt.part; nsplit = alt.nsplit; nz = alt.nz; nA = alt.nA; kp = alt.kp;
  }
  // 8 lanes per output: lane g sums the splits p = g (mod 8) in order, then a fixed
  // shuffle tree combines the 8 sums (deterministic)
  // inc = [N (k x nk) | Gamma (k x gk) | Omega (k x k) | f_w]  (gk = k for the sWLR increments)
  const int64_t nN = (int64_t)k * nk, nG = (int64_t)k * gk, nO = (int64_t)k * k;
  const int64_t tot = nN + nG + nO;
  const int64_t stride = (int64_t)k * nz;
#ifndef WLR_RED_L
#define WLR_RED_L 4
#endif
  constexpr int RL = WLR_RED_L;          // lanes per output (4, 8 or 16; same-box A/B: 4 best)
  static_assert(RL == 4 || RL == 8 || RL == 16, "reduce: the shuffle tree assumes 4, 8 or 16 lanes per output");
  const int g = threadIdx.x & (RL - 1);
  const int64_t per_block = blockDim.x / RL;
  for (int64_t i0 = blockIdx.x * per_block; i0 < tot; i0 += (int64_t)gridDim.x * per_block) {
    const int64_t i = i0 + threadIdx.x / RL;
    double s = 0.0;
    if (i < tot) {
      int l, zc;
      if (i < nN) { l = (int)(i / nk); zc = (int)(i % nk) + kshift; }
      else if (i < nN + nG) { const int64_t q = i - nN; l = (int)(q / gk); zc = nA + (int)(q % gk); }
      else { const int64_t q = i - nN - nG; l = (int)(q / k); zc = nA + kp + (int)(q % k); }
      const double* src = part + (int64_t)l * nz + zc;
      // batches of 8 splits per lane (64 per output), every load of a batch in flight at once
      for (int p0 = 0; p0 < nsplit; p0 += 8 * RL) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int p = p0 + g + RL * j;
          v[j] = p < nsplit ? __ldg(src + (int64_t)p * stride) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[j];
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (RL >= 8) s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (RL >= 16) s += __shfl_xor_sync(0xffffffffu, s, 8);
    if (g == 0 && i < tot) inc[i] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double s = 0.0;
    for (int p = threadIdx.x; p < nfw; p += 32) s += fw_part[p];
    s = warp_sum(s);                      // fixed lane order -> deterministic
    if (threadIdx.x == 0) inc[tot] = s;
  }
}

void launch_reduce_incr(const double* part, int nsplit, int k, int nk, int nz, int kshift, int nA,
                        int kp, const double* fw_part, int nfw, double* inc, cudaStream_t st,
                        const int* gate, ReduceLayout alt, bool pdl, int gk) {
  if (gk < 0) gk = k;
  const int64_t tot = (int64_t)k * nk + (int64_t)k * gk + (int64_t)k * k;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tot, (int64_t)(256 / WLR_RED_L)), 4096));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, reduce_incr_kernel, part, nsplit, k, nk, nz, kshift, nA, kp, fw_part, nfw, inc,
                     gate, alt, gk);
}

}  // namespace wlr
