// rowpass_tc.cu -- K2a on the 5th-generation tensor cores (uniform W1, fp32 data).
//
// The uniform-weight row update is one dense contraction over every pixel row
// (Algorithm 1 lines 7-9, as the linear update of DESIGN.md §2):
//     X1_{p+1}(i,:) = [A(i,:) | X1_p(i,:)] W',   W' = [w^2 K^{-1}; U K^{-1}; P K^{-1}]
// so a tile of 64 rows is a 64 x RP x (KA + KX) GEMM.  It runs as tcgen05.mma kind::tf32 with the
// 3xTF32 split
//     z w ~ z_hi w_hi + z_hi w_lo + z_lo w_hi,   z_hi = tf32(z) (the tensor core truncates),
// W'^T and W'^T_lo are written K-major by the small step; Z_lo is made here.  Per 32-column chunk:
//   warp 4 (1 thread)  : TMA (SWIZZLE_128B) Z = [A | X1_p] chunk (64 x 32), W'^T, W'^T_lo
//   warps 0-3          : Z_lo = Z - tf32(Z) into the lo ring (generic proxy), fence.proxy.async
//   warp 5 (1 thread)  : 4 k-steps x 3 MMAs into the TMEM accumulator; tcgen05.commit frees
//                        the raw and lo stages (and signals the epilogue after the last chunk)
// Epilogue (warps 0-3): TMEM lanes 32w..32w+15 hold rows 16w..16w+15 of the M = 64 tile
// (measured, profiles/r01_ubench_umma_m64_layout.log); writes X1_{p+1}, Delta and an fp64
// partial of f_w.  A1 and X1_p of the row are captured from the stream (chunks 0 and KA/32).
#include "kernels.h"
#include "umma.cuh"

namespace wlr {

// Warp roles (192 threads): warps 0-3 convert (lo parts) and run the epilogue (TMEM lanes
// 32w..32w+15 hold rows 16w..16w+15 of an M = 64 tile), warp 4 lane 0 issues TMA, warp 5
// lane 0 issues the MMAs.  Rings: NR raw stages (TMA -> smem) and NL lo stages.
constexpr int kTcThreads = 192;
constexpr int kTcNR = 3, kTcNL = 3;

template <int RP>
struct TcLayout {                                  // bytes; every block 1024-aligned
  static constexpr int ZB = kTcBM * 128;          // Z chunk (fp32 BM x 32)
  static constexpr int WB = RP * 128;             // W'^T chunk (RP x 32)
  static constexpr int STAGE = ZB + 2 * WB;       // raw stage = Z | W'^T | W'^T_lo (all TMA)
  static constexpr int TOTAL = kTcNR * STAGE + kTcNL * ZB;   // + lo ring of Z_lo
  static constexpr int NCOL = RP < 32 ? 32 : RP;  // TMEM columns (power of 2 >= 32)
};

template <int RP>
__global__ void __launch_bounds__(kTcThreads, 3) row_pass_tc_kernel(const __grid_constant__ RowPassTcArgs a) {
  using L = TcLayout<RP>;
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* rawst = sm;                               // [NR][Z | W | W_lo]
  unsigned char* lost = sm + kTcNR * L::STAGE;             // [NL][Z_lo]
  __shared__ __align__(8) uint64_t full[kTcNR], rawfree[kTcNR], lofull[kTcNL], lofree[kTcNL], accfull, accfree;
  __shared__ uint32_t tslot;
  __shared__ double wsum[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto stamp = [&](int i) {
    if (a.tstamp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.tstamp[(int64_t)blockIdx.x * 8 + i] = t;
    }
  };
  if (tid == 0) stamp(0);
  if (warp == 0) tmem_alloc<L::NCOL>(&tslot);
  if (tid == 32) {
    for (int s = 0; s < kTcNR; ++s) { mbar_init(&full[s], 1); mbar_init(&rawfree[s], 1); }
    for (int s = 0; s < kTcNL; ++s) { mbar_init(&lofull[s], 4); mbar_init(&lofree[s], 1); }
    mbar_init(&accfull, 1);
    mbar_init(&accfree, 4);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int nchA = a.KA / 32;
  const int nch = nchA + (a.kp + 31) / 32;
  const int64_t ntiles = ceil_div(a.m, kTcBM);
  const int myt = blockIdx.x < ntiles ? (int)ceil_div(ntiles - blockIdx.x, (int64_t)gridDim.x) : 0;
  const int64_t total = (int64_t)myt * nch;        // chunks this CTA streams

  if (warp == 4) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0, c = 0;
      uint32_t ph = 0;
      int64_t tile = blockIdx.x;
      for (int64_t g = 0; g < total; ++g) {
        if (g >= kTcNR) mbar_wait(&rawfree[s], ph ^ 1);
        if (g == 0) stamp(2);
        const int r0 = (int)(tile * kTcBM);
        unsigned char* st = rawst + s * L::STAGE;
        mbar_expect_tx(&full[s], (uint32_t)((a.dbg & 4) ? L::ZB : L::STAGE));
        if (c < nchA) tma_load_2d(st, &a.tmA, &full[s], c * 32, r0);
        else tma_load_2d(st, &a.tmX, &full[s], (c - nchA) * 32, r0);
        const int kw = c < nchA ? c * 32 : a.KA + (c - nchA) * 32;
        if (!(a.dbg & 4)) {
          tma_load_2d(st + L::ZB, &a.tmW, &full[s], kw, 0);
          tma_load_2d(st + L::ZB + L::WB, &a.tmW, &full[s], kw, RP);
        }
        if (++s == kTcNR) { s = 0; ph ^= 1; }
        if (++c == nch) { c = 0; tile += gridDim.x; }
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32<kTcBM, RP>();
      int r = 0, l = 0, c = 0;
      uint32_t phl = 0, pht = 0;
      int64_t tl = 0;
      for (int64_t g = 0; g < total; ++g) {
        if (c == 0 && tl > 0) { mbar_wait(&accfree, pht); pht ^= 1; }   // epilogue drained TMEM
        mbar_wait(&lofull[l], phl);
        tc_fence_after();
        const uint32_t zs = smem_u32(rawst + r * L::STAGE), ws = zs + L::ZB, wl = ws + L::WB;
        const uint32_t zl = smem_u32(lost + l * L::ZB);
#pragma unroll
        for (int kk = 0; kk < ((a.dbg & 2) ? 0 : 4); ++kk) {   // K = 8 tf32 (32 bytes) per MMA
          const uint64_t dzh = umma_desc_k_sw128(zs + kk * 32), dzl = umma_desc_k_sw128(zl + kk * 32);
          const uint64_t dwh = umma_desc_k_sw128(ws + kk * 32), dwl = umma_desc_k_sw128(wl + kk * 32);
          umma_tf32(tmem, dzh, dwh, idesc, c > 0 || kk > 0);
          umma_tf32(tmem, dzh, dwl, idesc, true);
          umma_tf32(tmem, dzl, dwh, idesc, true);
        }
        umma_commit(&rawfree[r]);
        umma_commit(&lofree[l]);
        if (c == nch - 1) umma_commit(&accfull);
        if (++r == kTcNR) r = 0;
        if (++l == kTcNL) { l = 0; phl ^= 1; }
        if (++c == nch) { c = 0; ++tl; }
      }
    }
  } else {
    // ---------------- warps 0-3: lo parts, then the epilogue of each tile
    double fw = 0.0;
    float4 a1r[8], xor_[8];                        // epilogue operands captured from the stream
    int r = 0, l = 0, c = 0;
    uint32_t phr = 0, phl = 0;
    int64_t tl = 0;
    for (int64_t g = 0; g < total; ++g) {
      mbar_wait(&full[r], phr);
      if (g == 0 && tid == 0) stamp(1);
      if (g >= kTcNL) mbar_wait(&lofree[l], phl ^ 1);
      const float4* src = reinterpret_cast<const float4*>(rawst + r * L::STAGE);
      float4* dst = reinterpret_cast<float4*>(lost + l * L::ZB);
      if (RP <= 32 && lane < 16 && (c == 0 || c == nchA)) {
        // this thread's epilogue row (16 warp + lane): A1 = chunk 0, X1_p = chunk nchA
        const int rr = 16 * warp + lane;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = src[rr * 8 + (q ^ (rr & 7))];   // SWIZZLE_128B: 16-byte unit q of row rr
          if (c == 0) a1r[q] = v;
          else xor_[q] = v;
        }
      }
#pragma unroll
      for (int i = tid; i < ((a.dbg & 1) ? 0 : L::ZB / 16); i += 128) {
        const float4 v = src[i];
        float4 o;
        float h;
        tf32_split(v.x, h, o.x); tf32_split(v.y, h, o.y); tf32_split(v.z, h, o.z); tf32_split(v.w, h, o.w);
        dst[i] = o;
      }
      fence_proxy_async();                         // generic-proxy writes -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&lofull[l]);
      if (++r == kTcNR) { r = 0; phr ^= 1; }
      if (++l == kTcNL) { l = 0; phl ^= 1; }
      if (c == nch - 1) {
        // ---- epilogue of tile tl: row 16 warp + lane (lanes < 16) of the M = 64 tile
        const int64_t r0 = (blockIdx.x + tl * gridDim.x) * kTcBM;
        if (tid == 0) stamp(3);
        mbar_wait(&accfull, (uint32_t)(tl & 1));
        if (tid == 0) stamp(4);
        tc_fence_after();
        const int64_t row = r0 + 16 * warp + lane;
        const bool live = lane < 16 && row < a.m && !(a.dbg & 8);
#pragma unroll 1
        for (int c0 = 0; c0 < RP && c0 < a.kp; c0 += 32) {
          // operands first (kp and lda are multiples of 4: 16-byte vectors), then the TMEM tile
          float4 xo[8], ar[8];
          const int nv = min(32, a.kp - c0) / 4;
          if (RP <= 32) {
#pragma unroll
            for (int q = 0; q < 8; ++q) { xo[q] = xor_[q]; ar[q] = a1r[q]; }
          } else if (live) {
            const float4* xp = reinterpret_cast<const float4*>(a.Xold + row * a.kp + c0);
            const float4* ap = reinterpret_cast<const float4*>(a.A + row * a.lda + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nv) { xo[q] = __ldg(xp + q); ar[q] = __ldg(ap + q); }
          }
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
          if (live) {
            float4* xn = reinterpret_cast<float4*>(a.Xnew + row * a.kp + c0);
            float4* dn = reinterpret_cast<float4*>(a.Dnew + row * a.kp + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (q < nv) {
                const float* xv = reinterpret_cast<const float*>(&xo[q]);
                const float* av = reinterpret_cast<const float*>(&ar[q]);
                float xq[4], dq[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int ll = c0 + 4 * q + e;
                  const float x = ll < a.k ? v[4 * q + e] : 0.f;
                  xq[e] = x;
                  dq[e] = x - xv[e];
                  if (ll < a.k) {
                    const double d = (double)av[e] - (double)x;
                    fw += (double)a.w2s * d * d;
                  }
                }
                xn[q] = make_float4(xq[0], xq[1], xq[2], xq[3]);
                dn[q] = make_float4(dq[0], dq[1], dq[2], dq[3]);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accfree);
        if (tid == 0) stamp(5);
      }
      if (++c == nch) { c = 0; ++tl; }
    }
    fw = warp_sum(fw);
    if (lane == 0) wsum[warp] = fw;
    if (warp == 0) {   // the small step that follows reads these: pull them into L2 (not earlier:
                       // bulk prefetches queue behind this CTA's first TMA loads)
      for (int r = 0; r < 6; ++r) {
        const char* base = reinterpret_cast<const char*>(a.pf_ptr[r]);
        const int64_t nb = a.pf_bytes[r] & ~(int64_t)15;
        if (!base || nb <= 0) continue;
        const int64_t chunk = 16384, nchunk = ceil_div(nb, chunk);   // spread over all CTAs
        for (int64_t c = blockIdx.x + (int64_t)gridDim.x * lane; c < nchunk; c += (int64_t)gridDim.x * 32) {
          const int64_t off = c * chunk;
          const unsigned sz = (unsigned)(nb - off < chunk ? nb - off : chunk);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base + off), "r"(sz) : "memory");
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) a.fw_part[blockIdx.x] = (wsum[0] + wsum[1]) + (wsum[2] + wsum[3]);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<L::NCOL>(tmem);
  }
  if (tid == 0) stamp(6);
}

template <int RP>
static cudaError_t launch_tc(const RowPassTcArgs& a, int grid, cudaStream_t st, int* occ) {
  auto kern = row_pass_tc_kernel<RP>;
  const size_t smem = TcLayout<RP>::TOTAL + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, kTcThreads, smem);
  kern<<<grid, kTcThreads, smem, st>>>(a);
  return cudaGetLastError();
}

int row_pass_tc_ctas_per_sm(int rp) {
  int bytes = 0;
  switch (rp) {
    case 16: bytes = TcLayout<16>::TOTAL; break;
    case 32: bytes = TcLayout<32>::TOTAL; break;
    case 64: bytes = TcLayout<64>::TOTAL; break;
    default: bytes = TcLayout<128>::TOTAL; break;
  }
  return std::max(1, std::min(3, (228 * 1024) / (bytes + 1024 + 1024)));   // + align pad + reserve
}

cudaError_t launch_row_pass_tc(const RowPassTcArgs& a, int rp, int grid, cudaStream_t st, int* occ) {
  switch (rp) {
    case 16: return launch_tc<16>(a, grid, st, occ);
    case 32: return launch_tc<32>(a, grid, st, occ);
    case 64: return launch_tc<64>(a, grid, st, occ);
    case 128: return launch_tc<128>(a, grid, st, occ);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wlr
