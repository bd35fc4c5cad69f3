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

// Warp roles (192 threads): warps 0-3 convert (lo parts) and run the epilogue (warp w reads TMEM
// lanes 32w.. : rows 32w..32w+31 of an M = 128 tile; rows 16w..16w+15 of an M = 64 tile), warp 4
// lane 0 issues TMA, warp 5 lane 0 issues the MMAs.  Rings: NR raw stages (TMA -> smem) and NL
// lo stages.  M = 128: a TF32 MMA with N = 32, K = 8 costs ~44 cycles whether M is 64 or 128
// (profiles/r01_ubench_umma_rate.log), so the 128-row tile halves the per-row MMA time.
// (+ warp 6 in the deep variant: the leftover rows)
template <int NR> constexpr int tc_threads() { return NR >= 8 ? 224 : 192; }
// The A operand lives in TMEM: each converter thread owns one row of the tile, reads its 32
// values of the chunk from the swizzled stage and writes Z_hi, Z_lo into TMEM (tcgen05.st);
// the MMAs read A from TMEM (the "TS" form) and only W'^T from shared memory.  Shared-memory
// traffic per chunk drops from ~100 KB (Z_lo staged in smem, Z read twice by the tensor core)
// to ~52 KB, which was the binding limit (profiles/r01_v7_rowpass_tc_roles.log).
// (Separate Z / W' rings with a polling producer were measured no faster: the MMA issue rate,
// ~90 cycles per N <= 64 MMA in situ, and the converter -> MMA handoff bound the chunk rate.)
constexpr int kTcNL = 3;
constexpr int kTcRPW = kTcBM / 4;                  // epilogue rows per warp

template <int RP, int NR>
struct TcLayout {                                  // bytes; every block 1024-aligned
  static constexpr int ZB = kTcBM * 128;          // Z chunk (fp32 BM x 32)
  static constexpr int WB = RP * 128;             // W'^T chunk (RP x 32)
  // deep variant: + the chunk of the CTA's <= 4 leftover rows (4 x 128 B, padded to 1 KB)
  static constexpr int XB = NR >= 8 ? 1024 : 0;
  static constexpr int STAGE = ZB + 2 * WB + XB;  // raw stage = Z | W'^T | W'^T_lo | leftover (TMA)
  static constexpr int TOTAL = NR * STAGE;
  // TMEM columns: accumulator [0, RP) z_hi w_hi + z_lo w_hi, [RP, 2 RP) z_hi w_lo; then NL slots
  // of 64 columns (Z_hi chunk | Z_lo chunk, 32 fp32 each)
  static constexpr int ACC = 2 * RP < 64 ? 64 : 2 * RP;
  static constexpr int NCOL = ACC + 64 * kTcNL <= 256 ? 256 : 512;
};

template <int RP, int NR>
__global__ void __launch_bounds__(tc_threads<NR>(), NR >= 8 ? 1 : 2) row_pass_tc_kernel(const __grid_constant__ RowPassTcArgs a) {
  if (a.stop && *a.stop) return;               // (eps mode: converged before this iteration)
  pdl_trigger();                               // the increments may be scheduled (they wait)
  using L = TcLayout<RP, NR>;
  constexpr int kTcNR = NR;
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round trip would turn
  // every access through sm into a generic load)
  unsigned char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
  unsigned char* rawst = sm;                               // [NR][Z | W | W_lo]
  __shared__ __align__(8) uint64_t full[kTcNR], rawfree[kTcNR], lofull[kTcNL], lofree[kTcNL], accfull, accfree;
  __shared__ uint32_t tslot;
  __shared__ double wsum[5];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto twait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
    if (a.tstamp) {
      const unsigned long long t0 = clock64();
      mbar_wait(bar, par);
      acc += clock64() - t0;
    } else {
      mbar_wait(bar, par);
    }
  };
  auto stamp = [&](int i) {
    if (a.tstamp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.tstamp[(int64_t)blockIdx.x * 8 + i] = t;
    }
  };
  if (tid == 0) stamp(0);
  const int nchA = a.KA / 32;
  const int nch = nchA + (a.kp + 31) / 32;
  const int64_t ntiles = ceil_div(a.m_main, kTcBM);
  const int myt = blockIdx.x < ntiles ? (int)ceil_div(ntiles - blockIdx.x, (int64_t)gridDim.x) : 0;
  const int64_t total = (int64_t)myt * nch;        // chunks this CTA streams
  // the producer thread initialises the barriers and puts the first stages in flight before the
  // block-wide barrier (the loads do not wait for the TMEM allocation)
  const bool xtra = L::XB > 0 && a.extra > 0;
  const int xr0 = (int)(a.m_main + (int64_t)a.extra * blockIdx.x);   // first leftover row
  auto issue = [&](int64_t g, int s, int lc, int64_t tile) {
    // chunk order 1, 2, ..., nch - 1, 0: the A1 chunk (whose w^2 K^{-1} term carries most of
    // x' in magnitude) is accumulated LAST, so the tensor core's fp32 accumulator holds only the
    // small terms while the other ~600 products are added (each MMA rounds its sum into the
    // accumulator: with the large term first, ~250 roundings at |x'| gave ~5e-6 relative error)
    const int c = lc + 1 == nch ? 0 : lc + 1;
    const int r0 = (int)(tile * kTcBM);
    unsigned char* st = rawst + s * L::STAGE;
    mbar_expect_tx(&full[s], (uint32_t)(L::ZB + 2 * L::WB + (xtra ? 512 : 0)));
    if (c < nchA) tma_load_2d(st, &a.tmA, &full[s], c * 32, r0);
    else tma_load_2d(st, &a.tmX, &full[s], (c - nchA) * 32, r0);
    const int kw = c < nchA ? c * 32 : a.KA + (c - nchA) * 32;
    tma_load_2d(st + L::ZB, &a.tmW, &full[s], kw, 0);
    tma_load_2d(st + L::ZB + L::WB, &a.tmW, &full[s], kw, RP);
    if (xtra) {
      if (c < nchA) tma_load_2d(st + L::ZB + 2 * L::WB, &a.tmAx, &full[s], c * 32, xr0);
      else tma_load_2d(st + L::ZB + 2 * L::WB, &a.tmXx, &full[s], (c - nchA) * 32, xr0);
    }
  };
  const int npre = (int)(total < kTcNR ? total : kTcNR);
  if (tid == 128) {
    for (int s = 0; s < kTcNR; ++s) { mbar_init(&full[s], 1); mbar_init(&rawfree[s], xtra ? 2 : 1); }
    for (int s = 0; s < kTcNL; ++s) { mbar_init(&lofull[s], 4); mbar_init(&lofree[s], 1); }
    mbar_init(&accfull, 1);
    mbar_init(&accfree, 4);
    mbar_init_fence();
    int c = 0;
    int64_t tile = blockIdx.x;
    for (int g = 0; g < npre; ++g) {               // stages 0 .. npre-1 of the first chunks
      issue(g, g, c, tile);
      if (++c == nch) { c = 0; tile += gridDim.x; }
    }
    stamp(2);
  }
  if (warp == 0) tmem_alloc<L::NCOL>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (warp == 4) {
    // ---------------- TMA producer
    unsigned long long w_prod = 0;
    if (lane == 0) {
      int s = 0, c = 0;
      uint32_t ph = 0;
      int64_t tile = blockIdx.x;
      for (int64_t g = 0; g < total; ++g) {
        if (g >= kTcNR) twait(&rawfree[s], ph ^ 1, w_prod);
        if (g >= npre) issue(g, s, c, tile);       // the first npre went out before the barrier
        if (++s == kTcNR) { s = 0; ph ^= 1; }
        if (++c == nch) { c = 0; tile += gridDim.x; }
      }
    }
    if (lane == 0 && a.tstamp) a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 0] = w_prod;
  } else if (warp == 5) {
    // ---------------- MMA issuer
    unsigned long long w_lof = 0, w_accf = 0;
    if (lane == 0) {
      // per k-step two MMAs: Z_hi against [W_hi; W_lo] (N = 2 RP, the two halves are adjacent in
      // the stage) and Z_lo against W_hi (N = RP) -- Z_hi is read once and the fixed per-MMA
      // cost (~44 cycles at N <= 64) is paid twice instead of three times
      const uint32_t idesc2 = umma_idesc_tf32<kTcBM, 2 * RP>();
      const uint32_t idesc1 = umma_idesc_tf32<kTcBM, RP>();
      int r = 0, l = 0, c = 0;
      uint32_t phl = 0, pht = 0;
      int64_t tl = 0;
      for (int64_t g = 0; g < total; ++g) {
        if (c == 0 && tl > 0) { twait(&accfree, pht, w_accf); pht ^= 1; }   // epilogue drained TMEM
        twait(&lofull[l], phl, w_lof);
        tc_fence_after();
        const uint32_t ws = smem_u32(rawst + r * L::STAGE) + L::ZB;
        const uint32_t ta = tmem + (uint32_t)(L::ACC + 64 * l);   // Z_hi | Z_lo of this chunk
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {           // K = 8 tf32 (8 TMEM columns) per MMA
          const uint64_t dw = umma_desc_k_sw128(ws + kk * 32);
          umma_tf32_ts(tmem, ta + 8 * kk, dw, idesc2, c > 0 || kk > 0);
          umma_tf32_ts(tmem, ta + 32 + 8 * kk, dw, idesc1, true);
        }
        umma_commit(&rawfree[r]);
        umma_commit(&lofree[l]);
        if (c == nch - 1) umma_commit(&accfull);
        if (++r == kTcNR) r = 0;
        if (++l == kTcNL) { l = 0; phl ^= 1; }
        if (++c == nch) { c = 0; ++tl; }
      }
      if (a.tstamp) {
        a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 1] = w_lof;
        a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 2] = w_accf;
      }
    }
  } else if (warp == 6) {
    // ---------------- warp 6: the CTA's leftover rows on the CUDA cores (fp32 FMA), lane = output
    // column l; Z(row e, chunk) comes with each stage (TMA box of 4 rows), W'^T row l from the
    // stage; the stage is released by this warp and the MMA (rawfree count 2)
    double fw = 0.0;
    if (xtra) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      int r = 0, c = 0;
      uint32_t phr = 0;
      for (int64_t g = 0; g < total; ++g) {
        mbar_wait(&full[r], phr);
        const unsigned char* st = rawst + r * L::STAGE;
        const float4* xb = reinterpret_cast<const float4*>(st + L::ZB + 2 * L::WB);   // [4 rows][8 units]
        const float4* wrow = reinterpret_cast<const float4*>(st + L::ZB) + (lane < RP ? lane : 0) * 8;
        const float4* wlow = reinterpret_cast<const float4*>(st + L::ZB + L::WB) + (lane < RP ? lane : 0) * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (lane < RP) {                                    // W' = hi + lo (the 3xTF32 pair)
            const float4 h4 = wrow[q ^ (lane & 7)], l4 = wlow[q ^ (lane & 7)];
            wv = make_float4(h4.x + l4.x, h4.y + l4.y, h4.z + l4.z, h4.w + l4.w);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4 z = xb[e * 8 + q];                   // broadcast
            acc[e] = fmaf(z.x, wv.x, acc[e]);
            acc[e] = fmaf(z.y, wv.y, acc[e]);
            acc[e] = fmaf(z.z, wv.z, acc[e]);
            acc[e] = fmaf(z.w, wv.w, acc[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rawfree[r]);
        if (++r == kTcNR) { r = 0; phr ^= 1; }
        if (++c == nch) {                                     // all chunks summed: epilogue
          c = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t xr = a.m_main + (int64_t)a.extra * blockIdx.x + e;
            if (e < a.extra && xr < a.m && lane < a.kp) {
              const float x = lane < a.k ? acc[e] : 0.f;
              a.Xnew[xr * a.kp + lane] = x;
              if (a.Dnew) a.Dnew[xr * a.kp + lane] = x - a.Xold[xr * a.kp + lane];
              if (lane < a.k) {
                const double d = (double)a.A[xr * a.lda + lane] - (double)x;
                fw += (double)a.w2s * d * d;
              }
            }
            acc[e] = 0.f;
          }
        }
      }
    }
    fw = warp_sum(fw);
    if (lane == 0) wsum[4] = fw;
  } else {
    // ---------------- warps 0-3: lo parts, then the epilogue of each tile
    double fw = 0.0;
    float4 a1r[8], xor_[8];                        // epilogue operands captured from the stream
    int r = 0, l = 0, c = 0;
    uint32_t phr = 0, phl = 0;
    int64_t tl = 0;
    unsigned long long w_full = 0, w_lofree = 0, w_acc = 0, t_conv = 0;
    for (int64_t g = 0; g < total; ++g) {
      twait(&full[r], phr, w_full);
      if (g == 0 && tid == 0) stamp(1);
      if (g >= kTcNL) twait(&lofree[l], phl ^ 1, w_lofree);
      const unsigned long long tc0 = a.tstamp ? clock64() : 0;
      const int pc = c + 1 == nch ? 0 : c + 1;      // physical chunk of logical chunk c (see issue)
      {   // this thread's row (32 warp + lane) of the chunk: 8 swizzled 16-byte units
        const int rr = 32 * warp + lane;
        const float4* src = reinterpret_cast<const float4*>(rawst + r * L::STAGE) + rr * 8;
        float hi[32], lo[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = src[q ^ (rr & 7)];
          if (RP <= 32 && pc == 0) a1r[q] = v;           // A1 (epilogue operand)
          if (RP <= 32 && pc == nchA) xor_[q] = v;       // X1_p
          tf32_split(v.x, hi[4 * q], lo[4 * q]);
          tf32_split(v.y, hi[4 * q + 1], lo[4 * q + 1]);
          tf32_split(v.z, hi[4 * q + 2], lo[4 * q + 2]);
          tf32_split(v.w, hi[4 * q + 3], lo[4 * q + 3]);
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(L::ACC + 64 * l);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lofull[l]);
      if (a.tstamp) t_conv += clock64() - tc0;
      if (++r == kTcNR) { r = 0; phr ^= 1; }
      if (++l == kTcNL) { l = 0; phl ^= 1; }
      if (c == nch - 1) {
        // ---- epilogue of tile tl: row kTcRPW warp + lane of the tile
        const int64_t r0 = (blockIdx.x + tl * gridDim.x) * kTcBM;
        if (tid == 0) stamp(3);
        twait(&accfull, (uint32_t)(tl & 1), w_acc);
        if (tid == 0) stamp(4);
        tc_fence_after();
        const int64_t row = r0 + kTcRPW * warp + lane;
        const bool live = lane < kTcRPW && row < a.m && !(a.dbg & 8);
#pragma unroll 1
        for (int c0 = 0; c0 < RP && c0 < a.kp; c0 += 32) {
          // operands first (kp and lda are multiples of 4: 16-byte vectors), then the TMEM tile
          float4 xo[8], ar[8];
          const int nv = min(32, a.kp - c0) / 4;
          if (RP <= 32) {
#pragma unroll
            for (int q = 0; q < 8; ++q) { xo[q] = xor_[q]; ar[q] = a1r[q]; }
          } else if (live && !a.E) {
            const float4* xp = reinterpret_cast<const float4*>(a.Xold + row * a.kp + c0);
            const float4* ap = reinterpret_cast<const float4*>(a.A + row * a.lda + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nv) {
                ar[q] = __ldg(ap + q);
                if (a.Dnew) xo[q] = __ldg(xp + q);   // (Gram-propagation mode: no Delta)
              }
          }
          float v[32];
          {
            float vl[32];
            tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
            tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(RP + c0), vl);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += vl[j];
          }
          if (live && a.E) {               // non-uniform: the linear part e - A1 . W1^2 (the per-row
            float4* en = reinterpret_cast<float4*>(a.E + row * a.kp + c0);   // solver adds A1 . W1^2:
#pragma unroll                                                           // no loads in this epilogue)
            for (int q = 0; q < 8; ++q) {
              if (q < nv) {
                float eq[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) eq[e] = c0 + 4 * q + e < a.k ? v[4 * q + e] : 0.f;
                en[q] = make_float4(eq[0], eq[1], eq[2], eq[3]);
              }
            }
          } else if (live) {
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
                if (a.Dnew) dn[q] = make_float4(dq[0], dq[1], dq[2], dq[3]);
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
    if (a.tstamp && tid == 0) {
      a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 3] = w_full;
      a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 4] = w_lofree;
      a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 5] = w_acc;
      a.tstamp[(int64_t)gridDim.x * 8 + blockIdx.x * 8 + 6] = t_conv;
    }
    fw = warp_sum(fw);
    if (lane == 0) wsum[warp] = fw;
    if (warp == 0) {   // the small step that follows reads these: pull them into L2 (not earlier:
                       // bulk prefetches queue behind this CTA's first TMA loads)
      for (int r = 0; r < kPf; ++r) {
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
  if (tid == 0) a.fw_part[blockIdx.x] = ((wsum[0] + wsum[1]) + (wsum[2] + wsum[3])) + wsum[4];
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<L::NCOL>(tmem);
  }
  if (tid == 0) stamp(6);
}

template <int RP, int NR>
static cudaError_t launch_tc(const RowPassTcArgs& a, int grid, cudaStream_t st, int* occ) {
  auto kern = row_pass_tc_kernel<RP, NR>;
  const size_t smem = TcLayout<RP, NR>::TOTAL + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, tc_threads<NR>(), smem);
  if (a.pdl) {   // programmatic dependent of the kernel before it on st (it never waits on that one)
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(grid);
    c.blockDim = dim3(tc_threads<NR>());
    c.dynamicSmemBytes = smem;
    c.stream = st;
    c.attrs = at;
    c.numAttrs = 1;
    return cudaLaunchKernelEx(&c, kern, a);
  }
  kern<<<grid, tc_threads<NR>(), smem, st>>>(a);
  return cudaGetLastError();
}

constexpr int kTcNRShallow = 4, kTcNRDeep = 8;

template <int RP, int NR>
static constexpr int tc_bytes_t() { return TcLayout<RP, NR>::TOTAL; }
static int tc_bytes(int rp, bool deep) {
  switch (rp) {
    case 16: return deep ? tc_bytes_t<16, kTcNRDeep>() : tc_bytes_t<16, kTcNRShallow>();
    case 32: return deep ? tc_bytes_t<32, kTcNRDeep>() : tc_bytes_t<32, kTcNRShallow>();
    case 64: return deep ? tc_bytes_t<64, kTcNRDeep>() : tc_bytes_t<64, kTcNRShallow>();
    default: return deep ? tc_bytes_t<128, kTcNRDeep>() : tc_bytes_t<128, kTcNRShallow>();
  }
}

int row_pass_tc_ctas_per_sm(int rp) {
  return std::max(1, std::min(2, (227 * 1024) / (tc_bytes(rp, false) + 1024 + 1024)));   // + align pad + reserve
}

bool row_pass_tc_deep_ok(int rp) { return tc_bytes(rp, true) + 2048 <= 227 * 1024; }

cudaError_t launch_row_pass_tc(const RowPassTcArgs& a, int rp, int grid, cudaStream_t st, int* occ, bool deep) {
  if (deep) {
    switch (rp) {
      case 16: return launch_tc<16, kTcNRDeep>(a, grid, st, occ);
      case 32: return launch_tc<32, kTcNRDeep>(a, grid, st, occ);
      case 64: return launch_tc<64, kTcNRDeep>(a, grid, st, occ);
    }
    return cudaErrorInvalidValue;
  }
  switch (rp) {
    case 16: return launch_tc<16, kTcNRShallow>(a, grid, st, occ);
    case 32: return launch_tc<32, kTcNRShallow>(a, grid, st, occ);
    case 64: return launch_tc<64, kTcNRShallow>(a, grid, st, occ);
    case 128: return launch_tc<128, kTcNRShallow>(a, grid, st, occ);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wlr
