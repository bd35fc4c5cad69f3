// incr_tc.cu -- K2b on the 5th-generation tensor cores (fp32 data, kp <= 128).
//
// The Gram increments are one contraction over the pixel rows:
//     [N | Gamma | Omega](l, j) = sum_i Delta(i, l) Z(i, j),   Z = [A(:, k0:n) | X1_p | Delta]
// computed here as D = Z^T Delta on tcgen05 with 3xTF32, one CTA per (128-column block of Z,
// row split):
//   warp 4 (lane 0): TMA per 32-row chunk: 4 boxes of Z (32 columns each, SWIZZLE_128B) + Delta
//   warps 0-3: thread c owns Z column c of the block: it reads its column of the chunk (32 rows,
//     conflict-free across the warp), splits it into tf32 hi / lo and stores both into TMEM
//     (tcgen05.st; the A operand, M = 128 columns x K = 32 rows, K-major); the four warps also
//     write Delta^T hi / lo (K-major, SWIZZLE_128B) into shared memory (the B operand)
//   warp 5 (lane 0): per 8-row k-step, Z_hi x [Delta_hi; Delta_lo] (N = 64) and
//     Z_lo x Delta_hi (N = 32) into the TMEM accumulator
// Epilogue: thread c reads its accumulator lane and writes the fp64 partial of column c for all
// l < k.  The column layout pads the A part to a multiple of 32 (nA32) and the X1_p and Delta
// parts to KPD = kp rounded up to 32, so that no 32-column TMA box straddles two sources; the
// reduce kernel reads that layout (nz' = nA32 + 2 KPD, kp' = KPD).  KPD = 64 .. 128 (k > 32,
// configs 4-5): the Delta^T operand is N = 2 KPD <= 256 wide, the accumulator 2 KPD TMEM columns;
// while the tensor-core gate is off those widths leave the chunk to the CUDA-core kernel.
#include "kernels.h"
#include "umma.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace wlr {

constexpr int kItThreads = 192;
#ifndef WLR_IT_NR
#define WLR_IT_NR 3
#endif
#ifndef WLR_IT_NL
#define WLR_IT_NL 3
#endif
constexpr int kItNR = WLR_IT_NR, kItNL = WLR_IT_NL;
constexpr int kItZB = 4 * 32 * 128;     // Z chunk: 4 boxes of 32 rows x 128 B (16 KB)
template <int KPD> struct ItLayout {
  static constexpr int DB = KPD * 128;                 // Delta chunk: 32 rows x KPD fp32 (KPD/32 boxes)
  static constexpr int ST = kItZB + DB;                // raw stage
  static constexpr int BT = 2 * KPD * 128;             // B operand slot: Delta^T hi | lo (2 KPD rows x 128 B)
  static constexpr int SMEM = kItNR * ST + kItNL * BT;
  static constexpr int ACC = 2 * KPD;                  // accumulator columns
  static constexpr int NCOL = ACC + 64 * kItNL <= 256 ? 256 : 512;
};

template <int KPD>
__global__ void __launch_bounds__(kItThreads, KPD <= 32 ? 2 : 1) incr_tc_kernel(const __grid_constant__ IncrTcArgs a) {
  using L = ItLayout<KPD>;
  constexpr int kItST = L::ST, kItBT = L::BT;
  // Programmatic dependent launch behind the row pass: only the producer waits for it, and only
  // before its Delta boxes -- the A and X1_p boxes of the first stages (not written by the row
  // pass) are requested while the row pass is still finishing.  The gate was written by the small
  // step before the row pass started.
  pdl_trigger();
  // gate: tensor cores once the X1 step is small; otherwise the same pipeline
  // feeds plain FP32 FMAs on the CUDA cores (fp32 sums over 32-row chunks, fp64 across chunks)
  const bool tc = *a.gate != 0;
  if (KPD > 32 && !tc) {                       // (gate off: the CUDA-core kernel computed this iteration;
    pdl_wait();                                //  complete only after it, for the reduce that follows)
    return;
  }
  auto stamp = [&](int i) {
    if (a.tstamp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.tstamp[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  extern __shared__ __align__(1024) unsigned char it_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round trip would turn
  // every access through sm into a generic load)
  unsigned char* sm = it_raw + ((1024u - (smem_u32(it_raw) & 1023u)) & 1023u);
  unsigned char* rawst = sm;                               // [NR][Z boxes | Delta]
  unsigned char* bst = sm + kItNR * kItST;                 // [NL][Delta^T hi | Delta^T lo]
  __shared__ __align__(8) uint64_t full[kItNR], rawfree[kItNR], lofull[kItNL], lofree[kItNL], accfull;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int ACC = L::ACC;                              // accumulator columns
  if (warp == 0) tmem_alloc<L::NCOL>(&tslot);              // ACC + NL x 64 (Z_hi | Z_lo)
  if (tid == 32) {
    for (int s = 0; s < kItNR; ++s) { mbar_init(&full[s], 1); mbar_init(&rawfree[s], tc ? 1 : 4); }
    for (int s = 0; s < kItNL; ++s) { mbar_init(&lofull[s], 4); mbar_init(&lofree[s], 1); }
    mbar_init(&accfull, 1);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  double acc64[32];                                        // CUDA-core path accumulators
  const int j0 = blockIdx.x * 128;                         // first Z column of this block
  const int64_t r0 = (int64_t)blockIdx.y * a.rows_per_split;
  const int64_t r1 = r0 + a.rows_per_split < a.m ? r0 + a.rows_per_split : a.m;
  const int nch = r1 > r0 ? (int)ceil_div(r1 - r0, (int64_t)32) : 0;

  if (warp == 4) {
    if (lane == 0) {
      // boxes of chunk ch in stage s: part 0 = A / X1_p (independent of the row pass), part 1 =
      // Delta (written by the row pass)
      auto issue = [&](int ch, int s, int part) {
        unsigned char* st = rawst + s * kItST;
        const int row = (int)(r0 + 32 * ch);
        if (part == 0) mbar_expect_tx(&full[s], (uint32_t)kItST);
        for (int b = 0; b < 4; ++b) {                      // Z column boxes
          const int zc = j0 + 32 * b;
          const bool dpart = zc >= a.nA32 + KPD;
          if (dpart != (part == 1)) continue;
          if (zc < a.nA32) tma_load_2d(st + b * 4096, &a.tmA, &full[s], a.k0 + zc, row);
          else if (zc < a.nA32 + KPD) tma_load_2d(st + b * 4096, &a.tmX, &full[s], zc - a.nA32, row);
          else tma_load_2d(st + b * 4096, &a.tmD, &full[s], zc - a.nA32 - KPD < KPD ? zc - a.nA32 - KPD : 0, row);
        }
        if (part == 1)
          for (int db = 0; db < KPD / 32; ++db) tma_load_2d(st + kItZB + db * 4096, &a.tmD, &full[s], 32 * db, row);
      };
      const int npre = nch < kItNR ? nch : kItNR;
      for (int ch = 0; ch < npre; ++ch) issue(ch, ch, 0);
      pdl_wait();                                          // the row pass: Delta is complete
      for (int ch = 0; ch < npre; ++ch) issue(ch, ch, 1);
      int s = npre == kItNR ? 0 : npre;
      uint32_t ph = npre == kItNR ? 1 : 0;
      for (int ch = npre; ch < nch; ++ch) {
        if (ch >= kItNR) mbar_wait(&rawfree[s], ph ^ 1);
        issue(ch, s, 0);
        issue(ch, s, 1);
        if (++s == kItNR) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && tc) {
      const uint32_t id2 = umma_idesc_tf32<128, 2 * KPD>(), id1 = umma_idesc_tf32<128, KPD>();
      int r = 0, l = 0;
      uint32_t phl = 0;
      for (int ch = 0; ch < nch; ++ch) {
        mbar_wait(&lofull[l], phl);
        tc_fence_after();
        const uint32_t ta = tmem + (uint32_t)(ACC + 64 * l);
        const uint32_t bs = smem_u32(bst + l * kItBT);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t db = umma_desc_k_sw128(bs + kk * 32);   // [Delta_hi^T; Delta_lo^T], N = 2 KPD
          umma_tf32_ts(tmem, ta + 8 * kk, db, id2, ch > 0 || kk > 0);
          umma_tf32_ts(tmem, ta + 32 + 8 * kk, db, id1, true);
        }
        umma_commit(&rawfree[r]);
        umma_commit(&lofree[l]);
        if (ch == nch - 1) umma_commit(&accfull);
        if (++r == kItNR) r = 0;
        if (++l == kItNL) { l = 0; phl ^= 1; }
      }
    }
  } else if (!tc) {
    // ---------------- warps 0-3, CUDA cores: thread c owns Z column c = 32 warp + lane;
    // per 32-row chunk acc32[l] = sum_i Delta(i, l) Z(i, c) in fp32, then added into fp64
    int r = 0;
    uint32_t phr = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) acc64[q] = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      mbar_wait(&full[r], phr);
      const unsigned char* st = rawst + r * kItST;
      const float* box = reinterpret_cast<const float*>(st + warp * 4096);
      const float4* dl = reinterpret_cast<const float4*>(st + kItZB);
      float acc32[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) acc32[q] = 0.f;
#pragma unroll 4
      for (int i = 0; i < 32; ++i) {
        const float z = box[i * 32 + ((((lane >> 2) ^ (i & 7)) << 2) | (lane & 3))];
#pragma unroll
        for (int q = 0; q < 8; ++q) {           // Delta(i, 4q..4q+3): unit q of row i (broadcast)
          const float4 d = dl[i * 8 + (q ^ (i & 7))];
          acc32[4 * q] = fmaf(d.x, z, acc32[4 * q]);
          acc32[4 * q + 1] = fmaf(d.y, z, acc32[4 * q + 1]);
          acc32[4 * q + 2] = fmaf(d.z, z, acc32[4 * q + 2]);
          acc32[4 * q + 3] = fmaf(d.w, z, acc32[4 * q + 3]);
        }
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) acc64[q] += (double)acc32[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&rawfree[r]);
      if (++r == kItNR) { r = 0; phr ^= 1; }
    }
  } else {
    // ---------------- warps 0-3: Z column c = 32 warp + lane -> TMEM; Delta^T -> smem
    const int c = 32 * warp + lane;
    int r = 0, l = 0;
    uint32_t phr = 0, phl = 0;
    for (int ch = 0; ch < nch; ++ch) {
      mbar_wait(&full[r], phr);
      if (ch == 0 && tid == 0) stamp(1);
      if (ch >= kItNL) mbar_wait(&lofree[l], phl ^ 1);
      const unsigned char* st = rawst + r * kItST;
      {   // column c: box warp, 16-byte unit (lane / 4) ^ (row & 7), word lane % 4
        const float* box = reinterpret_cast<const float*>(st + warp * 4096);
        float hi[32], lo[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float v = box[i * 32 + ((((lane >> 2) ^ (i & 7)) << 2) | (lane & 3))];
          tf32_split(v, hi[i], lo[i]);
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(ACC + 64 * l);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_st_wait();
      }
      {   // Delta^T hi (rows 0..KPD-1) | lo (rows KPD..) of the B slot: element (n, k) = Delta(k, n).
          // Task t = (kb, nb): the 4 x 4 block k = 4 kb.., n = 4 nb.. -- four 16-byte reads (one per
          // k row of the SWIZZLE_128B box), a register transpose, four 16-byte hi and four lo writes
          // (one per n row of the K-major SWIZZLE_128B operand).  A 128-bit access is served 8 lanes
          // at a time, so each 8-lane group takes u = lane % 8 and kb = (u + s) % 8 (s = the group):
          // the read position u ^ (k % 8) and the write position kb ^ (n % 8) are then 8 distinct
          // 16-byte units in every group, one wavefront each (lanes with kb = lane % 8 and a shared u
          // per group read with 4-way conflicts: 16 wavefronts per warp instead of 4, ncu source page)
        const unsigned char* dl = st + kItZB;
        unsigned char* bt = bst + l * kItBT;
#pragma unroll
        for (int t = tid; t < 2 * KPD; t += 128) {
          const int u = t & 7, kb = (u + (t >> 3)) & 7, bx = t >> 6;   // 16-byte unit of n, row block
          const int nb = 8 * bx + u;
          const unsigned char* box = dl + bx * 4096;          // 32-column box of the chunk
          float4 r[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = 4 * kb + i;
            r[i] = *reinterpret_cast<const float4*>(box + k * 128 + ((u ^ (k & 7)) << 4));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = 4 * nb + j;
            const float c[4] = {j == 0 ? r[0].x : j == 1 ? r[0].y : j == 2 ? r[0].z : r[0].w,
                                j == 0 ? r[1].x : j == 1 ? r[1].y : j == 2 ? r[1].z : r[1].w,
                                j == 0 ? r[2].x : j == 1 ? r[2].y : j == 2 ? r[2].z : r[2].w,
                                j == 0 ? r[3].x : j == 1 ? r[3].y : j == 2 ? r[3].z : r[3].w};
            float h[4], lo[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) tf32_split(c[i], h[i], lo[i]);
            const int pos = (kb ^ (n & 7)) << 4;                // (KPD + n) & 7 == n & 7
            *reinterpret_cast<float4*>(bt + n * 128 + pos) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(bt + (KPD + n) * 128 + pos) = make_float4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lofull[l]);
      if (++r == kItNR) { r = 0; phr ^= 1; }
      if (++l == kItNL) { l = 0; phl ^= 1; }
    }
  }
  // ---------------- epilogue: Z column c = tid (< 128), Delta columns l < 32, into an fp64 tile
  // [32][128] (the stages are free); the cs row splits of a cluster sum their tiles in rank order
  double* tile = reinterpret_cast<double*>(sm);
  if (!tc) {
    __syncthreads();                                       // every stage consumed
    if (warp < 4)
#pragma unroll
      for (int q = 0; q < 32; ++q) tile[q * 128 + tid] = acc64[q];
  } else if (warp < 4) {
    const int c = tid;
    if (tid == 0) stamp(2);                                // converters done
    if (nch > 0) {
      mbar_wait(&accfull, 0);
      if (tid == 0) stamp(3);                              // accumulator complete
      tc_fence_after();
    }
#pragma unroll 1
    for (int s0 = 0; s0 < KPD; s0 += 32) {                 // 32 Delta columns per TMEM load
      float v[32], v2[32];
      if (nch > 0) {
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)s0, v);
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(KPD + s0), v2);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) { v[q] = 0.f; v2[q] = 0.f; }
      }
      if (a.cs <= 1) {   // straight from the accumulator lanes: row q of the partial, coalesced over c
        double* out = a.part + (int64_t)blockIdx.y * a.k * a.nz;
        if (j0 + c < a.nz)
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (s0 + q < a.k) out[(int64_t)(s0 + q) * a.nz + j0 + c] = (double)v[q] + (double)v2[q];
      } else {           // (clusters: KPD = 32 only)
#pragma unroll
        for (int q = 0; q < 32; ++q) tile[q * 128 + c] = (double)v[q] + (double)v2[q];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (a.cs <= 1) {
    if (!tc) {   // CUDA-core path: the fp64 sums went through the tile
      double* out = a.part + (int64_t)blockIdx.y * a.k * a.nz;
      for (int idx = tid; idx < a.k * 128; idx += kItThreads) {
        const int q = idx >> 7, c = idx & 127;
        if (j0 + c < a.nz) out[(int64_t)q * a.nz + j0 + c] = tile[q * 128 + c];
      }
    }
  } else {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int rk = (int)cl.block_rank(), rows = 32 / a.cs;        // Delta columns per rank
    double* out = a.part + (int64_t)(blockIdx.y / a.cs) * a.k * a.nz;
    for (int idx = tid; idx < rows * 128; idx += kItThreads) {
      const int q = rk * rows + (idx >> 7), c = idx & 127;
      double s = 0.0;
      for (int r = 0; r < a.cs; ++r) s += cl.map_shared_rank(tile, r)[q * 128 + c];
      if (q < a.k && j0 + c < a.nz) out[(int64_t)q * a.nz + j0 + c] = s;
    }
    cl.sync();
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<L::NCOL>(tmem);
  }
  if (threadIdx.x == 0) stamp(4);
}

template <int KPD>
static cudaError_t launch_incr_tc_t(const IncrTcArgs& a, int nsplit, cudaStream_t st) {
  using L = ItLayout<KPD>;
  auto kern = incr_tc_kernel<KPD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM + 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int cs = (a.cs > 1 && KPD == 32) ? a.cs : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ceil_div(a.nz, 128), (unsigned)(ceil_div(nsplit, cs) * cs));
  cfg.blockDim = dim3(kItThreads);
  cfg.dynamicSmemBytes = L::SMEM + 1024;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = cs; at[0].val.clusterDim.z = 1;
  cudaLaunchAttribute atp[2] = {at[0], {}};
  int na = cs > 1 ? 1 : 0;
  atp[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  atp[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  cfg.attrs = atp;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

int incr_tc_kpd(int kp) { return kp <= 32 ? 32 : kp <= 64 ? 64 : kp <= 96 ? 96 : kp <= 128 ? 128 : -1; }

cudaError_t launch_incr_tc(const IncrTcArgs& a, int nsplit, cudaStream_t st) {
  switch (a.kpd) {
    case 32: return launch_incr_tc_t<32>(a, nsplit, st);
    case 64: return launch_incr_tc_t<64>(a, nsplit, st);
    case 96: return launch_incr_tc_t<96>(a, nsplit, st);
    case 128: return launch_incr_tc_t<128>(a, nsplit, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wlr
