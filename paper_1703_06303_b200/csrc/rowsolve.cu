// rowsolve.cu -- the per-row SPD solves of the non-uniform X1 half-step (PAPER.md:194,
// Algorithm 1 line 8):  x_i (diag(W1(i,:)^2) + C C^T) = e_i  for every pixel row i.
//
// The row pass (K2a, non-uniform W1) writes e_i; here ONE WARP solves one row problem at a time
// (one warp per CTA, grid-stride over rows, as many warps per SM as the factor storage allows).
//
// Method: left-looking (Crout) blocked Cholesky of the BORDERED matrix
//     [ K_i   e_i^T ]      K_i = C C^T + diag(W1(i,:)^2)  (k x k),
//     [ e_i    *    ]
// factoring its k columns only: row k of the factor is z = e_i L^{-T}, so the forward
// substitution comes for free; then x L = z by a blocked back substitution.  Rows 0..k are
// owned by the lanes in REVERSED cyclic order (q-block q holds rows k - 32 q - lane), so the
// rows that stay active longest fill whole q-blocks.
//   * Panel P (columns J = [8P, 8P + 8)): every own row a >= 8P accumulates
//       T[a, J] = K[a, J] - sum_{t < 8P} L[a, t] L[J, t]
//     in registers (8 x NQ accumulators per lane): per t one broadcast of the panel rows L[J, t]
//     (two LDS.128, the same address for all lanes) and one own-row load per q-block, i.e.
//     8 FMAs per shared-memory word -- the CUDA-core FMA pipe, not shared memory, is the bound.
//   * The 8 x 8 diagonal block T[J, J] goes through shared memory to every lane and is factored
//     redundantly in registers (no shuffle chain); rows below the panel then solve
//     L[a, J] = T[a, J] L_JJ^{-T} (36 FMAs per row) and store their 8 entries.
//   * Back substitution x L = z by 8-column blocks from the right: the block's z values are
//     published through shared memory, x_B = z_B L_BB^{-1} redundantly per lane, and every own
//     row b < 8P subtracts sum_i x_i L[8P + i, b] (one float4 pair per row; full blocks as two
//     packed FFMA2 chains of four).
// Storage per warp: the factor in 8-row blocks, block J = rows [8J, 8J + 8) stored [t][8]
// (t < 8J + 8; upper parts unused), block base 32 J (J + 1) + 8 J floats, so that any 32
// consecutive rows hit 32 distinct banks for a fixed column t; plus an 8 x 8 scratch, 1/L_jj
// and the solution vector.  k = 100: 24.8 KB per warp.
//
// Writes X1_{p+1}(i,:), Delta(i,:) and an fp64 partial of f_w = sum W1^2 (A1 - X1_{p+1})^2 per CTA.
#include "kernels.h"

namespace wlr {

__host__ __device__ inline int rs_nblk(int k) { return k / 8 + 1; }                // blocks of rows 0..k
__host__ __device__ inline int rs_base(int J) { return 32 * J * (J + 1) + 8 * J; }  // floats
__host__ __device__ inline int rs_k8(int k) { return (k + 7) & ~7; }
__host__ __device__ inline int rs_warp_floats(int k) { return rs_base(rs_nblk(k)) + 64 + 3 * rs_k8(k) + 8; }

WLR_DEVI float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
WLR_DEVI float lds1(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// (a0, a1) -= (x, x) * (b0, b1) as ONE packed FFMA2 (sm_100a): half the issue slots of two FFMAs
WLR_DEVI void ffma2_neg(float& a0, float& a1, float x, float b0, float b1) {
  unsigned long long A, X, B;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(X) : "f"(-x));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(A) : "l"(X), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(A));
}

// (a0, a1) += (x0, x1) * (b0, b1) as ONE packed FFMA2 (both operands per element)
WLR_DEVI void ffma2_vv(float& a0, float& a1, float x0, float x1, float b0, float b1) {
  unsigned long long A, X, B;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(X) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(A) : "l"(X), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(A));
}

template <int NQ, int NA>
WLR_DEVI void rs_fma4(float (&acc)[NQ][8], const float4 (&b)[8], const float (&o)[NA][4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float bb[8] = {b[2 * u].x, b[2 * u].y, b[2 * u].z, b[2 * u].w,
                         b[2 * u + 1].x, b[2 * u + 1].y, b[2 * u + 1].z, b[2 * u + 1].w};
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2) ffma2_neg(acc[q][jj], acc[q][jj + 1], o[q][u], bb[jj], bb[jj + 1]);
  }
}

template <int NA>
WLR_DEVI void rs_ld4(float4 (&b)[8], float (&o)[NA][4], uint32_t ob, const uint32_t* sa, uint32_t oa) {
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = lds4(ob + 16 * i);
#pragma unroll
  for (int q = 0; q < NA; ++q)
#pragma unroll
    for (int u = 0; u < 4; ++u) o[q][u] = lds1(sa[q] + oa + 32 * u);
}

// panel GEMM: acc[q][jj] -= sum_{t < J0} L[a_q, t] L[J0 + jj, t] for the NA first q-blocks.
// J0 is a multiple of 8: eight t per loop trip in two register stages of four (no copies), 32-bit
// shared addresses, the loads of one stage issued before the packed FMAs (FFMA2) of the other (the
// last trip over-reads four columns inside the factor storage; those values are never used).
template <int NQ, int NA>
WLR_DEVI void rs_gemm8(float (&acc)[NQ][8], const uint32_t (&sa)[NQ], uint32_t sb, int J0) {
  float4 b0[8], b1[8];
  float o0[NA][4], o1[NA][4];
  rs_ld4<NA>(b0, o0, sb, sa, 0);
  uint32_t oa = 0;
#pragma unroll 1
  for (int t = 0; t < J0; t += 8) {
    rs_ld4<NA>(b1, o1, sb + 128, sa, oa + 128);
    rs_fma4<NQ, NA>(acc, b0, o0);
    rs_ld4<NA>(b0, o0, sb + 256, sa, oa + 256);
    rs_fma4<NQ, NA>(acc, b1, o1);
    sb += 256;
    oa += 256;
  }
}

template <int NQ, int NA>
WLR_DEVI void rs_fma2(float (&acc)[NQ][8], const float4 (&b)[4], const float (&o)[NA][2]) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const float bb[8] = {b[2 * u].x, b[2 * u].y, b[2 * u].z, b[2 * u].w,
                         b[2 * u + 1].x, b[2 * u + 1].y, b[2 * u + 1].z, b[2 * u + 1].w};
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2) ffma2_neg(acc[q][jj], acc[q][jj + 1], o[q][u], bb[jj], bb[jj + 1]);
  }
}

template <int NA>
WLR_DEVI void rs_ld2(float4 (&b)[4], float (&o)[NA][2], uint32_t ob, const uint32_t* sa, uint32_t oa) {
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = lds4(ob + 16 * i);
#pragma unroll
  for (int q = 0; q < NA; ++q) { o[q][0] = lds1(sa[q] + oa); o[q][1] = lds1(sa[q] + oa + 32); }
}

// the same with four t per trip in two stages of two (fewer registers: the k <= 95 kernels, which
// run more warps per SM, are faster with it; measured at configs 4 / 5)
template <int NQ, int NA>
WLR_DEVI void rs_gemm4(float (&acc)[NQ][8], const uint32_t (&sa)[NQ], uint32_t sb, int J0) {
  float4 b0[4], b1[4];
  float o0[NA][2], o1[NA][2];
  rs_ld2<NA>(b0, o0, sb, sa, 0);
  uint32_t oa = 0;
#pragma unroll 1
  for (int t = 0; t < J0; t += 4) {
    rs_ld2<NA>(b1, o1, sb + 64, sa, oa + 64);
    rs_fma2<NQ, NA>(acc, b0, o0);
    rs_ld2<NA>(b0, o0, sb + 128, sa, oa + 128);
    rs_fma2<NQ, NA>(acc, b1, o1);
    sb += 128;
    oa += 128;
  }
}

template <int NQ, int NA>
WLR_DEVI void rs_gemm(float (&acc)[NQ][8], const uint32_t (&sa)[NQ], uint32_t sb, int J0) {
  if constexpr (NQ >= 4) rs_gemm8<NQ, NA>(acc, sa, sb, J0);
  else rs_gemm4<NQ, NA>(acc, sa, sb, J0);
}

// K entries of panel P for the own rows (rows of S = C C^T, ld k8 with zero padding, or e_i for
// the bordered row k), issued one panel ahead so that their L1 / L2 latency hides behind the
// current panel.  Rows below 8P are finished: nothing to load.
template <int NQ>
WLR_DEVI void rs_fetch_rc(float (&sn)[NQ][8], const int (&arow)[NQ], const float* __restrict__ S,
                          const float* __restrict__ er, int k, int k8, int P) {
  const int J0 = 8 * P;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int r = arow[q];
    if (r >= J0) {
      const float4* src = reinterpret_cast<const float4*>(r < k ? S + (int64_t)r * k8 + J0 : er + J0);
      const float4 u0 = __ldg(src), u1 = __ldg(src + 1);
      sn[q][0] = u0.x; sn[q][1] = u0.y; sn[q][2] = u0.z; sn[q][3] = u0.w;
      sn[q][4] = u1.x; sn[q][5] = u1.y; sn[q][6] = u1.z; sn[q][7] = u1.w;
    }
  }
}

// the same from per-pixel-row resolved row pointers (measured faster at NQ >= 4, slower at NQ = 2)
// src[q]: the own row's K row (row r of S, or e_i for r = k), resolved once per pixel row
template <int NQ>
WLR_DEVI void rs_fetch(float (&sn)[NQ][8], const int (&arow)[NQ], const float* const (&src)[NQ], int P) {
  const int J0 = 8 * P;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (arow[q] >= J0) {
      const float4* s4 = reinterpret_cast<const float4*>(src[q] + J0);
      const float4 u0 = __ldg(s4), u1 = __ldg(s4 + 1);
      sn[q][0] = u0.x; sn[q][1] = u0.y; sn[q][2] = u0.z; sn[q][3] = u0.w;
      sn[q][4] = u1.x; sn[q][5] = u1.y; sn[q][6] = u1.z; sn[q][7] = u1.w;
    }
  }
}

#ifndef WLR_RS_BS2_NQ
#define WLR_RS_BS2_NQ 1     // packed back substitution (measured faster at k = 50 and k = 100)
#endif
#ifndef WLR_RS_SROW_NQ
#define WLR_RS_SROW_NQ 4    // K-row pointers resolved once per pixel row
#endif

template <int NQ>
__global__ void __launch_bounds__(32) row_solve_kernel(const __grid_constant__ RowSolveArgs a) {
  if (a.stop && *a.stop) return;               // (eps mode: converged before this iteration)
  extern __shared__ __align__(16) float rs_sm[];
  const int k = a.k, kp = a.kp, k8 = rs_k8(k);
  const int lane = threadIdx.x;
  const float* __restrict__ S = a.S;                // k x k8  C C^T (L1 / L2-resident)
  float* Lw = rs_sm;
  float* T8 = Lw + rs_base(rs_nblk(k));             // 8 x 8 diagonal block / z_B
  float* invd = T8 + 64;                            // 1 / L_jj
  float* xo = invd + rs_k8(k);                      // solution row
  int arow[NQ];
  uint32_t sa[NQ];                                  // shared address of L[a_q, 0]
  float* Lwr[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    arow[q] = k - 32 * q - lane;
    const int ac = max(arow[q], 0);
    Lwr[q] = Lw + rs_base(ac >> 3) + (ac & 7);
    sa[q] = (uint32_t)__cvta_generic_to_shared(Lwr[q]);
  }
  float* w2s = xo + rs_k8(k);                       // W1(i,:)^2 of the row (the panel diagonals)
  float* ecor = xo;                                 // A1(i,:) . W1(i,:)^2 (e_lin: added to the bordered row
                                                    // during the factorisation; xo is written only after it)
  const float* Lk = Lw + rs_base(k >> 3) + (k & 7);   // row k: z = e L^{-T}
  const int npan = (k + 7) / 8;
  double fw = 0.0;
  bool spd = true;
  float sn[NQ][8];
  int64_t row = blockIdx.x;
  // own K rows: rows of S are fixed; the bordered row k points at e_i of the current / next pixel row
  const float* srow[NQ];
  const float* snext[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) srow[q] = arow[q] < k ? S + (int64_t)max(arow[q], 0) * k8 : a.E + row * kp;
  constexpr bool kSrow = NQ >= WLR_RS_SROW_NQ;
  if (row < a.m) {
    if constexpr (kSrow) rs_fetch<NQ>(sn, arow, srow, 0);
    else rs_fetch_rc<NQ>(sn, arow, S, a.E + row * kp, k, k8, 0);
  }
  // the row's X1_p, A1 and W1 values (lane + 32 q), software-pipelined one row ahead: W1^2 (the panel
  // diagonals) and A1 . W1^2 (e_lin) are needed at the start of a row, where a fresh load's DRAM
  // latency would be exposed; X1_p and A1 again at its end (Delta, f_w)
  float xon[NQ], a1n[NQ], w1n[NQ];
  auto load_row = [&](int64_t r) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int l = lane + 32 * q;
      xon[q] = r < a.m && l < kp ? a.Xold[r * kp + l] : 0.f;
      a1n[q] = r < a.m && l < k ? __ldg(a.A + r * a.lda + l) : 0.f;
      w1n[q] = r < a.m && l < k ? __ldg(a.W1 + r * a.ldw + l) : 0.f;
    }
  };
  load_row(row);
  for (; row < a.m; row += gridDim.x) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) snext[q] = arow[q] < k ? srow[q] : a.E + (row + gridDim.x) * kp;
    float xold[NQ], a1v[NQ], w1v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) { xold[q] = xon[q]; a1v[q] = a1n[q]; w1v[q] = w1n[q]; }
    load_row(row + gridDim.x);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int l = lane + 32 * q;
      if (l < k) w2s[l] = w1v[q] * w1v[q];
      if (a.e_lin && l < rs_k8(k)) ecor[l] = l < k ? a1v[q] * (w1v[q] * w1v[q]) : 0.f;
    }
    __syncwarp();
    // ---------------------------------------------------------------- factorisation
    for (int P = 0; P < npan; ++P) {
      const int J0 = 8 * P, nb = min(8, k - J0);
      float acc[NQ][8];
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) acc[q][jj] = sn[q][jj];
      if (a.e_lin) {                                 // row k = the bordered row e: lane 0 of q-block 0
        const float4 c0 = reinterpret_cast<const float4*>(ecor + J0)[0], c1 = reinterpret_cast<const float4*>(ecor + J0)[1];
        const float m0 = lane == 0 ? 1.f : 0.f;      // (no divergent branch: a broadcast and 8 FMAs)
        acc[0][0] = fmaf(m0, c0.x, acc[0][0]); acc[0][1] = fmaf(m0, c0.y, acc[0][1]);
        acc[0][2] = fmaf(m0, c0.z, acc[0][2]); acc[0][3] = fmaf(m0, c0.w, acc[0][3]);
        acc[0][4] = fmaf(m0, c1.x, acc[0][4]); acc[0][5] = fmaf(m0, c1.y, acc[0][5]);
        acc[0][6] = fmaf(m0, c1.z, acc[0][6]); acc[0][7] = fmaf(m0, c1.w, acc[0][7]);
      }
      {   // the next panel's K entries (or panel 0 of this warp's next row)
        if constexpr (kSrow) {
          if (P + 1 < npan) rs_fetch<NQ>(sn, arow, srow, P + 1);
          else if (row + gridDim.x < a.m) rs_fetch<NQ>(sn, arow, snext, 0);
        } else {
          const int64_t rn = P + 1 < npan ? row : row + gridDim.x;
          if (rn < a.m) rs_fetch_rc<NQ>(sn, arow, S, a.E + rn * kp, k, k8, P + 1 < npan ? P + 1 : 0);
        }
      }
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(Lw + rs_base(P));
      const int nqa = min(NQ, (k - J0) / 32 + 1);  // q-blocks holding a row >= J0
      if (J0 > 0) {
        if (nqa >= NQ) rs_gemm<NQ, NQ>(acc, sa, sb, J0);
        else if (NQ > 1 && nqa == NQ - 1) rs_gemm<NQ, (NQ > 1 ? NQ - 1 : 1)>(acc, sa, sb, J0);
        else if (NQ > 2 && nqa == NQ - 2) rs_gemm<NQ, (NQ > 2 ? NQ - 2 : 1)>(acc, sa, sb, J0);
        else if (NQ > 3 && nqa == NQ - 3) rs_gemm<NQ, (NQ > 3 ? NQ - 3 : 1)>(acc, sa, sb, J0);
        else rs_gemm<NQ, 1>(acc, sa, sb, J0);
      }
      // diagonal block: the panel rows publish T[J, J]
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = arow[q];
        if (r >= J0 && r < J0 + nb) {
          float4* d = reinterpret_cast<float4*>(T8 + 8 * (r - J0));
          d[0] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
          d[1] = make_float4(acc[q][4], acc[q][5], acc[q][6], acc[q][7]);
        }
      }
      __syncwarp();
      float Ld[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 u0 = reinterpret_cast<const float4*>(T8 + 8 * i)[0];
        const float4 u1 = reinterpret_cast<const float4*>(T8 + 8 * i)[1];
        const float u[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int c = 0; c <= i; ++c) Ld[i][c] = u[c];
        Ld[i][i] += w2s[J0 + i];                     // K = C C^T + diag(W1(i,:)^2)
      }
      if (nb < 8) {                                  // last, partial panel: identity padding
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int c = 0; c <= i; ++c)
            if (i >= nb) Ld[i][c] = i == c ? 1.f : 0.f;
      }
      float idg[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {                  // right-looking 8 x 8 Cholesky in registers
        const float d = Ld[j][j];
        spd = spd && (d > 0.f);
        const float rs = rsqrtf(d > 0.f ? d : 1.f);
        idg[j] = rs;
        Ld[j][j] = d * rs;
#pragma unroll
        for (int i = j + 1; i < 8; ++i) Ld[i][j] *= rs;
#pragma unroll
        for (int i = j + 1; i < 8; ++i)
#pragma unroll
          for (int c = j + 1; c <= i; ++c) Ld[i][c] = fmaf(-Ld[i][j], Ld[c][j], Ld[i][c]);
      }
      // rows below the panel: L[a, J] = T[a, J] L_JJ^{-T}; store
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = arow[q];
        if (r >= J0 + nb) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float v = acc[q][jj];
#pragma unroll
            for (int i = 0; i < jj; ++i) v = fmaf(-acc[q][i], Ld[jj][i], v);
            acc[q][jj] = v * idg[jj];
          }
          if (nb == 8) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) Lwr[q][8 * (J0 + jj)] = acc[q][jj];
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (jj < nb) Lwr[q][8 * (J0 + jj)] = acc[q][jj];
          }
        }
      }
      if (lane == 0) {                               // the panel rows' L_JJ and 1/L_jj
        float* Lc = Lw + rs_base(P) + 8 * J0;
        if (nb == 8) {
          reinterpret_cast<float4*>(invd + J0)[0] = make_float4(idg[0], idg[1], idg[2], idg[3]);
          reinterpret_cast<float4*>(invd + J0)[1] = make_float4(idg[4], idg[5], idg[6], idg[7]);
#pragma unroll
          for (int c = 0; c < 8; ++c) {              // column c: rows 0..7 (zeros above the diagonal)
            float col[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) col[i] = i >= c ? Ld[i][c] : 0.f;
            reinterpret_cast<float4*>(Lc + 8 * c)[0] = make_float4(col[0], col[1], col[2], col[3]);
            reinterpret_cast<float4*>(Lc + 8 * c)[1] = make_float4(col[4], col[5], col[6], col[7]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c < nb) invd[J0 + c] = idg[c];
#pragma unroll
            for (int i = c; i < 8; ++i)
              if (i < nb) Lc[8 * c + i] = Ld[i][c];
          }
        }
      }
      __syncwarp();
    }
    // ------------------------------------------------------------ back substitution x L = z
    float zr[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int r = arow[q];
      zr[q] = (r >= 0 && r < k) ? Lk[8 * r] : 0.f;
    }
    for (int P = npan - 1; P >= 0; --P) {
      const int J0 = 8 * P, nb = min(8, k - J0);
      const float* Lb = Lw + rs_base(P);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = arow[q];
        if (r >= J0 && r < J0 + nb) T8[r - J0] = zr[q];
      }
      __syncwarp();
      float zb[8], iv[8], Lc[8][8];
      {
        const float4 u0 = reinterpret_cast<const float4*>(T8)[0], u1 = reinterpret_cast<const float4*>(T8)[1];
        zb[0] = u0.x; zb[1] = u0.y; zb[2] = u0.z; zb[3] = u0.w; zb[4] = u1.x; zb[5] = u1.y; zb[6] = u1.z; zb[7] = u1.w;
        const float4 v0 = reinterpret_cast<const float4*>(invd + J0)[0], v1 = reinterpret_cast<const float4*>(invd + J0)[1];
        iv[0] = v0.x; iv[1] = v0.y; iv[2] = v0.z; iv[3] = v0.w; iv[4] = v1.x; iv[5] = v1.y; iv[6] = v1.z; iv[7] = v1.w;
#pragma unroll
        for (int i = 0; i < 8; ++i) {              // column J0 + i of the diagonal block
          const float4 c0 = reinterpret_cast<const float4*>(Lb + 8 * (J0 + i))[0];
          const float4 c1 = reinterpret_cast<const float4*>(Lb + 8 * (J0 + i))[1];
          Lc[i][0] = c0.x; Lc[i][1] = c0.y; Lc[i][2] = c0.z; Lc[i][3] = c0.w;
          Lc[i][4] = c1.x; Lc[i][5] = c1.y; Lc[i][6] = c1.z; Lc[i][7] = c1.w;
        }
      }
      // x_B from the right, column-oriented within the block (short dependency chain)
      float x[8];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        x[i] = 0.f;
        if (i < nb) {                                // (rows beyond k in the last block: never read)
          x[i] = zb[i] * iv[i];
#pragma unroll
          for (int i2 = 0; i2 < i; ++i2) zb[i2] = fmaf(-x[i], Lc[i2][i], zb[i2]);   // L[J0 + i, J0 + i2]
        }
      }
      if (lane == 0) {
        if (nb == 8) {
          reinterpret_cast<float4*>(xo + J0)[0] = make_float4(x[0], x[1], x[2], x[3]);
          reinterpret_cast<float4*>(xo + J0)[1] = make_float4(x[4], x[5], x[6], x[7]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i < nb) xo[J0 + i] = x[i];
        }
      }
      if (NQ >= WLR_RS_BS2_NQ && nb == 8) {          // full block: two packed chains of four FFMA2
        float nx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) nx[i] = -x[i];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = arow[q];
          if (r >= 0 && r < J0) {
            const float4 c0 = reinterpret_cast<const float4*>(Lb + 8 * r)[0];          // L[J0 + i, r]
            const float4 c1 = reinterpret_cast<const float4*>(Lb + 8 * r)[1];
            float v0 = zr[q], v1 = 0.f;
            ffma2_vv(v0, v1, nx[0], nx[1], c0.x, c0.y);
            ffma2_vv(v0, v1, nx[2], nx[3], c0.z, c0.w);
            ffma2_vv(v0, v1, nx[4], nx[5], c1.x, c1.y);
            ffma2_vv(v0, v1, nx[6], nx[7], c1.z, c1.w);
            zr[q] = v0 + v1;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = arow[q];
          if (r >= 0 && r < J0) {
            const float4 c0 = reinterpret_cast<const float4*>(Lb + 8 * r)[0];
            const float4 c1 = reinterpret_cast<const float4*>(Lb + 8 * r)[1];
            const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            float v = zr[q];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i < nb) v = fmaf(-x[i], cc[i], v);   // (entries beyond k in the last block: never set)
            zr[q] = v;
          }
        }
      }
      __syncwarp();
    }
    // ------------------------------------------------------------------------- outputs
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int l = lane + 32 * q;
      if (l < kp) {
        const float x = l < k ? xo[l] : 0.f;
        a.Xnew[row * kp + l] = x;
        a.Dnew[row * kp + l] = x - xold[q];
        const double w = (double)w1v[q];
        const double dd = (double)a1v[q] - (double)x;
        fw += w * w * dd * dd;
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) srow[q] = snext[q];
    __syncwarp();
  }
  if (!spd) raise_flag(a.flags, DF_ROWSPD);
  fw = warp_sum(fw);
  if (lane == 0) a.fw_part[blockIdx.x] = fw;
}

static int rs_nq(int k) { return (k + 1 + 31) / 32; }

size_t row_solve_smem(int k) { return sizeof(float) * (size_t)rs_warp_floats(k); }

bool row_solve_ok(int k) { return k >= 1 && rs_nq(k) <= 5 && row_solve_smem(k) <= 200 * 1024; }

template <int NQ>
static int rs_grid_t(int k, int nsm) {
  int occ = 0;
  const size_t smem = row_solve_smem(k);
  cudaFuncSetAttribute(row_solve_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(row_solve_kernel<NQ>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, row_solve_kernel<NQ>, 32, smem) != cudaSuccess || occ < 1)
    occ = 1;
  return nsm * occ;
}

int row_solve_grid(int k, int nsm) {
  switch (rs_nq(k)) {
    case 1: return rs_grid_t<1>(k, nsm);
    case 2: return rs_grid_t<2>(k, nsm);
    case 3: return rs_grid_t<3>(k, nsm);
    case 4: return rs_grid_t<4>(k, nsm);
    default: return rs_grid_t<5>(k, nsm);
  }
}

cudaError_t launch_row_solve(const RowSolveArgs& a, int grid, cudaStream_t st) {
  const size_t smem = row_solve_smem(a.k);
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(grid, a.m));
  switch (rs_nq(a.k)) {
    case 1: row_solve_kernel<1><<<g, 32, smem, st>>>(a); break;
    case 2: row_solve_kernel<2><<<g, 32, smem, st>>>(a); break;
    case 3: row_solve_kernel<3><<<g, 32, smem, st>>>(a); break;
    case 4: row_solve_kernel<4><<<g, 32, smem, st>>>(a); break;
    default: row_solve_kernel<5><<<g, 32, smem, st>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace wlr
