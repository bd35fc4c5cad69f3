// rowsolve.cu -- the per-row SPD solves of the non-uniform X1 half-step (PAPER.md:194,
// Algorithm 1 line 8):  x_i (diag(W1(i,:)^2) + C C^T) = e_i  for every pixel row i.
//
// The row pass (K2a, non-uniform W1) writes e_i; here one warp owns one row problem at a time
// (grid-stride over rows, many warps per SM).  K_i = C C^T + diag(W1(i,:)^2) is factored by a
// right-looking Cholesky in shared memory, stored "reverse packed": element (i, l), l <= i, at
// r = k-1-i, c = k-1-l (r <= c), offset c (c + 1) / 2 + r.  Then
//   * column j of L is the contiguous block c = M := k-1-j (offsets M(M+1)/2 + r, r < M; the
//     diagonal at r = M), and
//   * the trailing triangle of step j (i, l > j) is exactly the PREFIX [0, M(M+1)/2) of the
//     storage, so the rank-1 update runs over 32 consecutive elements per warp step, perfectly
//     balanced, with a per-CTA table e -> (r, c) (the same for every step and every row).
// Forward substitution L z = e by columns, back substitution L^T x = z by warp dot products.
// Writes X1_{p+1}(i,:), Delta(i,:) and an fp64 partial of f_w = sum W1^2 (A1 - X1_{p+1})^2.
#include "kernels.h"

namespace wlr {

constexpr int kRsWarps = 4;                      // warps (row problems in flight) per CTA

// floats of one warp's workspace: factor (rounded to 16 B) | vector | float4 panel rows
__host__ __device__ inline int rs_warp_floats(int k) {
  return ((k * (k + 1) / 2 + 3) & ~3) + ((k + 3) & ~3) + 4 * k;
}

__global__ void __launch_bounds__(32 * kRsWarps) row_solve_kernel(const __grid_constant__ RowSolveArgs a) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  const int k = a.k, kp = a.kp;
  const int ntri = k * (k + 1) / 2;
  const float* S = a.S;                                             // k x k  C C^T (L2-resident)
  uint16_t* tab = reinterpret_cast<uint16_t*>(rs_raw);              // ntri entries: r | c << 8
  float* wbase = reinterpret_cast<float*>(tab + ((ntri + 7) & ~7));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = rs_warp_floats(k);                             // multiple of 4 floats
  float* Lp = wbase + (size_t)warp * stride;                        // this warp's factor
  float* v = Lp + ((ntri + 3) & ~3);                                // e -> z -> x
  float4* P = reinterpret_cast<float4*>(v + ((k + 3) & ~3));        // panel: 4 columns per row r
  for (int c = warp; c < k; c += kRsWarps)
    for (int r = lane; r <= c; r += 32) tab[c * (c + 1) / 2 + r] = (uint16_t)(r | (c << 8));
  __syncthreads();
  double fw = 0.0;
  const int64_t nw = (int64_t)gridDim.x * kRsWarps;
  for (int64_t row = (int64_t)blockIdx.x * kRsWarps + warp; row < a.m; row += nw) {
    const float* w1 = a.W1 + row * a.ldw;
    // the row's W1^2 into the panel buffer first (one coalesced load, not one dependent global
    // load per diagonal element inside the build loop)
    float* w2r = reinterpret_cast<float*>(P);
    for (int l = lane; l < k; l += 32) { const float w = __ldg(w1 + l); w2r[l] = w * w; }
    for (int l = lane; l < k; l += 32) v[l] = a.E[row * kp + l];
    __syncwarp();
    // K_i in reverse packed form
    for (int e = lane; e < ntri; e += 32) {
      const int rc = tab[e], r = rc & 255, c = rc >> 8;
      const int i = k - 1 - r, l = k - 1 - c;
      float x = __ldg(S + i * k + l);
      if (i == l) x += w2r[i];
      Lp[e] = x;
    }
    __syncwarp();
    bool spd = true;
    // blocked right-looking Cholesky: panels of 4 columns, then one rank-4 update of the
    // trailing triangle (a storage prefix) with the panel staged as float4 per row
    for (int j0 = 0; j0 < k; j0 += 4) {
      const int nb = min(4, k - j0);
      for (int q = 0; q < nb; ++q) {                                // panel factorisation
        const int j = j0 + q, M = k - 1 - j, cb = M * (M + 1) / 2;
        const float djj = Lp[cb + M];
        spd = spd && (djj > 0.f);
        const float d = sqrtf(djj > 0.f ? djj : 1.f), inv = 1.f / d;
        for (int r = lane; r < M; r += 32) Lp[cb + r] *= inv;
        __syncwarp();
        if (lane == 0) Lp[cb + M] = d;
        for (int q2 = q + 1; q2 < nb; ++q2) {                       // later panel columns
          const int M2 = k - 1 - (j0 + q2), cb2 = M2 * (M2 + 1) / 2;
          const float ljj2 = Lp[cb + M2];                           // L(j0+q2, j)
          for (int r = lane; r <= M2; r += 32) Lp[cb2 + r] = fmaf(-Lp[cb + r], ljj2, Lp[cb2 + r]);
        }
        __syncwarp();
      }
      const int Mt = k - 1 - (j0 + nb - 1);                         // trailing rows r < Mt
      for (int r = lane; r < Mt; r += 32) {
        float c4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int M = k - 1 - (j0 + q);
          c4[q] = q < nb ? Lp[M * (M + 1) / 2 + r] : 0.f;
        }
        P[r] = make_float4(c4[0], c4[1], c4[2], c4[3]);
      }
      __syncwarp();
      const int tt = Mt * (Mt + 1) / 2;
      // 4 independent elements per lane per step: their shared-memory loads overlap
      int e = lane;
      for (; e + 96 < tt; e += 128) {
        int rcq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rcq[u] = tab[e + 32 * u];
        float4 pr[4], pc[4];
        float x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          pr[u] = P[rcq[u] & 255];
          pc[u] = P[rcq[u] >> 8];
          x[u] = Lp[e + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float y = x[u];
          y = fmaf(-pr[u].x, pc[u].x, y);
          y = fmaf(-pr[u].y, pc[u].y, y);
          y = fmaf(-pr[u].z, pc[u].z, y);
          y = fmaf(-pr[u].w, pc[u].w, y);
          Lp[e + 32 * u] = y;
        }
      }
      for (; e < tt; e += 32) {
        const int rc = tab[e], r = rc & 255, c = rc >> 8;
        const float4 pr = P[r], pc = P[c];
        float x = Lp[e];
        x = fmaf(-pr.x, pc.x, x);
        x = fmaf(-pr.y, pc.y, x);
        x = fmaf(-pr.z, pc.z, x);
        x = fmaf(-pr.w, pc.w, x);
        Lp[e] = x;
      }
      __syncwarp();
    }
    if (!spd && lane == 0) raise_flag(a.flags, DF_ROWSPD);
    // forward: L z = e (column j: z_j = v_j / L_jj, v_i -= L_ij z_j for i > j)
    for (int j = 0; j < k; ++j) {
      const int M = k - 1 - j, cb = M * (M + 1) / 2;
      const float zj = v[j] / Lp[cb + M];
      for (int r = lane; r < M; r += 32) v[k - 1 - r] = fmaf(-Lp[cb + r], zj, v[k - 1 - r]);
      __syncwarp();
      if (lane == 0) v[j] = zj;
      __syncwarp();
    }
    // back: L^T x = z (x_j = (z_j - sum_{i > j} L_ij x_i) / L_jj, warp dot product)
    for (int j = k - 1; j >= 0; --j) {
      const int M = k - 1 - j, cb = M * (M + 1) / 2;
      float s = 0.f;
      for (int r = lane; r < M; r += 32) s = fmaf(Lp[cb + r], v[k - 1 - r], s);
      s = warp_sum(s);
      if (lane == 0) v[j] = (v[j] - s) / Lp[cb + M];
      __syncwarp();
    }
    for (int l = lane; l < kp; l += 32) {
      const float x = l < k ? v[l] : 0.f;
      a.Xnew[row * kp + l] = x;
      a.Dnew[row * kp + l] = x - a.Xold[row * kp + l];
      if (l < k) {
        const double w = (double)w1[l];
        const double dd = (double)a.A[row * a.lda + l] - (double)x;
        fw += w * w * dd * dd;
      }
    }
    __syncwarp();
  }
  fw = warp_sum(fw);
  __shared__ double ws[kRsWarps];
  if (lane == 0) ws[warp] = fw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kRsWarps; ++w) s += ws[w];
    a.fw_part[blockIdx.x] = s;
  }
}

size_t row_solve_smem(int k) {
  const int ntri = k * (k + 1) / 2;
  return sizeof(uint16_t) * (size_t)((ntri + 7) & ~7) +
         sizeof(float) * (size_t)kRsWarps * rs_warp_floats(k);
}

bool row_solve_ok(int k) { return k >= 1 && k <= 255 && row_solve_smem(k) <= 220 * 1024; }

int row_solve_grid(int k, int nsm) {
  int occ = 0;
  const size_t smem = row_solve_smem(k);
  cudaFuncSetAttribute(row_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, row_solve_kernel, 32 * kRsWarps, smem) != cudaSuccess || occ < 1)
    occ = 1;
  return std::min(1184, nsm * occ);
}

cudaError_t launch_row_solve(const RowSolveArgs& a, int grid, cudaStream_t st) {
  const size_t smem = row_solve_smem(a.k);
  row_solve_kernel<<<grid, 32 * kRsWarps, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace wlr
