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

__global__ void __launch_bounds__(32 * kRsWarps) row_solve_kernel(const __grid_constant__ RowSolveArgs a) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  const int k = a.k, kp = a.kp;
  const int ntri = k * (k + 1) / 2;
  const float* S = a.S;                                             // k x k  C C^T (L2-resident)
  uint16_t* tab = reinterpret_cast<uint16_t*>(rs_raw);              // ntri entries: r | c << 8
  float* wbase = reinterpret_cast<float*>(tab + ((ntri + 7) & ~7));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Lp = wbase + (size_t)warp * (ntri + 2 * (k + 4));           // this warp's factor
  float* v = Lp + ntri;                                             // e -> z -> x
  for (int c = warp; c < k; c += kRsWarps)
    for (int r = lane; r <= c; r += 32) tab[c * (c + 1) / 2 + r] = (uint16_t)(r | (c << 8));
  __syncthreads();
  double fw = 0.0;
  const int64_t nw = (int64_t)gridDim.x * kRsWarps;
  for (int64_t row = (int64_t)blockIdx.x * kRsWarps + warp; row < a.m; row += nw) {
    const float* w1 = a.W1 + row * a.ldw;
    // K_i in reverse packed form
    for (int e = lane; e < ntri; e += 32) {
      const int rc = tab[e], r = rc & 255, c = rc >> 8;
      const int i = k - 1 - r, l = k - 1 - c;
      float x = __ldg(S + i * k + l);
      if (i == l) { const float w = w1[i]; x += w * w; }
      Lp[e] = x;
    }
    for (int l = lane; l < k; l += 32) v[l] = a.E[row * kp + l];
    __syncwarp();
    bool spd = true;
    for (int j = 0; j < k; ++j) {
      const int M = k - 1 - j, cb = M * (M + 1) / 2;
      const float djj = Lp[cb + M];
      spd = spd && (djj > 0.f);
      const float d = sqrtf(djj > 0.f ? djj : 1.f), inv = 1.f / d;
      for (int r = lane; r < M; r += 32) Lp[cb + r] *= inv;          // column j below the diagonal
      __syncwarp();
      if (lane == 0) Lp[cb + M] = d;
      for (int e = lane; e < cb; e += 32) {                         // trailing triangle = prefix
        const int rc = tab[e], r = rc & 255, c = rc >> 8;
        Lp[e] = fmaf(-Lp[cb + r], Lp[cb + c], Lp[e]);
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
         sizeof(float) * (size_t)kRsWarps * (ntri + 2 * (k + 4));
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
