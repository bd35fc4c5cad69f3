// result.cu -- K4: Algorithm 1 output: X2 = X1 C + B D with D = V^T,
// B = P^perp_{X1} A2 V (B itself is produced by the row-pass kernel in result mode).
#include "kernels.h"

namespace wlr {

// X2[i][c] = sum_l X1[i][l] C[l][c] + sum_j B[i][j] V[c][j]   (C, V in fp64)
template <typename T>
__global__ void assemble_x2_kernel(const T* __restrict__ X1, int kp, const T* __restrict__ B,
                                   int64_t ldb, const double* __restrict__ C,
                                   const double* __restrict__ V, int64_t m, int k, int nk, int t,
                                   T* __restrict__ X2, int64_t ldx2) {
  const int64_t tot = m * nk;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / nk;
    const int c = (int)(idx % nk);
    double v = 0.0;
    for (int l = 0; l < k; ++l) v = fma((double)X1[i * kp + l], C[(int64_t)l * nk + c], v);
    for (int j = 0; j < t; ++j) v = fma((double)B[i * ldb + j], V[(int64_t)c * t + j], v);
    X2[i * ldx2 + c] = (T)v;
  }
}

template <typename T>
void launch_assemble_x2(const T* X1, int kp, const T* B, int64_t ldb, const double* C,
                        const double* V, int64_t m, int k, int nk, int t, T* X2, int64_t ldx2,
                        cudaStream_t st) {
  const int64_t tot = m * nk;
  assemble_x2_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(tot, 256), 16384), 256, 0, st>>>(
      X1, kp, B, ldb, C, V, m, k, nk, t, X2, ldx2);
}
template void launch_assemble_x2<float>(const float*, int, const float*, int64_t, const double*,
                                        const double*, int64_t, int, int, int, float*, int64_t,
                                        cudaStream_t);
template void launch_assemble_x2<double>(const double*, int, const double*, int64_t, const double*,
                                         const double*, int64_t, int, int, int, double*, int64_t,
                                         cudaStream_t);

template <typename T>
__global__ void copy_x1_kernel(const T* __restrict__ X, int kp, int64_t m, int k, T* __restrict__ out,
                               int64_t ldo) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < m * k;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / k;
    const int l = (int)(idx % k);
    out[i * ldo + l] = X[i * kp + l];
  }
}

template <typename T>
void launch_copy_x1(const T* X, int kp, int64_t m, int k, T* out, int64_t ldo, cudaStream_t st) {
  copy_x1_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(m * k, 256), 16384), 256, 0, st>>>(
      X, kp, m, k, out, ldo);
}
template void launch_copy_x1<float>(const float*, int, int64_t, int, float*, int64_t, cudaStream_t);
template void launch_copy_x1<double>(const double*, int, int64_t, int, double*, int64_t, cudaStream_t);

}  // namespace wlr
