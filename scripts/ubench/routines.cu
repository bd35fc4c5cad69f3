// Time individual K3 device routines (cycles, one CTA of 512 threads).
#include <cstdio>
#include "small_step.cuh"
using namespace wlr;

__global__ void __launch_bounds__(512, 1) k_routines(double* out, int n, int b) {
  __shared__ double A[60 * 60];
  __shared__ double T[32 * 32], U[32 * 32], th[32], d0[128], rb[128];
  __shared__ int ok_s;
  // SPD test matrix: diag dominant
  for (int idx = threadIdx.x; idx < n * n; idx += 512) {
    const int i = idx / n, j = idx % n;
    A[idx] = (i == j ? n + 1.0 : 0.0) + 1.0 / (1.0 + i + j);
  }
  for (int idx = threadIdx.x; idx < b * b; idx += 512) {
    const int i = idx / b, j = idx % b;
    T[idx] = (i == j ? 10.0 * (b - i) : 0.0) + 0.01 / (1.0 + i + j);
  }
  __syncthreads();
  long long t0 = clock64();
  bool ok = spd_inverse_cta(A, n, 0.0, d0, rb);
  long long t1 = clock64();
  jacobi_warp0(T, U, th, b);
  long long t2 = clock64();
  for (int idx = threadIdx.x; idx < b * b; idx += 512) {
    const int i = idx / b, j = idx % b;
    T[idx] = (i == j ? 10.0 * (b - i) : 0.0) + 0.01 / (1.0 + i + j);
  }
  __syncthreads();
  long long t3 = clock64();
  bool ok2 = chol_small(T, b, &ok_s);
  long long t4 = clock64();
  __syncthreads();
  long long t5 = clock64();
  double v = block_sum((double)threadIdx.x, th);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t4 - t3; out[3] = t6 - t5; out[4] = ok + ok2 + A[0] + U[0] + v;
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 64 * 8);
  int ns[3] = {10, 30, 60};
  for (int q = 0; q < 3; ++q) {
    for (int rep = 0; rep < 2; ++rep) k_routines<<<1, 512>>>(out, ns[q], 8);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    double h[5];
    cudaMemcpy(h, out, 5 * 8, cudaMemcpyDeviceToHost);
    printf("n=%d b=8: spd_inverse %.0f cyc (%.0f/step) | jacobi(b=8) %.0f | chol_small(b=8) %.0f | block_sum %.0f\n",
           ns[q], h[0], h[0] / ns[q], h[1], h[2], h[3]);
  }
  return 0;
}
