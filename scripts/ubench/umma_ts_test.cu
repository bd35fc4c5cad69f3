// Unit test of the TS form (A in TMEM written by tcgen05.st, B in smem via TMA SWIZZLE_128B):
// D (128 x 32) = A (128 x 32) . B (32 x 32)^T with 3xTF32, against an fp64 host product.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;
constexpr int M = 128, N = 32, K = 32;
__global__ void k_ts(const float* A, const __grid_constant__ CUtensorMap tmB, const float* Blo_g, float* D) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  float* Bs = (float*)sm;                // [32][32] swizzled (hi = raw)
  float* Bl = Bs + N * K;                // lo (same swizzled positions)
  __shared__ __align__(8) uint64_t full, done, stb;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<128>(&tslot);
  if (tid == 0) { mbar_init(&full, 1); mbar_init(&done, 1); mbar_init(&stb, 4); mbar_init_fence(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;           // cols [0,32) D, [32,64) A_hi, [64,96) A_lo
  if (tid == 0) { mbar_expect_tx(&full, N * K * 4); tma_load_2d(Bs, &tmB, &full, 0, 0); }
  // row r = 32 warp + lane of A into TMEM (hi and lo)
  {
    const int r = 32 * warp + lane;
    float hi[32], lo[32];
    for (int c = 0; c < 32; ++c) tf32_split(A[r * K + c], hi[c], lo[c]);
    tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 32, hi);
    tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + 64, lo);
    tmem_st_wait();
  }
  mbar_wait(&full, 0);
  for (int i = tid; i < N * K; i += blockDim.x) { float h, l; tf32_split(Bs[i], h, l); Bl[i] = l; }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    const uint32_t id = umma_idesc_tf32<M, N>();
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t bh = umma_desc_k_sw128(smem_u32(Bs) + kk * 32), bl = umma_desc_k_sw128(smem_u32(Bl) + kk * 32);
      umma_tf32_ts(tmem, tmem + 32 + 8 * kk, bh, id, kk > 0);
      umma_tf32_ts(tmem, tmem + 32 + 8 * kk, bl, id, true);
      umma_tf32_ts(tmem, tmem + 64 + 8 * kk, bh, id, true);
    }
    umma_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
  for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * N + j] = v[j];
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<128>(tmem);
}
int main() {
  std::mt19937 g(2); std::normal_distribution<float> nd;
  std::vector<float> A(M * K), B(N * K);
  for (auto& x : A) x = nd(g);
  for (auto& x : B) x = nd(g);
  float *dA, *dB, *dD; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tB; make_tmap_2d(&tB, dB, 4, K, N, K * 4, 32, N, true);
  cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k_ts<<<1, 128, 32768>>>(dA, tB, nullptr, dD);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> D(M * N); cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double emax = 0, ref = 0;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
    double s = 0; for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
    emax = fmax(emax, fabs(D[i * N + j] - s)); ref = fmax(ref, fabs(s));
  }
  printf("TS 3xTF32: max|D - exact| = %.3e (rel %.2e)  D[0]=%f D[last]=%f\n", emax, emax / ref, D[0], D[M * N - 1]);
  return 0;
}
