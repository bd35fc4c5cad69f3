// Unit test of the tcgen05 TF32 path (descriptors, TMA SWIZZLE_128B, TMEM load, 3xTF32):
// D (128 x 32) = A (128 x K) . B (32 x K)^T with K = 64, against an fp64 host product.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;

constexpr int M = 128, N = 32, K = 64;
__global__ void k_test(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* D, int mode) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  float* Ahi = (float*)sm;                 // [2 chunks][128][32] swizzled
  float* Alo = Ahi + 2 * M * 32;
  float* Bhi = Alo + 2 * M * 32;           // [2 chunks][32][32]
  float* Blo = Bhi + 2 * N * 32;
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<32>(&tslot);
  if (tid == 0) { mbar_init(&full, 1); mbar_init(&done, 1); mbar_init_fence(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    mbar_expect_tx(&full, (2 * M * 32 + 2 * N * 32) * 4);
    for (int c = 0; c < 2; ++c) {
      tma_load_2d(Ahi + c * M * 32, &tmA, &full, c * 32, 0);
      tma_load_2d(Bhi + c * N * 32, &tmB, &full, c * 32, 0);
    }
  }
  mbar_wait(&full, 0);
  for (int i = tid; i < 2 * M * 32; i += blockDim.x) { float h, l; tf32_split(Ahi[i], h, l); if (mode != 2) Ahi[i] = h; Alo[i] = l; }
  for (int i = tid; i < 2 * N * 32; i += blockDim.x) { float h, l; tf32_split(Bhi[i], h, l); if (mode != 2) Bhi[i] = h; Blo[i] = l; }
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    const uint32_t id = umma_idesc_tf32<M, N>();
    for (int c = 0; c < 2; ++c)
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ah = umma_desc_k_sw128(smem_u32(Ahi + c * M * 32) + kk * 32);
        const uint64_t al = umma_desc_k_sw128(smem_u32(Alo + c * M * 32) + kk * 32);
        const uint64_t bh = umma_desc_k_sw128(smem_u32(Bhi + c * N * 32) + kk * 32);
        const uint64_t bl = umma_desc_k_sw128(smem_u32(Blo + c * N * 32) + kk * 32);
        umma_tf32(tmem, ah, bh, id, c > 0 || kk > 0);
        if (mode == 1) { umma_tf32(tmem, ah, bl, id, true); umma_tf32(tmem, al, bh, id, true); }
      }
    umma_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
  for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * N + j] = v[j];
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

int main() {
  std::mt19937 g(1); std::normal_distribution<float> nd;
  std::vector<float> A(M * K), B(N * K);
  for (auto& x : A) x = nd(g);
  for (auto& x : B) x = nd(g);
  float *dA, *dB, *dD; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  if (!make_tmap_2d(&tA, dA, 4, K, M, K * 4, 32, M, true) || !make_tmap_2d(&tB, dB, 4, K, N, K * 4, 32, N, true)) { printf("tmap fail\n"); return 1; }
  const size_t smem = (2 * M * 32 * 2 + 2 * N * 32 * 2) * 4 + 1024;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[3] = {"1xTF32(masked hi)", "3xTF32", "1xTF32(raw fp32 operands)"};
  for (int mode : {0, 1, 2}) {
    cudaMemset(dD, 0, M * N * 4);
    k_test<<<1, 128, smem>>>(tA, tB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(M * N); cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double emax = 0, ref = 0, etr = 0, ern = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
      double s = 0, st = 0, sr = 0;
      for (int k = 0; k < K; ++k) {
        s += (double)A[i * K + k] * B[j * K + k];
        auto tr = [](float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return (double)y; };
        auto rn = [](float x) { unsigned u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xFFFFE000u; float y; memcpy(&y, &u, 4); return (double)y; };
        st += tr(A[i * K + k]) * tr(B[j * K + k]);
        sr += rn(A[i * K + k]) * rn(B[j * K + k]);
      }
      emax = fmax(emax, fabs(D[i * N + j] - s)); ref = fmax(ref, fabs(s));
      etr = fmax(etr, fabs(D[i * N + j] - st)); ern = fmax(ern, fabs(D[i * N + j] - sr));
    }
    printf("%-26s err %s: max|D-exact|=%.3e (rel %.2e)  vs trunc-ref %.3e  vs rne-ref %.3e\n", names[mode], cudaGetErrorString(e), emax, emax / ref, etr, ern);
  }
  return 0;
}
