// Where does a cta_group::1 M=64 tf32 accumulator land in TMEM?  D = A (64 x 32) . B (32 x 32)^T
// with A[i][k] = (k == 0) * (i + 1), B[j][k] = (k == 0) * (j == 0): D[i][0] = i + 1, else 0.
#include <cstdio>
#include <vector>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;
__global__ void k64(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  float* As = (float*)sm; float* Bs = As + 64 * 32;
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<32>(&tslot);
  if (tid == 0) { mbar_init(&full, 1); mbar_init(&done, 1); mbar_init_fence(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) { mbar_expect_tx(&full, (64 * 32 + 32 * 32) * 4); tma_load_2d(As, &tmA, &full, 0, 0); tma_load_2d(Bs, &tmB, &full, 0, 0); }
  mbar_wait(&full, 0);
  if (tid == 0) {
    tc_fence_after();
    umma_tf32(tmem, umma_desc_k_sw128(smem_u32(As)), umma_desc_k_sw128(smem_u32(Bs)), umma_idesc_tf32<64, 32>(), false);
    umma_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
  out[tid] = v[0];
  out[128 + tid] = v[1];
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<32>(tmem);
}
int main() {
  std::vector<float> A(64 * 32, 0.f), B(32 * 32, 0.f);
  for (int i = 0; i < 64; ++i) A[i * 32] = (float)(i + 1);
  B[0] = 1.f; B[1 * 32 + 0] = 1000.f;   // D[i][1] = 1000 (i+1)
  float *dA, *dB, *dO; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dO, 256 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  make_tmap_2d(&tA, dA, 4, 32, 64, 128, 32, 64, true); make_tmap_2d(&tB, dB, 4, 32, 32, 128, 32, 32, true);
  cudaFuncSetAttribute(k64, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k64<<<1, 128, 64 * 1024>>>(tA, tB, dO);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> o(256); cudaMemcpy(o.data(), dO, 1024, cudaMemcpyDeviceToHost);
  for (int l = 0; l < 128; ++l) printf("lane %3d: col0 %6.0f col1 %8.0f%s", l, o[l], o[128 + l], (l % 4 == 3) ? "\n" : " | ");
  return 0;
}
