// Unit test of MN-major operands (SWIZZLE_128B): D (128 x 64) = Zt (128 x K) . Dl (64 x K)^T with
// Z stored row-major K x 128 (rows = K, columns = M contiguous) and Dl stored K x 64 (N contiguous),
// i.e. D[c][l] = sum_k Z[k][c] Dl[k][l] -- the increment contraction Z^T Delta.
// Layout: TMA boxes of {32 columns, 32 rows}; MN atom (32 columns) stride LBO = 4096 B,
// K atom (8 rows) stride SBO = 1024 B.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;
constexpr int M = 128, N = 64, K = 32;
__host__ __device__ constexpr uint32_t idesc_mn(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__global__ void k_mn(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmD, float* out, uint32_t lbo, uint32_t sbo, uint32_t id, uint32_t kstep) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  unsigned char* Zs = sm;                 // 4 boxes x 4 KB (32 rows x 128 B each)
  unsigned char* Ds = sm + 16384;         // 2 boxes x 4 KB
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<64>(&tslot);
  if (tid == 0) { mbar_init(&full, 1); mbar_init(&done, 1); mbar_init_fence(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    mbar_expect_tx(&full, 16384 + 8192);
    for (int b = 0; b < 4; ++b) tma_load_2d(Zs + b * 4096, &tmZ, &full, b * 32, 0);
    for (int b = 0; b < 2; ++b) tma_load_2d(Ds + b * 4096, &tmD, &full, b * 32, 0);
  }
  mbar_wait(&full, 0);
  if (tid == 0) {
    tc_fence_after();
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t da = desc_mn(smem_u32(Zs) + kk * kstep, lbo, sbo);
      const uint64_t db = desc_mn(smem_u32(Ds) + kk * kstep, lbo, sbo);
      umma_tf32(tmem, da, db, id, kk > 0);
    }
    umma_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  float v[32];
  for (int c0 = 0; c0 < N; c0 += 32) {
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int j = 0; j < 32; ++j) out[(32 * warp + lane) * N + c0 + j] = v[j];
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<64>(tmem);
}
int main(int argc, char** argv) {
  std::mt19937 g(3); std::normal_distribution<float> nd;
  std::vector<float> Z(K * M), Dl(K * N);
  for (auto& x : Z) x = nd(g);
  for (auto& x : Dl) x = nd(g);
  float *dZ, *dD, *dO; cudaMalloc(&dZ, Z.size() * 4); cudaMalloc(&dD, Dl.size() * 4); cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dZ, Z.data(), Z.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dD, Dl.data(), Dl.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tZ, tD;
  make_tmap_2d(&tZ, dZ, 4, M, K, M * 4, 32, 32, true);
  make_tmap_2d(&tD, dD, 4, N, K, N * 4, 32, 32, true);
  cudaFuncSetAttribute(k_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  struct V { uint32_t lbo, sbo, kstep; int am, bm; };
  std::vector<V> vs;
  vs.push_back({(uint32_t)atoi(argv[1]), (uint32_t)atoi(argv[2]), (uint32_t)atoi(argv[5]), atoi(argv[3]), atoi(argv[4])});
  for (auto v : vs) {
    cudaMemset(dO, 0, M * N * 4);
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)v.am << 15) | ((uint32_t)v.bm << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    k_mn<<<1, 128, 40000>>>(tZ, tD, dO, v.lbo, v.sbo, id, v.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> O(M * N); cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double emax = 0, ref = 0;
    for (int c = 0; c < M; ++c) for (int l = 0; l < N; ++l) {
      double s = 0; for (int k = 0; k < K; ++k) {
        auto tr = [](float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return (double)y; };
        s += tr(Z[k * M + c]) * tr(Dl[k * N + l]);
      }
      emax = fmax(emax, fabs(O[c * N + l] - s)); ref = fmax(ref, fabs(s));
    }
    printf("am=%d bm=%d LBO=%5u SBO=%5u: err %.3e (ref %.2f) D00=%.4f\n", v.am, v.bm, v.lbo, v.sbo, emax, ref, O[0]);
  }
  return 0;
}
