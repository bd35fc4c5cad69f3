// tcgen05 TF32 issue rate in the row pass's pattern (M = 128; per 8-column k-step one N = 64 and
// one N = 32 MMA), one CTA per SM on every SM:
//   mode 0: SS (A and B from shared memory)
//   mode 1: TS (A from TMEM, B from shared memory)
//   mode 2: TS while warps 0-3 keep storing 64 TMEM columns per "chunk" (tcgen05.st), as the
//           row pass's converters do
//   mode 3: SS while warps 0-3 keep storing into TMEM
#include <cstdio>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;
constexpr int NCHUNK = 400;
template <int MODE>
__global__ void k(unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  if (warp == 0) tmem_alloc<256>(&tslot);
  if (tid == 0) { mbar_init(&bar, 1); mbar_init_fence(); done = 0; }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 4) {
    if ((tid & 31) == 0) {
      const uint32_t id2 = umma_idesc_tf32<128, 64>(), id1 = umma_idesc_tf32<128, 32>();
      const uint64_t da = umma_desc_k_sw128(smem_u32(sm)), db = umma_desc_k_sw128(smem_u32(sm + 16384));
      unsigned long long t0 = clock64();
      for (int c = 0; c < NCHUNK; ++c) {
        const uint32_t ta = tmem + 64 + 64 * (c % 3);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (MODE == 1 || MODE == 2) {
            umma_tf32_ts(tmem, ta + 8 * kk, db + 2 * kk, id2, c > 0 || kk > 0);
            umma_tf32_ts(tmem, ta + 32 + 8 * kk, db + 2 * kk, id1, true);
          } else {
            umma_tf32(tmem, da + 2 * kk, db + 2 * kk, id2, c > 0 || kk > 0);
            umma_tf32(tmem, da + 2 * kk, db + 2 * kk, id1, true);
          }
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      unsigned long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      done = 1;
    }
  } else if (MODE >= 2) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = (float)i;
    int c = 0;
    while (!done) {
      const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + 64 + 64 * (c % 3);
      tmem_st32(ta, v);
      tmem_st32(ta + 32, v);
      tmem_st_wait();
      ++c;
      // pace: about one chunk's conversion work between stores
      for (int q = 0; q < 64; ++q) v[q & 31] = v[q & 31] * 1.0000001f + 1e-7f;
    }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(tmem);
}
template <int MODE>
void run(unsigned long long* d) {
  unsigned long long h = 0;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int r = 0; r < 2; ++r) { k<MODE><<<148, 160, 70000>>>(d); cudaDeviceSynchronize(); }
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d: %.1f cycles per chunk (8 MMAs), %.1f per MMA  [%s]\n", MODE, h / (double)NCHUNK, h / (8.0 * NCHUNK),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  run<0>(d); run<1>(d); run<2>(d); run<3>(d);
  return 0;
}
