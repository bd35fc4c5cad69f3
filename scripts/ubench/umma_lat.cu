// tcgen05 TF32 MMA latency / throughput on one CTA: M = 64 or 128, N = 32, K = 8 per MMA.
//  (a) latency: 12 MMAs + commit, wait on the mbarrier (repeat, average)
//  (b) throughput: 1200 MMAs back to back, one commit
//  (c) commit + mbarrier round trip with no MMA
#include <cstdio>
#include "../../paper_1703_06303_b200/csrc/umma.cuh"
using namespace wlr;
template <int M, int N = 32>
__global__ void k(unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  if (tid < 32) tmem_alloc<256>(&tslot);
  if (tid == 0) { mbar_init(&bar, 1); mbar_init_fence(); }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t id = umma_idesc_tf32<M, N>();
    const uint64_t da = umma_desc_k_sw128(smem_u32(sm)), db = umma_desc_k_sw128(smem_u32(sm + 16384));
    uint32_t ph = 0;
    unsigned long long t0, t1;
    // (c) commit round trip
    t0 = clock64();
    for (int r = 0; r < 100; ++r) { umma_commit(&bar); mbar_wait(&bar, ph); ph ^= 1; }
    t1 = clock64(); out[0] = (t1 - t0) / 100;
    // (a) 12 MMAs + commit + wait
    t0 = clock64();
    for (int r = 0; r < 100; ++r) {
      for (int q = 0; q < 12; ++q) umma_tf32(tmem, da, db, id, q > 0);
      umma_commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
    }
    t1 = clock64(); out[1] = (t1 - t0) / 100;
    // (b) 1200 MMAs, one commit
    t0 = clock64();
    for (int q = 0; q < 1200; ++q) umma_tf32(tmem, da, db, id, q > 0);
    umma_commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
    t1 = clock64(); out[2] = (t1 - t0);
    // (d) issue cost only: 1200 MMAs, time to issue
    t0 = clock64();
    for (int q = 0; q < 1200; ++q) umma_tf32(tmem, da, db, id, true);
    t1 = clock64(); out[3] = (t1 - t0);
    umma_commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc<256>(tmem);
}
template <int M, int N>
void run(unsigned long long* d) {
  unsigned long long h[4];
  cudaFuncSetAttribute(k<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<M, N><<<1, 128, 70000>>>(d); cudaDeviceSynchronize();
  k<M, N><<<1, 128, 70000>>>(d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("M=%3d N=%3d: commit rt %llu | 12 MMA+commit %llu | 1200 MMA %.1f cyc/MMA = %.0f MAC/cyc  [%s]\n", M, N, h[0], h[1],
         h[2] / 1200.0, (double)M * N * 8 / (h[2] / 1200.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  run<64, 32>(d); run<128, 32>(d); run<64, 64>(d); run<64, 128>(d); run<64, 136>(d); run<64, 256>(d);
  run<128, 64>(d); run<128, 128>(d); run<128, 256>(d);
  return 0;
}
