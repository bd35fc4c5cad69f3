"""Generate icache_pf.cu: can instruction fetch after an L2 flush be sped up by prefetching the
code into L2 (cp.async.bulk.prefetch.L2 on the address of a __noinline__ device function)?
A 256 KB straight-line device function is timed (clock64, one warp) cold, cold after a code
prefetch issued by another kernel, and warm."""
import sys

N = 16384
body = ['__device__ __noinline__ float big(float a) {',
        '  float r0=a,r1=a+1,r2=a+2,r3=a+3,r4=a+4,r5=a+5,r6=a+6,r7=a+7;']
for i in range(N):
    body.append('  asm volatile("fma.rn.f32 %%0, %%0, %%1, %%2;" : "+f"(r%d) : "f"(r%d), "f"(r%d) : "memory");'
                % (i % 8, (i + 1) % 8, (i + 3) % 8))
body.append('  return r0+r1+r2+r3+r4+r5+r6+r7;\n}')
src = ["#include <cstdio>", "#include <cstdint>"] + body + ["""
__device__ uintptr_t g_fp;
__global__ void k_addr() { g_fp = (uintptr_t)(void*)&big; }
__global__ void k_run(float* out, float a) {
  long long t0 = clock64();
  float r = big(a + (float)(t0 & 0));
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (float)(t1 - t0); out[1] = r; }
}
// prefetch [fp - before, fp + bytes) into L2 in 16 KB pieces spread over the grid
__global__ void k_pf(size_t before, size_t bytes) {
  const char* base = (const char*)g_fp - before;
  const size_t tot = before + bytes, chunk = 16384;
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c * chunk < tot; c += (size_t)gridDim.x * blockDim.x) {
    const size_t off = c * chunk, sz = tot - off < chunk ? tot - off : chunk;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(base + off), "r"((unsigned)sz) : "memory");
  }
}
// plain loads of the code bytes (does reading code memory even work?)
__global__ void k_rd(size_t bytes, float* out) {
  const uint32_t* p = (const uint32_t*)g_fp;
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes / 4; i += (size_t)gridDim.x * blockDim.x) acc ^= p[i];
  if (acc == 0x12345678u) out[2] = 1.f;
}
__global__ void k_flush(float* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] = 1.0f;
}
int main() {
  float *out, *buf; size_t nf = 256ull << 20;
  cudaMalloc(&out, 64); cudaMalloc(&buf, nf * 4);
  k_addr<<<1, 1>>>(); uintptr_t fp; cudaMemcpyFromSymbol(&fp, g_fp, sizeof(fp));
  printf("device address of big(): %#lx  (%s)\\n", (unsigned long)fp, cudaGetErrorString(cudaDeviceSynchronize()));
  float h[2];
  const char* names[4] = {"cold (L2 flushed)", "cold + L2 prefetch of the code", "cold + ld.global of the code", "warm rerun"};
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      if (mode < 3) k_flush<<<1184, 256>>>(buf, nf);
      if (mode == 1) k_pf<<<64, 32>>>(0, %d * 16 + 4096);
      if (mode == 2) k_rd<<<148, 256>>>(%d * 16 + 4096, out);
      cudaDeviceSynchronize();
      k_run<<<1, 32>>>(out, 1.0f);
      cudaError_t e = cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
      printf("%%-34s %%9.0f cycles = %%6.2f cycles/instr  (%%s)\\n", names[mode], h[0], h[0] / %d, cudaGetErrorString(e));
    }
  return 0;
}""".replace("%d", str(N)).replace("%%", "%")]
open(sys.argv[1], "w").write("\n".join(src))
