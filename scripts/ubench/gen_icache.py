"""Generate icache.cu: kernels with N straight-line FMAs, timed with clock64 (cold after an
L2 flush, and warm) -- measures instruction-fetch cost of code executed once."""
import sys

def kernel(n):
    out = ["__global__ void k_code_%d(float* out, float a) {" % n,
           "  float r0=a,r1=a+1,r2=a+2,r3=a+3,r4=a+4,r5=a+5,r6=a+6,r7=a+7;",
           '  long long t0; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");',
           '  r0 += (float)(t0 & 0);']
    for i in range(n):
        out.append('  asm volatile("fma.rn.f32 %%0, %%0, %%1, %%2;" : "+f"(r%d) : "f"(r%d), "f"(r%d) : "memory");'
                   % (i % 8, (i + 1) % 8, (i + 3) % 8))
    out.append('  long long t1; asm volatile("add.f32 %1, %1, %2;\\n\\tmov.u64 %0, %%clock64;" : "=l"(t1), "+f"(r0) : "f"(r1+r2+r3+r4+r5+r6+r7) : "memory");')
    out.append("  if (threadIdx.x == 0) { out[0] = (float)(t1 - t0); out[1] = r0+r1+r2+r3+r4+r5+r6+r7; }")
    out.append("}")
    return "\n".join(out)

sizes = [1024, 4096, 16384]
src = ["#include <cstdio>"] + [kernel(n) for n in sizes]
src.append("""__global__ void k_flush(float* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] = 1.0f;
}
int main() {
  float *out, *buf; size_t nf = 256ull << 20;
  cudaMalloc(&out, 64); cudaMalloc(&buf, nf * 4);
  float h[2];""")
for n in sizes:
    src.append("""  for (int rep = 0; rep < 3; ++rep) {
    if (rep < 2) k_flush<<<1184, 256>>>(buf, nf);
    k_code_%d<<<1, 32>>>(out, 1.0f); cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("N=%%6d instr (%%4d KB): %%s %%9.0f cycles = %%6.2f cycles/instr\\n", %d, %d, rep < 2 ? "after L2 flush" : "warm rerun    ", h[0], h[0] / %d);
  }""" % (n, n, n * 16 // 1024, n))
src.append('  printf("%s\\n", cudaGetErrorString(cudaDeviceSynchronize()));\n  return 0;\n}')
open(sys.argv[1], "w").write("\n".join(src))
