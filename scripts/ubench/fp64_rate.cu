// Per-SM throughput of DFMA, F2F.F64.F32 and FFMA on sm_100a: one CTA of W warps, 8 independent
// chains per thread, clock64 around the loop; prints ops/clk/SM.
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(double* out, float* outf, int iters, long long* cyc) {
  double d[8]; float f[8];
  for (int i = 0; i < 8; ++i) { d[i] = threadIdx.x * 1e-3 + i; f[i] = (float)d[i]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) d[i] = fma(d[i], 0.999999, 1e-7);
      else if (KIND == 1) { d[i] += (double)f[i]; f[i] = f[i] * 1.0000001f; }
      else f[i] = fmaf(f[i], 0.999999f, 1e-7f);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; float sf = 0;
  for (int i = 0; i < 8; ++i) { s += d[i]; sf += f[i]; }
  out[threadIdx.x] = s; outf[threadIdx.x] = sf;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; float* of; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&of, 8192); cudaMalloc(&c, 8);
  const int iters = 4096;
  for (int W : {4, 8, 16, 32}) {
    long long h;
    k<0><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    k<0><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double dfma = 32.0 * W * iters * 8 / h;
    k<1><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    k<1><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double cvt = 32.0 * W * iters * 8 / h;   // (one F2F + one DADD + one FMUL per element)
    k<2><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    k<2><<<1, 32 * W>>>(o, of, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double ffma = 32.0 * W * iters * 8 / h;
    printf("warps %2d: DFMA %.1f /clk/SM, (F2F.F64.F32 + DADD + FMUL) %.1f /clk/SM, FFMA %.1f /clk/SM\n", W, dfma, cvt, ffma);
  }
  return 0;
}
