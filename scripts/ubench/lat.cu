// Latency micro-benchmarks for the K3 design (B200): cluster barrier, DSMEM load, L2 load,
// fp64 div / sqrt / rsqrt chains, __syncthreads with 512 threads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ long long clk() { return clock64(); }

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(512) k_cluster(double* out, const double* g, int iters) {
  __shared__ double sm[4096];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 4096; i += 512) sm[i] = i * 1.0;
  cl.sync();
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clk();
  // DSMEM dependent chain
  double* rem = cl.map_shared_rank(sm, (cl.block_rank() + 1) % 16);
  int idx = threadIdx.x;
  double acc = 0;
  long long t2 = clk();
  for (int i = 0; i < iters; ++i) { double v = rem[idx & 4095]; idx = (int)v + 1; acc += v; }
  long long t3 = clk();
  // L2 dependent chain
  int gi = threadIdx.x;
  long long t4 = clk();
  for (int i = 0; i < iters; ++i) { double v = __ldcg(g + (gi & 1048575)); gi = (int)v + 33; acc += v; }
  long long t5 = clk();
  // fp64 div chain
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t6 = clk();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);
  long long t7 = clk();
  double y = 2.0 + threadIdx.x;
  long long t8 = clk();
  for (int i = 0; i < iters; ++i) y = sqrt(y + 1.0);
  long long t9 = clk();
  double z = 2.0 + threadIdx.x;
  long long t10 = clk();
  for (int i = 0; i < iters; ++i) z = rsqrt(z + 1.0);
  long long t11 = clk();
  long long t12 = clk();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t13 = clk();
  double f = 1.0 + threadIdx.x;
  long long t14 = clk();
  for (int i = 0; i < iters; ++i) f = fma(f, 1.0000001, 0.5);
  long long t15 = clk();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[0] = (double)(t1 - t0) / iters; out[1] = (double)(t3 - t2) / iters; out[2] = (double)(t5 - t4) / iters;
    out[3] = (double)(t7 - t6) / iters; out[4] = (double)(t9 - t8) / iters; out[5] = (double)(t11 - t10) / iters;
    out[6] = (double)(t13 - t12) / iters; out[7] = (double)(t15 - t14) / iters;
    out[8] = acc + x + y + z + f;
  }
}

int main() {
  double *out, *g;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&g, (1 << 20) * 8 + 64 * 8);
  cudaMemset(g, 0, (1 << 20) * 8);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 2; ++rep) {
    k_cluster<<<16, 512>>>(out, g, 200);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  }
  double h[9];
  cudaMemcpy(h, out, 9 * 8, cudaMemcpyDeviceToHost);
  printf("cycles: cluster.sync %.0f | DSMEM load chain %.0f | L2 load chain %.0f | fp64 div %.0f | sqrt %.0f | rsqrt %.0f | syncthreads(512) %.0f | dfma chain %.0f\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  return 0;
}
