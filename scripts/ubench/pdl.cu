// Does a programmatic dependent launch overlap a cluster-launched primary that triggers at
// its first instruction?  (stream and graph-capture variants)
#include <cstdio>
#include <cuda_runtime.h>
__device__ void spin(long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}
__global__ void primary(int trig, long long ns) {
  if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ char sm[];
  sm[threadIdx.x] = 0;
  spin(ns);
}
__global__ void secondary(long long ns) { spin(ns); }
int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t psm = 150 * 1024;
  cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
  cudaFuncSetAttribute(primary, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 8; ++mode) {
    const int trig = mode & 1, cl = (mode >> 1) & 1 ? 16 : 1, graph = mode >= 4;
    auto enq = [&]() {
      cudaLaunchConfig_t c = {}; c.gridDim = dim3(16); c.blockDim = dim3(512); c.dynamicSmemBytes = psm; c.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      c.attrs = at; c.numAttrs = 1;
      cudaLaunchKernelEx(&c, primary, trig, 50000LL);
      cudaLaunchConfig_t d = {}; d.gridDim = dim3(400); d.blockDim = dim3(256); d.stream = st;
      cudaLaunchAttribute bt[1]; bt[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      bt[0].val.programmaticStreamSerializationAllowed = 1;
      d.attrs = bt; d.numAttrs = 1;
      cudaLaunchKernelEx(&d, secondary, 40000LL);
    };
    cudaGraphExec_t ge = nullptr;
    if (graph) {
      cudaGraph_t g;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      enq();
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
    }
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a, st);
      if (graph) cudaGraphLaunch(ge, st); else enq();
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("trig=%d cluster=%d graph=%d: %.1f us (serial ~90, overlapped ~50) %s\n", trig, cl, graph, ms * 1e3,
                           cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
