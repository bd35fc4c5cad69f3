// small_step.cu -- dispatch of the K3 cluster kernel (templates in small_step.cuh, one
// translation unit per eigen-block width BT so the build parallelises).
#include "small_step.cuh"

namespace wlr {

extern template cudaError_t launch_ss<4>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<4>(int, size_t);
extern template cudaError_t launch_ss<8>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<8>(int, size_t);
extern template cudaError_t launch_ss<12>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<12>(int, size_t);
extern template cudaError_t launch_ss<16>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<16>(int, size_t);
extern template cudaError_t launch_ss<24>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<24>(int, size_t);
extern template cudaError_t launch_ss<32>(const SmallArgs&, int, size_t, int, cudaStream_t);
extern template int ss_max_clusters<32>(int, size_t);

// exchange-slot payload (doubles) large enough for every round
int64_t small_step_xchg_stride(int k, int nk, int t, int b) {
  int64_t fin = 5 + 7LL * k * t + 4LL * t * t + (int64_t)k * k + 8;
  int64_t prod = (int64_t)k * b;
  int64_t gram = (int64_t)b * b + b;
  int64_t s = std::max(fin, std::max(prod, gram));
  return round_up(s, 32);
}

static int bt_of(int b) { return b <= 4 ? 4 : b <= 8 ? 8 : b <= 12 ? 12 : b <= 16 ? 16 : b <= 24 ? 24 : 32; }
int small_step_bt(int b) { return bt_of(b); }

static int max_clusters(int bt, int CL, size_t smem) {
  switch (bt) {
    case 4: return ss_max_clusters<4>(CL, smem);
    case 8: return ss_max_clusters<8>(CL, smem);
    case 12: return ss_max_clusters<12>(CL, smem);
    case 16: return ss_max_clusters<16>(CL, smem);
    case 24: return ss_max_clusters<24>(CL, smem);
    default: return ss_max_clusters<32>(CL, smem);
  }
}

// Choose the cluster size (largest of 16, 8, 4, 2, 1 the device can co-schedule) and
// whether G_A rows fit in shared memory.
int small_step_cluster_size(const SmallArgs& a, size_t* smem_out, int* flags_out) {
  const int bt = bt_of(a.b);
  const int want = (int)std::max<int64_t>(1, std::min<int64_t>(16, ceil_div(a.nk, 24)));
  for (int CL = 16; CL >= 1; CL /= 2) {
    if (CL > want && CL > 1) continue;
    for (int fl = 3; fl >= 0; --fl) {
      const size_t smem = ss_smem_bytes(a, CL, fl);
      if (smem > 220 * 1024) continue;
      if (max_clusters(bt, CL, smem) >= 1) {
        *smem_out = smem;
        *flags_out = fl;
        return CL;
      }
    }
  }
  return 0;
}

cudaError_t launch_small_step(const SmallArgs& a, int CL, size_t smem, int fl, cudaStream_t st) {
  switch (bt_of(a.b)) {
    case 4: return launch_ss<4>(a, CL, smem, fl, st);
    case 8: return launch_ss<8>(a, CL, smem, fl, st);
    case 12: return launch_ss<12>(a, CL, smem, fl, st);
    case 16: return launch_ss<16>(a, CL, smem, fl, st);
    case 24: return launch_ss<24>(a, CL, smem, fl, st);
    default: return launch_ss<32>(a, CL, smem, fl, st);
  }
}

}  // namespace wlr
