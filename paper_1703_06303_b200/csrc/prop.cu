// prop.cu -- Gram propagation for the LINEAR X1 half-step (uniform W1).
//
// With uniform W1 every row of the X1 half-step (Algorithm 1 lines 7-9) is the
// same linear map of z = [A(i,:) | X1_p(i,:)]:  X1_{p+1} = A W'_A + X1_p W'_X  (W' built by K3).
// The small step only needs Grams of X1_{p+1}, and those follow EXACTLY from the n x n Gram
// A^T A (fp64, computed once at init) and the running Q_p = A^T X1_p, G_p = X1_p^T X1_p:
//     Q_{p+1} = A^T A W'_A + Q_p W'_X                          (n x k)
//     H       = X1_{p+1}^T X1_p = W'_A^T Q_p + W'_X^T G_p       (k x k)
//     G_{p+1} = Q_{p+1}^T W'_A + H W'_X                         (k x k)
//     M_{p+1} = X1_{p+1}^T A2 = Q_{p+1}(k:n, :)^T
// They are written in the packed increment format the small step consumes
// [N = M_{p+1} - M_p | Gamma = H - G_p | Omega = G_{p+1} - H - H^T + G_p | (f_w)], so K3 is
// unchanged and no pass over the m rows is on its path (the row pass materialises X1_{p+1}
// beside it and supplies f_w = sum W1^2 (A1 - X1_{p+1})^2 from the stored rows: the closed form
// w^2 (||A1||^2 - 2 tr Q + tr G) cancels to ~1e-16 ||A1||^2 / ||A1 - X1||^2, too coarse in fp64 mode).
// W' is read in the storage dtype the row pass uses (fp32 in fp32 mode), upcast exactly.
//
// prop1: CTA b of nb = min(n, #SMs) owns RB = ceil(n / nb) (or RB - 1) consecutive rows of the n
//        index: Q_{p+1} rows (A^T A rows and all of W' staged in shared memory), N columns, the
//        per-block partials Hp[b] = W'_A(rows)^T Q_p(rows), Gp[b] = Q_{p+1}(rows)^T W'_A(rows)
//        (k x k each), and G_A Y of the warm Ritz block for the small step's first S-product.
// prop2: CTA a sums row a (and column a) of the partials in block order and adds the k x k terms:
//        row a of H, of H^T, of G_{p+1}; writes row a of Gamma and Omega.
// fp64 throughout; every sum has a fixed order (replicas and reruns bitwise identical).
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace wlr {

constexpr int kPropT = 256;        // prop2 threads
constexpr int kPropT1 = 512;       // prop1 threads (16 warps: one CTA per SM)
constexpr int kPropRBmax = 8;      // max n-index rows per prop1 CTA (the grid is min(n, #SMs) CTAs)

template <typename T>
WLR_DEVI double wld(const void* W, int64_t i) { return (double)reinterpret_cast<const T*>(W)[i]; }

WLR_DEVI void pstamp(const PropArgs& a, int i, int base = 0) {   // (diagnostics: wlr_debug_state "proptime")
  if (a.ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.ts[(base + blockIdx.x) * 8 + i] = t;
  }
}

// rows of prop1 CTA b of nb: n = nb * base + ext, the first ext CTAs take base + 1 rows
WLR_DEVI void prop1_rows(int n, int nb, int b, int& i0, int& nr) {
  const int base = n / nb, ext = n - base * nb;
  i0 = b * base + min(b, ext);
  nr = base + (b < ext ? 1 : 0);
}
// Q column blocks of 4, rounded up to a power of 2 (lanes of one column block are reduced by shuffles)
__host__ __device__ inline int prop1_ncbp(int k) {
  const int ncb = (k + 3) / 4;
  int p = 1;
  while (p < ncb) p *= 2;
  return p;
}
// G_A Y in prop1: thread (output o = (row, column), lane g of tpo threads per output) sums
// l = g, g + tpo, ... < n - k
__host__ __device__ inline int prop1_gay_tpo(int nout) {
  int t = kPropT1 / (nout > 0 ? nout : 1);
  return t >= 32 ? 32 : t >= 16 ? 16 : t >= 8 ? 8 : t >= 4 ? 4 : t >= 2 ? 2 : 1;
}
int prop1_rb(int n, int nsm) { return (n + std::min(n, nsm) - 1) / std::min(n, nsm); }

// shared layout of prop1 (RB rows): A^T A rows (RB x n doubles; reused for the j-group reduction,
// 16 warps x RB x 4 ncbp doubles, once the rows are consumed) | Q_p, Q_{p+1} rows (RB x k each) |
// Y ((n - k) x b doubles, when G_A Y is computed here) | W'_A rows 0..n-1 and W'_X rows (k), RP
// elements each in the storage dtype, bulk-copied (fp32: RP = 32 for k <= 32, so W' is 80 KB at
// config 3) | mbarriers
static size_t prop1_wbytes(int n, int k, int RP, int es) { return (size_t)(n + k) * RP * es; }
__host__ __device__ inline int prop1_even(int x) { return (x + 1) & ~1; }   // (16-byte region starts)
__host__ __device__ inline int prop1_rows_doubles(int n, int k, int rb) {
  return prop1_even(rb * (n > (kPropT1 / 32) * 4 * prop1_ncbp(k) ? n : (kPropT1 / 32) * 4 * prop1_ncbp(k)));
}
size_t prop1_smem(int n, int k, int RP, int es, int rb, int ys) {
  return sizeof(double) * ((size_t)prop1_rows_doubles(n, k, rb) + prop1_even(2 * rb * k) + prop1_even(ys)) +
         prop1_wbytes(n, k, RP, es) + 32;
}
// with G_A Y (the warm block Y, (n - k) x b doubles, staged in shared memory) when it fits
size_t prop1_smem(int n, int k, int nsm, int b) {
  const int RP = (k + 31) / 32 * 32, rb = prop1_rb(n, nsm);
  const size_t with = prop1_smem(n, k, RP, 4, rb, (n - k) * b);
  return with <= 227 * 1024 ? with : prop1_smem(n, k, RP, 4, rb, 0);
}
bool prop_gay_ok(int n, int k, int b, int nsm) {
  const int RP = (k + 31) / 32 * 32, rb = prop1_rb(n, nsm);
  return b >= 1 && rb * b <= kPropT1 && prop1_smem(n, k, RP, 4, rb, (n - k) * b) <= 227 * 1024;
}

// prop1: CTA b owns RB (or RB - 1) consecutive rows i0.. of the n index (FP64 CUDA cores; the
// m8n8k4 DMMA chain measured 3x slower for these shapes, profiles/r02_prop_dmma.log):
//   G_A Y rows (the small step's first S-product operand; needs only the A^T A rows, so it runs
//   while W' is still in flight), Q_{p+1} rows = [A^T A rows | Q_p rows] . [W'_A ; W'_X], N columns,
//   and the per-block partials Hp = W'_A(rows)^T Q_p(rows), Gp = Q_{p+1}(rows)^T W'_A(rows).
template <typename T, int RB>
__global__ void __launch_bounds__(kPropT1, 1) prop1_kernel(const __grid_constant__ PropArgs a) {
  if (a.stop && *a.stop) return;               // (eps mode: converged before this iteration)
  pstamp(a, 0);
  extern __shared__ __align__(16) double pr_sm[];
  const int n = a.n, k = a.k, nk = n - k, RP = a.RP, kk = k * k;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int b = blockIdx.x;
  int i0, nr;
  prop1_rows(n, a.nb, b, i0, nr);
  const int ncbp = prop1_ncbp(k), ncb = (k + 3) / 4;
  double* rows = pr_sm;                                  // nr x n rows of A^T A (then the reduction)
  double* Qps = rows + prop1_rows_doubles(n, k, RB);     // RB x k  Q_p rows
  double* Qns = Qps + RB * k;                            // RB x k  Q_{p+1} rows
  double* Ys = Qps + prop1_even(2 * RB * k);             // (n - k) x b  Y (G_A Y only)
  T* Wr = reinterpret_cast<T*>(Ys + prop1_even(a.GAY ? nk * a.b : 0));   // (n + k) x RP  [W'_A ; W'_X], storage dtype
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(Wr) + (size_t)(n + k) * RP * sizeof(T));
  const uint32_t wa_bytes = (uint32_t)((size_t)n * RP * sizeof(T)), wx_bytes = (uint32_t)((size_t)k * RP * sizeof(T));
  // G_A Y for the small step's first S-product (Y = the warm Ritz block K3a(p-1) left, complete
  // before this kernel starts; G_A = the A2 block of A^T A, whose rows this CTA stages): rows i >= k
  // of the block, (n-k) x b.  Y is staged in shared memory now (coalesced, rounds of 8 loads in
  // flight); the sums run while W' is still in flight.
  const int gbw = a.b, gnout = a.GAY ? nr * gbw : 0, gtpo = prop1_gay_tpo(gnout);
  if (gnout > 0) {
    const int ny = nk * gbw;
    for (int r0 = 0; r0 < ny; r0 += 8 * kPropT1) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int idx = r0 + u * kPropT1 + tid; v[u] = idx < ny ? a.Y[idx] : 0.0; }
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int idx = r0 + u * kPropT1 + tid; if (idx < ny) Ys[idx] = v[u]; }
    }
  }
  const bool bulk_rows = ((size_t)n * 8) % 16 == 0 && ((size_t)i0 * n * 8) % 16 == 0;   // 16-byte aligned
  // two barriers, each used for ONE phase: a parity wait on a barrier that has since moved two
  // phases on (rows, then W') would wait for a phase that never completes
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init_fence();
    if (bulk_rows) {                                     // (init data: before the dependency wait)
      mbar_expect_tx(bar + 1, (uint32_t)(nr * n * 8));
      bulk_load_1d(rows, a.AtA + (int64_t)i0 * n, (uint32_t)(nr * n * 8), bar + 1);
    }
  }
  if (!bulk_rows) {
    for (int r0 = 0; r0 < nr * n; r0 += 8 * kPropT1) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = r0 + u * kPropT1 + tid;
        v[u] = idx < nr * n ? a.AtA[(int64_t)i0 * n + idx] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = r0 + u * kPropT1 + tid;
        if (idx < nr * n) rows[idx] = v[u];
      }
    }
  }
  __syncthreads();
  pstamp(a, 1);
  pdl_wait();                                            // W' (K3) and Q_p (previous prop)
  pstamp(a, 2);
  if (tid == 0) {                                        // W' rows by two bulk copies
    mbar_expect_tx(bar, wa_bytes + wx_bytes);
    bulk_load_1d(Wr, a.Wt, wa_bytes, bar);
    bulk_load_1d(Wr + (size_t)n * RP, reinterpret_cast<const T*>(a.Wt) + (size_t)a.KA * RP, wx_bytes, bar);
  }
  for (int idx = tid; idx < RB * k; idx += kPropT1) Qps[idx] = idx < nr * k ? a.Qp[(int64_t)i0 * k + idx] : 0.0;
  if (w == 15) {   // the small step (K3a) that follows reads these: pull them into L2 now (the
    for (int r = 0; r < kPf; ++r) {              // bench flushes L2 before every iteration)
      const char* base = reinterpret_cast<const char*>(a.pf_ptr[r]);
      const int64_t nbt = a.pf_bytes[r] & ~(int64_t)15;
      if (!base || nbt <= 0) continue;
      const int64_t chunk = 8192, nchunk = (nbt + chunk - 1) / chunk;   // spread over all CTAs
#pragma unroll 1
      for (int64_t c = blockIdx.x + (int64_t)gridDim.x * lane; c < nchunk; c += (int64_t)gridDim.x * 32) {
        const int64_t off = c * chunk;
        const unsigned sz = (unsigned)(nbt - off < chunk ? nbt - off : chunk);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base + off), "r"(sz) : "memory");
      }
    }
  }
  if (bulk_rows) mbar_wait(bar + 1, 0);                  // the A^T A rows
  if (gnout > 0) {
    for (int o0 = 0; o0 < gnout; o0 += kPropT1 / gtpo) {
      const int o = o0 + tid / gtpo, g = tid % gtpo, r = o / gbw, j = o - r * gbw;
      const bool valid = o < gnout && i0 + r >= k;
      double v4[4] = {0.0, 0.0, 0.0, 0.0};
      if (valid) {
        const double* ar = rows + r * n + k;
        int l = g;
        for (; l + 3 * gtpo < nk; l += 4 * gtpo) {
#pragma unroll
          for (int q = 0; q < 4; ++q) v4[q] = fma(ar[l + q * gtpo], Ys[(l + q * gtpo) * gbw + j], v4[q]);
        }
        for (; l < nk; l += gtpo) v4[0] = fma(ar[l], Ys[l * gbw + j], v4[0]);
      }
      double v = (v4[0] + v4[1]) + (v4[2] + v4[3]);
      for (int sft = gtpo >> 1; sft > 0; sft >>= 1) v += __shfl_xor_sync(0xffffffffu, v, sft);
      if (g == 0 && valid) a.GAY[(int64_t)(i0 + r - k) * gbw + j] = v;
    }
  }
  pstamp(a, 3);
  mbar_wait(bar, 0);                                     // W'
  __syncthreads();
  pstamp(a, 4);
  // Q_{p+1} rows: thread = (column block cb of 4 columns, j group jg); RB rows x 4 columns of
  // accumulators.  The j groups split the combined sum over [A^T A rows | Q_p rows] . [W'_A ; W'_X]
  // (n + k terms) evenly; they are summed in a fixed order: within a warp by shuffles (the lanes
  // of one column block), then over the 16 warps through shared memory (in the rows' place).
  {
    const int njg = kPropT1 / ncbp;                      // (ncbp <= 32: 16 or more j groups)
    const int cb = tid % ncbp, jg = tid / ncbp;
    double acc[RB][4];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    if (cb < ncb) {
      const int nj = n + k;
      const int jlo = (int)((int64_t)nj * jg / njg), jhi = (int)((int64_t)nj * (jg + 1) / njg);
      const int jae = min(jhi, n);
#pragma unroll 2
      for (int j = jlo; j < jae; ++j) {
        double wv[4];
        const float4 w4 = *reinterpret_cast<const float4*>(Wr + (int64_t)j * RP + 4 * cb);
        wv[0] = w4.x; wv[1] = w4.y; wv[2] = w4.z; wv[3] = w4.w;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const double av = rows[r * n + j];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fma(av, wv[c], acc[r][c]);
        }
      }
      for (int j = max(jlo, n); j < jhi; ++j) {          // + Q_p W'_X (rows n.. of W')
        const int q = j - n;
        double wv[4];
        const float4 w4 = *reinterpret_cast<const float4*>(Wr + (int64_t)j * RP + 4 * cb);
        wv[0] = w4.x; wv[1] = w4.y; wv[2] = w4.z; wv[3] = w4.w;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const double qv = Qps[r * k + q];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fma(qv, wv[c], acc[r][c]);
        }
      }
    }
    for (int sft = ncbp; sft < 32; sft *= 2)
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], sft);
    const int w4n = 4 * ncbp, nsl = kPropT1 / 32;
    __syncthreads();                                     // (every warp is done with the rows)
    double* red = rows;                                  // [warp][r][4 ncbp]
    if (lane < ncbp)
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[((int64_t)w * RB + r) * w4n + 4 * cb + c] = acc[r][c];
    __syncthreads();
    for (int o = tid; o < RB * k; o += kPropT1) {
      const int r = o / k, ll = o - r * k;
      double v = 0.0;
      for (int g = 0; g < nsl; ++g) v += red[((int64_t)g * RB + r) * w4n + ll];
      Qns[o] = v;
      if (r < nr) {
        const int i = i0 + r;
        a.Qn[(int64_t)i * k + ll] = v;
        if (i >= k) a.inc[(int64_t)ll * nk + (i - k)] = v - Qps[o];   // N = M_{p+1} - M_p
      }
    }
    __syncthreads();
  }
  pstamp(a, 5);
  // per-block partials of H and of Q_{p+1}^T W'_A over the block's rows, stored for prop2's CTA a
  // as three contiguous [nb][k] panels: row a of Hp, column a of Hp, row a of Gp
  const int nb = a.nb;
#define Ws(j, l) ((double)Wr[(int64_t)(j) * RP + (l)])
  for (int idx = tid; idx < kk; idx += kPropT1) {
    const int ar = idx / k, l = idx - ar * k;
    double h = 0.0, g = 0.0;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < nr) {
        h = fma(Ws(i0 + r, ar), Qps[r * k + l], h);
        g = fma(Qns[r * k + ar], Ws(i0 + r, l), g);
      }
    }
    a.part[(((int64_t)ar * 3 + 0) * nb + b) * k + l] = h;     // H row ar
    a.part[(((int64_t)l * 3 + 1) * nb + b) * k + ar] = h;     // H column l (entry ar)
    a.part[(((int64_t)ar * 3 + 2) * nb + b) * k + l] = g;     // Gp row ar
  }
#undef Ws
  pstamp(a, 6);
  pdl_trigger();
}

// prop2: CTA a (of k) finishes row a: 15 warps sum the three [nb][k] partial panels of row a (row a
// of Hp, column a of Hp, row a of Gp; 5 warps per panel over the block range, one round of loads),
// then the k x k terms: row a of H, of H^T and of G_{p+1}; writes row a of Gamma and Omega.
constexpr int kPropT2 = 512;
constexpr int kP2Sub = 5;                      // warps per panel
template <typename T>
__global__ void __launch_bounds__(kPropT2) prop2_kernel(const __grid_constant__ PropArgs a) {
  if (a.stop && *a.stop) return;
  pstamp(a, 0, a.nb);
  __shared__ double hrow[128], hcol[128], grow[128];
  extern __shared__ __align__(16) double p2_sm[];
  const int n = a.n, k = a.k, nk = n - k, RP = a.RP, kk = k * k;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int ar = blockIdx.x;
  const int nb = a.nb;
  double* Wx = p2_sm;                                      // k x k   W'_X
  double* Gs = Wx + kk;                                    // k x k   G_p
  double* wred = Gs + kk;                                  // 3 x kP2Sub x k  panel partial sums
  for (int r0 = 0; r0 < kk; r0 += 2 * kPropT2) {          // (G_p, W': not written by prop1)
    double v[2], x[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = r0 + u * kPropT2 + tid, q = idx / k;
      v[u] = idx < kk ? a.Gp[idx] : 0.0;
      x[u] = idx < kk ? wld<T>(a.Wt, (int64_t)(a.KA + q) * RP + (idx - q * k)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = r0 + u * kPropT2 + tid;
      if (idx < kk) { Gs[idx] = v[u]; Wx[idx] = x[u]; }
    }
  }
  pstamp(a, 1, a.nb);
  pdl_wait();
  pstamp(a, 2, a.nb);
  if (w < 3 * kP2Sub) {
    const int pn = w / kP2Sub, sub = w - pn * kP2Sub;
    const int b0 = (int)((int64_t)nb * sub / kP2Sub), b1 = (int)((int64_t)nb * (sub + 1) / kP2Sub);
    const double* P = a.part + ((int64_t)ar * 3 + pn) * nb * k;
    for (int c0 = 0; c0 < k; c0 += 32) {
      const int c = c0 + lane;
      double v = 0.0;
      if (c < k) {
        for (int bb = b0; bb < b1; bb += 32) {           // (nb <= 160: one round)
          double x[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) x[u] = bb + u < b1 ? __ldcg(P + (int64_t)(bb + u) * k + c) : 0.0;
#pragma unroll
          for (int u = 0; u < 32; ++u) v += x[u];
        }
        wred[(pn * kP2Sub + sub) * k + c] = v;
      }
    }
  }
  __syncthreads();
  pstamp(a, 3, a.nb);
  for (int o = tid; o < 3 * k; o += kPropT2) {             // fixed-order sums over the sub-ranges
    const int pn = o / k, c = o - pn * k;
    double v = 0.0;
    for (int sub = 0; sub < kP2Sub; ++sub) v += wred[(pn * kP2Sub + sub) * k + c];
    (pn == 0 ? hrow : pn == 1 ? hcol : grow)[c] = v;
  }
  __syncthreads();
  pstamp(a, 4, a.nb);
  // + W'_X^T G_p terms of H (row a) and H^T (column a): 8 lanes per output, q split, shuffle sum
  for (int o0 = 0; o0 < 2 * k; o0 += kPropT2 / 8) {
    const int o = o0 + tid / 8, g = tid & 7;
    const int c = o < k ? o : o - k;
    double v = 0.0;
    if (o < 2 * k) {
      if (o < k) for (int q = g; q < k; q += 8) v = fma(Wx[q * k + ar], Gs[q * k + c], v);
      else       for (int q = g; q < k; q += 8) v = fma(Wx[q * k + c], Gs[q * k + ar], v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    if (o < 2 * k && g == 0) (o < k ? hrow : hcol)[c] += v;
  }
  __syncthreads();
  pstamp(a, 5, a.nb);
  double* gam = a.inc + (int64_t)k * nk;
  double* om = gam + (int64_t)kk;
  for (int c0 = 0; c0 < k; c0 += kPropT2 / 8) {
    const int c = c0 + tid / 8, g = tid & 7;
    double v = 0.0;                                        // (H W'_X)[a][c]
    if (c < k)
      for (int q = g; q < k; q += 8) v = fma(hrow[q], Wx[q * k + c], v);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    if (c < k && g == 0) {
      const double gv = grow[c] + v;                       // G_{p+1}[a][c]
      const double gp = Gs[ar * k + c];
      gam[ar * k + c] = hrow[c] - gp;
      om[ar * k + c] = gv - hrow[c] - hcol[c] + gp;
      if (c == ar) a.dg[ar] = gv - 2.0 * a.Qn[(int64_t)ar * k + ar];   // f_w's diagonal terms
    }
  }
  // (f_w = w^2 (||A1||^2 + sum_a dg[a]) is summed by the small step's CTA 0, which runs next)
  pdl_trigger();
  pstamp(a, 6, a.nb);
}

cudaError_t launch_prop(const PropArgs& a, bool f64, int pdl, cudaStream_t st, cudaEvent_t after1) {
  if (f64) return cudaErrorNotSupported;       // (Gram propagation is the fp32 path, api.cu)
  const int rb = (a.n + a.nb - 1) / a.nb;
  if (rb < 1 || rb > kPropRBmax) return cudaErrorInvalidValue;
  const size_t sm1 = prop1_smem(a.n, a.k, a.RP, 4, rb, a.GAY ? (a.n - a.k) * a.b : 0);
  const size_t sm2 = sizeof(double) * (2 * (size_t)a.k * a.k + 3 * kP2Sub * (size_t)a.k);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cudaLaunchConfig_t c1{};
  c1.gridDim = dim3(a.nb);
  c1.blockDim = dim3(kPropT1);
  c1.dynamicSmemBytes = sm1;
  c1.stream = st;
  c1.attrs = at;
  c1.numAttrs = 1;
  cudaError_t e;
  auto go1 = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    return cudaLaunchKernelEx(&c1, kern, a);
  };
  switch (rb) {
    case 1: e = go1(prop1_kernel<float, 1>); break;
    case 2: e = go1(prop1_kernel<float, 2>); break;
    case 3: e = go1(prop1_kernel<float, 3>); break;
    case 4: e = go1(prop1_kernel<float, 4>); break;
    case 5: e = go1(prop1_kernel<float, 5>); break;
    case 6: e = go1(prop1_kernel<float, 6>); break;
    case 7: e = go1(prop1_kernel<float, 7>); break;
    default: e = go1(prop1_kernel<float, 8>); break;
  }
  if (e != cudaSuccess) return e;
  if (after1 && (e = cudaEventRecord(after1, st)) != cudaSuccess) return e;   // (prop1 done)
  cudaLaunchAttribute at2[1];
  at2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at2[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t c2{};
  c2.gridDim = dim3(a.k);
  c2.blockDim = dim3(kPropT2);
  c2.dynamicSmemBytes = sm2;
  c2.stream = st;
  c2.attrs = at2;
  c2.numAttrs = 1;
  cudaFuncSetAttribute(prop2_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  return cudaLaunchKernelEx(&c2, prop2_kernel<float>, a);
}

__global__ void stop_latch_kernel(int* flags) { flags[6] = flags[2]; }

__global__ void noop_kernel() {}
cudaError_t launch_noop(cudaStream_t st) {
  noop_kernel<<<1, 32, 0, st>>>();
  return cudaGetLastError();
}

cudaError_t launch_stop_latch(int* flags, cudaStream_t st) {
  stop_latch_kernel<<<1, 1, 0, st>>>(flags);
  return cudaGetLastError();
}

__global__ void vsum_kernel(double* __restrict__ out, const double* __restrict__ in, int G, size_t stride, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += in[(size_t)g * stride + i];
    out[i] = s;
  }
}

cudaError_t launch_vsum(double* out, const double* in, int G, size_t stride, size_t count, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>(1024, (count + 255) / 256);
  vsum_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(out, in, G, stride, count);
  return cudaGetLastError();
}

size_t prop_part_doubles(int nb, int k) { return (size_t)nb * 3 * k * k; }

}  // namespace wlr
