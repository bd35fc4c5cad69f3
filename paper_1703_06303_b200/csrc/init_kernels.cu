// init_kernels.cu -- one-time kernels of wlr_init:
//   * gram64: fp64 Gram L^T R over rows, used for A^T A at init.  With X1_0 = A1 this
//     yields G_0 = A1^T A1, M_0 = A1^T A2 and G_A = A2^T A2 at once.  Inputs are fp32
//     or fp64; products are formed in fp64, so fp32 inputs give exact products and the
//     incremental Grams of the row pass add onto exact bases.
//   * X1 buffer initialisation (X1_0 = A1 for the GHS start, PAPER.md:203 / R5, or a
//     caller-supplied X1_0) and the initial weighted residual f_w(X1_0).
#include "kernels.h"

namespace wlr {

// Tile: 64 x 64 outputs per CTA, 256 threads (4 x 4 each), rows staged 16 at a time.
template <typename T>
__global__ void __launch_bounds__(256) gram64_kernel(const T* __restrict__ L, int64_t ldl, int nl,
                                                     const T* __restrict__ R, int64_t ldr, int nr,
                                                     int64_t m, int64_t rows_per_split,
                                                     double* __restrict__ part, int sym) {
  // sym (L == R): only the tiles on or above the diagonal; sum_splits mirrors the rest
  if (sym && blockIdx.x > blockIdx.y) return;
  __shared__ double Ls[16][64];
  __shared__ double Rs[16][64];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int i0 = blockIdx.x * 64, j0 = blockIdx.y * 64;
  const int64_t rb0 = (int64_t)blockIdx.z * rows_per_split;
  const int64_t re = rb0 + rows_per_split < m ? rb0 + rows_per_split : m;
  double acc[4][4] = {};
  // the next 16 rows' operands are loaded into registers while this step computes (software
  // pipelined: the step's global-load latency was exposed once per 16 rows)
  T lv[4], rv[4];
  auto fetch = [&](int64_t rb) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = threadIdx.x + e * 256;
      const int rr = idx / 64, cc = idx % 64;
      const int64_t row = rb + rr;
      const bool ok = row < re;
      lv[e] = (ok && i0 + cc < nl) ? L[row * ldl + i0 + cc] : T(0);
      rv[e] = (ok && j0 + cc < nr) ? R[row * ldr + j0 + cc] : T(0);
    }
  };
  if (rb0 < re) fetch(rb0);
  for (int64_t rb = rb0; rb < re; rb += 16) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = threadIdx.x + e * 256;
      Ls[idx / 64][idx % 64] = (double)lv[e];
      Rs[idx / 64][idx % 64] = (double)rv[e];
    }
    __syncthreads();
    if (rb + 16 < re) fetch(rb + 16);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Ls[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Rs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = part + (int64_t)blockIdx.z * nl * nr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = i0 + ty * 4 + i;
    if (gi >= nl) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = j0 + tx * 4 + j;
      if (gj < nr) out[(int64_t)gi * nr + gj] = acc[i][j];
    }
  }
}

__global__ void sum_splits_kernel(const double* __restrict__ part, int nsplit, int64_t len,
                                  double* __restrict__ out, int sym_n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t src = i;
    if (sym_n > 0) {   // square symmetric product: tiles below the diagonal read their mirror
      const int64_t r = i / sym_n, c = i - r * sym_n;
      if (r / 64 > c / 64) src = c * sym_n + r;
    }
    double s = 0.0;
    for (int p = 0; p < nsplit; ++p) s += part[(int64_t)p * len + src];   // fixed order
    out[i] = s;
  }
}

template <typename T>
void launch_gram64(const T* L, int64_t ldl, int nl, const T* R, int64_t ldr, int nr, int64_t m,
                   double* part, int nsplit, double* out, cudaStream_t st) {
  const int64_t rps = round_up(ceil_div(m, nsplit), 16);
  dim3 grid((unsigned)ceil_div(nl, 64), (unsigned)ceil_div(nr, 64), (unsigned)nsplit);
  const int sym = (L == R && ldl == ldr && nl == nr) ? 1 : 0;
  gram64_kernel<T><<<grid, 256, 0, st>>>(L, ldl, nl, R, ldr, nr, m, rps, part, sym);
  const int64_t len = (int64_t)nl * nr;
  sum_splits_kernel<<<(unsigned)std::min<int64_t>(ceil_div(len, 256), 4096), 256, 0, st>>>(
      part, nsplit, len, out, sym ? nr : 0);
}
template void launch_gram64<float>(const float*, int64_t, int, const float*, int64_t, int, int64_t,
                                   double*, int, double*, cudaStream_t);
template void launch_gram64<double>(const double*, int64_t, int, const double*, int64_t, int,
                                    int64_t, double*, int, double*, cudaStream_t);

// Zero a list of buffers (pool allocations: 256-byte aligned): every thread of the grid strides
// over each buffer in turn in 16-byte stores, the tail bytes singly
__global__ void zero_list_kernel(const __grid_constant__ ZeroList z) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < z.n; ++j) {
    const int64_t nb = z.bytes[j], n16 = nb / 16;
    int4* p = reinterpret_cast<int4*>(z.ptr[j]);
    for (int64_t i = tid; i < n16; i += nt) p[i] = make_int4(0, 0, 0, 0);
    char* c = reinterpret_cast<char*>(z.ptr[j]);
    for (int64_t i = 16 * n16 + tid; i < nb; i += nt) c[i] = 0;
  }
}
cudaError_t launch_zero_list(const ZeroList& z, cudaStream_t st) {
  if (z.n <= 0) return cudaSuccess;
  zero_list_kernel<<<1184, 256, 0, st>>>(z);
  return cudaGetLastError();
}

// X1 buffer (m x kp, zero padded) := first k columns of src (ld lds)
template <typename T>
__global__ void init_x1_kernel(const T* __restrict__ src, int64_t lds, int64_t m, int k, int kp,
                               T* __restrict__ x) {
  const int64_t tot = m * kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / kp;
    const int l = (int)(i % kp);
    x[i] = l < k ? src[row * lds + l] : T(0);
  }
}

template <typename T>
void launch_init_x1(const T* src, int64_t lds, int64_t m, int k, int kp, T* x, cudaStream_t st) {
  const int64_t tot = m * kp;
  init_x1_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(tot, 256), 8192), 256, 0, st>>>(
      src, lds, m, k, kp, x);
}
template void launch_init_x1<float>(const float*, int64_t, int64_t, int, int, float*, cudaStream_t);
template void launch_init_x1<double>(const double*, int64_t, int64_t, int, int, double*, cudaStream_t);

// f_w(X1) = sum_i sum_l W1_il^2 (A1_il - X1_il)^2  (weighted term), one
// fp64 partial per CTA (summed in fixed order later).
template <typename T>
__global__ void fw_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ W1, int64_t ldw,
                          double w2s, const T* __restrict__ x, int kp, int64_t m, int k,
                          double* __restrict__ part) {
  double s = 0.0;
  const int64_t tot = m * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / k;
    const int l = (int)(i % k);
    const double d = (double)A[row * lda + l] - (double)x[row * kp + l];
    const double w2 = W1 ? (double)W1[row * ldw + l] * (double)W1[row * ldw + l] : w2s;
    s += w2 * d * d;
  }
  s = warp_sum(s);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    part[blockIdx.x] = t;
  }
}

template <typename T>
void launch_fw(const T* A, int64_t lda, const T* W1, int64_t ldw, double w2s, const T* x, int kp,
               int64_t m, int k, double* part, int nblk, cudaStream_t st) {
  fw_kernel<T><<<nblk, 256, 0, st>>>(A, lda, W1, ldw, w2s, x, kp, m, k, part);
}
template void launch_fw<float>(const float*, int64_t, const float*, int64_t, double, const float*,
                               int, int64_t, int, double*, int, cudaStream_t);
template void launch_fw<double>(const double*, int64_t, const double*, int64_t, double,
                                const double*, int, int64_t, int, double*, int, cudaStream_t);

// W1 > 0 and finite-input validation: flags[1] |= 1 on a
// non-positive weight, flags[1] |= 2 on a non-finite A or W1 entry.
template <typename T>
__global__ void validate_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int n,
                                const T* __restrict__ W1, int64_t ldw, int k, int* flags) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = A[(i / n) * lda + (i % n)];
    if (!isfinite((double)v)) bad |= 2;
  }
  if (W1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * k;
         i += (int64_t)gridDim.x * blockDim.x) {
      const T v = W1[(i / k) * ldw + (i % k)];
      if (!isfinite((double)v)) bad |= 2;
      else if (!(v > T(0))) bad |= 1;
    }
  }
  if (bad) atomicOr(flags + 1, bad);
}

template <typename T>
void launch_validate(const T* A, int64_t lda, int64_t m, int n, const T* W1, int64_t ldw, int k,
                     int* flags, cudaStream_t st) {
  validate_kernel<T><<<1184, 256, 0, st>>>(A, lda, m, n, W1, ldw, k, flags);
}
template void launch_validate<float>(const float*, int64_t, int64_t, int, const float*, int64_t,
                                     int, int*, cudaStream_t);
template void launch_validate<double>(const double*, int64_t, int64_t, int, const double*, int64_t,
                                      int, int*, cudaStream_t);

}  // namespace wlr
