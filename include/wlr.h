/*
 * wlr.h -- C ABI of libwlr.so, the B200 (sm_100a) implementation of the per-iteration
 * sWLR update of Dutta & Li, "A Fast Algorithm for a Weighted Low Rank Approximation"
 * (arXiv 1703.06303).  Citations "PAPER.md:a-b" refer to the LaTeX source of the paper.
 *
 * Problem (Eq. (5); reparameterised as Eq. (8)):
 *     min_{X1, C, D : rank(D) <= r-k}  ||(A1 - X1) . W1||_F^2 + ||A2 - X1 C - D||_F^2
 * with A = (A1 A2) m x n split at column k, W = (W1 1), W1 > 0.
 *
 * Algorithm 1 is executed as: one (C, D) half-step at init (the
 * GHS / Theorem 1 closed form when X1_0 = A1), then per iteration one
 * X1 half-step (row formula) followed by one (C, D) half-step
 * (Theorem 2).  D is kept factored as D = B V^T (V: (n-k) x (r-k),
 * orthonormal columns; B = P^perp_{X1} A2 V, m x (r-k)).
 *
 * Conventions for every entry point:
 *   - Matrices are ROW-MAJOR with an explicit leading dimension (elements, >= #cols).
 *     Rows of A, W1, X1, B, X2 are pixels; this rank owns rows [row_offset,
 *     row_offset + m_local) of the global m x n problem.
 *   - Element type is double when opts.dtype == WLR_F64, float when WLR_F32; the
 *     (C, D) half-step always runs in fp64 internally.  C and D are returned as double.
 *   - Pointers may be host or device memory (detected with cudaPointerGetAttributes);
 *     host buffers are copied on opts.stream inside the call.
 *   - Every call returns a wlr_status; on failure wlr_last_error() describes it.  There
 *     is no silent fallback and no CPU fallback: if the GPU cannot run, calls fail.
 *   - One handle is used from one host thread at a time; distinct handles are
 *     independent.
 */
#ifndef WLR_H
#define WLR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WLR_VERSION 1

typedef struct wlr_ctx* wlr_handle;

typedef enum {
  WLR_OK = 0,
  WLR_EINVAL = 1,      /* bad argument: k<1, k>=n, r<=k (Theorem 2 needs r>k),
                          r>min(m,n), W1<=0, ld < cols, bad pointer;
                          build limits: n-k > 1024, r-k > 32                            */
  WLR_ERANK = 2,       /* X1 numerically rank deficient: Cholesky of X1^T X1 failed
                          (PAPER.md:133 assumes rank(X1)=k)                  */
  WLR_EEIG = 3,        /* top-(r-k) eigensolver exceeded its iteration budget            */
  WLR_EINTERNAL = 4,   /* a per-row system (diag(W1(i,:)^2)+CC^T) was not SPD            */
  WLR_ENONFINITE = 5,  /* non-finite input or non-finite objective                        */
  WLR_ECUDA = 6,       /* CUDA runtime error (message in wlr_last_error)                 */
  WLR_ENCCL = 7,       /* NCCL error (multi-rank only)                                   */
  WLR_ENOMEM = 8       /* device allocation failed                                        */
} wlr_status;

enum { WLR_F32 = 0, WLR_F64 = 1 };
enum { WLR_INIT_GHS = 0, WLR_INIT_GIVEN = 1 };

typedef struct {
  int32_t dtype;          /* WLR_F32 | WLR_F64: storage + row-pass precision              */
  int32_t init;           /* WLR_INIT_GHS: X1_0 = A1 (step 0 = Theorem 1)
                             WLR_INIT_GIVEN: X1_0 = x1_0 (random init PAPER.md:234; resume) */
  const void* x1_0;       /* INIT_GIVEN only: m_local x k, row-major, ld = k, dtype      */
  double w1_scalar;       /* used iff W1 == NULL: uniform weight value (> 0)             */
  double eps;             /* stopping threshold: stop when Error_p < eps or
                             Error_p/||X_p||_F < eps.  0 = run the requested count.      */
  double eig_tol;         /* eigensolver relative residual target, relative to lambda_1
                             (0 -> 1e-12 for WLR_F64, 1e-7 for WLR_F32; R17)   */
  int32_t eig_block;      /* eigensolver block width b >= r-k (0 -> r-k+2; capped at
                             min(32, n-k))                                               */
  int32_t eig_max_outer;  /* eigensolver restart budget per (C,D) step (0 -> 60; init x4)*/
  int64_t m_global;       /* total rows over all ranks (0 -> m_local)                    */
  int64_t row_offset;     /* first global row owned by this rank                          */
  int32_t nranks, rank;   /* row sharding over ranks (1, 0 for single GPU)                */
  const void* nccl_id;    /* 128-byte ncclUniqueId shared by all ranks (NULL if nranks==1;
                             with nranks==1 a one-rank communicator: tests the NCCL path)  */
  void* stream;           /* cudaStream_t for all work; NULL = a BLOCKING stream owned by
                             the handle (ordered after the legacy default stream).  With a
                             caller stream, the caller orders device inputs before wlr_init. */
  int32_t use_graph;      /* 1: replay each iteration as a captured CUDA graph (default)  */
  int32_t seed;           /* seed of the eigensolver's cold-start block (host PCG)        */
  void* vgroup;           /* wlr_vgroup (see wlr_vgroup_create) or NULL: virtual ranks      */
  int32_t check_every;    /* eps > 0: host checks the stop flag every this many iterations
                             (0 -> 8).  The stopping rule itself is applied on the device: the
                             iterations launched after the converged state do no work, so the
                             result is the converged state whatever this value              */
} wlr_opts;

/* Virtual ranks (validation hook for the row-sharded path on ONE GPU).  A group of G members:
 * member g is a handle created with opts.vgroup = group, opts.nranks = G, opts.rank = g,
 * opts.m_global / opts.row_offset of its contiguous row shard, each handle
 * driven by its own host thread (like one process per GPU).  Every sum that the NCCL path
 * all-reduces over ranks (the init Grams; per iteration, the Gram increments [N, Gamma, Omega,
 * f_w] of non-uniform W1 -- uniform W1 exchanges nothing per iteration) is formed
 * instead by a fixed-order device sum over the members' buffers, so the replicated small-step state
 * (C, V, F) must come out bitwise identical on every member.  Graph capture is disabled for
 * members.  Every member must make the same sequence of calls; a member that fails leaves the
 * others waiting (test use only).  Errors: WLR_EINVAL (G < 1), WLR_ENOMEM.                    */
typedef struct wlr_vgroup_s* wlr_vgroup;
wlr_status wlr_vgroup_create(int32_t G, wlr_vgroup* out);
void wlr_vgroup_destroy(wlr_vgroup g);

/* Fill *o with defaults (dtype F32, GHS init, eps 0, single rank, graphs on). */
void wlr_opts_default(wlr_opts* o);

/* Create a handle and run the initial (C, D) half-step.
 *   A   : m_local x n (ld lda) data matrix rows of this rank, A1 = columns [0,k).
 *         BORROWED when it is device memory: it must stay alive and unmodified until
 *         wlr_destroy.  A host A is copied into a handle-owned device buffer.
 *   W1  : m_local x k (ld ldw) weights > 0, or NULL for the uniform weight w1_scalar.
 *         Same ownership rule as A.
 * On success *h owns every iterate (X1, C, V, Grams) and the state is the canonical
 * X_0 = (X1_0, X1_0 C_0 + D_0) (reading R1).                               */
wlr_status wlr_init(wlr_handle* h, const void* A, int64_t lda, const void* W1, int64_t ldw,
                    int64_t m_local, int64_t n, int64_t k, int64_t r, const wlr_opts* o);

/* Run up to max_iters iterations (each = X1 half-step, then (C,D)
 * half-step).  Stops early when opts.eps > 0 and the stopping rule
 * holds (R3): the state is then the first one that satisfies it, and later calls
 * do not move it.  *iters_done / *converged may be NULL.  Synchronises the stream.       */
wlr_status wlr_iterate(wlr_handle h, int32_t max_iters, int32_t* iters_done, int32_t* converged);

/* Enqueue exactly n_iters iterations on the stream WITHOUT synchronising and without
 * checking convergence (benchmark / graph path).  Errors surface at the next wlr_sync. */
wlr_status wlr_iterate_async(wlr_handle h, int32_t n_iters);

/* Synchronise the handle's stream and report any device-side error flag. */
wlr_status wlr_sync(wlr_handle h);

/* Objective F_p = F(X1_p, C_p, D_p), step Error_{p-1} =
 * ||X_p - X_{p-1}||_F and relative error Error_{p-1}/||X_{p-1}||_F of
 * the latest canonical state (step = rel = -1 at p = 0).                              */
wlr_status wlr_objective(wlr_handle h, double* F, double* step_norm, double* rel_error);

/* Copy the convergence trace: out[4*i + {0,1,2,3}] = {F_p, step, rel, p} for the last
 * min(cap, n_states) canonical states in order.  *count = number written.             */
wlr_status wlr_trace(wlr_handle h, double* out, int32_t cap, int32_t* count);

/* Results of this rank (any pointer may be NULL to skip it; host or device):
 *   X1 : m_local x k   (ld ldx1)        dtype
 *   C  : k x (n-k)     (row-major)      double   (replicated on all ranks)
 *   B  : m_local x (r-k) (ld ldb)       dtype    B = P^perp_{X1} A2 V
 *   D  : (r-k) x (n-k) (row-major)      double   D = V^T, so that D_p = B D
 *   X2 : m_local x (n-k) (ld ldx2)      dtype    X2 = X1 C + B D (Algorithm 1 output)   */
wlr_status wlr_result(wlr_handle h, void* X1, int64_t ldx1, void* C, void* B, int64_t ldb,
                      void* D, void* X2, int64_t ldx2);

/* the factorised WLR (X2 = X1 C + B D, B m x (r-k), D (r-k) x (n-k)) as a
 * one-sweep block ALS (reading R21), starting from the handle's GHS state (p = 0,
 * before any wlr_iterate).  A sweep is X1 <- the row formula of PAPER.md:184-196 with
 * D_p := B_p D_p, then C, B and D by least squares.  Runs n_iters sweeps on the handle's stream
 * and copies the objectives F_0 .. F_N of all states so far (up to cap doubles) into F (host or
 * device).  With F = NULL the call only enqueues the sweeps (no host synchronisation; errors
 * surface at the next wlr_sync).  Single rank only; needs r - k <= round_up(k, 4) (B shares X1's row
 * layout).  The sWLR state is consumed: wlr_iterate on the same
 * handle afterwards returns WLR_EINVAL.  Errors: WLR_EINVAL (p != 0, nranks > 1, k too large
 * for the small steps), WLR_ERANK (X1^T X1 or B^T B singular), WLR_ECUDA.                    */
wlr_status wlr_als_iterate(wlr_handle h, int32_t n_iters, double* F, int32_t cap);

/* Block-ALS state (host or device pointers, NULL to skip): X1 m x k (ld ldx1, dtype),
 * C k x (n-k) double, B m x (r-k) (ld ldb, dtype), D (r-k) x (n-k) double.                   */
wlr_status wlr_als_result(wlr_handle h, void* X1, int64_t ldx1, void* C, void* B, int64_t ldb,
                          void* D);

/* Small replicated state for tests: name in {"G","M","C","V","lam","GA"}; copies up to
 * cap doubles to host out, *count = element count.  G = X1^T X1 (k x k), M = X1^T A2
 * (k x (n-k)), C (k x (n-k)), V ((n-k) x (r-k) row-major), lam (r-k), GA (n-k)^2.      */
wlr_status wlr_debug_state(wlr_handle h, const char* name, double* out, int64_t cap,
                           int64_t* count);

/* Per-kernel device time accumulated (CUDA events on the handle's stream) while profiling is
 * on; profiling runs every kernel of an iteration serially (no graph, no overlap).  Order of
 * ms[] (nms <= 6): row pass, increment GEMM (uniform W1: the Gram propagation), reduce, small
 * step (critical half), deferred small-step half (objective / step norm), per-row solves
 * (non-uniform W1; included in neither the row pass nor the increments).
 * launches = number of library kernel launches since the last reset.                 */
wlr_status wlr_profile(wlr_handle h, int32_t enable, int32_t reset, double* ms, int32_t nms,
                       int64_t* launches, int64_t* timed_iters);

/* Allocate a 128-byte ncclUniqueId into out (rank 0), to be broadcast by the caller. */
wlr_status wlr_nccl_unique_id(void* out128);

const char* wlr_last_error(wlr_handle h);   /* message of the last failing call       */
const char* wlr_status_string(int32_t s);
void wlr_destroy(wlr_handle h);             /* frees everything the handle owns       */
int32_t wlr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WLR_H */
