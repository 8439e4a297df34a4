/*
 * tb_pairwise.h — C-ABI of the B200-native memory-safe pairwise-kernel hot
 * path (kNN + SGPR statistics + kernel MVM).  Plain pointers and sizes only;
 * no torch or C++ types cross this boundary.
 *
 * The reference ("tensorbudget", /root/reference/pkg/src/tensorbudget) is a
 * pure-Python package whose operator API for this path is the graph builder
 * + interpreter pair.  Each entry point below replaces the piece of that API
 * named beside it; INTEGRATION.md shows the ctypes binding a maintainer adds.
 *
 * Conventions (mirroring the reference):
 *   - row-major, C-contiguous device buffers (interpreter.py:35-38,543);
 *   - dtype TB_F32 / TB_F64 only (ir.py:32-51);
 *   - kNN parameters: database first, queries second (frontend.py:108-109);
 *   - results ascending, equal distances resolve to the lower data index
 *     (interpreter.py:379-381);
 *   - inputs are read-only; the library never allocates device memory: the
 *     caller passes a workspace whose size the planner returns;
 *   - every function returns a status code; tb_last_error() gives the
 *     thread-local message (the reference raises BudgetExceeded /
 *     EvaluationError / ValueError / UnsplittableCandidate instead,
 *     interpreter.py:40-54, frontend.py:103-106, split.py:31-32).
 *   - all device work is stream-ordered on the given cudaStream_t (passed as
 *     void*); there is no global mutable state besides the error string.
 */
#ifndef TB_PAIRWISE_H
#define TB_PAIRWISE_H

#include <stdint.h>

#if defined(__GNUC__)
#define TB_API __attribute__((visibility("default")))
#else
#define TB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define TB_OK 0
#define TB_ERR_ARG 1          /* EvaluationError / ValueError analogue      */
#define TB_ERR_BUDGET 2       /* BudgetExceeded analogue                    */
#define TB_ERR_UNSPLITTABLE 3 /* UnsplittableCandidate analogue             */
#define TB_ERR_CUDA 4         /* CUDA runtime / launch failure              */
#define TB_ERR_UNSUPPORTED 5  /* shape outside the compiled kernel set      */
#define TB_ERR_NO_DEVICE 6    /* no sm_100 device visible                   */

/* element types (ir.py:32-51) */
#define TB_F32 0
#define TB_F64 1

/* kNN metrics (frontend.py:19) */
#define TB_METRIC_L2 0
#define TB_METRIC_L1 1
#define TB_METRIC_COSINE 2

/* kNN candidate engines */
#define TB_ENGINE_AUTO 0
#define TB_ENGINE_TC3 1   /* tcgen05 bf16x3 split cross term (fp32-class)   */
#define TB_ENGINE_SIMT 2  /* CUDA-core fp32 cross term                      */
#define TB_ENGINE_TC1 3   /* tcgen05 single-pass fp16 (power-of-two scaled), bound from the measured rounding residuals, certified re-rank (AUTO) */

/* SGPR kernels */
#define TB_KERNEL_RBF 0
#define TB_KERNEL_MATERN32 1

/*
 * kNN plan: the runtime replacement of the reference's compile-time
 * memory tiler (PassConfig pipeline.py:18-41, plan_split split.py:285-301).
 * Filled by tb_knn_plan_create; treat as opaque except for the documented outputs.
 */
typedef struct tb_knn_plan {
  /* problem */
  int64_t n, m, d, k;
  int32_t metric, dtype, out_dtype, engine;
  /* memory contract */
  int64_t memory_limit;    /* bytes; <= 0 means unlimited                    */
  int64_t resident_bytes;  /* caller-owned device bytes counted in the limit */
  /* planner outputs */
  int32_t cand;            /* K': candidates kept per (slice, query)         */
  int32_t slices;          /* database slices per chunk (CTA columns)        */
  int64_t chunk_rows;      /* database rows staged per chunk                 */
  int64_t n_chunks;
  int64_t d_pad, m_pad;    /* tensor-core padded extents                     */
  int64_t workspace_bytes; /* caller must pass at least this much           */
  int64_t output_bytes;    /* dist[m,k] (out_dtype) + idx[m,k] (int64)        */
  int64_t peak_bytes;      /* resident + workspace + output: <= memory_limit */
  int64_t off[16];         /* workspace carve-up (internal)                  */
} tb_knn_plan;

/* Replaces build_knn(n, m, d, k, metric, dtype) + run_pipeline(PassConfig)
 * (frontend.py:98-114, pipeline.py:44-60): validates arguments exactly as
 * build_knn does (k in [1, n], known metric) and sizes every tile so that
 * resident_bytes + workspace + outputs <= memory_limit.  Fails with
 * TB_ERR_BUDGET when no tiling fits (the reference would raise
 * BudgetExceeded at run time, interpreter.py:149-151). */
TB_API int tb_knn_plan_create(int64_t n, int64_t m, int64_t d, int64_t k, int32_t metric,
                int32_t dtype, int32_t out_dtype, int32_t engine,
                int64_t memory_limit, int64_t resident_bytes,
                tb_knn_plan* plan);

/* tb_knn_plan_create with an upper bound on the database rows staged per
 * chunk (max_chunk_rows <= 0: none).  Smaller chunks let tb_knn_run_host
 * overlap more of the host->device copy with compute. */
TB_API int tb_knn_plan_create_ex(int64_t n, int64_t m, int64_t d, int64_t k, int32_t metric,
                int32_t dtype, int32_t out_dtype, int32_t engine,
                int64_t memory_limit, int64_t resident_bytes,
                int64_t max_chunk_rows, tb_knn_plan* plan);

/* Replaces evaluate(knn_graph, [x, q], budget) (interpreter.py:522-551) for
 * the kNN graph family: x[n,d], q[m,d] (plan dtype, C-contiguous, 16-byte
 * aligned base pointers; TB_ERR_ARG otherwise) -> out_dist[m,k]
 * (plan out_dtype, squared L2 as the reference's rewritten graph computes,
 * match_replace.py:149-155) and out_idx[m,k] (int64, + index_base so a
 * database shard reports global indices).  Asynchronous on `stream`. */
TB_API int tb_knn_run(const tb_knn_plan* plan, const void* x, const void* q,
               int64_t index_base, void* out_dist, int64_t* out_idx,
               void* workspace, int64_t workspace_bytes, void* stream);

/* tb_knn_run plus timing hooks: when events != NULL it records
 * events[2c] / events[2c+1] (cudaEvent_t) on `stream` immediately before /
 * after the candidate-engine launch of database chunk c (c < n_events/2),
 * so a caller can time the dominant kernel inside a larger timed region. */
TB_API int tb_knn_run_ex(const tb_knn_plan* plan, const void* x, const void* q,
                         int64_t index_base, void* out_dist, int64_t* out_idx,
                         void* workspace, int64_t workspace_bytes, void* stream,
                         void** events, int32_t n_events);

/* The same call with HOST inputs/outputs (the reference's evaluate() takes
 * host numpy arrays, interpreter.py:522-551): x_host[n,d], q_host[m,d] are
 * copied into the caller's device buffers x_dev / q_dev (database chunk by
 * chunk on a side stream, so chunk c+1's copy overlaps chunk c's compute),
 * results land in dist_dev / idx_dev and are copied to dist_host /
 * idx_host.  Host buffers should be pinned for the copies to be
 * asynchronous.  Completes asynchronously on `stream`. */
TB_API int tb_knn_run_host(const tb_knn_plan* plan, const void* x_host, const void* q_host,
                           int64_t index_base, void* dist_host, int64_t* idx_host,
                           void* x_dev, void* q_dev, void* dist_dev, int64_t* idx_dev,
                           void* workspace, int64_t workspace_bytes, void* stream);

/* Merge L per-shard result lists (each [m,k], ascending, dtype `dtype`) into
 * the global top-k with ties -> lower global index.  No reference
 * counterpart: the reference splits queries, never the database
 * (split.py:221-222), so this is the cross-GPU merge the north star adds. */
TB_API int tb_topk_merge(const void* dist_lists, const int64_t* idx_lists,
                  int32_t n_lists, int64_t m, int64_t k, int32_t dtype,
                  void* out_dist, int64_t* out_idx, void* stream);

/* Number of queries the last tb_knn_run on this plan sent to the exact fp64
 * fallback (read from the workspace; synchronises the stream). */
TB_API int tb_knn_fallback_count(const tb_knn_plan* plan, const void* workspace,
                          void* stream, int64_t* count);

/* Input check of the last tb_knn_run / tb_knn_run_host on this plan:
 * TB_ERR_ARG ("cosine distance is undefined for zero rows") when the cosine
 * operand prep met an all-zero database or query row, else TB_OK.  Replaces
 * the reference's host-side zero-norm scan (frontend.py:126-135): the prep
 * kernels flag the rows while they normalise, so the check costs no pass over
 * the inputs.  Synchronises the stream. */
TB_API int tb_knn_check(const tb_knn_plan* plan, const void* workspace, void* stream);

/* ---------------- SGPR sufficient statistics ----------------------------
 * Sigma = Kuf Kuf^T (M x M, fp64), v = Kuf y (M, fp64), yy = y^T y, for
 * X[N,dim], y[N], Z[M,dim] (dtype), accumulated over N in ascending order.
 * No reference counterpart; the nearest is the
 * contracted-dim running add of split.py:322-324,539-547, which the
 * reference cannot apply to Kuf Kuf^T (split.py:210-214).  accumulate != 0
 * adds into Sigma/v/yy instead of overwriting (for N streamed in calls).
 *
 * Engines:
 *   TB_SGPR_ENGINE_I8   exact Gram of Kuf rounded once to 24-bit fixed point
 *                       (Sigma = var^2 2^-48 Q Q^T, v = var 2^-24 Q y, both
 *                       exact for that Q) on the INT8 tensor cores; Sigma is
 *                       returned as packed lower tiles (TB_SIGMA_TILES);
 *   TB_SGPR_ENGINE_F64  fp64 products + fp64 accumulation on the FP64 tensor
 *                       cores (DMMA); Sigma full symmetric (TB_SIGMA_FULL);
 *   TB_SGPR_ENGINE_F64_SIMT  the same numerics on CUDA cores (cross-check).
 *   TB_SGPR_ENGINE_AUTO = I8. */
#define TB_SGPR_ENGINE_AUTO 0
#define TB_SGPR_ENGINE_I8 1
#define TB_SGPR_ENGINE_F64 2
#define TB_SGPR_ENGINE_F64_SIMT 3

/* Sigma layouts: FULL = row-major symmetric [M, M]; TILES = lower 128x128
 * tiles (a >= b) packed at index a(a+1)/2 + b, each tile column-major,
 * M_pad = round_up(M, 128); rows/cols >= M are zero. */
#define TB_SIGMA_FULL 0
#define TB_SIGMA_TILES 1

typedef struct tb_sgpr_plan {
  int64_t N, M, dim;
  int32_t kernel, dtype;
  int64_t memory_limit, resident_bytes;
  int32_t engine;           /* engine actually used (never AUTO)            */
  int32_t sigma_layout;     /* TB_SIGMA_FULL / TB_SIGMA_TILES               */
  int64_t M_pad;
  int64_t sigma_bytes;      /* size of the Sigma buffer tb_sgpr_stats_run writes */
  int64_t chunk_n;          /* training points per streamed chunk           */
  int64_t workspace_bytes;
  int64_t output_bytes;     /* Sigma + v + yy                               */
  int64_t peak_bytes;       /* resident + outputs + workspace <= limit; for the
                               fixed-point engine also the packed tail's peak */
  int64_t off[8];           /* internal; off[5] = tail workspace bytes,
                               off[6] = tail peak (TB_SIGMA_TILES plans)     */
} tb_sgpr_plan;

TB_API int tb_sgpr_plan_create(int64_t N, int64_t M, int64_t dim, int32_t kernel,
                 int32_t dtype, int32_t engine, int64_t memory_limit,
                 int64_t resident_bytes, tb_sgpr_plan* plan);

TB_API int tb_sgpr_stats_run(const tb_sgpr_plan* plan, const void* X, const void* y,
                      const void* Z, double variance,
                      const double* lengthscales, double* Sigma, double* v,
                      double* yy, int32_t accumulate, void* workspace,
                      int64_t workspace_bytes, void* stream);

/* Expand a TB_SIGMA_TILES Sigma into the full symmetric [M, M] matrix the
 * O(M^3) tail (cuSOLVER) consumes; for TB_SIGMA_FULL plans it is a copy. */
TB_API int tb_sgpr_sigma_unpack(const tb_sgpr_plan* plan, const double* Sigma,
                                double* full, void* stream);

/* ---------------- SGPR tail on the packed tiles --------------------------
 * The O(M^3) part of the ELBO on a TB_SIGMA_TILES Sigma, in place, so the
 * whole evaluation fits memory_limit (two packed M x M matrices):
 *   Kuu = L L^T,  Kuu + Sigma/s2 = P P^T (P overwrites Sigma),  X = L^-1 P
 * out4 = {sum log diag L, sum log diag P, |P^-1 v|^2, ||X||_F^2,
 *         min diag(L)^2, max diag(L)^2} (6 device doubles: the last two
 *         bound cond(Kuu) from below, a conditioning indicator) and w_out[M] = P^-T P^-1 v / s2 (the predictive-mean weights).
 * Then (GPflow SGPR.elbo): sum log diag LB = out4[1] - out4[0],
 * c^T c = out4[2] / s2^2, tr(AAT) = out4[3] - M_pad.  Synchronises `stream`
 * (reports a failed Cholesky as TB_ERR_ARG). */
TB_API int64_t tb_sgpr_tail_workspace(const tb_sgpr_plan* plan);
TB_API int tb_sgpr_tail_run(const tb_sgpr_plan* plan, const void* Z, double variance,
                            const double* lengthscales, double jitter, double noise_variance,
                            double* Sigma, const double* v, double* w_out, double* out4,
                            void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------- SGPR ELBO gradient inside memory_limit -----------------
 * The whole GPflow 2.3.1 SGPR training gradient (paper §5.3, Table 2) from
 * the packed statistics (TB_SIGMA_TILES, consumed: Sigma becomes the factor
 * P of Kuu + Sigma/s2 in place).  Only L = chol(Kuu) and P stay resident;
 * 2 dELBO/dKuu and 2 dELBO/dSigma are produced one 128-column panel at a
 * time and consumed at once (the data side streams all N rows of X, y
 * through a fused generate-Kuf / DMMA / derivative kernel), so the device
 * footprint is two packed M x M triangles + 3 column panels.
 * out8: [0] sum log diag L, [1] sum log diag P, [2] |P^-1 v|^2,
 * [3] tr(Kuu^-1 A), [4] tr(A^-1 Kuu), [5] w^T Kuu w (A = Kuu + Sigma/s2,
 * w = A^-1 v / s2), [6] min diag(L)^2, [7] max diag(L)^2 (a lower bound on
 * cond(Kuu)).  grad_hyp[2 (1 + dim)]: data-side (variance,
 * lengthscales) then Kuu-side sums (the latter doubled: halve them);
 * grad_Z[2 M dim]: data side then Kuu side.  Both are accumulated into
 * (zero them first).  dim <= 16.  No reference counterpart. */
TB_API int64_t tb_sgpr_grad_workspace(const tb_sgpr_plan* plan);
TB_API int tb_sgpr_grad_run(const tb_sgpr_plan* plan, const void* X, const void* y, const void* Z,
                            double variance, const double* lengthscales, double jitter,
                            double noise_variance, double* Sigma, const double* v, double* out8,
                            double* grad_hyp, double* grad_Z, void* workspace,
                            int64_t workspace_bytes, void* stream);

/* ---------------- SGPR ELBO gradient (N-streaming half) ------------------
 * GPflow 2.3.1 SGPR training-loss gradient (paper §5.3).  With
 * G = dELBO/dSigma and g = dELBO/dv from the O(M^3) tail (autodiff), the
 * data enter only through W = 2 G Kuf + g y^T, and
 *   grad_hyp[0]      += sum_in W_in dK_in/d variance
 *   grad_hyp[1 + t]  += sum_in W_in dK_in/d lengthscale_t
 *   grad_Z[i, t]     += sum_n  W_in dK_in/d Z_it
 * for one chunk: Xc[nc, dim], Z[M, dim] (dtype), W and K = k(Z, Xc) fp64
 * [M, nc] row-major.  Fixed-order reductions (deterministic).  No reference
 * counterpart. */
TB_API int64_t tb_sgpr_kuf_grad_workspace(int64_t nc, int64_t M, int64_t dim);
TB_API int tb_sgpr_kuf_grad(const void* Xc, const void* Z, const double* W, const double* K,
                            int64_t nc, int64_t M, int64_t dim, int32_t kernel, int32_t dtype,
                            double variance, const double* lengthscales, double* grad_hyp,
                            double* grad_Z, void* workspace, int64_t workspace_bytes,
                            void* stream);

/* ---------------- kernel MVM --------------------------------------------
 * out[i] = sum_j k(X_i, Z_j) w_j in fp64 accumulation, X[n,dim], Z[M,dim]
 * (dtype), w[M] fp64 -> out[n] fp64.  Replaces evaluate(build_kernel_mvm)
 * (frontend.py:34-54: 1-D inputs, SE kernel, op order scale->exp->variance)
 * and is the SGPR predictive mean K*u w.  Streams Z tiles; never forms K. */
TB_API int tb_kernel_mvm(const void* X, const void* Z, const double* w, int64_t n,
                  int64_t M, int64_t dim, int32_t kernel, int32_t dtype,
                  double variance, const double* lengthscales, double* out,
                  void* stream);

/* out[i, j] = k(A_i, B_j), fp64 [na, nb]; the same kernel code as the
 * statistics (so Kuu and Kuf agree bit for bit).  Feeds the O(M^3) tail. */
TB_API int tb_kernel_matrix(const void* A, const void* B, int64_t na, int64_t nb,
                            int64_t dim, int32_t kernel, int32_t dtype, double variance,
                            const double* lengthscales, double* out, void* stream);

/* ---------------- misc ---------------------------------------------------*/
TB_API const char* tb_last_error(void);
/* compiled-in capabilities: bit0 tcgen05 kNN, bit1 SIMT kNN, bit2 SGPR,
 * bit3 kernel MVM; returns the library version in the high 16 bits. */
TB_API int32_t tb_capabilities(void);

#ifdef __cplusplus
}
#endif
#endif /* TB_PAIRWISE_H */
