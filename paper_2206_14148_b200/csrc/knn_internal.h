// knn_internal.h — launchers shared between the C-ABI layer and kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace tb {

// workspace slots of tb_knn_plan::off
enum KnnSlot {
  kQn64 = 0,    // double[m]        ||q||^2 (fp64, exact)
  kQnorm = 1,   // float[m]         ||q||   (for the error bound)
  kStats = 2,   // u32[64]          [0] = max ||x|| bits, [1] = fallback count
  kFbList = 3,  // int[m]           queries sent to the exact fallback
  kXn = 4,      // float[chunk_pad] ||x||^2 of the staged chunk (fp32)
  kCandS = 5,   // float[L][m][K']  per-(slice,query) candidate scores
  kCandI = 6,   // int  [L][m][K']
  kRunS = 7,    // float[2][m][K']  running merged candidates (ping-pong)
  kRunI = 8,    // int  [2][m][K']
  kQHi = 9,     // bf16[m_pad][d_pad]   (tensor-core engines)
  kQLo = 10,
  kXHi = 11,    // bf16[chunk_pad][d_pad]
  kXLo = 12,
  kGThr = 13,   // u32[m]           per-query shared K'-th score bound (ordered key)
  kXExt = 14,   // bf16[chunk_pad][16] augmented-K rows -(h,m,l) of ||x||^2 (core matrices)
  kQln = 15,    // float[m]         ||q - fp16 q|| (engine tc1's certified bound)
  kNumSlots = 16
};
// stats (u32[64]): [0] max ||x|| bits, [1] fallback count, [2] max ||x - fp16 x||
// bits, [3] max |q| bits, [4] max |x| bits of the current chunk, [5] the
// chunk's max ||x - fp16 x||, [kF16Slot..+3] fp16 engine scales (floats:
// s, t, alpha, 1/(s t)), [12] redo flag of the chunk conversion, [13] max 1/t,
// [14] centring flag, [15] max |mu|, [16] cosine zero-row flag, [17] count
// of queries the fallback's hit-buffer path hands on; words 64..
// hold mu (fp64 [d]) for tc1
constexpr int kF16Slot = 8;
constexpr int kFbOverWord = 17;      // count of fallback queries the hit-buffer path hands on

// kFbList region: int fb_list[m] (uncertified query rows), then (8-byte
// aligned) double bounds[m]: the exact k-th candidate distance of each, an
// upper bound on its true k-th distance (the fallback scans below it), then
// int hits[m]: the fallback's hit counts (zeroed by the re-rank as it
// appends a query, so the common no-fallback call needs no memset)
inline int64_t fb_region_bytes(int64_t m) { return ((m * 4 + 7) & ~(int64_t)7) + m * 12; }
__host__ __device__ __forceinline__ double* fb_bounds(int* fb, int64_t m) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(fb) + ((m * 4 + 7) & ~(int64_t)7));
}
__host__ __device__ __forceinline__ int* fb_hits(int* fb, int64_t m) {
  return reinterpret_cast<int*>(fb_bounds(fb, m) + m);
}

// kGThr region: per-query thresholds (u32[m], padded to 32 words) followed by
// the per-query insertion pools of the tcgen05 engine (tc_pool_slots(K')
// hashed slots per query; 2 K' for K' = 16, see knn_tc.cu)
constexpr int tc_pool_slots(int cand) { return cand == 16 ? 32 : cand; }
inline int64_t tc_thr_words(int64_t m) { return (m + 31) / 32 * 32; }
inline int64_t tc_gthr_words(int64_t m, int cand) {
  return tc_thr_words(m) + m * (int64_t)tc_pool_slots(cand);
}
constexpr int kZeroRowWord = 16;

struct KnnDims {
  int64_t n, m, d, k;
  int cand;
  int64_t d_pad, m_pad;
};

// prep
int launch_query_prep(int dtype, int metric, const void* q, int64_t m, int64_t d,
                      double* qn64, float* qnorm, __nv_bfloat16* qhi,
                      __nv_bfloat16* qlo, int64_t m_pad, int64_t d_pad,
                      cudaStream_t st, unsigned* centre = nullptr);
int launch_db_prep(int dtype, int metric, const void* x, int64_t rows, int64_t d,
                   float* xn, unsigned* xmax_bits, __nv_bfloat16* xhi,
                   __nv_bfloat16* xlo, int64_t rows_pad, int64_t d_pad,
                   uint8_t* xext, cudaStream_t st);
int launch_query_prep_f16(int dtype, int metric, const void* q, int64_t m, int64_t d,
                          double* qn64, float* qnorm, float* qln, unsigned* stats,
                          __half* qhi, int64_t m_pad, int64_t d_pad, cudaStream_t st);
// l2 + tc1: sample mean of the first rows of x and the centring decision
// (stats[14], mu as fp64 at stats + 64 words, max |mu| in stats[15])
int launch_f16_center(int dtype, const void* x, int64_t rows, int64_t d, unsigned* stats,
                      cudaStream_t st);
int launch_db_prep_f16(int dtype, int metric, const void* x, int64_t rows, int64_t d,
                       float* xn, unsigned* stats, __half* xhi, int64_t rows_pad,
                       int64_t d_pad, uint8_t* xext, cudaStream_t st);
// SIMT candidate engine: writes lists [2*slices][m][cand]
int launch_knn_simt(int dtype, int metric, int cand, const void* x_chunk, const void* q,
                    const float* xn, int64_t rows, int64_t m, int64_t d,
                    int slices, int idx_base, float* cand_s, int* cand_i,
                    cudaStream_t st);
// tcgen05 candidate engine (persistent): writes tc_lists(...) lists
// [lists][m][cand]; gthr[m] is the shared per-query threshold (ordered keys)
int launch_knn_tc(int passes, int cand, const __nv_bfloat16* xhi,
                  const __nv_bfloat16* xlo, const __nv_bfloat16* qhi,
                  const __nv_bfloat16* qlo, const uint8_t* xext, int64_t rows,
                  int64_t rows_pad, int64_t m, int64_t m_pad, int64_t d_pad,
                  int lists, int idx_base, float* cand_s, int* cand_i,
                  unsigned* gthr, const float* f16p, cudaStream_t st);
int tc_lists(int64_t m, int64_t rows_pad, int sms, int passes, int64_t d_pad);
int tc_max_dpad();
// merge L lists (+ optional previous running list) into out
int launch_knn_merge(int cand, const float* in_s, const int* in_i, int lists,
                     const float* prev_s, const int* prev_i, int64_t m,
                     float* out_s, int* out_i, cudaStream_t st);
// exact fp64 re-rank + certification
int launch_knn_refine(int dtype, int out_dtype, int metric, int cand, const float* cs,
                      const int* ci, const void* x, const void* q,
                      const double* qn64, const float* qnorm, const float* qln,
                      const unsigned* stats, int64_t n, int64_t m, int64_t d,
                      int64_t k, double c1, double c2, void* out_dist,
                      int64_t* out_idx, int64_t index_base, int* fb_list,
                      cudaStream_t st);
int launch_knn_fallback(int dtype, int out_dtype, int metric, const void* x, const void* q,
                        int64_t n, int64_t m, int64_t d, int64_t k,
                        const unsigned* stats, const int* fb_list, void* scratch,
                        int64_t scratch_bytes, void* out_dist, int64_t* out_idx,
                        int64_t index_base, cudaStream_t st);
int launch_topk_merge(const void* dist_lists, const int64_t* idx_lists,
                      int n_lists, int64_t m, int64_t k, int dtype,
                      void* out_dist, int64_t* out_idx, cudaStream_t st);

}  // namespace tb
