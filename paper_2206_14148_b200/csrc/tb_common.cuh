// tb_common.cuh — shared device helpers for the pairwise-kernel hot path.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <float.h>
#include <limits.h>
#include <string>

#include "../../include/tb_pairwise.h"

namespace tb {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define TB_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess)                                                  \
      return ::tb::fail(TB_ERR_CUDA, std::string(#expr) + ": " +            \
                                         cudaGetErrorString(_e));           \
  } while (0)

#define TB_LAUNCH_CHECK(what)                                               \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess)                                                  \
      return ::tb::fail(TB_ERR_CUDA, std::string("launch ") + (what) +      \
                                         ": " + cudaGetErrorString(_e));    \
  } while (0)

constexpr int kInvalidIdx = INT_MAX;
// invalid-slot marker per index type (the cross-shard merge keeps int64
// global indices: index_base + local can pass 2^31 on a sharded database)
template <typename I>
__host__ __device__ constexpr I invalid_idx() {
  return sizeof(I) == 8 ? (I)INT64_MAX : (I)INT_MAX;
}

// ------------------------------------------------------- (score, index) --
// Ordering used everywhere: ascending score, ties -> lower index
// (the reference TopK's stable argsort, interpreter.py:379-381).
template <typename S, typename I>
__device__ __forceinline__ bool lex_less(S a, I ia, S b, I ib) {
  // non-short-circuit: compiles to compares + one predicate op, no branches
  return (a < b) | ((a == b) & (ia < ib));
}

// K-th smallest (K <= 16) of 32 keys: Batcher odd-even merge sort of each
// half (63 comparators each), then min over i of max(a[i-1], b[K-1-i]) for
// the two sorted halves a, b (~290 integer min/max, registers only)
template <int N>
__host__ __device__ __forceinline__ void oem_sort(unsigned* a) {
#pragma unroll
  for (int p = 1; p < N; p <<= 1)
#pragma unroll
    for (int k = p; k >= 1; k >>= 1)
#pragma unroll
      for (int j = k % p; j + k < N; j += 2 * k)
#pragma unroll
        for (int i = 0; i < k && i + j + k < N; ++i)
          if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
            const unsigned lo = a[i + j] < a[i + j + k] ? a[i + j] : a[i + j + k];
            const unsigned hi = a[i + j] < a[i + j + k] ? a[i + j + k] : a[i + j];
            a[i + j] = lo;
            a[i + j + k] = hi;
          }
}
template <int K>
__host__ __device__ __forceinline__ unsigned kth_of_32(unsigned (&v)[32]) {
  static_assert(K >= 1 && K <= 16, "kth_of_32: K in [1, 16]");
  oem_sort<16>(v);
  oem_sort<16>(v + 16);
  unsigned best = v[16 + K - 1] < v[K - 1] ? v[16 + K - 1] : v[K - 1];   // i = 0 and i = K
#pragma unroll
  for (int i = 1; i < K; ++i) {
    const unsigned m = v[i - 1] < v[16 + K - 1 - i] ? v[16 + K - 1 - i] : v[i - 1];
    best = m < best ? m : best;
  }
  return best;
}

// Sorted top-K list held in registers (fully unrolled -> no local memory).
template <typename S, int K, typename I = int>
struct TopList {
  S s[K];
  I i[K];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      s[p] = (S)INFINITY;
      i[p] = invalid_idx<I>();
    }
  }
  __device__ __forceinline__ S worst() const { return s[K - 1]; }
  __device__ __forceinline__ I worst_idx() const { return i[K - 1]; }

  // Insert (v, j); caller guarantees (v, j) < (s[K-1], i[K-1]).
  // Branch-free parallel network on the OLD list: c[p] = (v,j) < entry p;
  // slot p takes entry p-1 if c[p-1] (shift down), else (v,j) if c[p],
  // else keeps its entry.  All K compares are independent (ILP, no
  // divergence-serialised branch chain).
  __device__ __forceinline__ void insert(S v, I j) {
    bool c[K];
#pragma unroll
    for (int p = 0; p < K; ++p) c[p] = lex_less(v, j, s[p], i[p]);
#pragma unroll
    for (int p = K - 1; p > 0; --p) {
      const S ns = c[p - 1] ? s[p - 1] : (c[p] ? v : s[p]);
      const I ni = c[p - 1] ? i[p - 1] : (c[p] ? j : i[p]);
      s[p] = ns;
      i[p] = ni;
    }
    if (c[0]) {
      s[0] = v;
      i[0] = j;
    }
  }
  // Insert (v, j) when j is larger than every index in the list (columns
  // scanned in ascending order): a score tie then ranks after the entry,
  // so the lexicographic compare reduces to one strict float compare.
  __device__ __forceinline__ void insert_after(S v, I j) {
    bool c[K];
#pragma unroll
    for (int p = 0; p < K; ++p) c[p] = v < s[p];
#pragma unroll
    for (int p = K - 1; p > 0; --p) {
      const S ns = c[p - 1] ? s[p - 1] : (c[p] ? v : s[p]);
      const I ni = c[p - 1] ? i[p - 1] : (c[p] ? j : i[p]);
      s[p] = ns;
      i[p] = ni;
    }
    if (c[0]) {
      s[0] = v;
      i[0] = j;
    }
  }
  __device__ __forceinline__ void offer(S v, I j) {
    if (lex_less(v, j, s[K - 1], i[K - 1])) insert(v, j);
  }
  // remove the head (smallest); shifts the rest up
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int p = 0; p < K - 1; ++p) {
      s[p] = s[p + 1];
      i[p] = i[p + 1];
    }
    s[K - 1] = (S)INFINITY;
    i[K - 1] = invalid_idx<I>();
  }
};

// Offer the scores sc[j] whose bit is set in `mask` (ascending j, index
// base + j).  Kept out of line with a dynamic index so that one copy of the
// insertion network serves all 32 columns (I-cache friendliness).  Every
// caller scans columns in ascending index order within a list's lifetime,
// so base + j exceeds every index already held (TopList::insert_after).
template <int K>
__device__ __forceinline__ void insert_masked(TopList<float, K>& L, const float (&sc)[32],
                                           uint32_t mask, int base, float cap = INFINITY) {
  float tmp[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) tmp[j] = sc[j];
  while (mask) {
    const int j = __ffs(mask) - 1;
    mask &= mask - 1;
    const float v = tmp[j];
    if (v < L.worst() && v < cap) L.insert_after(v, base + j);
  }
}

// Warp-wide lexicographic argmin of per-lane (v, j); returns the winner in
// every lane.
template <typename S, typename I>
__device__ __forceinline__ void warp_lex_min(S& v, I& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const S ov = __shfl_xor_sync(0xffffffffu, v, o);
    const I oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (lex_less(ov, oj, v, j)) {
      v = ov;
      j = oj;
    }
  }
}

// Drains `count` smallest entries of the per-lane sorted lists (warp-wide
// k-way merge).  out(t, v, j) is called by lane 0 for t = 0..count-1.
template <typename S, int K, typename I, typename Out>
__device__ __forceinline__ void warp_drain(TopList<S, K, I>& L, int count, Out out) {
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < count; ++t) {
    S v = L.s[0];
    I j = L.i[0];
    warp_lex_min(v, j);
    if (L.i[0] == j && L.s[0] == v && j != invalid_idx<I>()) L.pop();
    if (lane == 0) out(t, v, j);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return (double)v; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
// Device bytes the caller's caching allocator charges for one b-byte buffer
// (PyTorch: 512-B granules up to 1 MiB, 2 MiB granules above).  Planners
// count buffers this way so measured max_memory_allocated <= peak_bytes.
inline int64_t alloc_bytes(int64_t b) {
  return b <= ((int64_t)1 << 20) ? round_up(b, 512) : round_up(b, (int64_t)2 << 20);
}

// Raise a kernel's dynamic shared-memory limit once per (kernel, device,
// size): cudaFuncSetAttribute is a driver round trip, and the host-buffer
// path launches the engines once per database chunk.
int set_smem_once(const void* kernel, int bytes);

}  // namespace tb
