// knn_kernels.cu — data prep, SIMT candidate engine, candidate merge, exact
// fp64 re-rank + certification, and the exact fp64 fallback.
//
// Pipeline per shard:
//   query_prep -> [per chunk: db_prep -> candidate engine -> merge]
//   -> refine (exact fp64 distances of the K' candidates, ties -> lower
//      index, certification against the engine's error bound)
//   -> fallback (exact fp64 brute force for uncertified queries; normally 0)
//
// The reference computes the distances as ``norms + (-2)·dot`` in the input
// dtype (match_replace.py:149-155) and selects with a full stable argsort
// (interpreter.py:371-390).  Here candidates are *selected* with the fast
// approximate score s_j = ||x_j||^2 - 2 q·x_j (||q||^2 is constant per row),
// and the returned distances/ordering come from an exact fp64 re-rank.
#include "tb_common.cuh"
#include "knn_internal.h"

namespace tb {

// ------------------------------------------------------------------ prep --

// One warp per row: ||row||^2 in fp64 and optional bf16 hi/lo split with
// zero padding to [rows_pad, d_pad] (tensor-core operand layout, K-major).
// L1 (metric == TB_METRIC_L1): acc = sum |v| and norm32 = ||row||_1 (for
// the L1 error bound) instead of the squared L2 norm.
template <typename T>
__global__ void rows_prep_kernel(const T* __restrict__ src, int64_t rows,
                                 int64_t d, double* __restrict__ n64,
                                 float* __restrict__ n32,
                                 float* __restrict__ norm32,
                                 unsigned* __restrict__ max_bits,
                                 __nv_bfloat16* __restrict__ hi,
                                 __nv_bfloat16* __restrict__ lo,
                                 int64_t rows_pad, int64_t d_pad, int metric) {
  const int lane = threadIdx.x & 31;
  const int64_t limit = hi ? rows_pad : rows;
  const int64_t cols = hi ? d_pad : d;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  float wmax = 0.f;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < limit;
       r += nwarps) {
    double acc = 0.0;
    for (int64_t j = lane; j < cols; j += 32) {
      const double v = (r < rows && j < d) ? (double)src[r * d + j] : 0.0;
      acc += metric == TB_METRIC_L1 ? fabs(v) : v * v;
      if (hi) {
        const __nv_bfloat16 h = __double2bfloat16(v);
        const __nv_bfloat16 l = __double2bfloat16(v - (double)__bfloat162float(h));
        hi[r * d_pad + j] = h;
        lo[r * d_pad + j] = l;
      }
    }
    acc = warp_sum(acc);
    if (lane == 0 && r < rows) {
      if (n64) n64[r] = acc;
      if (n32) n32[r] = (float)acc;
      const float nrm = (float)(metric == TB_METRIC_L1 ? acc : sqrt(acc)) * (1.0f + 1e-6f);
      if (norm32) norm32[r] = nrm;
      wmax = fmaxf(wmax, nrm);
    }
  }
  // one atomic per warp (a per-row atomic on one address serialises)
  if (max_bits && lane == 0 && wmax > 0.f) atomicMax(max_bits, __float_as_uint(wmax));
}

// Tensor-core operand prep, G threads per row (G = d_pad / 8 for d_pad 64 /
// 128, a full warp looping over 8-element segments beyond), 8 elements per
// thread and step: 16-byte loads/stores of the bf16 hi/lo split, fp64 norms
// reduced over the row's lanes, and one max-norm atomic per block.
// NORM (cosine): rows are first scaled to unit L2 norm (a pre-pass over the
// row computes it), so the engine's ||x||^2 - 2 q.x ranks by cosine.
template <typename T, int G, bool NORM>
__global__ void __launch_bounds__(256)
rows_split_kernel(const T* __restrict__ src, int64_t rows, int64_t d,
                  double* __restrict__ n64, float* __restrict__ n32,
                  float* __restrict__ norm32, unsigned* __restrict__ max_bits,
                  __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                  int64_t rows_pad, int64_t d_pad, double scale,
                  uint8_t* __restrict__ ext, unsigned* __restrict__ centre) {
  __shared__ float wmax[8];
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = gt / G;
  // l2 centring on the sample mean (decided on the device, f16_center_*):
  // rows become x - mu (fp64) before the split; padding rows stay zero
  const bool centred = !NORM && centre != nullptr && centre[14] != 0u;
  const double* mu = centred ? reinterpret_cast<const double*>(centre + 64) : nullptr;
  const int seg = (int)(gt % G);
  double inv = 1.0;
  if (NORM) {
    double nn = 0.0;
    for (int64_t c = (int64_t)seg; r < rows && c < d; c += G) {
      const double v = (double)src[r * d + c];
      nn = fma(v, v, nn);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
    inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
    // cosine is undefined for an all-zero row: flag it (stats word
    // kZeroRowWord, read back by tb_knn_check) instead of a separate pass
    if (centre && seg == 0 && r < rows && nn == 0.0) centre[kZeroRowWord] = 1u;
  }
  double acc = 0.0;
  for (int64_t c0 = (int64_t)seg * 8; r < rows_pad && c0 < d_pad; c0 += 8 * G) {
    double v[8];
    if (r < rows && c0 + 8 <= d && sizeof(T) == 4 && (d & 3) == 0) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + r * d + c0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(src + r * d + c0 + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = (r < rows && c0 + j < d) ? (double)src[r * d + c0 + j] : 0.0;
    }
    if (centred && r < rows) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + j < d) v[j] -= mu[c0 + j];
    }
    __align__(16) __nv_bfloat16 h[8];
    __align__(16) __nv_bfloat16 l[8];
    if (sizeof(T) == 4 && !NORM && scale == 1.0 && !centred) {
      // f32 rows: x - bf16(x) is exact in f32, so the split needs no fp64
      // (same bits as the fp64 path); only the norm accumulates in fp64
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float f = (float)v[j];
        acc = fma(v[j], v[j], acc);
        h[j] = __float2bfloat16_rn(f);
        l[j] = __float2bfloat16_rn(f - __bfloat162float(h[j]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double u = NORM ? v[j] * inv : v[j];
        acc = fma(u, u, acc);
        const double sv = scale * u;             // scale: exact power of two
        h[j] = __double2bfloat16(sv);
        l[j] = __double2bfloat16(sv - (double)__bfloat162float(h[j]));
      }
    }
    *reinterpret_cast<uint4*>(hi + r * d_pad + c0) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(lo + r * d_pad + c0) = *reinterpret_cast<const uint4*>(l);
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (ext && seg == 0 && r < rows_pad) {
    // augmented-K row for the tensor-core engine: -(h, m, l) with
    // h + m + l = ||x||^2 to ~2^-24 (padding rows: -inf, never selected),
    // stored as 8-row x 16-byte core matrices (SWIZZLE_NONE, K-major)
    __nv_bfloat16 e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = __float2bfloat16(0.f);
    if (r < rows) {
      const __nv_bfloat16 h0 = __double2bfloat16(acc);
      const double r1 = acc - (double)__bfloat162float(h0);
      const __nv_bfloat16 h1 = __double2bfloat16(r1);
      const __nv_bfloat16 h2 = __double2bfloat16(r1 - (double)__bfloat162float(h1));
      e[0] = __hneg(h0);
      e[1] = __hneg(h1);
      e[2] = __hneg(h2);
    } else {
      e[0] = __float2bfloat16(-INFINITY);
    }
    uint8_t* base = ext + (r >> 8) * 8192 + ((r & 255) >> 3) * 256 + (r & 7) * 16;
    *reinterpret_cast<uint4*>(base) = *reinterpret_cast<const uint4*>(e);
    *reinterpret_cast<uint4*>(base + 128) = make_uint4(0u, 0u, 0u, 0u);
  }
  float nrm = 0.f;
  if (seg == 0 && r < rows) {
    if (n64) n64[r] = acc;
    if (n32) n32[r] = (float)acc;
    nrm = (float)sqrt(acc) * (1.0f + 1e-6f);
    if (norm32) norm32[r] = nrm;
  }
  if (max_bits) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm = fmaxf(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      float m = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wmax[w]);
      atomicMax(max_bits, __float_as_uint(m));
    }
  }
}

template <typename T>
static int rows_prep(const void* src, int64_t rows, int64_t d, double* n64,
                     float* n32, float* norm32, unsigned* max_bits,
                     __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t rows_pad,
                     int64_t d_pad, cudaStream_t st, int metric, double scale = 1.0,
                     uint8_t* ext = nullptr, unsigned* centre = nullptr) {
  const int64_t limit = hi ? rows_pad : rows;
  if (limit <= 0) return TB_OK;
  if (hi && d_pad % 64 == 0) {
    const int G = d_pad == 64 ? 8 : d_pad == 128 ? 16 : 32;
    const int64_t threads = rows_pad * G;
    const unsigned blocks = (unsigned)ceil_div(threads, 256);
    const bool norm = metric == TB_METRIC_COSINE;
#define TB_SPLIT(GG, NN)                                                                     \
  rows_split_kernel<T, GG, NN><<<blocks, 256, 0, st>>>((const T*)src, rows, d, n64, n32,     \
                                                       norm32, max_bits, hi, lo, rows_pad,   \
                                                       d_pad, scale, ext, centre)
    if (G == 8) {
      if (norm) TB_SPLIT(8, true); else TB_SPLIT(8, false);
    } else if (G == 16) {
      if (norm) TB_SPLIT(16, true); else TB_SPLIT(16, false);
    } else {
      if (norm) TB_SPLIT(32, true); else TB_SPLIT(32, false);
    }
#undef TB_SPLIT
    TB_LAUNCH_CHECK("rows_split");
    return TB_OK;
  }
  if (hi) return fail(TB_ERR_UNSUPPORTED, "tensor-core prep needs d_pad % 64 == 0");
  const int warps = 8;
  const int64_t blocks = std::min<int64_t>(ceil_div(limit, warps), 148 * 16);
  rows_prep_kernel<T><<<(unsigned)blocks, warps * 32, 0, st>>>(
      (const T*)src, rows, d, n64, n32, norm32, max_bits, hi, lo, rows_pad, d_pad, metric);
  TB_LAUNCH_CHECK("rows_prep");
  return TB_OK;
}

// ------------------------------------------ fp16 single-pass operand prep --
// Engine tc1: one fp16 x fp16 -> fp32 MMA pass with a TIGHT certified bound.
// Operands are scaled by powers of two (exact) into fp16 range: A = fp16(2 s q),
// B = fp16(t x), A_ext = alpha, B_ext = -(h, m, l) with h + m + l =
// s t ||x||^2 / alpha, so the accumulator is s t (2 q.x - ||x||^2) and the
// engine unscales by 1 / (s t).  The rounding residuals are measured exactly
// (fp64): ||ql|| per query, max ||xl|| per database (stats), and the refine
// step's bound uses them (Cauchy-Schwarz) instead of a worst-case relative
// error: |q.x - q'.x'| <= ||q|| XL + ||ql|| (X + 3 XL).
// Scale slots (floats, stats + kF16Slot): [0] s, [1] t, [2] alpha, [3] 1/(s t).

// Block-wide max of non-negative floats, then ONE atomicMax per block (one
// per warp serialised ~10k atomics on a single word: 10 us for the C2 queries).
__device__ __forceinline__ void block_atomic_max(float mx, unsigned* bits) {
  __shared__ float wm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, wm[w]);
    if (mx > 0.f) atomicMax(bits, __float_as_uint(mx));
  }
}

__global__ void absmax_f32_kernel(const float* __restrict__ src, int64_t n,
                                  unsigned* __restrict__ bits) {
  float mx = 0.f;
  const int64_t n4 = n / 4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(src) + e);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int64_t e = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, fabsf(src[e]));
  block_atomic_max(mx, bits);
}

__global__ void absmax_f64_kernel(const double* __restrict__ src, int64_t n,
                                  unsigned* __restrict__ bits) {
  float mx = 0.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, __double2float_ru(fabs(src[e])));
  block_atomic_max(mx, bits);
}

__device__ __forceinline__ float pow2_floor(float v) {      // largest 2^e <= v
  return exp2f(floorf(log2f(v)));
}

// which = 0: queries (s from max|q| in stats[3]).  which = 1: database chunk,
// after the provisional pass (t = 1) recorded max|x| in stats[4]: t = 1 is
// kept when max|x| is in [2^-3, 2^14] (no overflow, normal fp16 values for all
// but tiny elements) and s d max|x|^2 <= 2^29 (the ||x||^2 block fits fp16
// with alpha <= 2^15); otherwise t is recomputed and stats[12] asks the second
// pass to redo the conversion.
__global__ void f16_scales_kernel(unsigned* __restrict__ stats, int64_t d, int which,
                                  int metric) {
  float* sc = reinterpret_cast<float*>(stats + kF16Slot);
  if (which == 0) {
    float qm = metric == TB_METRIC_COSINE ? 1.f : __uint_as_float(stats[3]);
    if (metric != TB_METRIC_COSINE && stats[14]) qm += __uint_as_float(stats[15]);   // |q - mu|
    // |2 s q| <= 256; s, t in [2^-60, 2^60] keep 1/(s t) a normal float
    sc[0] = qm > 0.f ? fminf(fmaxf(pow2_floor(128.f / qm), 0x1p-60f), 0x1p60f) : 1.f;
    return;
  }
  const float xm = metric == TB_METRIC_COSINE ? 1.f : __uint_as_float(stats[4]);
  const double s = sc[0];
  const double cap = 536870912.0;                            // 2^29
  float t = 1.f;
  unsigned redo = 0;
  if (!(xm >= 0.125f && xm <= 16384.f && s * (double)d * (double)xm * (double)xm <= cap)) {
    t = xm > 0.f ? fminf(fmaxf(pow2_floor(256.f / xm), 0x1p-60f), 0x1p60f) : 1.f;
    const double V = s * (double)t * (double)d * (double)xm * (double)xm;
    if (V > cap) t = (float)((double)t / exp2(ceil(log2(V / cap))));
    redo = t != 1.f;
  }
  const double V = s * (double)t * (double)d * (double)xm * (double)xm;
  double a = exp2(ceil(log2(fmax(V, 1e-30) / 16384.0)));
  a = fmin(fmax(a, 1.0 / 16384.0), 32768.0);
  sc[1] = t;
  sc[2] = (float)a;
  sc[3] = (float)(1.0 / (s * (double)t));
  stats[12] = redo;
  atomicMax(stats + 13, __float_as_uint(1.f / t));   // max 1/t over chunks (refine)
  if (redo) stats[5] = 0u;                 // the chunk's residual max is redone
}

// MODE 0: queries, A = fp16(2 s q), ||ql|| per row (rounded up).
// MODE 1: database, provisional t = 1; records max |x| (stats[4]).
// MODE 2: database, t = sc[1]; only when stats[12] asks for it.
// Database modes: fp32 ||x||^2 (xn), max ||x|| (stats[0]), chunk max ||xl||
// (stats[5]).  f32 rows without normalisation take an exact fp32 path: t is
// a power of two, so x t and fp16(x t) / t are exact and x - fp16(x t) / t
// is exact (Sterbenz); the residual norm is summed in fp32 and rounded up by
// (1 + (d + 2) 2^-23) so it stays an upper bound.
template <typename T, int G, bool NORM, int MODE, bool CENTRED>
__global__ void __launch_bounds__(256)
rows_f16_kernel(const T* __restrict__ src, int64_t rows, int64_t d,
                double* __restrict__ n64, float* __restrict__ n32, float* __restrict__ norm32,
                float* __restrict__ resid, unsigned* __restrict__ stats,
                __half* __restrict__ hi, int64_t rows_pad, int64_t d_pad) {
  __shared__ float wmax[8], wres[8], wabs[8];
  const float* sc = reinterpret_cast<const float*>(stats + kF16Slot);
  if (MODE == 2 && *reinterpret_cast<volatile unsigned*>(stats + 12) == 0u) return;
  const float mulf = MODE == 0 ? 2.f * sc[0] : MODE == 1 ? 1.f : sc[1];
  const double mul = mulf, imul = 1.0 / (double)mulf;       // powers of two: exact
  const float imulf = 1.f / mulf;
  // centred rows (l2 only, translation invariant): x - mu, q - mu with the
  // sample mean mu chosen by f16_center_kernel; fp64 path then
  // both variants are launched; the one that does not match the device-side
  // centring decision exits at once
  if (!NORM && (*reinterpret_cast<volatile unsigned*>(stats + 14) != 0u) != CENTRED) return;
  constexpr bool centred = CENTRED && !NORM;
  const double* mu = reinterpret_cast<const double*>(stats + 64);
  constexpr bool FAST = sizeof(T) == 4 && !NORM && !centred;
  // grid-stride over rows (the stride keeps a row's G lanes in one warp)
  float nrm = 0.f, res = 0.f, amax = 0.f;
  const int64_t total = rows_pad * G;
  for (int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       gt - threadIdx.x < total; gt += (int64_t)gridDim.x * blockDim.x) {
  const int64_t r = gt < total ? gt / G : rows_pad;
  const int seg = (int)(gt % G);
  double inv = 1.0;
  if (NORM) {
    double nn = 0.0;
    for (int64_t c = (int64_t)seg; r < rows && c < d; c += G) {
      const double v = (double)src[r * d + c];
      nn = fma(v, v, nn);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
    inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
    if (seg == 0 && r < rows && nn == 0.0) stats[kZeroRowWord] = 1u;   // see rows_split_kernel
  }
  double acc = 0.0, rn = 0.0;
  float rnf = 0.f, accf = 0.f;
#pragma unroll 2
  for (int64_t c0 = (int64_t)seg * 8; r < rows_pad && c0 < d_pad; c0 += 8 * G) {
    double v[8];
    float f[8];
    if (r < rows && c0 + 8 <= d && sizeof(T) == 4 && (d & 3) == 0) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + r * d + c0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(src + r * d + c0 + 4));
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
      f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = f[j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = (r < rows && c0 + j < d) ? (double)src[r * d + c0 + j] : 0.0;
        f[j] = (float)v[j];
      }
    }
    if (centred && r >= rows) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = c0 + j < d ? mu[c0 + j] : 0.0;   // u = 0 on padding
    }
    __align__(16) __half h[8];
    if (FAST) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 0) acc = fma(v[j], v[j], acc);       // ||q||^2 exact for the re-rank
        else accf = fmaf(f[j], f[j], accf);               // ||x||^2: fp32, bounded below
        amax = fmaxf(amax, fabsf(f[j]));
        h[j] = __float2half_rn(f[j] * mulf);
        const float e = f[j] - __half2float(h[j]) * imulf;
        rnf = fmaf(e, e, rnf);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double u = NORM ? v[j] * inv : (centred && c0 + j < d ? v[j] - mu[c0 + j] : v[j]);
        acc = fma(u, u, acc);
        amax = fmaxf(amax, __double2float_ru(fabs(u)));
        h[j] = __double2half(mul * u);
        const double e = u - (double)__half2float(h[j]) * imul;
        rn = fma(e, e, rn);
      }
    }
    *reinterpret_cast<uint4*>(hi + r * d_pad + c0) = *reinterpret_cast<const uint4*>(h);
  }
  // fp32 sums of d non-negative terms: relative error <= (d + 2) 2^-24
  const double up = 1.0 + (double)(d + 2) * 0x1p-23;
  if (FAST) rn = (double)rnf * up;
  if (FAST && MODE != 0) acc = (double)accf;
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    rn += __shfl_xor_sync(0xffffffffu, rn, o);
  }
  if (seg == 0 && r < rows) {
    if (n64) n64[r] = acc;
    if (n32) n32[r] = (float)acc;
    const float nr = (float)(sqrt(acc) * (FAST && MODE != 0 ? up : 1.0)) * (1.0f + 1e-6f);
    nrm = fmaxf(nrm, nr);
    if (norm32) norm32[r] = nr;
    const float rs = __double2float_ru(sqrt(rn) * (1.0 + 1e-12));
    res = fmaxf(res, rs);
    if (MODE == 0 && resid) resid[r] = rs;
  }
  }
  if (MODE != 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nrm = fmaxf(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
      res = fmaxf(res, __shfl_xor_sync(0xffffffffu, res, o));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      wmax[threadIdx.x >> 5] = nrm;
      wres[threadIdx.x >> 5] = res;
      wabs[threadIdx.x >> 5] = amax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float m = 0.f, mr = 0.f, ma = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        m = fmaxf(m, wmax[w]);
        mr = fmaxf(mr, wres[w]);
        ma = fmaxf(ma, wabs[w]);
      }
      if (MODE == 1) {
        atomicMax(stats, __float_as_uint(m));
        atomicMax(stats + 4, __float_as_uint(ma));
      }
      atomicMax(stats + 5, __float_as_uint(mr));
    }
  }
}

// -(h, m, l) of s t ||x||^2 / alpha in fp16 (core-matrix layout) from the
// fp32 norms; padding rows -inf.  Also folds the chunk's residual max into
// the global one (stats[2]).
__global__ void ext_f16_kernel(const float* __restrict__ xn, int64_t rows, int64_t rows_pad,
                               unsigned* __restrict__ stats, uint8_t* __restrict__ ext) {
  const float* sc = reinterpret_cast<const float*>(stats + kF16Slot);
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) atomicMax(stats + 2, stats[5]);
  if (r >= rows_pad) return;
  __half e[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) e[j] = __float2half(0.f);
  if (r < rows) {
    const double V = (double)sc[0] * (double)sc[1] * (double)xn[r] / (double)sc[2];
    const __half h0 = __double2half(V);
    const double r1 = V - (double)__half2float(h0);
    const __half h1 = __double2half(r1);
    const __half h2 = __double2half(r1 - (double)__half2float(h1));
    e[0] = __hneg(h0);
    e[1] = __hneg(h1);
    e[2] = __hneg(h2);
  } else {
    e[0] = __float2half(-INFINITY);
  }
  uint8_t* base = ext + (r >> 8) * 8192 + ((r & 255) >> 3) * 256 + (r & 7) * 16;
  *reinterpret_cast<uint4*>(base) = *reinterpret_cast<const uint4*>(e);
  *reinterpret_cast<uint4*>(base + 128) = make_uint4(0u, 0u, 0u, 0u);
}

// Grid of a grid-stride kernel: at most one full wave of resident blocks
// (occupancy queried once per kernel), so no partial second wave runs at a
// fraction of the SMs' bandwidth.
template <auto Kern>
static unsigned resident_grid(int threads, int64_t want) {
  static int cap = 0;
  if (!cap) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, Kern, threads, 0);
    cap = std::max(1, per_sm) * sms;
  }
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, cap));
}

template <typename T, int MODE>
static void f16_rows_launch(const void* src, int64_t rows, int64_t d, double* n64, float* n32,
                            float* norm32, float* resid, unsigned* stats, __half* hi,
                            int64_t rows_pad, int64_t d_pad, bool norm, cudaStream_t st) {
  // lanes per row: at d_pad = 128 each lane converts two 8-column groups
  // (loads of both issued together): 150 -> 116 us at C2 against 16 lanes x 1
  const int G = d_pad <= 128 ? 8 : 32;
  const int64_t want = ceil_div(rows_pad * G, 256);
#define TB_F16(GG, NN)                                                                   \
  do {                                                                                     \
    rows_f16_kernel<T, GG, NN, MODE, false>                                                \
        <<<resident_grid<rows_f16_kernel<T, GG, NN, MODE, false>>(256, want), 256, 0, st>>>( \
            (const T*)src, rows, d, n64, n32, norm32, resid, stats, hi, rows_pad, d_pad);  \
    if (!NN)                                                                               \
      rows_f16_kernel<T, GG, false, MODE, true>                                            \
          <<<resident_grid<rows_f16_kernel<T, GG, false, MODE, true>>(256, want), 256, 0,  \
             st>>>((const T*)src, rows, d, n64, n32, norm32, resid, stats, hi, rows_pad,   \
                   d_pad);                                                                 \
  } while (0)
  if (G == 8) {
    if (norm) TB_F16(8, true); else TB_F16(8, false);
  } else {
    if (norm) TB_F16(32, true); else TB_F16(32, false);
  }
#undef TB_F16
}

// Sample mean of the first S database rows and the decision to centre
// (one block): centre when ||mu||^2 exceeds half the mean ||x - mu||^2 of the
// sample, i.e. when a common offset would dominate the norms that scale the
// certified rounding bound.  mu is stored as fp64 at stats + 64 words.
constexpr int kCenterBlocks = 64, kCenterRows = 32;       // sample = 2048 rows
// stage 1: block b sums rows [b*128, b*128+128) of the sample per column
// (coalesced) and the squared norms; partials at stats + 64 + 2 d words
template <typename T>
__global__ void __launch_bounds__(1024)
f16_center_partial_kernel(const T* __restrict__ x, int64_t S, int64_t d,
                          unsigned* __restrict__ stats) {
  double* part = reinterpret_cast<double*>(stats + 64) + d;      // [kCenterBlocks][d + 1]
  __shared__ double colsum[1024];
  __shared__ double sq;
  const int tid = threadIdx.x;
  const int P = (int)blockDim.x / (int)d;
  const int c = tid % (int)d, lp = tid / (int)d;
  if (tid == 0) sq = 0.0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kCenterRows;
  const int64_t r1 = std::min<int64_t>(S, r0 + kCenterRows);
  double sx = 0.0, sxx = 0.0;
  if (lp < P)
    for (int64_t r = r0 + lp; r < r1; r += P) {
      const double v = (double)x[r * d + c];
      sx += v;
      sxx = fma(v, v, sxx);
    }
  colsum[tid] = lp < P ? sx : 0.0;
  const double wsq = warp_sum(lp < P ? sxx : 0.0);        // one shared atomic per warp
  if ((tid & 31) == 0) atomicAdd(&sq, wsq);
  __syncthreads();
  if (tid < d) {
    double a = 0.0;
    for (int pp = 0; pp < P; ++pp) a += colsum[pp * d + tid];
    part[blockIdx.x * (d + 1) + tid] = a;
  }
  if (tid == 0) part[blockIdx.x * (d + 1) + d] = sq;
}

// stage 2 (one block): fixed-order combination -> mu, ||mu||^2, mean
// ||x - mu||^2 over the sample, the centring decision and max |mu|
__global__ void __launch_bounds__(1024)
f16_center_final_kernel(int64_t S, int64_t d, int nb, unsigned* __restrict__ stats) {
  double* mu = reinterpret_cast<double*>(stats + 64);
  const double* part = mu + d;
  __shared__ double red[2];
  __shared__ double acc[1024];
  const int tid = threadIdx.x;
  const int P = (int)blockDim.x / (int)d;
  const int c = tid % (int)d, lp = tid / (int)d;
  if (tid == 0) red[0] = red[1] = 0.0;
  double a = 0.0;
  if (lp < P)
    for (int bb = lp; bb < nb; bb += P) a += part[bb * (d + 1) + c];   // fixed order
  acc[tid] = a;
  __syncthreads();
  double mm = 0.0;
  float am = 0.f;
  if (tid < d) {
    double t = 0.0;
    for (int pp = 0; pp < P; ++pp) t += acc[pp * d + tid];
    t /= (double)S;
    mu[tid] = t;
    mm = t * t;
    am = __double2float_ru(fabs(t));
  }
  mm = warp_sum(mm);
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  if ((tid & 31) == 0) {
    atomicAdd(&red[0], mm);
    atomicMax(stats + 15, __float_as_uint(am));
  }
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
    for (int bb = 0; bb < nb; ++bb) sq += part[bb * (d + 1) + d];
    const double spread = sq / (double)S - red[0];        // mean ||x_r - mu||^2
    stats[14] = red[0] > 0.5 * spread ? 1u : 0u;
  }
}

int launch_f16_center(int dtype, const void* x, int64_t rows, int64_t d, unsigned* stats,
                      cudaStream_t st) {
  const int64_t S = std::min<int64_t>(rows, (int64_t)kCenterBlocks * kCenterRows);
  if (S <= 0 || d > 1024) return TB_OK;
  const unsigned threads = (unsigned)(1024 / d * d);
  const int nb = (int)ceil_div(S, kCenterRows);
  if (dtype == TB_F32)
    f16_center_partial_kernel<float><<<nb, threads, 0, st>>>((const float*)x, S, d, stats);
  else
    f16_center_partial_kernel<double><<<nb, threads, 0, st>>>((const double*)x, S, d, stats);
  f16_center_final_kernel<<<1, threads, 0, st>>>(S, d, nb, stats);
  TB_LAUNCH_CHECK("f16_center");
  return TB_OK;
}

template <typename T>
static int f16_query_prep(const void* q, int64_t m, int64_t d, double* qn64, float* qnorm,
                          float* qln, unsigned* stats, __half* qhi, int64_t m_pad,
                          int64_t d_pad, int metric, cudaStream_t st) {
  if (d_pad % 64) return fail(TB_ERR_UNSUPPORTED, "tensor-core prep needs d_pad % 64 == 0");
  TB_CUDA_TRY(cudaMemsetAsync(stats + 3, 0, 4, st));
  if (metric != TB_METRIC_COSINE && m > 0) {
    const int64_t n = m * d;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, 256 * 4), 148 * 2);
    if (sizeof(T) == 4)
      absmax_f32_kernel<<<blocks, 256, 0, st>>>((const float*)q, n, stats + 3);
    else
      absmax_f64_kernel<<<blocks, 256, 0, st>>>((const double*)q, n, stats + 3);
    TB_LAUNCH_CHECK("absmax");
  }
  f16_scales_kernel<<<1, 1, 0, st>>>(stats, d, 0, metric);
  TB_LAUNCH_CHECK("f16_scales");
  f16_rows_launch<T, 0>(q, m, d, qn64, nullptr, qnorm, qln, stats, qhi, m_pad, d_pad,
                        metric == TB_METRIC_COSINE, st);
  TB_LAUNCH_CHECK("rows_f16");
  return TB_OK;
}

template <typename T>
static int f16_db_prep(const void* x, int64_t rows, int64_t d, float* xn, unsigned* stats,
                       __half* xhi, int64_t rows_pad, int64_t d_pad, uint8_t* ext, int metric,
                       cudaStream_t st) {
  if (d_pad % 64) return fail(TB_ERR_UNSUPPORTED, "tensor-core prep needs d_pad % 64 == 0");
  TB_CUDA_TRY(cudaMemsetAsync(stats + 4, 0, 8, st));          // chunk max |x|, max ||xl||
  const bool norm = metric == TB_METRIC_COSINE;
  f16_rows_launch<T, 1>(x, rows, d, nullptr, xn, nullptr, nullptr, stats, xhi, rows_pad,
                        d_pad, norm, st);
  f16_scales_kernel<<<1, 1, 0, st>>>(stats, d, 1, metric);
  f16_rows_launch<T, 2>(x, rows, d, nullptr, xn, nullptr, nullptr, stats, xhi, rows_pad,
                        d_pad, norm, st);
  ext_f16_kernel<<<(unsigned)ceil_div(rows_pad, 256), 256, 0, st>>>(xn, rows, rows_pad, stats,
                                                                    ext);
  TB_LAUNCH_CHECK("rows_f16");
  return TB_OK;
}

int launch_query_prep_f16(int dtype, int metric, const void* q, int64_t m, int64_t d,
                          double* qn64, float* qnorm, float* qln, unsigned* stats,
                          __half* qhi, int64_t m_pad, int64_t d_pad, cudaStream_t st) {
  if (dtype == TB_F32)
    return f16_query_prep<float>(q, m, d, qn64, qnorm, qln, stats, qhi, m_pad, d_pad, metric, st);
  return f16_query_prep<double>(q, m, d, qn64, qnorm, qln, stats, qhi, m_pad, d_pad, metric, st);
}

int launch_db_prep_f16(int dtype, int metric, const void* x, int64_t rows, int64_t d,
                       float* xn, unsigned* stats, __half* xhi, int64_t rows_pad,
                       int64_t d_pad, uint8_t* xext, cudaStream_t st) {
  if (dtype == TB_F32)
    return f16_db_prep<float>(x, rows, d, xn, stats, xhi, rows_pad, d_pad, xext, metric, st);
  return f16_db_prep<double>(x, rows, d, xn, stats, xhi, rows_pad, d_pad, xext, metric, st);
}

int launch_query_prep(int dtype, int metric, const void* q, int64_t m, int64_t d,
                      double* qn64, float* qnorm, __nv_bfloat16* qhi,
                      __nv_bfloat16* qlo, int64_t m_pad, int64_t d_pad,
                      cudaStream_t st, unsigned* centre) {
  // the tensor-core engines use 2q (exact) so that acc' = 2 q.x - ||x||^2
  if (dtype == TB_F32)
    return rows_prep<float>(q, m, d, qn64, nullptr, qnorm, nullptr, qhi, qlo, m_pad, d_pad, st,
                            metric, 2.0, nullptr, centre);
  return rows_prep<double>(q, m, d, qn64, nullptr, qnorm, nullptr, qhi, qlo, m_pad, d_pad, st,
                           metric, 2.0, nullptr, centre);
}

int launch_db_prep(int dtype, int metric, const void* x, int64_t rows, int64_t d,
                   float* xn, unsigned* xmax_bits, __nv_bfloat16* xhi,
                   __nv_bfloat16* xlo, int64_t rows_pad, int64_t d_pad,
                   uint8_t* xext, cudaStream_t st) {
  // xmax_bits is the stats block, which also carries the centring decision
  if (dtype == TB_F32)
    return rows_prep<float>(x, rows, d, nullptr, xn, nullptr, xmax_bits, xhi, xlo, rows_pad, d_pad,
                            st, metric, 1.0, xext, xhi ? xmax_bits : nullptr);
  return rows_prep<double>(x, rows, d, nullptr, xn, nullptr, xmax_bits, xhi, xlo, rows_pad, d_pad,
                           st, metric, 1.0, xext, xhi ? xmax_bits : nullptr);
}

// ------------------------------------------------- SIMT candidate engine --
// CTA = 128 queries x one database slice; 256 threads, 8x8 fp32 micro-tile
// per thread over 128x128 score tiles; the score tile is staged in shared
// memory and scanned by 256 threads (query row tid&127, column half tid>>7)
// that each keep a register top-K' list.  Output: 2 lists per slice.
constexpr int kSimtTile = 128;
constexpr int kSimtLd = 132;   // padded k-major operand rows
constexpr int kSimtSt = 129;   // padded score rows
constexpr size_t kSimtSmem = (2 * 16 * kSimtLd + kSimtTile * kSimtSt) * sizeof(float);

// L1 = true: the tile accumulates sum |q - x| (no tensor-core form) and the
// score is that sum; otherwise the L2 cross term and ||x||^2 - 2 q.x.
template <typename T, int KC, bool L1>
__global__ void __launch_bounds__(256, 1)
knn_simt_kernel(const T* __restrict__ x, const T* __restrict__ q,
                const float* __restrict__ xn, int64_t rows, int m, int d,
                int64_t rows_per_slice, int idx_base, float* __restrict__ cand_s,
                int* __restrict__ cand_i) {
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                    // [16][kSimtLd]  queries, k-major
  float* Bs = As + 16 * kSimtLd;       // [16][kSimtLd]  database rows
  float* St = Bs + 16 * kSimtLd;       // [128][kSimtSt] scores

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int q0 = blockIdx.x * kSimtTile;
  const int64_t r_begin = (int64_t)blockIdx.y * rows_per_slice;
  const int64_t r_end = min(rows, r_begin + rows_per_slice);
  const int srow = tid & 127, shalf = tid >> 7;
  const int lr = tid >> 1, lc = (tid & 1) * 8;
  const bool qvalid = (q0 + lr) < m;
  const T* qrow = q + (int64_t)(q0 + (qvalid ? lr : 0)) * d;

  TopList<float, KC> L;
  L.init();

  for (int64_t t0 = r_begin; t0 < r_end; t0 += kSimtTile) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    const bool xvalid = (t0 + lr) < r_end;
    const T* xrow = x + (t0 + (xvalid ? lr : 0)) * d;
    float ra[8], rb[8];
    auto load = [&](int kk) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = kk + lc + j;
        ra[j] = (qvalid && c < d) ? (float)qrow[c] : 0.f;
        rb[j] = (xvalid && c < d) ? (float)xrow[c] : 0.f;
      }
    };
    load(0);
    for (int kk = 0; kk < d; kk += 16) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        As[(lc + j) * kSimtLd + lr] = ra[j];
        Bs[(lc + j) * kSimtLd + lr] = rb[j];
      }
      __syncthreads();
      if (kk + 16 < d) load(kk + 16);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[c * kSimtLd + ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[c * kSimtLd + ty * 8 + 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[c * kSimtLd + tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[c * kSimtLd + 64 + tx * 4]);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            acc[i][j] = L1 ? acc[i][j] + fabsf(a[i] - b[j]) : fmaf(a[i], b[j], acc[i][j]);
      }
    }
    // epilogue: score = ||x||^2 - 2 q.x, staged for the scan
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4);
        const int64_t g = t0 + col;
        St[(ty * 8 + i) * kSimtSt + col] =
            g < r_end ? (L1 ? acc[i][j] : fmaf(-2.f, acc[i][j], xn[g])) : INFINITY;
      }
    __syncthreads();
    if (q0 + srow < m) {
      const float* srow_p = St + srow * kSimtSt + shalf * 64;
      const int base = idx_base + (int)(t0 + shalf * 64);
#pragma unroll 1
      for (int cb = 0; cb < 64; cb += 32) {
        const float thr = L.worst();
        float sc[32];
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sc[j] = srow_p[cb + j];
          mask |= (sc[j] < thr ? 1u : 0u) << j;
        }
        if (mask) insert_masked(L, sc, mask, base + cb);
      }
    }
  }
  if (q0 + srow < m) {
    const int64_t o = (((int64_t)blockIdx.y * 2 + shalf) * m + q0 + srow) * KC;
#pragma unroll
    for (int p = 0; p < KC; ++p) {
      cand_s[o + p] = L.s[p];
      cand_i[o + p] = L.i[p];
    }
  }
}

template <typename T, int KC, bool L1>
static int simt_launch(const void* x, const void* q, const float* xn,
                       int64_t rows, int64_t m, int64_t d, int slices,
                       int idx_base, float* cs, int* ci, cudaStream_t st) {
  TB_CUDA_TRY(cudaFuncSetAttribute(knn_simt_kernel<T, KC, L1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kSimtSmem));
  const int64_t rps = round_up(ceil_div(rows, slices), kSimtTile);
  dim3 grid((unsigned)ceil_div(m, kSimtTile), (unsigned)slices);
  knn_simt_kernel<T, KC, L1><<<grid, 256, kSimtSmem, st>>>(
      (const T*)x, (const T*)q, xn, rows, (int)m, (int)d, rps, idx_base, cs, ci);
  TB_LAUNCH_CHECK("knn_simt");
  return TB_OK;
}

int launch_knn_simt(int dtype, int metric, int cand, const void* x, const void* q,
                    const float* xn, int64_t rows, int64_t m, int64_t d,
                    int slices, int idx_base, float* cs, int* ci,
                    cudaStream_t st) {
  if (metric == TB_METRIC_COSINE)
    return fail(TB_ERR_UNSUPPORTED, "SIMT engine: cosine runs on the tensor-core engine");
  const bool l1 = metric == TB_METRIC_L1;
#define TB_SIMT_CASE(KC)                                                                     \
  case KC:                                                                                   \
    if (dtype == TB_F32)                                                                     \
      return l1 ? simt_launch<float, KC, true>(x, q, xn, rows, m, d, slices, idx_base, cs, ci, st) \
                : simt_launch<float, KC, false>(x, q, xn, rows, m, d, slices, idx_base, cs, ci, st); \
    return l1 ? simt_launch<double, KC, true>(x, q, xn, rows, m, d, slices, idx_base, cs, ci, st) \
              : simt_launch<double, KC, false>(x, q, xn, rows, m, d, slices, idx_base, cs, ci, st);
  switch (cand) {
    TB_SIMT_CASE(16)
    TB_SIMT_CASE(32)
    TB_SIMT_CASE(64)
  }
#undef TB_SIMT_CASE
  return fail(TB_ERR_UNSUPPORTED, "SIMT engine: unsupported candidate count");
}

// ------------------------------------------------------- candidate merge --
template <int KC>
__global__ void knn_merge_kernel(const float* __restrict__ in_s,
                                 const int* __restrict__ in_i, int lists,
                                 const float* __restrict__ prev_s,
                                 const int* __restrict__ prev_i, int64_t m,
                                 float* __restrict__ out_s, int* __restrict__ out_i) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= m) return;
  const int total = lists + (prev_s ? 1 : 0);
  float* os = out_s + r * KC;
  int* oi = out_i + r * KC;
  if (KC <= 32 && total <= 32) {
    // one sorted list per lane, held in registers: KC rounds of a warp-wide
    // lexicographic argmin over the list heads; the winning lane pops
    float v[KC];
    int j[KC];
    if (lane < total) {
      const float* s = lane < lists ? in_s + ((int64_t)lane * m + r) * KC : prev_s + r * KC;
      const int* ix = lane < lists ? in_i + ((int64_t)lane * m + r) * KC : prev_i + r * KC;
#pragma unroll
      for (int u = 0; u < KC / 4; ++u) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(s) + u);
        const int4 b = __ldg(reinterpret_cast<const int4*>(ix) + u);
        v[4 * u] = a.x; v[4 * u + 1] = a.y; v[4 * u + 2] = a.z; v[4 * u + 3] = a.w;
        j[4 * u] = b.x; j[4 * u + 1] = b.y; j[4 * u + 2] = b.z; j[4 * u + 3] = b.w;
      }
    } else {
#pragma unroll
      for (int p = 0; p < KC; ++p) {
        v[p] = INFINITY;
        j[p] = kInvalidIdx;
      }
    }
#pragma unroll 1
    for (int t = 0; t < KC; ++t) {
      float bv = v[0];
      int bj = j[0];
      warp_lex_min(bv, bj);
      if (bj != kInvalidIdx && j[0] == bj && v[0] == bv) {   // indices are unique
#pragma unroll
        for (int p = 0; p < KC - 1; ++p) {
          v[p] = v[p + 1];
          j[p] = j[p + 1];
        }
        v[KC - 1] = INFINITY;
        j[KC - 1] = kInvalidIdx;
      }
      if (lane == 0) {
        os[t] = bv;
        oi[t] = bj;
      }
    }
    return;
  }
  TopList<float, KC> L;
  L.init();
  for (int l = lane; l < total; l += 32) {
    const float* s = l < lists ? in_s + ((int64_t)l * m + r) * KC : prev_s + r * KC;
    const int* ix = l < lists ? in_i + ((int64_t)l * m + r) * KC : prev_i + r * KC;
    for (int p = 0; p < KC; ++p) {
      const float v = s[p];
      const int j = ix[p];
      if (!lex_less(v, j, L.worst(), L.worst_idx())) break;  // lists are sorted
      L.insert(v, j);
    }
  }
  warp_drain(L, KC, [&](int t, float v, int j) {
    os[t] = v;
    oi[t] = j;
  });
}

int launch_knn_merge(int cand, const float* in_s, const int* in_i, int lists,
                     const float* prev_s, const int* prev_i, int64_t m,
                     float* out_s, int* out_i, cudaStream_t st) {
  if (m <= 0) return TB_OK;
  const int warps = 4;
  const unsigned blocks = (unsigned)ceil_div(m, warps);
  switch (cand) {
    case 16: knn_merge_kernel<16><<<blocks, warps * 32, 0, st>>>(in_s, in_i, lists, prev_s, prev_i, m, out_s, out_i); break;
    case 32: knn_merge_kernel<32><<<blocks, warps * 32, 0, st>>>(in_s, in_i, lists, prev_s, prev_i, m, out_s, out_i); break;
    case 64: knn_merge_kernel<64><<<blocks, warps * 32, 0, st>>>(in_s, in_i, lists, prev_s, prev_i, m, out_s, out_i); break;
    default: return fail(TB_ERR_UNSUPPORTED, "merge: unsupported candidate count");
  }
  TB_LAUNCH_CHECK("knn_merge");
  return TB_OK;
}

// Exact fp64 distance of one (query row, data row) pair in the reference
// graph's formula (frontend.py:57-73): sum (q-x)^2, sum |q-x|, or
// 1 - q.x / (|q| |x|).  Warp-cooperative (lane-strided over d); every lane
// returns the same value.
template <typename T, int MET>
__device__ __forceinline__ double exact_dist_warp(const T* __restrict__ qr,
                                                  const T* __restrict__ xr, int64_t d,
                                                  int lane) {
  if (MET == TB_METRIC_COSINE) {
    double dot = 0.0, qq = 0.0, xx = 0.0;
    for (int64_t t = lane; t < d; t += 32) {
      const double a = (double)qr[t], b = (double)xr[t];
      dot = fma(a, b, dot);
      qq = fma(a, a, qq);
      xx = fma(b, b, xx);
    }
    dot = warp_sum(dot);
    qq = warp_sum(qq);
    xx = warp_sum(xx);
    return 1.0 - dot / (sqrt(qq) * sqrt(xx));
  }
  double acc = 0.0;
  for (int64_t t = lane; t < d; t += 32) {
    const double df = (double)qr[t] - (double)xr[t];
    acc = MET == TB_METRIC_L1 ? acc + fabs(df) : fma(df, df, acc);
  }
  return warp_sum(acc);
}

// --------------------------------------------- exact re-rank + certify --
// One warp per query.  Exact fp64 sum((q - x)^2) for the K' candidates,
// sorted by (distance, index); the k best are the answer.  Certified when
// every point outside the candidate set provably ranks after the k-th:
//   approx(j) >= T* (K'-th merged approx score)   and
//   |approx - exact| <= E = c1 ||q|| max||x|| + c2 max||x||^2
// => need T* - E > exact_score(k-th).  Otherwise the query goes to the
// exact fallback.  Per metric (engine score s~ vs exact distance):
//   l2:     s~ = ||x||^2 - 2q.x,        E = c1 |q| X + c2 X^2, score_k = kth - ||q||^2
//   cosine: s~ = 1 - 2 q^.x^ (unit rows), same E with |q| = X = 1, score_k = 2 kth - 1
//   l1:     s~ = fp32 sum |q-x| (SIMT):  outside s >= s~/(1+c1) - c2 (|q|_1 + X_1)
template <typename T, typename OT, int KC, int MET>
__global__ void knn_refine_kernel(const float* __restrict__ cs,
                                  const int* __restrict__ ci,
                                  const T* __restrict__ x, const T* __restrict__ q,
                                  const double* __restrict__ qn64,
                                  const float* __restrict__ qnorm,
                                  const float* __restrict__ qln,
                                  unsigned* __restrict__ stats, int64_t m,
                                  int64_t d, int k, double c1, double c2,
                                  OT* __restrict__ out_dist,
                                  int64_t* __restrict__ out_idx,
                                  int64_t index_base, int* __restrict__ fb_list) {
  constexpr int PER = (KC + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= m) return;
  const T* qr = q + r * d;
  double ds[PER];
  int js[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    ds[p] = INFINITY;
    js[p] = kInvalidIdx;
  }
  if (sizeof(T) == 4 && MET == TB_METRIC_L2 && d <= 128 && (d & 3) == 0) {
    // f32 rows of <= 128 columns: one float4 per lane per row, and the rows
    // of 8 candidates in flight at once (the generic loop below waits for
    // each gathered row in turn)
    const bool act = lane * 4 < d;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 qv = act ? __ldg(reinterpret_cast<const float4*>(qr) + lane) : z4;
    int jv[PER];
#pragma unroll
    for (int p = 0; p < PER; ++p)
      jv[p] = p * 32 + lane < KC ? ci[r * KC + p * 32 + lane] : kInvalidIdx;
    constexpr int B = KC < 8 ? KC : 8;
#pragma unroll
    for (int c0 = 0; c0 < KC; c0 += B) {
      float4 xv[B];
      int jj[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int c = c0 + u;
        jj[u] = __shfl_sync(0xffffffffu, jv[c >> 5], c & 31);
        xv[u] = act && jj[u] != kInvalidIdx
                    ? __ldg(reinterpret_cast<const float4*>(
                                reinterpret_cast<const float*>(x) + (int64_t)jj[u] * d) + lane)
                    : z4;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int c = c0 + u;
        const double e0 = (double)qv.x - (double)xv[u].x, e1 = (double)qv.y - (double)xv[u].y;
        const double e2 = (double)qv.z - (double)xv[u].z, e3 = (double)qv.w - (double)xv[u].w;
        const double acc = warp_sum(fma(e3, e3, fma(e2, e2, fma(e1, e1, e0 * e0))));
        if ((c & 31) == lane) {
          ds[c >> 5] = jj[u] != kInvalidIdx ? acc : INFINITY;
          js[c >> 5] = jj[u];
        }
      }
    }
  } else {
    for (int c = 0; c < KC; ++c) {
      const int j = ci[r * KC + c];
      double acc = 0.0;
      if (j != kInvalidIdx) acc = exact_dist_warp<T, MET>(qr, x + (int64_t)j * d, d, lane);
      if ((c & 31) == lane) {
#pragma unroll
        for (int p = 0; p < PER; ++p)
          if (p == (c >> 5)) {
            ds[p] = j != kInvalidIdx ? acc : INFINITY;
            js[p] = j;
          }
      }
    }
  }
  double kth = INFINITY;
  for (int t = 0; t < k; ++t) {
    double v = INFINITY;
    int j = kInvalidIdx;
#pragma unroll
    for (int p = 0; p < PER; ++p)
      if (lex_less(ds[p], js[p], v, j)) {
        v = ds[p];
        j = js[p];
      }
    warp_lex_min(v, j);
#pragma unroll
    for (int p = 0; p < PER; ++p)
      if (js[p] == j && ds[p] == v) {
        ds[p] = INFINITY;
        js[p] = kInvalidIdx;
      }
    if (lane == 0) {
      out_dist[r * k + t] = (OT)v;
      out_idx[r * k + t] = (int64_t)j + index_base;
    }
    kth = v;
  }
  if (lane == 0) {
    const float tstar = cs[r * KC + KC - 1];
    if (isfinite(tstar)) {
      const double X = (double)__uint_as_float(stats[0]);
      bool ok;
      if (MET == TB_METRIC_L1) {
        ok = (double)tstar / (1.0 + c1) - c2 * ((double)qnorm[r] + X) > kth;
      } else {
        // Norm split (l2): every row with ||x|| > R >= ||q|| has exact score
        // ||x||^2 - 2 q.x >= R^2 - 2 ||q|| R, which exceeds the k-th exact
        // score kth - ||q||^2 once R > ||q|| + sqrt(kth); only rows with
        // ||x|| <= R need the rounding bound, evaluated at R instead of the
        // largest norm in the database (outliers no longer widen E).
        const double qn = (double)qnorm[r];
        double R = X;
        if (MET == TB_METRIC_L2) {
          const double Rq = (qn + sqrt(fmax(kth, 0.0))) * (1.0 + 1e-9);
          if (Rq < X) R = Rq;
        }
        double E = c1 * qn * R + c2 * R * R;
        if (qln) {
          // fp16 single pass: measured rounding residuals (Cauchy-Schwarz),
          // |q.x - q'.x'| <= ||q|| XL + ||ql|| (R + 3 XL), times 2 for -2 q.x;
          // rows with ||x|| <= R have ||xl|| <= 2^-11 ||x|| + sqrt(d) 2^-25 / t
          double XL = (double)__uint_as_float(stats[2]);
          if (R < X)
            XL = fmin(XL, (0x1p-11 * R + sqrt((double)d) * 0x1p-25 *
                                             (double)__uint_as_float(stats[13])) * (1.0 + 1e-6));
          E += 2.0 * (1.0 + 1e-6) * (qn * XL + (double)qln[r] * (R + 3.0 * XL));
        }
        const double exact_score_k = MET == TB_METRIC_COSINE ? 2.0 * kth - 1.0 : kth - qn64[r];
        ok = (double)tstar - E > exact_score_k;
      }
      if (!ok) {
        const int pos = atomicAdd(reinterpret_cast<int*>(&stats[1]), 1);
        fb_list[pos] = (int)r;
        fb_bounds(fb_list, m)[pos] = kth;     // the true k-th distance is <= kth
        fb_hits(fb_list, m)[pos] = 0;
      }
    }
  }
}

template <typename T, typename OT, int MET>
static int refine_dispatch(int cand, const float* cs, const int* ci,
                           const void* x, const void* q, const double* qn64,
                           const float* qnorm, const float* qln, unsigned* stats, int64_t m,
                           int64_t d, int64_t k, double c1, double c2,
                           void* od, int64_t* oi, int64_t base, int* fb,
                           cudaStream_t st) {
  const int warps = 4;
  const unsigned blocks = (unsigned)ceil_div(m, warps);
#define TB_REFINE_CASE(KC)                                                   \
  case KC:                                                                   \
    knn_refine_kernel<T, OT, KC, MET><<<blocks, warps * 32, 0, st>>>(        \
        cs, ci, (const T*)x, (const T*)q, qn64, qnorm, qln, stats, m, d, (int)k,  \
        c1, c2, (OT*)od, oi, base, fb);                                      \
    break;
  switch (cand) {
    TB_REFINE_CASE(16)
    TB_REFINE_CASE(32)
    TB_REFINE_CASE(64)
    default: return fail(TB_ERR_UNSUPPORTED, "refine: unsupported candidate count");
  }
#undef TB_REFINE_CASE
  TB_LAUNCH_CHECK("knn_refine");
  return TB_OK;
}

int launch_knn_refine(int dtype, int out_dtype, int metric, int cand, const float* cs,
                      const int* ci, const void* x, const void* q,
                      const double* qn64, const float* qnorm, const float* qln,
                      const unsigned* stats, int64_t n, int64_t m, int64_t d,
                      int64_t k, double c1, double c2, void* out_dist,
                      int64_t* out_idx, int64_t index_base, int* fb_list,
                      cudaStream_t st) {
  (void)n;
  if (m <= 0) return TB_OK;
  unsigned* s = const_cast<unsigned*>(stats);
#define TB_REF(T, OT, MET)                                                                  \
  return refine_dispatch<T, OT, MET>(cand, cs, ci, x, q, qn64, qnorm, qln, s, m, d, k, c1, c2,   \
                                     out_dist, out_idx, index_base, fb_list, st)
#define TB_REF_MET(T, OT)                                        \
  if (metric == TB_METRIC_L1) TB_REF(T, OT, TB_METRIC_L1);       \
  if (metric == TB_METRIC_COSINE) TB_REF(T, OT, TB_METRIC_COSINE); \
  TB_REF(T, OT, TB_METRIC_L2)
  if (dtype == TB_F32) {
    if (out_dtype == TB_F32) { TB_REF_MET(float, float); }
    TB_REF_MET(float, double);
  }
  if (out_dtype == TB_F32) { TB_REF_MET(double, float); }
  TB_REF_MET(double, double);
#undef TB_REF_MET
#undef TB_REF
}

// ------------------------------------------------- exact fp64 fallback --
// Uncertified queries (count = stats[1], normally 0) are brute-forced in
// fp64 with direct differences.  The grid is sized on the host without
// knowing count: each of the G blocks derives S = max(1, G / count) database
// slices per query and takes units u = slice * count + p (slice-major, so
// concurrently running blocks scan the same rows for different queries and
// share them through L2).  One warp per database row (lane-strided over d,
// coalesced), a per-warp top-KC, merged per block into scratch[u]; then
// knn_fallback_merge combines the S lists of each query.
template <typename T, int KC, int MET>
__global__ void __launch_bounds__(256)
knn_fallback_partial_kernel(const T* __restrict__ x, const T* __restrict__ q, int64_t n,
                            int64_t d, const unsigned* __restrict__ stats,
                            const int* __restrict__ fb_list, double* __restrict__ sc_d,
                            int* __restrict__ sc_i) {
  __shared__ double sd[8][KC];
  __shared__ int si[8][KC];
  const int count = *reinterpret_cast<const volatile int*>(stats);
  if (count == 0) return;
  const int S = max(1, (int)gridDim.x / count);
  const int units = count * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int slice = u / count, p = u - slice * count;
    const int64_t r = fb_list[p];
    const T* qr = q + r * d;
    const int64_t j0 = n * slice / S, j1 = n * (slice + 1) / S;
    TopList<double, KC> L;
    L.init();
    for (int64_t j = j0 + warp; j < j1; j += 8)
      L.offer(exact_dist_warp<T, MET>(qr, x + j * d, d, lane), (int)j);   // same in every lane
    if (lane == 0)
      for (int t = 0; t < KC; ++t) {
        sd[warp][t] = L.s[t];
        si[warp][t] = L.i[t];
      }
    __syncthreads();
    if (warp == 0) {
      TopList<double, KC> M;
      M.init();
      if (lane < 8)
        for (int t = 0; t < KC; ++t) M.offer(sd[lane][t], si[lane][t]);
      warp_drain(M, KC, [&](int t, double v, int j) {
        sc_d[(int64_t)u * KC + t] = v;
        sc_i[(int64_t)u * KC + t] = j;
      });
    }
    __syncthreads();
  }
}

// Short rows (d <= 64): one database row per THREAD (the query staged in
// shared memory, the row read from L1/L2 element by element, no shuffles),
// a register top-K' per lane, the warp's K' best by a warp-wide k-way merge,
// then the block's K' best as above.  Same fp64 formulas as
// exact_dist_warp, summed serially.  ~10x fewer instructions per row than
// the warp-per-row kernel for small d, where uncertified queries are usually
// many (e.g. clustered data).
template <typename T, int KC, int MET, int DMAX>
__global__ void __launch_bounds__(256)
knn_fallback_rows_kernel(const T* __restrict__ x, const T* __restrict__ q, int64_t n,
                         int64_t d, const unsigned* __restrict__ stats,
                         const int* __restrict__ fb_list, double* __restrict__ sc_d,
                         int* __restrict__ sc_i) {
  __shared__ double qs[DMAX];
  __shared__ double qq_s;
  __shared__ double sd[8][KC];
  __shared__ int si[8][KC];
  const int count = *reinterpret_cast<const volatile int*>(stats);
  if (count == 0) return;
  const int S = max(1, (int)gridDim.x / count);
  const int units = count * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int slice = u / count, p = u - slice * count;
    const int64_t r = fb_list[p];
    for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = (double)q[r * d + c];
    __syncthreads();
    if (threadIdx.x == 0 && MET == TB_METRIC_COSINE) {
      double a = 0.0;
      for (int c = 0; c < d; ++c) a = fma(qs[c], qs[c], a);
      qq_s = a;
    }
    __syncthreads();
    const int64_t j0 = n * slice / S, j1 = n * (slice + 1) / S;
    TopList<double, KC> L;
    L.init();
    for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const T* xr = x + j * d;
      double acc = 0.0, xx = 0.0;
      auto term = [&](int c, double b) {
        if (MET == TB_METRIC_COSINE) {
          acc = fma(qs[c], b, acc);
          xx = fma(b, b, xx);
        } else {
          const double df = qs[c] - b;
          acc = MET == TB_METRIC_L1 ? acc + fabs(df) : fma(df, df, acc);
        }
      };
      if (sizeof(T) == 4 && (d & 15) == 0) {
        // 16-byte loads, four in flight per step (rows are 16-byte aligned)
        for (int c = 0; c < d; c += 16) {
          float4 v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = __ldg(reinterpret_cast<const float4*>(xr + c) + e);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            term(c + 4 * e, v[e].x);
            term(c + 4 * e + 1, v[e].y);
            term(c + 4 * e + 2, v[e].z);
            term(c + 4 * e + 3, v[e].w);
          }
        }
      } else {
        for (int c = 0; c < d; ++c) term(c, (double)xr[c]);
      }
      const double dist = MET == TB_METRIC_COSINE ? 1.0 - acc / (sqrt(qq_s) * sqrt(xx)) : acc;
      L.offer(dist, (int)j);
    }
    warp_drain(L, KC, [&](int t, double v, int jj) {
      sd[warp][t] = v;
      si[warp][t] = jj;
    });
    __syncthreads();
    if (warp == 0) {
      TopList<double, KC> M;
      M.init();
      if (lane < 8)
        for (int t = 0; t < KC; ++t) M.offer(sd[lane][t], si[lane][t]);
      warp_drain(M, KC, [&](int t, double v, int jj) {
        sc_d[(int64_t)u * KC + t] = v;
        sc_i[(int64_t)u * KC + t] = jj;
      });
    }
    __syncthreads();
  }
}

template <typename OT, int KC>
__global__ void knn_fallback_merge_kernel(const unsigned* __restrict__ stats,
                                          const int* __restrict__ fb_list, int G, int k,
                                          const double* __restrict__ sc_d,
                                          const int* __restrict__ sc_i,
                                          OT* __restrict__ out_dist,
                                          int64_t* __restrict__ out_idx, int64_t index_base) {
  const int count = *reinterpret_cast<const volatile int*>(stats);
  const int S = count ? max(1, G / count) : 1;
  const int lane = threadIdx.x & 31;
  for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < count;
       p += gridDim.x * (blockDim.x >> 5)) {
    const int64_t r = fb_list[p];
    TopList<double, KC> M;
    M.init();
    for (int sl = lane; sl < S; sl += 32) {
      const int64_t u = (int64_t)sl * count + p;
      for (int t = 0; t < KC; ++t) M.offer(sc_d[u * KC + t], sc_i[u * KC + t]);
    }
    warp_drain(M, k, [&](int t, double v, int j) {
      out_dist[r * k + t] = (OT)v;
      out_idx[r * k + t] = (int64_t)j + index_base;
    });
  }
}

// Bounded fallback (the first, fast stage).  The re-rank already holds, for
// every uncertified query, the exact distance of its k-th candidate: an
// upper bound on its true k-th distance.  Blocks take QB such queries (in
// shared memory, fp64) against a slice of the database, one database row
// per thread: each row is read once for the QB queries, QB fp64 distances
// in registers (the re-rank's formulas, summed serially), and a row at or
// below a query's bound is appended to that query's hit buffer - usually
// just its k true neighbours, so no per-row top-K' work.  (The warp-per-row
// brute force below took 0.33 ms per query at 1e6 x 128.)
constexpr int kFbQB = 8;
template <typename T, int MET>
__global__ void __launch_bounds__(256)
knn_fallback_tile_kernel(const T* __restrict__ x, const T* __restrict__ q, int64_t n,
                         int64_t d, const unsigned* __restrict__ cntp,
                         const int* __restrict__ fb_list, const double* __restrict__ fb_bnd,
                         int* __restrict__ hit_cnt, double* __restrict__ hit_d,
                         int* __restrict__ hit_i, int hcap) {
  extern __shared__ __align__(16) double fq[];      // [kFbQB][d]
  __shared__ double bnd[kFbQB], qq[kFbQB];
  const int count = *reinterpret_cast<const volatile int*>(cntp);
  if (count == 0) return;
  const int groups = (count + kFbQB - 1) / kFbQB;
  const int S = max(1, (int)gridDim.x / groups);
  for (int u = blockIdx.x; u < groups * S; u += gridDim.x) {
    const int g = u % groups, slice = u / groups;   // concurrent blocks share a slice (L2)
    __syncthreads();
    for (int64_t e = threadIdx.x; e < kFbQB * d; e += blockDim.x) {
      const int qi = (int)(e / d);
      const int p = g * kFbQB + qi;
      fq[e] = p < count ? (double)q[(int64_t)fb_list[p] * d + (e - (int64_t)qi * d)] : 0.0;
    }
    if (threadIdx.x < kFbQB) {
      const int p = g * kFbQB + threadIdx.x;
      // slack for the summation order (<= 2 d 2^-53 relative for sums of
      // non-negative terms; an absolute 1e-12 for the cosine's 1 - c)
      const double b = p < count ? fb_bnd[p] : -INFINITY;
      bnd[threadIdx.x] = b + 1e-12 * fabs(b) + (MET == TB_METRIC_COSINE ? 1e-12 : 0.0);
    }
    __syncthreads();
    if (MET == TB_METRIC_COSINE && threadIdx.x < kFbQB) {
      double a = 0.0;
      for (int64_t c = 0; c < d; ++c) a = fma(fq[threadIdx.x * d + c], fq[threadIdx.x * d + c], a);
      qq[threadIdx.x] = a;
    }
    __syncthreads();
    const int64_t j0 = n * slice / S, j1 = n * (slice + 1) / S;
    for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const T* xr = x + j * d;
      double acc[kFbQB], xx = 0.0;
#pragma unroll
      for (int qi = 0; qi < kFbQB; ++qi) acc[qi] = 0.0;
      auto term = [&](int64_t c, double b) {
        if (MET == TB_METRIC_COSINE) xx = fma(b, b, xx);
#pragma unroll
        for (int qi = 0; qi < kFbQB; ++qi) {
          const double a = fq[qi * d + c];
          if (MET == TB_METRIC_COSINE) {
            acc[qi] = fma(a, b, acc[qi]);
          } else {
            const double df = a - b;
            acc[qi] = MET == TB_METRIC_L1 ? acc[qi] + fabs(df) : fma(df, df, acc[qi]);
          }
        }
      };
      if (sizeof(T) == 4 && (d & 3) == 0) {
        // 4 row elements per step; each query's 4 values as two 16-byte
        // shared loads (one load per two fp64 updates)
        for (int64_t c = 0; c < d; c += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(xr + c));
          const double b0 = v.x, b1 = v.y, b2 = v.z, b3 = v.w;
          if (MET == TB_METRIC_COSINE) xx = fma(b3, b3, fma(b2, b2, fma(b1, b1, fma(b0, b0, xx))));
#pragma unroll
          for (int qi = 0; qi < kFbQB; ++qi) {
            const double2 a01 = *reinterpret_cast<const double2*>(fq + qi * d + c);
            const double2 a23 = *reinterpret_cast<const double2*>(fq + qi * d + c + 2);
            double t = acc[qi];
            if (MET == TB_METRIC_COSINE) {
              t = fma(a23.y, b3, fma(a23.x, b2, fma(a01.y, b1, fma(a01.x, b0, t))));
            } else if (MET == TB_METRIC_L1) {
              t = (((t + fabs(a01.x - b0)) + fabs(a01.y - b1)) + fabs(a23.x - b2)) + fabs(a23.y - b3);
            } else {
              const double d0 = a01.x - b0, d1 = a01.y - b1, d2 = a23.x - b2, d3 = a23.y - b3;
              t = fma(d3, d3, fma(d2, d2, fma(d1, d1, fma(d0, d0, t))));
            }
            acc[qi] = t;
          }
        }
      } else {
        for (int64_t c = 0; c < d; ++c) term(c, (double)xr[c]);
      }
#pragma unroll
      for (int qi = 0; qi < kFbQB; ++qi) {
        const double dist =
            MET == TB_METRIC_COSINE ? 1.0 - acc[qi] / (sqrt(qq[qi]) * sqrt(xx)) : acc[qi];
        if (dist <= bnd[qi]) {
          const int p = g * kFbQB + qi;
          const int pos = atomicAdd(hit_cnt + p, 1);
          if (pos < hcap) {
            hit_d[(int64_t)p * hcap + pos] = dist;
            hit_i[(int64_t)p * hcap + pos] = (int)j;
          }
        }
      }
    }
  }
}

// The k best hits of each query (ties -> lower index); a query whose hits
// overflowed the buffer (many rows tied at its bound) or came short goes on
// to the exhaustive kernels through the overflow list.
template <typename OT, int KC>
__global__ void knn_fallback_hits_kernel(const unsigned* __restrict__ cntp,
                                         const int* __restrict__ fb_list,
                                         const int* __restrict__ hit_cnt,
                                         const double* __restrict__ hit_d,
                                         const int* __restrict__ hit_i, int hcap, int k,
                                         unsigned* __restrict__ over_cnt,
                                         int* __restrict__ over_list,
                                         OT* __restrict__ out_dist,
                                         int64_t* __restrict__ out_idx, int64_t index_base) {
  const int count = *reinterpret_cast<const volatile int*>(cntp);
  const int lane = threadIdx.x & 31;
  for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < count;
       p += gridDim.x * (blockDim.x >> 5)) {
    const int64_t r = fb_list[p];
    const int h = hit_cnt[p];
    if (h > hcap || h < k) {
      if (lane == 0) over_list[atomicAdd(reinterpret_cast<int*>(over_cnt), 1)] = (int)r;
      continue;
    }
    TopList<double, KC> M;
    M.init();
    for (int t = lane; t < h; t += 32) M.offer(hit_d[(int64_t)p * hcap + t], hit_i[(int64_t)p * hcap + t]);
    warp_drain(M, k, [&](int t, double v, int j) {
      out_dist[r * k + t] = (OT)v;
      out_idx[r * k + t] = (int64_t)j + index_base;
    });
  }
}

template <typename T, typename OT, int KC, int MET>
static int fallback_launch(const void* x, const void* q, int64_t n, int64_t d, int64_t k,
                           const unsigned* stats, const int* fb, void* scratch,
                           int64_t scratch_bytes, int64_t m, void* od, int64_t* oi,
                           int64_t base, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // scratch holds max(G, count) lists of KC (double, int); count <= m
  const int64_t cap = scratch_bytes / (12 * KC);
  if (cap < m) return fail(TB_ERR_ARG, "fallback scratch too small");
  const unsigned* list_cnt = stats + 1;
  const int* list = fb;
  // stage 1: bounded scan into per-query hit buffers (hcap (distance, row)
  // slots per query in the scratch); what it cannot settle goes
  // on through stats[kFbOverWord] and the overflow list (the bounds' space,
  // dead once the scan has run)
  // (up to 1024 slots: on clustered data the k-th candidate's distance can
  // enclose hundreds of rows of the query's cluster)
  const int64_t hcap = std::min<int64_t>(1024, scratch_bytes / std::max<int64_t>(m, 1) / 12);
  const size_t fq_bytes = (size_t)kFbQB * d * 8;
  if (hcap >= k + 4 && fq_bytes <= 48 * 1024) {
    int* hit_cnt = fb_hits(const_cast<int*>(fb), m);        // zeroed by the re-rank
    double* hit_d = (double*)scratch;
    int* hit_i = (int*)(hit_d + m * hcap);
    knn_fallback_tile_kernel<T, MET><<<4 * sms, 256, fq_bytes, st>>>(
        (const T*)x, (const T*)q, n, d, list_cnt, fb, fb_bounds(const_cast<int*>(fb), m), hit_cnt,
        hit_d, hit_i, (int)hcap);
    TB_LAUNCH_CHECK("knn_fallback_tile");
    unsigned* over_cnt = const_cast<unsigned*>(stats) + kFbOverWord;
    int* over_list = reinterpret_cast<int*>(fb_bounds(const_cast<int*>(fb), m));
    knn_fallback_hits_kernel<OT, KC><<<(unsigned)ceil_div(m, 8), 256, 0, st>>>(
        list_cnt, fb, hit_cnt, hit_d, hit_i, (int)hcap, (int)k, over_cnt, over_list, (OT*)od, oi,
        base);
    TB_LAUNCH_CHECK("knn_fallback_hits");
    list_cnt = over_cnt;
    list = over_list;
  }
  // stage 2 (exhaustive; normally nothing left): per-block top-K' over
  // database slices, then one merge
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(4 * sms, cap));
  double* sc_d = (double*)scratch;
  int* sc_i = (int*)(sc_d + cap * KC);
  if (d <= 64)
    knn_fallback_rows_kernel<T, KC, MET, 64><<<G, 256, 0, st>>>((const T*)x, (const T*)q, n, d,
                                                                list_cnt, list, sc_d, sc_i);
  else
    knn_fallback_partial_kernel<T, KC, MET><<<G, 256, 0, st>>>((const T*)x, (const T*)q, n, d,
                                                               list_cnt, list, sc_d, sc_i);
  TB_LAUNCH_CHECK("knn_fallback_partial");
  knn_fallback_merge_kernel<OT, KC><<<(unsigned)ceil_div(m, 8), 256, 0, st>>>(
      list_cnt, list, G, (int)k, sc_d, sc_i, (OT*)od, oi, base);
  TB_LAUNCH_CHECK("knn_fallback_merge");
  return TB_OK;
}

template <typename T, typename OT, int MET>
static int fallback_dispatch(const void* x, const void* q, int64_t n, int64_t d, int64_t k,
                             const unsigned* stats, const int* fb, void* scratch,
                             int64_t scratch_bytes, int64_t m, void* od, int64_t* oi,
                             int64_t base, cudaStream_t st) {
  if (k <= 16)
    return fallback_launch<T, OT, 16, MET>(x, q, n, d, k, stats, fb, scratch, scratch_bytes, m,
                                           od, oi, base, st);
  if (k <= 32)
    return fallback_launch<T, OT, 32, MET>(x, q, n, d, k, stats, fb, scratch, scratch_bytes, m,
                                           od, oi, base, st);
  if (k <= 64)
    return fallback_launch<T, OT, 64, MET>(x, q, n, d, k, stats, fb, scratch, scratch_bytes, m,
                                           od, oi, base, st);
  return fail(TB_ERR_UNSUPPORTED, "fallback: k > 64");
}

int launch_knn_fallback(int dtype, int out_dtype, int metric, const void* x, const void* q,
                        int64_t n, int64_t m, int64_t d, int64_t k,
                        const unsigned* stats, const int* fb_list, void* scratch,
                        int64_t scratch_bytes, void* out_dist, int64_t* out_idx,
                        int64_t index_base, cudaStream_t st) {
  if (m <= 0) return TB_OK;
#define TB_FB(T, OT, MET)                                                                     \
  return fallback_dispatch<T, OT, MET>(x, q, n, d, k, stats, fb_list, scratch, scratch_bytes, \
                                       m, out_dist, out_idx, index_base, st)
#define TB_FB_MET(T, OT)                                          \
  if (metric == TB_METRIC_L1) TB_FB(T, OT, TB_METRIC_L1);         \
  if (metric == TB_METRIC_COSINE) TB_FB(T, OT, TB_METRIC_COSINE); \
  TB_FB(T, OT, TB_METRIC_L2)
  if (dtype == TB_F32) {
    if (out_dtype == TB_F32) { TB_FB_MET(float, float); }
    TB_FB_MET(float, double);
  }
  if (out_dtype == TB_F32) { TB_FB_MET(double, float); }
  TB_FB_MET(double, double);
#undef TB_FB_MET
#undef TB_FB
}

// ------------------------------------------------ cross-shard top-k merge --
template <typename T, int KC>
__global__ void topk_merge_kernel(const T* __restrict__ dl,
                                  const int64_t* __restrict__ il, int lists,
                                  int64_t m, int k, T* __restrict__ od,
                                  int64_t* __restrict__ oi) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= m) return;
  // int64 global indices end to end: index_base + local may pass 2^31 on a
  // sharded database, and ties must still resolve to the lower global index
  TopList<T, KC, int64_t> L;
  L.init();
  for (int l = lane; l < lists; l += 32) {
    const T* s = dl + ((int64_t)l * m + r) * k;
    const int64_t* ix = il + ((int64_t)l * m + r) * k;
    for (int p = 0; p < k; ++p) {
      const T v = s[p];
      const int64_t j = ix[p];
      if (!lex_less(v, j, L.worst(), L.worst_idx())) break;
      L.insert(v, j);
    }
  }
  warp_drain(L, k, [&](int t, T v, int64_t j) {
    od[r * k + t] = v;
    oi[r * k + t] = j;
  });
}

int launch_topk_merge(const void* dist_lists, const int64_t* idx_lists,
                      int n_lists, int64_t m, int64_t k, int dtype,
                      void* out_dist, int64_t* out_idx, cudaStream_t st) {
  if (m <= 0) return TB_OK;
  const int warps = 4;
  const unsigned blocks = (unsigned)ceil_div(m, warps);
#define TB_TM(TT, KC)                                                        \
  topk_merge_kernel<TT, KC><<<blocks, warps * 32, 0, st>>>(                  \
      (const TT*)dist_lists, idx_lists, n_lists, m, (int)k, (TT*)out_dist, out_idx)
  if (dtype == TB_F32) {
    if (k <= 16) TB_TM(float, 16); else if (k <= 32) TB_TM(float, 32); else if (k <= 64) TB_TM(float, 64);
    else return fail(TB_ERR_UNSUPPORTED, "topk_merge: k > 64");
  } else {
    if (k <= 16) TB_TM(double, 16); else if (k <= 32) TB_TM(double, 32); else if (k <= 64) TB_TM(double, 64);
    else return fail(TB_ERR_UNSUPPORTED, "topk_merge: k > 64");
  }
#undef TB_TM
  TB_LAUNCH_CHECK("topk_merge");
  return TB_OK;
}

}  // namespace tb
