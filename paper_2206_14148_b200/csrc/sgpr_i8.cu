// sgpr_i8.cu — SGPR sufficient statistics with an EXACT fixed-point Gram on
// the INT8 tensor cores (tcgen05.mma kind::i8, s32 accumulators in TMEM).
//
// Why fixed point (re-checked in DESIGN.md §4): an
// error in Sigma = Kuf Kuf^T that is not itself of Gram form (K+d)(K+d)^T is
// amplified by cond(Kuu); every fp32-class product scheme (fp32, 3xTF32)
// misses the 1e-4 predictive-mean tolerance at cond ~1e5.  Here Kuf is
// rounded ONCE to 24-bit fixed point, q = rint(k / variance * 2^24), and
//     Sigma = variance^2 * 2^-48 * Q Q^T,   v = variance * 2^-24 * Q y
// are computed EXACTLY for that Q (integer products, no rounding inside a
// chunk), i.e. the statistics of a consistently perturbed Kuf.  Q is split
// into three u8 digit planes, Q = a2 2^16 + a1 2^8 + a0, and
//     Q_a Q_b^T = sum_{s,t} 2^{8(s+t)} A_s B_t^T
// is 9 u8 x u8 products grouped into 5 weight levels l = s + t.
//
// Per streamed chunk of Nc training points (planner, <= kI8MaxChunk so no
// s32 level can overflow):
//   kuf_quant   q[i, n] from fp64 direct differences (the same kernel code
//               as Kuu), written as 3 planes [3][M_pad][Nc] u8 (n contiguous:
//               K-major for both MMA operands); v partial sums per
//               128-point segment from the SAME q (exact products q*y in fp64);
//   v_reduce    v[i] += variance 2^-24 sum_seg vpart[seg][i] (fixed order);
//   gram_i8     persistent, one CTA per SM, units = lower 128x128 Sigma tiles.
//     warp 0    TMA producer: per 64-point k-block the plane tiles
//               (A_p rows of tile a, B_p rows of tile b), 64-B swizzle,
//               through a 4-stage mbarrier ring (48 KB per stage: one
//               phase-A k-block, or plane 0 of three k-blocks in phase B);
//               Units are ordered in 12x12 super-blocks of tiles (L2 reuse);
//     warp 1    TMEM (512 columns = 4 accumulators x 128) + MMA issuer:
//               phase A: levels 4..1 (8 products per k-block):
//                 acc0 = A2B2, acc1 = A2B1 + A1B2, acc2 = A2B0 + A1B1 + A0B2,
//                 acc3 = A1B0 + A0B1;
//               phase B (after the epilogue drained acc0): acc0 = A0B0
//               (plane 0 streamed a second time);
//     warps 2-9 epilogue: P = ((((L4 256 + L3) 256 + L2) 256 + L1) 256 + L0
//               in fp64 registers (64 per thread), then one read-modify-write
//               of the fp64 Sigma tile: Sigma += variance^2 2^-48 P.
// Sigma is kept as packed lower tiles (column-major 128x128, tile (a, b),
// a >= b, at index a(a+1)/2 + b): 414 MB at M = 1e4 instead of 800 MB, so a
// 10880-point chunk fits the 1 GB budget of C4.  tb_sgpr_sigma_unpack
// expands it for the O(M^3) tail.
#include <cmath>
#include <cstdlib>

#include "sgpr_internal.h"
#include "sm100.cuh"

namespace tb {
using namespace sm100;

constexpr int kI8Stages = 4;
constexpr uint32_t kI8TileBytes = kI8Tile * kI8KB;        // 8 KB
constexpr uint32_t kI8StageBytes = 6 * kI8TileBytes;      // 3 x (A + B) = 48 KB
constexpr int kI8EpiWarps = 8;
constexpr int kI8Threads = 64 + 32 * kI8EpiWarps;
constexpr size_t kI8Smem = 1024 + (size_t)kI8Stages * kI8StageBytes + 512;   // + barriers

// ------------------------------------------------------------ kuf_quant --
// Block: 32 inducing rows x 128 points, 128 threads.  Lane l owns inducing
// row i0 + l (its scaled z in registers) and warp w the points w*32..+31, so
// that
//   * the scaled points x_c / l are staged once per block in shared memory
//     and read as broadcast 16-byte loads (one per two dimensions),
//   * v_i = sum_c q_ic y_c accumulates in the owning thread's register (no
//     per-element warp reductions), the 4 warps' partials combined in a fixed
//     order,
//   * q = rint(k 2^24 / variance) comes from the low word of
//     min(k qscale, 2^24 - 1) + 1.5 * 2^52 (round-to-nearest-even in the add,
//     no float->int conversion), and (double) q is that sum minus the magic,
//   * the three digit bytes are staged in shared memory (rows padded to 132
//     bytes against bank conflicts) and written out as coalesced 128-byte
//     rows.
// r^2 and k are the same fp64 expressions, in the same order, as before and
// as oracle.sgpr.sufficient_stats_fixed24.  EXACT: DMAX is the dimension
// (no predicated-off dimensions issue).
constexpr int kI8QuantThreads = 128;
constexpr int kQRows = 32, kQPts = 128, kQLd = kQPts + 4;
template <int KERN>
__device__ __forceinline__ double kern_r2_t(double variance, double r2) {
  // kern_from_r2 with the kernel type fixed at compile time (same
  // expressions, same order: identical results)
  if (KERN == TB_KERNEL_RBF) return variance * exp(-0.5 * r2);
  const double r = sqrt(fmax(r2, 1e-36));
  const double s3 = 1.7320508075688772 * r;
  return variance * (1.0 + s3) * exp(-s3);
}

template <typename T, int DMAX, bool EXACT, int KERN>
__global__ void __launch_bounds__(kI8QuantThreads)
kuf_quant_kernel(const T* __restrict__ X, const T* __restrict__ y, const T* __restrict__ Z,
                 int64_t n0, int64_t cur, int64_t M, int64_t M_pad, int64_t nc, KernParams p,
                 double qscale, uint8_t* __restrict__ planes, double* __restrict__ vpart) {
  constexpr int DP = (DMAX + 1) & ~1;
  extern __shared__ __align__(16) double xs_dyn[];     // [kQPts][DP]
  double (*xs)[DP] = reinterpret_cast<double (*)[DP]>(xs_dyn);
  __shared__ double ys[kQPts];
  __shared__ __align__(16) uint8_t qb[3][kQRows][kQLd];
  __shared__ double vred[4][kQRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * kQPts;
  const int i0 = blockIdx.y * kQRows;
  const int dim = EXACT ? DMAX : p.dim;
  for (int e = tid; e < kQPts * DP; e += kI8QuantThreads) {
    const int pc = e / DP, t = e % DP;
    const int64_t c = c0 + pc;
    xs[pc][t] = (c < cur && t < dim) ? (double)X[(n0 + c) * p.dim + t] * p.inv_ls[t] : 0.0;
  }
  for (int pc = tid; pc < kQPts; pc += kI8QuantThreads) {
    const int64_t c = c0 + pc;
    ys[pc] = c < cur ? (double)y[n0 + c] : 0.0;
  }
  const int64_t i = i0 + lane;
  const bool row_ok = i < M;
  double zr[DP];
#pragma unroll
  for (int t = 0; t < DP; ++t)
    zr[t] = (row_ok && t < dim) ? (double)Z[i * p.dim + t] * p.inv_ls[t] : 0.0;
  __syncthreads();
  const double magic = 6755399441055744.0;            // 1.5 * 2^52
  const int ncol = (int)(cur - c0 < kQPts ? cur - c0 : kQPts);   // valid points of this block
  double vacc = 0.0;
  // 4 points in flight per thread (independent r^2 / exp chains; per point
  // the r^2 / k expressions and their order are unchanged): 0.49 -> 0.46 ms
  // per C4 chunk.  (Generating the next chunk inside the Gram kernel with its
  // idle epilogue warps was tried: 8 warps per SM cannot hide the fp64
  // latencies, the Gram stretched from 2.45 to 4.7-5.0 ms; reverted.)
  // Branch-free validity (selects) and the 4 points' digit bytes packed
  // into one 32-bit shared store per plane (byte permutes): ncu had the
  // kernel issue-bound (76 % of issue slots) with 110 instructions per
  // evaluation, a third of them fp64.
  for (int k = 0; k < 32; k += 4) {
    double r2[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < DP; t += 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 xv = *reinterpret_cast<const double2*>(&xs[warp * 32 + k + u][t]);
        if (EXACT || t < dim) {
          const double d0 = zr[t] - xv.x;
          r2[u] = fma(d0, d0, r2[u]);
        }
        if (t + 1 < DMAX && (EXACT || t + 1 < dim)) {
          const double d1 = zr[t + 1] - xv.y;
          r2[u] = fma(d1, d1, r2[u]);
        }
      }
    }
    uint32_t q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pc = warp * 32 + k + u;
      const bool ok = row_ok && pc < ncol;
      const double qm = fmin(kern_r2_t<KERN>(p.variance, r2[u]) * qscale, 16777215.0) + magic;
      q[u] = ok ? (uint32_t)__double2loint(qm) : 0u;
      vacc = fma(ok ? qm - magic : 0.0, ys[pc], vacc);   // exact q * y products
    }
    const uint32_t t01 = __byte_perm(q[0], q[1], 0x5140), t23 = __byte_perm(q[2], q[3], 0x5140);
    const uint32_t u01 = __byte_perm(q[0], q[1], 0x0062), u23 = __byte_perm(q[2], q[3], 0x0062);
    const int pc0 = warp * 32 + k;
    *reinterpret_cast<uint32_t*>(&qb[0][lane][pc0]) = __byte_perm(t01, t23, 0x5410);
    *reinterpret_cast<uint32_t*>(&qb[1][lane][pc0]) = __byte_perm(t01, t23, 0x7632);
    *reinterpret_cast<uint32_t*>(&qb[2][lane][pc0]) = __byte_perm(u01, u23, 0x5410);
  }
  vred[warp][lane] = vacc;
  __syncthreads();
  if (tid < kQRows)
    vpart[(int64_t)blockIdx.x * M_pad + i0 + tid] =
        ((vred[0][tid] + vred[1][tid]) + vred[2][tid]) + vred[3][tid];
  const int64_t plane = M_pad * nc;
  for (int e = tid; e < 3 * kQRows * (kQPts / 4); e += kI8QuantThreads) {
    const int pl = e / (kQRows * (kQPts / 4));
    const int rr = (e / (kQPts / 4)) % kQRows, seg = e % (kQPts / 4);
    *reinterpret_cast<uint32_t*>(planes + pl * plane + (int64_t)(i0 + rr) * nc + c0 + seg * 4) =
        *reinterpret_cast<const uint32_t*>(&qb[pl][rr][seg * 4]);
  }
}

__global__ void v_reduce_kernel(const double* __restrict__ vpart, int nseg, int64_t M,
                                int64_t M_pad, double scale, double* __restrict__ v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  double s = 0.0;
  for (int g = 0; g < nseg; ++g) s += vpart[(int64_t)g * M_pad + i];
  v[i] += s * scale;
}

// ------------------------------------------------------------- gram_i8 --
__device__ __forceinline__ void tri_of(int u, int& a, int& b) {
  a = (int)((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
  while ((a + 1) * (a + 2) / 2 <= u) ++a;
  while (a * (a + 1) / 2 > u) --a;
  b = u - a * (a + 1) / 2;
}
// Unit u -> lower tile (ta, tb).  Units are grouped in 12 x 12 super-blocks
// of tiles (lower ones, row-major), so the ~148 units running at once touch
// ~24 row blocks of the chunk instead of up to nt + 2: far fewer L2 misses
// (each wave re-streams every row block it touches).
constexpr int kI8SuperBlock = 12;
__device__ __forceinline__ void tile_of_unit(int u, int nt, int& ta, int& tb) {
  const int nsb = (nt + kI8SuperBlock - 1) / kI8SuperBlock;
  for (int I = 0; I < nsb; ++I) {
    const int r0 = I * kI8SuperBlock, r1 = min(nt, r0 + kI8SuperBlock);
    for (int J = 0; J <= I; ++J) {
      const int c0 = J * kI8SuperBlock, c1 = min(nt, c0 + kI8SuperBlock);
      const int cnt = I > J ? (r1 - r0) * (c1 - c0) : (r1 - r0) * (r1 - r0 + 1) / 2;
      if (u < cnt) {
        if (I > J) {
          ta = r0 + u / (c1 - c0);
          tb = c0 + u % (c1 - c0);
        } else {
          int a, b;
          tri_of(u, a, b);
          ta = r0 + a;
          tb = c0 + b;
        }
        return;
      }
      u -= cnt;
    }
  }
  ta = tb = 0;
}

// A/B timing modes (TB_I8_DEBUG) only in a study build (-DTB_I8_STUDY): in
// the product library they are compile-time zero and leave no branches in
// the tcgen05 loops.
#ifdef TB_I8_STUDY
#define TB_I8_DBG(x) (x)
#else
#define TB_I8_DBG(x) 0
#endif

__global__ void __launch_bounds__(kI8Threads, 1)
sgpr_gram_i8_kernel(const __grid_constant__ CUtensorMap tm, int units, int nkb, int m_pad,
                    double scale, double* __restrict__ sig, int dbg) {
  // dbg (TB_I8_DEBUG, A/B timing only): 1 = producer skips the TMA loads
  // (MMA-issue bound), 2 = issuer skips the MMAs (TMA-feed bound), 3 = no
  // phase B (level 0);
  // results are garbage in both modes
  const int nt = m_pad / kI8Tile;
  constexpr int S = kI8Stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kI8StageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull_a = empty + S;      // levels 4..1 ready
  uint64_t* acc0_free = tfull_a + 1;  // epilogue drained acc0 (level 4)
  uint64_t* tfull_b = acc0_free + 1;  // level 0 ready
  uint64_t* tempty = tfull_b + 1;     // all accumulators drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull_a, 1);
    mbar_init(acc0_free, 32 * kI8EpiWarps);
    mbar_init(tfull_b, 1);
    mbar_init(tempty, 32 * kI8EpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    // phase A stage = one k-block, tiles [A2 B2 A1 B1 A0 B0];
    // phase B stage = plane 0 of up to 3 k-blocks, tiles [A0 B0] x 3.
    // The whole warp runs the loop and one elected lane issues (uniform
    // registers, no per-instruction broadcast loop), as in the issuer below.
    if (elect_one_sync()) tma_prefetch(&tm);
    __syncwarp();
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int ta, tb;
      tile_of_unit(u, nt, ta, tb);
      const int ra = ta * kI8Tile, rb = tb * kI8Tile;
      for (int phase = 0; phase < (TB_I8_DBG(dbg) == 3 ? 1 : 2); ++phase) {
        const int step = phase ? 3 : 1;
        for (int kb = 0; kb < nkb; kb += step) {
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one_sync()) {
            if (TB_I8_DBG(dbg) == 1) {
              mbar_arrive(&full[s]);
            } else {
              uint8_t* st = smem + (size_t)s * kI8StageBytes;
              if (phase == 0) {
                mbar_expect_tx(&full[s], kI8StageBytes);
                for (int pl = 2; pl >= 0; --pl) {
                  uint8_t* t = st + (2 - pl) * 2 * kI8TileBytes;
                  tma_load_2d(t, &tm, &full[s], kb * kI8KB, pl * m_pad + ra);
                  tma_load_2d(t + kI8TileBytes, &tm, &full[s], kb * kI8KB, pl * m_pad + rb);
                }
              } else {
                const int nk = min(3, nkb - kb);
                mbar_expect_tx(&full[s], nk * 2 * kI8TileBytes);
                for (int j = 0; j < nk; ++j) {
                  uint8_t* t = st + j * 2 * kI8TileBytes;
                  tma_load_2d(t, &tm, &full[s], (kb + j) * kI8KB, ra);
                  tma_load_2d(t + kI8TileBytes, &tm, &full[s], (kb + j) * kI8KB, rb);
                }
              }
            }
          }
          __syncwarp();
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    // Issue rate is this kernel's limiter (64-cycle MMAs), so: the whole
    // warp runs the loop (waits included) and one elected lane issues from
    // uniform registers - each MMA is one 64-bit add of a precomputed UMMA
    // descriptor, with no per-instruction register->uniform broadcast loop -
    // and each barrier handshake covers 16 MMAs (phase A) or 6 (phase B).
    constexpr uint32_t idesc = idesc_u8_s32(kI8Tile, kI8Tile);
    const uint32_t acc0 = tmem, acc1 = tmem + 128, acc2 = tmem + 256, acc3 = tmem + 384;
    // UMMA descriptor of stage s, tile j: d0 + s * kStageD + j * kTileD
    // (16-byte units); the second K=32 step of a 64-byte row is +2
    const uint64_t d0 = desc_k_sw64(smem_u32(smem));
    constexpr uint64_t kStageD = kI8StageBytes >> 4, kTileD = kI8TileBytes >> 4;
    int s = 0;
    uint32_t ph = 0;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      mbar_wait(tempty, (i & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t a2 = d0 + (uint64_t)s * kStageD, b2 = a2 + kTileD;
        const uint64_t a1 = a2 + 2 * kTileD, b1 = a2 + 3 * kTileD;
        const uint64_t a0 = a2 + 4 * kTileD, b0 = a2 + 5 * kTileD;
        if (elect_one_sync()) {
          if (TB_I8_DBG(dbg) != 2) {
            const uint32_t acc = kb ? 1u : 0u;
            mma_i8(acc0, a2, b2, idesc, acc);
            mma_i8(acc1, a2, b1, idesc, acc);
            mma_i8(acc1, a1, b2, idesc, 1);
            mma_i8(acc2, a2, b0, idesc, acc);
            mma_i8(acc2, a1, b1, idesc, 1);
            mma_i8(acc2, a0, b2, idesc, 1);
            mma_i8(acc3, a1, b0, idesc, acc);
            mma_i8(acc3, a0, b1, idesc, 1);
            mma_i8(acc0, a2 + 2, b2 + 2, idesc, 1);
            mma_i8(acc1, a2 + 2, b1 + 2, idesc, 1);
            mma_i8(acc1, a1 + 2, b2 + 2, idesc, 1);
            mma_i8(acc2, a2 + 2, b0 + 2, idesc, 1);
            mma_i8(acc2, a1 + 2, b1 + 2, idesc, 1);
            mma_i8(acc2, a0 + 2, b2 + 2, idesc, 1);
            mma_i8(acc3, a1 + 2, b0 + 2, idesc, 1);
            mma_i8(acc3, a0 + 2, b1 + 2, idesc, 1);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one_sync()) mma_commit(tfull_a);
      __syncwarp();
      mbar_wait(acc0_free, i & 1);
      tc_fence_after();
      for (int kb = 0; kb < (TB_I8_DBG(dbg) == 3 ? 0 : nkb); kb += 3) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t a = d0 + (uint64_t)s * kStageD;
        const int nk = min(3, nkb - kb);
        if (elect_one_sync()) {
          if (TB_I8_DBG(dbg) != 2) {
            for (int j = 0; j < nk; ++j) {
              const uint64_t aj = a + 2 * j * kTileD, bj = aj + kTileD;
              mma_i8(acc0, aj, bj, idesc, (kb | j) ? 1u : 0u);
              mma_i8(acc0, aj + 2, bj + 2, idesc, 1);
            }
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one_sync()) mma_commit(tfull_b);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int quad = warp & 3;          // TMEM lane quadrant this warp may read
    const int half = ew >> 2;           // 64-column half of the tile
    const int row = quad * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + half * 64;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      double P[64];
      uint32_t r[32];
      mbar_wait_sleep(tfull_a, i & 1, 256);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tbase + h * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) P[h * 32 + j] = (double)(int)r[j];
      }
      tc_fence_before();
      mbar_arrive(acc0_free);
#pragma unroll
      for (int a = 1; a < 4; ++a) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld32(tbase + a * 128 + h * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) P[h * 32 + j] = fma(P[h * 32 + j], 256.0, (double)(int)r[j]);
        }
      }
      mbar_wait_sleep(tfull_b, i & 1, 256);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tbase + h * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) P[h * 32 + j] = fma(P[h * 32 + j], 256.0, (double)(int)r[j]);
      }
      tc_fence_before();
      mbar_arrive(tempty);
      // column-major tile: lanes (consecutive rows) hit consecutive doubles
      int ta, tb;
      tile_of_unit(u, nt, ta, tb);
      const int64_t slot = (int64_t)ta * (ta + 1) / 2 + tb;
      double* t = sig + slot * (kI8Tile * kI8Tile) + (int64_t)(half * 64) * kI8Tile + row;
#pragma unroll
      for (int j = 0; j < 64; ++j) t[j * kI8Tile] += P[j] * scale;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------- gram_i8, CTA pairs --
// The same statistics with tcgen05.mma.cta_group::2: a cluster of two CTAs
// on one TPC computes a 256 x 128 pair tile (rows 256 I + 128 rank, cols
// 128 J); the leader (rank 0) issues M256.N128.K32 MMAs that use both SMs'
// tensor cores, each CTA holding its 128 rows of A and half (64 rows) of B.
// Per SM this halves the MMA instructions the single issuing thread must
// push (the 1-SM kernel's limiter) and cuts TMA bytes per k-block from 48 to
// 36 KB.  TMEM per CTA is unchanged: 4 s32 accumulators x 128 columns.
// Protocol: "full" barriers live in the leader and receive the tx bytes of
// both CTAs' loads (leader arms expect_tx for both); "empty" and the
// accumulator-ready barriers are arrived in both CTAs by multicast commits;
// the epilogue warps of both CTAs arrive on the leader's acc0_free / tempty.
constexpr int kP2Stages = 6;
constexpr uint32_t kP2ATile = kI8Tile * kI8KB;             // 8 KB: 128 rows x 64 B
constexpr uint32_t kP2BTile = (kI8Tile / 2) * kI8KB;       // 4 KB: 64 rows x 64 B
constexpr uint32_t kP2Stage = 3 * (kP2ATile + kP2BTile);   // 36 KB
constexpr size_t kP2Smem = 1024 + (size_t)kP2Stages * kP2Stage + 512;
constexpr int kP2SbI = 6, kP2SbJ = 12;                     // super-block of pair tiles

// pair unit u -> (I, J), J <= 2I + 1, grouped in 6 x 12 super-blocks
__device__ __forceinline__ void pair_of_unit(int u, int nI, int& I, int& J) {
  for (int I0 = 0; I0 < nI; I0 += kP2SbI) {
    const int I1 = min(nI, I0 + kP2SbI);
    for (int J0 = 0; J0 <= 2 * (I1 - 1) + 1; J0 += kP2SbJ) {
      const int J1 = min(2 * nI, J0 + kP2SbJ);
      for (int i = I0; i < I1; ++i) {
        const int c = max(0, min(J1, 2 * i + 2) - J0);
        if (u < c) {
          I = i;
          J = J0 + u;
          return;
        }
        u -= c;
      }
    }
  }
  I = J = 0;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kI8Threads, 1)
sgpr_gram_i8_pair_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                         int units, int nkb, int m_pad, double scale, double* __restrict__ sig,
                         int dbg) {
  constexpr int S = kP2Stages;
  const int nt = m_pad / kI8Tile, nI = m_pad / (2 * kI8Tile);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kP2Stage);
  uint64_t* empty = full + S;
  uint64_t* tfull_a = empty + S;
  uint64_t* acc0_free = tfull_a + 1;
  uint64_t* tfull_b = acc0_free + 1;
  uint64_t* tempty = tfull_b + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull_a, 1);
    mbar_init(acc0_free, 2 * kI8EpiWarps);   // one arrive per epilogue warp, both CTAs
    mbar_init(tfull_b, 1);
    mbar_init(tempty, 2 * kI8EpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();               // barriers of both CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tma);
      tma_prefetch(&tmb);
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < units; u += npairs) {
        int I, J;
        pair_of_unit(u, nI, I, J);
        const int ra = I * 2 * kI8Tile + rank * kI8Tile;
        const int rb = J * kI8Tile + rank * (kI8Tile / 2);
        for (int phase = 0; phase < 2; ++phase) {
          const int step = phase ? 3 : 1;
          for (int kb = 0; kb < nkb; kb += step) {
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t fb = mapa_shared(&full[s], 0);     // the leader's barrier
            uint8_t* st = smem + (size_t)s * kP2Stage;
            const int nk = phase ? min(3, nkb - kb) : 1;
            if (TB_I8_DBG(dbg) == 1) {
              if (rank == 0) mbar_arrive(&full[s]);
            } else {
            // the leader arms its own barrier for both CTAs' bytes
            if (rank == 0) mbar_expect_tx(&full[s], 2 * (phase ? nk * (kP2ATile + kP2BTile) : kP2Stage));
            if (phase == 0) {
              for (int pl = 2; pl >= 0; --pl) {
                uint8_t* t = st + (2 - pl) * (kP2ATile + kP2BTile);
                tma_load_2d_2sm(t, &tma, fb, kb * kI8KB, pl * m_pad + ra);
                tma_load_2d_2sm(t + kP2ATile, &tmb, fb, kb * kI8KB, pl * m_pad + rb);
              }
            } else {
              for (int j = 0; j < nk; ++j) {
                uint8_t* t = st + j * (kP2ATile + kP2BTile);
                tma_load_2d_2sm(t, &tma, fb, (kb + j) * kI8KB, ra);
                tma_load_2d_2sm(t + kP2ATile, &tmb, fb, (kb + j) * kI8KB, rb);
              }
            }
            }
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_u8_s32(2 * kI8Tile, kI8Tile);   // M256 N128
      const uint32_t acc0 = tmem, acc1 = tmem + 128, acc2 = tmem + 256, acc3 = tmem + 384;
      const uint64_t d0 = desc_k_sw64(smem_u32(smem));
      constexpr uint64_t kStageD = kP2Stage >> 4, kAD = kP2ATile >> 4, kPairD = (kP2ATile + kP2BTile) >> 4;
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int u = pair; u < units; u += npairs, ++i) {
        mbar_wait(tempty, (i & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a2 = d0 + (uint64_t)s * kStageD, b2 = a2 + kAD;
          const uint64_t a1 = a2 + kPairD, b1 = a1 + kAD;
          const uint64_t a0 = a1 + kPairD, b0 = a0 + kAD;
          const uint32_t acc = kb ? 1u : 0u;
          if (TB_I8_DBG(dbg) != 2) {
          mma_i8_2sm(acc0, a2, b2, idesc, acc);
          mma_i8_2sm(acc1, a2, b1, idesc, acc);
          mma_i8_2sm(acc1, a1, b2, idesc, 1);
          mma_i8_2sm(acc2, a2, b0, idesc, acc);
          mma_i8_2sm(acc2, a1, b1, idesc, 1);
          mma_i8_2sm(acc2, a0, b2, idesc, 1);
          mma_i8_2sm(acc3, a1, b0, idesc, acc);
          mma_i8_2sm(acc3, a0, b1, idesc, 1);
          mma_i8_2sm(acc0, a2 + 2, b2 + 2, idesc, 1);
          mma_i8_2sm(acc1, a2 + 2, b1 + 2, idesc, 1);
          mma_i8_2sm(acc1, a1 + 2, b2 + 2, idesc, 1);
          mma_i8_2sm(acc2, a2 + 2, b0 + 2, idesc, 1);
          mma_i8_2sm(acc2, a1 + 2, b1 + 2, idesc, 1);
          mma_i8_2sm(acc2, a0 + 2, b2 + 2, idesc, 1);
          mma_i8_2sm(acc3, a1 + 2, b0 + 2, idesc, 1);
          mma_i8_2sm(acc3, a0 + 2, b1 + 2, idesc, 1);
          }
          mma_commit_2sm(&empty[s], 3);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_2sm(tfull_a, 3);
        mbar_wait(acc0_free, i & 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; kb += 3) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a = d0 + (uint64_t)s * kStageD;
          const int nk = min(3, nkb - kb);
          for (int j = 0; j < nk && TB_I8_DBG(dbg) != 2; ++j) {
            const uint64_t aj = a + j * kPairD, bj = aj + kAD;
            mma_i8_2sm(acc0, aj, bj, idesc, (kb | j) ? 1u : 0u);
            mma_i8_2sm(acc0, aj + 2, bj + 2, idesc, 1);
          }
          mma_commit_2sm(&empty[s], 3);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_2sm(tfull_b, 3);
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int quad = warp & 3;
    const int half = ew >> 2;
    const int row = quad * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + half * 64;
    const uint32_t acc0_free_l = mapa_shared(acc0_free, 0), tempty_l = mapa_shared(tempty, 0);
    int i = 0;
    for (int u = pair; u < units; u += npairs, ++i) {
      double P[64];
      uint32_t r[32];
      mbar_wait_sleep(tfull_a, i & 1, 256);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tbase + h * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) P[h * 32 + j] = (double)(int)r[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc0_free_l);
#pragma unroll
      for (int a = 1; a < 4; ++a) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld32(tbase + a * 128 + h * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) P[h * 32 + j] = fma(P[h * 32 + j], 256.0, (double)(int)r[j]);
        }
      }
      mbar_wait_sleep(tfull_b, i & 1, 256);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tbase + h * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) P[h * 32 + j] = fma(P[h * 32 + j], 256.0, (double)(int)r[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_l);
      int I, J;
      pair_of_unit(u, nI, I, J);
      const int ta = 2 * I + (int)rank, tb = J;
      if (ta >= tb && ta < nt) {     // rank 0 of J = 2I + 1 lies above the diagonal
        const int64_t slot = (int64_t)ta * (ta + 1) / 2 + tb;
        double* t = sig + slot * (kI8Tile * kI8Tile) + (int64_t)(half * 64) * kI8Tile + row;
#pragma unroll
        for (int j = 0; j < 64; ++j) t[j * kI8Tile] += P[j] * scale;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_2sm(tmem, 512);
}

// ------------------------------------------------------------ unpack --
// full[r, c] (M x M, symmetric) from the packed lower tiles.
__global__ void sigma_unpack_kernel(const double* __restrict__ tiles, int64_t M,
                                    double* __restrict__ full) {
  const int64_t r = (int64_t)blockIdx.y * 32 + threadIdx.y;
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (r >= M || c >= M) return;
  const int64_t lo = r >= c ? r : c, hi = r >= c ? c : r;   // (row, col) in the lower half
  const int64_t ta = lo / kI8Tile, tb = hi / kI8Tile;
  const int64_t u = ta * (ta + 1) / 2 + tb;
  full[r * M + c] = tiles[u * (kI8Tile * kI8Tile) + (hi % kI8Tile) * kI8Tile + (lo % kI8Tile)];
}

// --------------------------------------------------------------- host --
static int make_plane_map(CUtensorMap* map, const uint8_t* base, int64_t M_pad, int64_t nc,
                          uint32_t box_rows = kI8Tile) {
  auto fn = tensor_map_encoder();
  if (!fn) return fail(TB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)nc, (cuuint64_t)(3 * M_pad)};
  cuuint64_t strides[1] = {(cuuint64_t)nc};
  cuuint32_t box[2] = {(cuuint32_t)kI8KB, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TB_ERR_CUDA, "cuTensorMapEncodeTiled (u8 planes) failed: " + std::to_string((int)r));
  return TB_OK;
}

int i8_gen_chunk(const void* X, const void* y, const void* Z, int dtype, int64_t n0,
                 int64_t cur, int64_t M, int64_t M_pad, int64_t nc, const KernParams& kp,
                 uint8_t* planes, double* vpart, double* v, cudaStream_t st) {
  const int64_t ncur = round_up(cur, 128);           // columns written this chunk
  const double qscale = std::ldexp(1.0, kI8FracBits) / kp.variance;
  dim3 g((unsigned)(ncur / 128), (unsigned)(M_pad / 32));
#define TB_KQK(T, D, EX, KK)                                                               \
  do {                                                                                     \
    const int xs_bytes = kQPts * ((D + 1) & ~1) * 8;                                       \
    if (xs_bytes > 32768)                                                                  \
      TB_CUDA_TRY(cudaFuncSetAttribute(kuf_quant_kernel<T, D, EX, KK>,                     \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                       xs_bytes));                                         \
    kuf_quant_kernel<T, D, EX, KK><<<g, kI8QuantThreads, xs_bytes, st>>>(                  \
        (const T*)X, (const T*)y, (const T*)Z, n0, cur, M, M_pad, nc, kp, qscale, planes,  \
        vpart);                                                                            \
  } while (0)
#define TB_KQ(T, D, EX)                                                                    \
  do {                                                                                     \
    if (kp.kernel == TB_KERNEL_RBF) TB_KQK(T, D, EX, TB_KERNEL_RBF);                       \
    else TB_KQK(T, D, EX, TB_KERNEL_MATERN32);                                             \
  } while (0)
#define TB_KQ_DIM(T)                                                      \
  switch (kp.dim) {                                                       \
    case 1: TB_KQ(T, 1, true); break;   case 2: TB_KQ(T, 2, true); break; \
    case 3: TB_KQ(T, 3, true); break;   case 4: TB_KQ(T, 4, true); break; \
    case 5: TB_KQ(T, 5, true); break;   case 6: TB_KQ(T, 6, true); break; \
    case 7: TB_KQ(T, 7, true); break;   case 8: TB_KQ(T, 8, true); break; \
    case 11: TB_KQ(T, 11, true); break; case 16: TB_KQ(T, 16, true); break; \
    default:                                                              \
      if (kp.dim <= 16) TB_KQ(T, 16, false);                              \
      else if (kp.dim <= 32) TB_KQ(T, 32, false);                         \
      else TB_KQ(T, 64, false);                                           \
  }
  if (dtype == TB_F32) {
    TB_KQ_DIM(float);
  } else {
    TB_KQ_DIM(double);
  }
#undef TB_KQ_DIM
#undef TB_KQ
#undef TB_KQK
  TB_LAUNCH_CHECK("kuf_quant");
  v_reduce_kernel<<<(unsigned)ceil_div(M, 256), 256, 0, st>>>(
      vpart, (int)(ncur / 128), M, M_pad, kp.variance * std::ldexp(1.0, -kI8FracBits), v);
  TB_LAUNCH_CHECK("v_reduce");
  return TB_OK;
}

int i8_gram_chunk(int64_t cur, int64_t M_pad, int64_t nc, double variance, const uint8_t* planes,
                  double* Sigma_tiles, cudaStream_t st) {
  CUtensorMap tm;
  int rc = make_plane_map(&tm, planes, M_pad, nc);
  if (rc) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nkb = (int)ceil_div(cur, kI8KB);
  const double scale = variance * variance * std::ldexp(1.0, -2 * kI8FracBits);
  const char* dbg_env = std::getenv("TB_I8_DEBUG");
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
  // CTA-pair engine: opt-in (TB_I8_PAIR=1, needs M_pad % 256 == 0).  Both
  // kernels run into the 1 kW power cap (sw_power_cap, SM ~1.7 GHz) on C4;
  // there the 1-SM kernel is ~7% faster (no 256-row padding, 22 vs 23
  // rounds), so it stays the default.
  const char* pair_env = std::getenv("TB_I8_PAIR");
  if (M_pad % (2 * kI8Tile) == 0 && pair_env && pair_env[0] == '1') {
    CUtensorMap tmb;
    if ((rc = make_plane_map(&tmb, planes, M_pad, nc, kI8Tile / 2))) return rc;
    const int nI = (int)(M_pad / (2 * kI8Tile));
    const int units = nI * (nI + 1);
    TB_CUDA_TRY(cudaFuncSetAttribute(sgpr_gram_i8_pair_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kP2Smem));
    const int pairs = std::min(units, sms / 2);
    sgpr_gram_i8_pair_kernel<<<2 * pairs, kI8Threads, kP2Smem, st>>>(tm, tmb, units, nkb,
                                                                     (int)M_pad, scale,
                                                                     Sigma_tiles, dbg);
    TB_LAUNCH_CHECK("sgpr_gram_i8_pair");
    return TB_OK;
  }
  const int units = (int)i8_tiles(M_pad);
  TB_CUDA_TRY(cudaFuncSetAttribute(sgpr_gram_i8_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8Smem));
  // the whole 228 KB as shared memory: with the Gram CTA's ~199 KB there is
  // room beside it for a digit-plane producer block (kuf_quant, ~6 KB, 56
  // registers x 128 threads fit the Gram's unused register file), so the
  // next chunk's generation can run on the CUDA cores next to the Gram
  TB_CUDA_TRY(cudaFuncSetAttribute(sgpr_gram_i8_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  sgpr_gram_i8_kernel<<<std::min(units, sms), kI8Threads, kI8Smem, st>>>(tm, units, nkb,
                                                                         (int)M_pad, scale,
                                                                         Sigma_tiles, dbg);
  TB_LAUNCH_CHECK("sgpr_gram_i8");
  return TB_OK;
}

int i8_unpack(const double* tiles, int64_t M, int64_t M_pad, double* full, cudaStream_t st) {
  (void)M_pad;
  dim3 g((unsigned)ceil_div(M, 32), (unsigned)ceil_div(M, 32));
  sigma_unpack_kernel<<<g, dim3(32, 32), 0, st>>>(tiles, M, full);
  TB_LAUNCH_CHECK("sigma_unpack");
  return TB_OK;
}

}  // namespace tb
