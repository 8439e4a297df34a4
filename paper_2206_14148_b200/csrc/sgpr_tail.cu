// sgpr_tail.cu — the O(M^3) SGPR tail on the packed lower-tile storage the
// fixed-point statistics engine produces, so the whole ELBO evaluation stays
// inside memory_limit (two packed M x M matrices instead of ~4 dense ones).
//
// Formulation (algebraically GPflow 2.3.1 SGPR.elbo / predict_f, Titsias):
//   Kuu = L L^T,   Kuu + Sigma / s2 = P P^T
//   (then L^-1 P P^T L^-T = I + AAT = B, so with X = L^-1 P)
//   sum log diag LB = sum log diag P - sum log diag L
//   c^T c            = |P^-1 v|^2 / s2^2
//   tr(AAT)          = ||X||_F^2 - M
//   w (pred. mean)   = P^-T P^-1 v / s2
// Cost 4/3 M^3 (3 Choleskys-worth) vs 8/3 M^3 for the dense two-sided solve.
// Storage: 128 x 128 tiles, lower tiles (a >= b) packed at a(a+1)/2 + b,
// column-major inside; padding rows/cols (>= M) are identity blocks.
// Kernels: tile Cholesky + triangular inverse of the diagonal tile (one
// CTA, shared memory); every off-diagonal triangular solve and update is a
// DMMA tile GEMM (mma.sync m8n8k4 fp64) with that inverse; blocked vector
// solves (diagonal inverse + parallel matvec updates); fixed-order
// reductions.
#include <cmath>
#include <string>
#include <cooperative_groups.h>

#include "sgpr_internal.h"

namespace tb {

constexpr int kTT = 128;               // tile edge
constexpr int kTLd = kTT + 1;          // padded shared-memory row
constexpr int64_t kTE = kTT * kTT;     // doubles per tile

__host__ __device__ __forceinline__ int64_t tslot(int a, int b) {
  return (int64_t)a * (a + 1) / 2 + b;
}
__device__ __forceinline__ void tri_idx(int u, int& a, int& b) {
  a = (int)((sqrt(8.0 * u + 1.0) - 1.0) * 0.5);
  while ((a + 1) * (a + 2) / 2 <= u) ++a;
  while (a * (a + 1) / 2 > u) --a;
  b = u - a * (a + 1) / 2;
}

// ---------------------------------------------------------------- Kuu --
// dst tile = alpha * dst + k(Z_rows, Z_cols) (+ jitter on the diagonal);
// padding: identity.  Diagonal tiles: upper part left untouched (ignored).
__global__ void __launch_bounds__(256)
tail_kuu_kernel(const double* __restrict__ Zs, int64_t M, KernParams p, double jitter,
                double alpha, double* __restrict__ dst) {
  int a, b;
  tri_idx(blockIdx.x, a, b);
  double* t = dst + tslot(a, b) * kTE;
  for (int e = threadIdx.x; e < kTE; e += blockDim.x) {
    const int c = e / kTT, r = e % kTT;
    const int64_t i = (int64_t)a * kTT + r, j = (int64_t)b * kTT + c;
    if (a == b && r < c) continue;
    double val;
    if (i < M && j < M) {
      double r2 = 0.0;
      for (int d = 0; d < p.dim; ++d) {
        const double df = Zs[i * p.dim + d] - Zs[j * p.dim + d];
        r2 = fma(df, df, r2);
      }
      val = kern_from_r2(p, r2) + (i == j ? jitter : 0.0);
    } else {
      val = i == j ? 1.0 : 0.0;
    }
    t[e] = alpha == 0.0 ? val : fma(alpha, t[e], val);
  }
}

// Z scaled by 1/l (fp64) once, for the Kuu tiles
template <typename T>
__global__ void scale_z_kernel(const T* __restrict__ Z, int64_t M, KernParams p,
                               double* __restrict__ Zs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < M * p.dim) Zs[e] = (double)Z[e] * p.inv_ls[e % p.dim];
}

// ------------------------------------------------- potrf + tri. inverse --
// Diagonal tile k: in-place Cholesky (lower, upper zeroed), then its
// inverse L_kk^-1 into inv (column-major).  The off-diagonal triangular
// solves become DMMA tile GEMMs with this inverse (the usual GPU TRSM
// blocking; cond(L_kk) <= sqrt(cond(Kuu)) keeps it accurate).
// One CTA; the lower triangle lives in registers as 4x4 blocks, one block
// per thread (528 blocks).  Both factorisations are right-looking over
// 4-wide block columns / rows, three (two) barriers per block:
//   Cholesky, block column jb:  the owner of (jb, jb) factors it in
//   registers and publishes it; the owners of (bi, jb) solve their panel
//   block against it and publish it; every trailing block applies the
//   rank-4 update (16 shared loads, 64 FMAs from registers).
//   Inverse (X = L^-1 from L X = I), block row jb:  the owners of (jb, bc)
//   finalise X_jb,bc = L_jb,jb^-1 R_jb,bc and publish it; every block below
//   subtracts L_bi,jb X_jb,bc.
constexpr int kPB = 4;                              // register block edge
constexpr int kPNB = kTT / kPB;                     // 32 block rows
constexpr int kPBlocks = kPNB * (kPNB + 1) / 2;     // 528 lower blocks
constexpr int kPThreads = (kPBlocks + 31) / 32 * 32;

__global__ void __launch_bounds__(kPThreads)
tail_potrf_inv_kernel(double* __restrict__ base, int k, double* __restrict__ inv,
                      int* __restrict__ info) {
  extern __shared__ double sL[];                    // [kTT][kTLd] row-major, final L
  __shared__ __align__(16) double pan[kTT][kPB];    // panel block column / X block row
  __shared__ double sld[kPB][kPB], srd[kPB];        // factored diagonal block, 1/diag
  __shared__ double rdiag[kTT];
  __shared__ int sfail;
  double* t = base + tslot(k, k) * kTE;
  const int tid = threadIdx.x;
  const bool own = tid < kPBlocks;
  int bi = 0, bj = 0;
  if (own) tri_idx(tid, bi, bj);
  const int r0 = bi * kPB, c0 = bj * kPB;
  double a[kPB][kPB];
#pragma unroll
  for (int r = 0; r < kPB; ++r)
#pragma unroll
    for (int c = 0; c < kPB; ++c)
      a[r][c] = own && r0 + r >= c0 + c ? t[(int64_t)(c0 + c) * kTT + r0 + r] : 0.0;
  if (tid == 0) sfail = 0;
  __syncthreads();
  for (int jb = 0; jb < kPNB; ++jb) {
    if (own && bi == jb && bj == jb) {      // diagonal block: factor in registers
      int bad = 0;
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const double d = a[q][q];
        if (!(d > 0.0) && !bad) bad = q + 1;
        const double rl = rsqrt(d);
        a[q][q] = d * rl;
        srd[q] = rl;
#pragma unroll
        for (int r = q + 1; r < kPB; ++r) a[r][q] *= rl;
#pragma unroll
        for (int r = q + 1; r < kPB; ++r)
#pragma unroll
          for (int c = q + 1; c <= r; ++c) a[r][c] = fma(-a[r][q], a[c][q], a[r][c]);
      }
#pragma unroll
      for (int r = 0; r < kPB; ++r)
#pragma unroll
        for (int c = 0; c < kPB; ++c) sld[r][c] = r >= c ? a[r][c] : 0.0;
      if (bad) {
        sfail = 1;
        atomicExch(info, k * kTT + jb * kPB + bad);
      }
    }
    __syncthreads();
    if (sfail) return;                      // uniform
    if (own && bj == jb && bi > jb) {       // panel: A_bi,jb <- A_bi,jb L_jb,jb^-T
#pragma unroll
      for (int r = 0; r < kPB; ++r) {
#pragma unroll
        for (int q = 0; q < kPB; ++q) {
          double x = a[r][q];
#pragma unroll
          for (int p = 0; p < q; ++p) x = fma(-a[r][p], sld[q][p], x);
          a[r][q] = x * srd[q];
        }
        *reinterpret_cast<double4*>(&pan[r0 + r][0]) = make_double4(a[r][0], a[r][1], a[r][2], a[r][3]);
      }
    }
    __syncthreads();
    if (own && bj > jb) {                   // trailing rank-4 update
      double u[kPB][kPB];
#pragma unroll
      for (int r = 0; r < kPB; ++r) {
        const double4 pu = *reinterpret_cast<const double4*>(&pan[r0 + r][0]);
        u[r][0] = pu.x; u[r][1] = pu.y; u[r][2] = pu.z; u[r][3] = pu.w;
      }
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        const double4 pw = *reinterpret_cast<const double4*>(&pan[c0 + c][0]);
#pragma unroll
        for (int r = 0; r < kPB; ++r) {
          if (bi == bj && c > r) continue;
          double x = a[r][c];
          x = fma(-u[r][0], pw.x, x);
          x = fma(-u[r][1], pw.y, x);
          x = fma(-u[r][2], pw.z, x);
          a[r][c] = fma(-u[r][3], pw.w, x);
        }
      }
    }
    __syncthreads();
  }
  // L out (global, column-major, upper zeroed) and to shared for the inverse
  if (own) {
#pragma unroll
    for (int r = 0; r < kPB; ++r)
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        const int row = r0 + r, col = c0 + c;
        const double v = row >= col ? a[r][c] : 0.0;
        sL[row * kTLd + col] = v;
        t[(int64_t)col * kTT + row] = v;
        if (bi != bj) t[(int64_t)row * kTT + col] = 0.0;      // mirrored upper block
      }
  }
  __syncthreads();
  if (tid < kTT) rdiag[tid] = 1.0 / sL[tid * kTLd + tid];
#pragma unroll
  for (int r = 0; r < kPB; ++r)
#pragma unroll
    for (int c = 0; c < kPB; ++c) a[r][c] = own && r0 + r == c0 + c ? 1.0 : 0.0;
  __syncthreads();
  double (*xs)[kTT] = reinterpret_cast<double (*)[kTT]>(&pan[0][0]);   // [4][128]
  for (int jb = 0; jb < kPNB; ++jb) {
    if (own && bi == jb) {                  // X_jb,bc = L_jb,jb^-1 R_jb,bc
#pragma unroll
      for (int r = 0; r < kPB; ++r) {
        const double* lr = sL + (r0 + r) * kTLd + r0;
#pragma unroll
        for (int c = 0; c < kPB; ++c) {
          double x = a[r][c];
#pragma unroll
          for (int p = 0; p < r; ++p) x = fma(-lr[p], a[p][c], x);
          a[r][c] = x * rdiag[r0 + r];
        }
        *reinterpret_cast<double4*>(&xs[r][c0]) = make_double4(a[r][0], a[r][1], a[r][2], a[r][3]);
      }
    }
    __syncthreads();
    if (own && bi > jb && bj <= jb) {       // R_bi,bc -= L_bi,jb X_jb,bc
      double xv[kPB][kPB];
#pragma unroll
      for (int p = 0; p < kPB; ++p) {
        const double4 v = *reinterpret_cast<const double4*>(&xs[p][c0]);
        xv[p][0] = v.x; xv[p][1] = v.y; xv[p][2] = v.z; xv[p][3] = v.w;
      }
#pragma unroll
      for (int r = 0; r < kPB; ++r) {
        const double* lr = sL + (r0 + r) * kTLd + jb * kPB;
        const double l0 = lr[0], l1 = lr[1], l2 = lr[2], l3 = lr[3];
#pragma unroll
        for (int c = 0; c < kPB; ++c) {
          double x = a[r][c];
          x = fma(-l0, xv[0][c], x);
          x = fma(-l1, xv[1][c], x);
          x = fma(-l2, xv[2][c], x);
          a[r][c] = fma(-l3, xv[3][c], x);
        }
      }
    }
    __syncthreads();
  }
  if (own) {
#pragma unroll
    for (int r = 0; r < kPB; ++r)
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        const int row = r0 + r, col = c0 + c;
        inv[(int64_t)col * kTT + row] = row >= col ? a[r][c] : 0.0;
        if (bi != bj) inv[(int64_t)row * kTT + col] = 0.0;
      }
  }
}

// ------------------------------------------------------ DMMA GEMM update --
// mode 0 (Cholesky trailing update at step k): blocks over pairs
//   k < j <= i:  C_ij -= A_ik A_jk^T
// mode 1 (left-TRSM update after row s of X): blocks over (l > s, j <= s):
//   P_lj -= L_ls X_sj
// mode 2 (panel solve at step k, i > k):   C_ik  = C_ik Inv_k^T   (in place)
// mode 3 (row solve at row s, j <= s):     X_sj  = Inv_s P_sj     (in place)
// (in place is safe: all global reads of the operand happen before the
// epilogue's stores)
constexpr int kGKc = 16;
constexpr int kGLd = kTT + 4;
constexpr size_t kGSmem = 2 * 2 * kGKc * kGLd * sizeof(double);

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 1)
tail_gemm_kernel(double* base_c, const double* base_a, const double* base_b, int k, int nt,
                 int mode) {      // operands may alias C (modes 0, 2, 3): no __restrict__
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + 2 * kGKc * kGLd;
  const double *A, *B;
  double* C;
  if (mode == 0 || mode >= 4) {
    // 0: whole trailing triangle; 4: its first column (j = k + 1) only;
    // 5: the rest (j >= k + 2), so that the next diagonal tile can be
    // factored while mode 5 runs (look-ahead)
    int a, b;
    if (mode == 4) {
      a = blockIdx.x;
      b = 0;
    } else {
      tri_idx(blockIdx.x, a, b);
      if (mode == 5) {
        ++a;
        ++b;
      }
    }
    const int i = k + 1 + a, j = k + 1 + b;
    C = base_c + tslot(i, j) * kTE;
    A = base_a + tslot(i, k) * kTE;
    B = base_a + tslot(j, k) * kTE;
  } else if (mode == 1) {
    const int l = k + 1 + blockIdx.x / (k + 1), j = blockIdx.x % (k + 1);
    C = base_c + tslot(l, j) * kTE;
    A = base_a + tslot(l, k) * kTE;
    B = base_b + tslot(k, j) * kTE;
  } else if (mode == 2) {
    C = base_c + tslot(k + 1 + blockIdx.x, k) * kTE;
    A = C;
    B = base_b + (int64_t)k * kTE;          // inverse of diagonal tile k
  } else {
    C = base_c + tslot(k, blockIdx.x) * kTE;
    A = base_a + (int64_t)k * kTE;          // inverse of diagonal tile k
    B = C;
  }
  const bool bt = mode == 0 || mode == 2 || mode >= 4;   // B operand used transposed
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, tg = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // loaders: A (and B in mode 0) column-major m-panels: thread -> row
  // tid & 127, 8 k values; mode 1 B[m][c]: thread -> col tid >> 1, 8 k
  const int lr = tid & 127, lk = (tid >> 7) * 8;
  const int bc = tid >> 1, bk = (tid & 1) * 8;
  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      ra[q] = A[(int64_t)(k0 + lk + q) * kTT + lr];
      rb[q] = bt ? B[(int64_t)(k0 + lk + q) * kTT + lr] : B[(int64_t)bc * kTT + k0 + bk + q];
    }
  };
  load(0);
  int stage = 0;
  for (int k0 = 0; k0 < kTT; k0 += kGKc) {
    double* as = As + stage * kGKc * kGLd;
    double* bs = Bs + stage * kGKc * kGLd;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      as[(lk + q) * kGLd + lr] = ra[q];
      if (bt) bs[(lk + q) * kGLd + lr] = rb[q];
      else bs[(bk + q) * kGLd + bc] = rb[q];
    }
    __syncthreads();
    if (k0 + kGKc < kTT) load(k0 + kGKc);
#pragma unroll
    for (int ks = 0; ks < kGKc / 4; ++ks) {
      double af[8], bf[4];
      const double* ak = as + (ks * 4 + tg) * kGLd + wr * 64 + g;
      const double* bk2 = bs + (ks * 4 + tg) * kGLd + wc * 32 + g;
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = ak[a * 8];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bk2[b * 8];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    stage ^= 1;
  }
  // C[r][c] (column-major) -= acc
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int r = wr * 64 + a * 8 + g;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wc * 32 + b * 8 + 2 * tg + e;
        if (mode <= 1 || mode >= 4) C[(int64_t)c * kTT + r] -= acc[a][b][e];
        else C[(int64_t)c * kTT + r] = acc[a][b][e];
      }
  }
}

// ------------------------------------------------------ vector solves --
// Blocked forward / backward substitution with the diagonal inverses:
//   forward  (L y = b):   y_i = Inv_i acc_i;     acc_l -= L_li y_i   (l > i)
//   backward (L^T y = b): y_i = Inv_i^T acc_i;   acc_l -= L_il^T y_i (l < i)
// diag: one CTA; update: one CTA per remaining tile row (128 threads each).
__global__ void __launch_bounds__(kTT)
tail_vec_diag_kernel(const double* __restrict__ inv, int i, const double* __restrict__ acc,
                     double* __restrict__ y, int trans) {
  __shared__ double sa[kTT];
  const int r = threadIdx.x;
  sa[r] = acc[(int64_t)i * kTT + r];
  __syncthreads();
  const double* Iv = inv + (int64_t)i * kTE;
  double s = 0.0;
  for (int c = 0; c < kTT; ++c)
    s = fma(trans ? Iv[(int64_t)r * kTT + c] : Iv[(int64_t)c * kTT + r], sa[c], s);
  y[(int64_t)i * kTT + r] = s;
}

__global__ void __launch_bounds__(kTT)
tail_vec_update_kernel(const double* __restrict__ base, int i, const double* __restrict__ y,
                       double* __restrict__ acc, int trans) {
  __shared__ double sy[kTT];
  const int r = threadIdx.x;
  sy[r] = y[(int64_t)i * kTT + r];
  __syncthreads();
  const int l = trans ? blockIdx.x : i + 1 + blockIdx.x;
  double s = 0.0;
  if (!trans) {
    const double* T = base + tslot(l, i) * kTE;      // L_li[r][c]
    for (int c = 0; c < kTT; ++c) s = fma(T[(int64_t)c * kTT + r], sy[c], s);
  } else {
    const double* T = base + tslot(i, l) * kTE;      // L_il^T[r][c] = L_il[c][r]
    for (int c = 0; c < kTT; ++c) s = fma(T[(int64_t)r * kTT + c], sy[c], s);
  }
  acc[(int64_t)l * kTT + r] -= s;
}

// ------------------------------------------------------------ reductions --
// out[blk] = sum over tile u of (mode 0) log diag, (mode 1) squares (lower)
__global__ void __launch_bounds__(256)
tail_reduce_kernel(const double* __restrict__ base, int mode, double* __restrict__ part) {
  __shared__ double red[8];
  int a, b;
  tri_idx(blockIdx.x, a, b);
  const double* t = base + tslot(a, b) * kTE;
  double s = 0.0;
  if (mode == 0) {
    if (a == b && threadIdx.x < kTT) s = log(t[(int64_t)threadIdx.x * kTT + threadIdx.x]);
  } else {
    for (int e = threadIdx.x; e < kTE; e += blockDim.x) {
      const int c = e / kTT, r = e % kTT;
      if (a != b || r >= c) s = fma(t[e], t[e], s);
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w];
    part[blockIdx.x] = v;
  }
}

// min and max of diag(L)^2 over the M real rows (padding rows are identity):
// cond(Kuu) >= max/min, the conditioning indicator the Python layer uses to
// move engine "auto" to fp64 statistics (one block, 128 threads)
__global__ void tail_diag_range_kernel(const double* __restrict__ L, int nt, int64_t M,
                                       double* __restrict__ out2) {
  __shared__ double smin[kTT], smax[kTT];
  double lo = INFINITY, hi = 0.0;
  for (int a = 0; a < nt; ++a) {
    const int64_t row = (int64_t)a * kTT + threadIdx.x;
    if (row < M) {
      const double d = L[tslot(a, a) * kTE + (int64_t)threadIdx.x * kTT + threadIdx.x];
      lo = fmin(lo, d * d);
      hi = fmax(hi, d * d);
    }
  }
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < kTT; ++t) {
      lo = fmin(lo, smin[t]);
      hi = fmax(hi, smax[t]);
    }
    out2[0] = lo;
    out2[1] = hi;
  }
}

__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  // fixed order: lane-strided partial sums, then a fixed shuffle tree
  double s = 0.0;
  for (int q = threadIdx.x; q < n; q += 32) s += part[q];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

__global__ void dot_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) s = fma(a[e], a[e], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
    *out = v;
  }
}

__global__ void scale_copy_kernel(const double* __restrict__ a, int64_t n, int64_t n_pad,
                                  double s, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_pad) out[e] = e < n ? a[e] * s : 0.0;
}

// ------------------------------------------------------------------ host --
// Blocked right-looking Cholesky with one step of look-ahead: after the
// panel of step k, the first trailing column is updated alone, then the
// diagonal tile k+1 is factored on a high-priority side stream while the rest
// of the trailing update runs on `st`.
static int tail_cholesky(double* base, double* inv, int nt, int* info, cudaStream_t st,
                         cudaStream_t side, cudaEvent_t e_col, cudaEvent_t e_diag) {
  tail_potrf_inv_kernel<<<1, kPThreads, (size_t)kTT * kTLd * 8, st>>>(base, 0, inv, info);
  TB_LAUNCH_CHECK("tail_potrf_inv");
  for (int k = 0; k + 1 < nt; ++k) {
    const int below = nt - k - 1;
    if (k > 0) TB_CUDA_TRY(cudaStreamWaitEvent(st, e_diag, 0));     // potrf(k) done
    tail_gemm_kernel<<<below, 256, kGSmem, st>>>(base, base, inv, k, nt, 2);       // panel
    TB_LAUNCH_CHECK("tail_panel");
    tail_gemm_kernel<<<below, 256, kGSmem, st>>>(base, base, base, k, nt, 4);      // column k+1
    TB_LAUNCH_CHECK("tail_update_col");
    TB_CUDA_TRY(cudaEventRecord(e_col, st));
    TB_CUDA_TRY(cudaStreamWaitEvent(side, e_col, 0));
    tail_potrf_inv_kernel<<<1, kPThreads, (size_t)kTT * kTLd * 8, side>>>(
        base, k + 1, inv + (int64_t)(k + 1) * kTE, info);
    TB_LAUNCH_CHECK("tail_potrf_inv");
    TB_CUDA_TRY(cudaEventRecord(e_diag, side));
    if (below > 1) {
      tail_gemm_kernel<<<below * (below - 1) / 2, 256, kGSmem, st>>>(base, base, base, k, nt, 5);
      TB_LAUNCH_CHECK("tail_update_rest");
    }
  }
  if (nt > 1) TB_CUDA_TRY(cudaStreamWaitEvent(st, e_diag, 0));
  return TB_OK;
}

// y = L^-1 b (trans = 0) or L^-T b (trans = 1); acc is scratch [M_pad]
static int tail_solve(const double* base, const double* inv, int nt, const double* b,
                      double* acc, double* y, int trans, cudaStream_t st) {
  TB_CUDA_TRY(cudaMemcpyAsync(acc, b, (size_t)nt * kTT * 8, cudaMemcpyDeviceToDevice, st));
  for (int s = 0; s < nt; ++s) {
    const int i = trans ? nt - 1 - s : s;
    tail_vec_diag_kernel<<<1, kTT, 0, st>>>(inv, i, acc, y, trans);
    const int rest = trans ? i : nt - 1 - i;
    if (rest) tail_vec_update_kernel<<<rest, kTT, 0, st>>>(base, i, y, acc, trans);
  }
  TB_LAUNCH_CHECK("tail_solve");
  return TB_OK;
}

int64_t tail_workspace_bytes(int64_t M, int64_t M_pad, int64_t dim) {
  const int64_t nt = M_pad / kTT, tiles = nt * (nt + 1) / 2;
  return round_up(tiles * kTE * 8, 256)            // L (packed)
         + round_up(2 * nt * kTE * 8, 256)         // inverses of the diagonal tiles of L, P
         + round_up(M * dim * 8, 256)              // scaled Z
         + round_up(4 * M_pad * 8, 256)            // u, w, v copy, solve scratch
         + round_up((tiles + 8) * 8, 256) + 256;   // partials, scalars, info
}

int tail_run(int64_t M, int64_t M_pad, const void* Z, int dtype, const KernParams& kp,
             double jitter, double noise, double* sigma, const double* v, double* w_out,
             double* out4, void* workspace, cudaStream_t st) {
  const int nt = (int)(M_pad / kTT);
  const int tiles = nt * (nt + 1) / 2;
  char* ws = (char*)workspace;
  double* L = (double*)ws;
  ws += round_up((int64_t)tiles * kTE * 8, 256);
  double* invL = (double*)ws;
  double* invP = invL + (int64_t)nt * kTE;
  ws += round_up(2 * (int64_t)nt * kTE * 8, 256);
  double* Zs = (double*)ws;
  ws += round_up(M * kp.dim * 8, 256);
  double* u = (double*)ws;
  double* w = u + M_pad;
  double* vv = w + M_pad;
  double* scratch = vv + M_pad;
  ws += round_up(4 * M_pad * 8, 256);
  double* part = (double*)ws;
  double* scal = part + tiles;            // [0] logdet L, [1] logdet P, [2] |u|^2, [3] ||X||^2,
                                          // [4] min diag(L)^2, [5] max diag(L)^2
  int* info = (int*)(scal + 6);
  TB_CUDA_TRY(cudaFuncSetAttribute(tail_potrf_inv_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((size_t)kTT * kTLd * 8)));
  TB_CUDA_TRY(cudaFuncSetAttribute(tail_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kGSmem));
  TB_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int), st));
  const unsigned zb = (unsigned)ceil_div(std::max<int64_t>(M * kp.dim, 1), 256);
  if (dtype == TB_F32)
    scale_z_kernel<float><<<zb, 256, 0, st>>>((const float*)Z, M, kp, Zs);
  else
    scale_z_kernel<double><<<zb, 256, 0, st>>>((const double*)Z, M, kp, Zs);
  TB_LAUNCH_CHECK("scale_z");
  // L = chol(Kuu)
  tail_kuu_kernel<<<tiles, 256, 0, st>>>(Zs, M, kp, jitter, 0.0, L);
  TB_LAUNCH_CHECK("tail_kuu");
  cudaStream_t side = nullptr;
  cudaEvent_t e_col = nullptr, e_diag = nullptr;
  int lo_p = 0, hi_p = 0;
  TB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
  TB_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi_p));
  TB_CUDA_TRY(cudaEventCreateWithFlags(&e_col, cudaEventDisableTiming));
  TB_CUDA_TRY(cudaEventCreateWithFlags(&e_diag, cudaEventDisableTiming));
  struct Cleanup {
    cudaStream_t s;
    cudaEvent_t a, b;
    ~Cleanup() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaStreamDestroy(s);
    }
  } cleanup{side, e_col, e_diag};
  int rc = tail_cholesky(L, invL, nt, info, st, side, e_col, e_diag);
  if (rc) return rc;
  // P = chol(Kuu + Sigma / s2), in place over Sigma
  tail_kuu_kernel<<<tiles, 256, 0, st>>>(Zs, M, kp, jitter, 1.0 / noise, sigma);
  TB_LAUNCH_CHECK("tail_kuu_add");
  if ((rc = tail_cholesky(sigma, invP, nt, info, st, side, e_col, e_diag))) return rc;
  // log dets
  tail_reduce_kernel<<<tiles, 256, 0, st>>>(L, 0, part);
  sum_kernel<<<1, 32, 0, st>>>(part, tiles, scal + 0);
  tail_diag_range_kernel<<<1, kTT, 0, st>>>(L, nt, M, scal + 4);
  tail_reduce_kernel<<<tiles, 256, 0, st>>>(sigma, 0, part);
  sum_kernel<<<1, 32, 0, st>>>(part, tiles, scal + 1);
  TB_LAUNCH_CHECK("tail_logdet");
  // u = P^-1 v,  |u|^2,  w = P^-T u / s2
  scale_copy_kernel<<<(unsigned)ceil_div(M_pad, 256), 256, 0, st>>>(v, M, M_pad, 1.0, vv);
  if ((rc = tail_solve(sigma, invP, nt, vv, scratch, u, 0, st))) return rc;
  dot_kernel<<<1, 256, 0, st>>>(u, M_pad, scal + 2);
  if ((rc = tail_solve(sigma, invP, nt, u, scratch, w, 1, st))) return rc;
  scale_copy_kernel<<<(unsigned)ceil_div(M, 256), 256, 0, st>>>(w, M, M, 1.0 / noise, w_out);
  TB_LAUNCH_CHECK("tail_vec");
  // X = L^-1 P in place over P, row by row: X_ij = Inv_i P_ij (j <= i), then
  // P_lj -= L_li X_ij for the rows below; then ||X||_F^2
  for (int i = 0; i < nt; ++i) {
    tail_gemm_kernel<<<i + 1, 256, kGSmem, st>>>(sigma, invL, sigma, i, nt, 3);
    TB_LAUNCH_CHECK("tail_row_solve");
    const int below = nt - i - 1;
    if (below == 0) break;
    tail_gemm_kernel<<<below * (i + 1), 256, kGSmem, st>>>(sigma, L, sigma, i, nt, 1);
    TB_LAUNCH_CHECK("tail_row_update");
  }
  tail_reduce_kernel<<<tiles, 256, 0, st>>>(sigma, 1, part);
  sum_kernel<<<1, 32, 0, st>>>(part, tiles, scal + 3);
  TB_LAUNCH_CHECK("tail_frob");
  TB_CUDA_TRY(cudaMemcpyAsync(out4, scal, 6 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int h_info = 0;
  TB_CUDA_TRY(cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  TB_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info)
    return fail(TB_ERR_ARG, "sgpr tail: Cholesky failed at row " + std::to_string(h_info - 1) +
                                " (matrix not positive definite)");
  return TB_OK;
}

// ======================================================= gradient tail ==
// The GPflow training gradient of the ELBO inside memory_limit (DESIGN.md §4
// "Gradient").  With Kuu = L L^T, A = Kuu + Sigma/s2 = P P^T, w = A^-1 v / s2:
//   G2 = 2 dELBO/dSigma = (Kuu^-1 - A^-1 - w w^T) / s2
//   H2 = 2 dELBO/dKuu   = 2 Kuu^-1 - A^-1 - Kuu^-1 A Kuu^-1 - w w^T
// Only the two packed factors L and P stay resident; both M x M matrices are
// produced one 128-column panel at a time (E_P = identity columns of tile P):
//   Kuu^-1[:,P] = L^-T L^-1 E_P,   A^-1[:,P] = P^-T P^-1 E_P,
//   (Kuu^-1 A Kuu^-1)[:,P] = L^-T L^-1 P P^T Kuu^-1[:,P]
// and consumed at once: H2[:,P] against the kernel derivatives over Z x Z_P
// (tb_sgpr_kuf_grad with K recomputed), G2[:,P] by the fused data kernel
// below, which streams all N points, generating the Kuf tiles it multiplies
// on the fly (W[P,:] = G2[:,P]^T Kuf + g_P y^T never exists in memory) and
// contracting W with the kernel derivatives in its epilogue.
namespace cg = cooperative_groups;

// acc(r, c) += sum_k opA(r, k) opB(k, c) over one 128 x 128 x 128 tile
// product, column-major tiles, the DMMA fragment layout of tail_gemm_kernel:
//   opA(r, k) = ta ? A[r*128 + k] : A[k*128 + r]
//   opB(k, c) = tb ? B[k*128 + c] : B[c*128 + k]
// GEN (data kernel): opB is generated by gen(k, c) instead of loaded.
template <typename Gen>
__device__ __forceinline__ void tile_mma_impl(double (&acc)[8][4][2], const double* A, bool ta,
                                              const double* B, bool tb, double* sm, Gen gen,
                                              bool use_gen) {
  double* As = sm;
  double* Bs = sm + 2 * kGKc * kGLd;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, tg = lane & 3;
  const int cr = tid & 127, ck = (tid >> 7) * 8;      // "column" pattern (row fastest)
  const int rr = tid >> 1, rk = (tid & 1) * 8;        // "row" pattern (k fastest)
  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      ra[q] = ta ? A[(int64_t)rr * kTT + k0 + rk + q] : A[(int64_t)(k0 + ck + q) * kTT + cr];
      if (use_gen) rb[q] = gen(k0 + ck + q, cr);
      else rb[q] = tb ? B[(int64_t)(k0 + ck + q) * kTT + cr] : B[(int64_t)rr * kTT + k0 + rk + q];
    }
  };
  const bool bcol = use_gen || tb;
  load(0);
  int stage = 0;
  for (int k0 = 0; k0 < kTT; k0 += kGKc) {
    double* as = As + stage * kGKc * kGLd;
    double* bs = Bs + stage * kGKc * kGLd;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (ta) as[(rk + q) * kGLd + rr] = ra[q];
      else as[(ck + q) * kGLd + cr] = ra[q];
      if (bcol) bs[(ck + q) * kGLd + cr] = rb[q];
      else bs[(rk + q) * kGLd + rr] = rb[q];
    }
    __syncthreads();
    if (k0 + kGKc < kTT) load(k0 + kGKc);
#pragma unroll
    for (int ks = 0; ks < kGKc / 4; ++ks) {
      double af[8], bf[4];
      const double* ak = as + (ks * 4 + tg) * kGLd + wr * 64 + g;
      const double* bk2 = bs + (ks * 4 + tg) * kGLd + wc * 32 + g;
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = ak[a * 8];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bk2[b * 8];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    stage ^= 1;
  }
  __syncthreads();
}
struct NoGen {
  __device__ double operator()(int, int) const { return 0.0; }
};
__device__ __forceinline__ void tile_mma(double (&acc)[8][4][2], const double* A, bool ta,
                                         const double* B, bool tb, double* sm) {
  tile_mma_impl(acc, A, ta, B, tb, sm, NoGen{}, false);
}
__device__ __forceinline__ void acc_zero(double (&acc)[8][4][2]) {
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
}
// C (column-major tile) = acc (mode 0) or C -= acc (mode 1)
__device__ __forceinline__ void acc_store(const double (&acc)[8][4][2], double* C, int mode) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, tg = lane & 3;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int r = wr * 64 + a * 8 + g;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wc * 32 + b * 8 + 2 * tg + e;
        if (mode) C[(int64_t)c * kTT + r] -= acc[a][b][e];
        else C[(int64_t)c * kTT + r] = acc[a][b][e];
      }
  }
}

// Panel triangular solve in place, one cooperative launch:
//   TRANS = 0: L Y = B (forward from tile row i0; the rows above are zero)
//   TRANS = 1: L^T Y = B (backward over all tile rows)
// step i: CTA 0 applies the diagonal inverse, grid sync, every CTA updates
// its share of the remaining tile rows, grid sync.
template <int TRANS>
__global__ void __launch_bounds__(256, 1)
gp_trsm_kernel(const double* __restrict__ L, const double* __restrict__ inv, double* Y, int nt,
               int i0) {
  extern __shared__ __align__(16) double gsm[];
  cg::grid_group grid = cg::this_grid();
  double acc[8][4][2];
  const int steps = TRANS ? nt : nt - i0;
  for (int s = 0; s < steps; ++s) {
    const int i = TRANS ? nt - 1 - s : i0 + s;
    double* Yi = Y + (int64_t)i * kTE;
    if (blockIdx.x == 0) {
      acc_zero(acc);
      tile_mma(acc, inv + (int64_t)i * kTE, TRANS, Yi, false, gsm);
      acc_store(acc, Yi, 0);
    }
    grid.sync();
    const int cnt = TRANS ? i : nt - 1 - i;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
      const int k = TRANS ? q : i + 1 + q;
      acc_zero(acc);
      tile_mma(acc, L + (TRANS ? tslot(i, k) : tslot(k, i)) * kTE, TRANS, Yi, false, gsm);
      acc_store(acc, Y + (int64_t)k * kTE, 1);
    }
    grid.sync();
  }
}

// out = L Y (TRANS = 0) or L^T Y (TRANS = 1), out of place; CTA = out tile row
template <int TRANS>
__global__ void __launch_bounds__(256, 1)
gp_trmm_kernel(const double* __restrict__ L, const double* __restrict__ Y,
               double* __restrict__ out, int nt) {
  extern __shared__ __align__(16) double gsm[];
  const int k = blockIdx.x;
  double acc[8][4][2];
  acc_zero(acc);
  if (!TRANS) {
    for (int j = 0; j <= k; ++j)
      tile_mma(acc, L + tslot(k, j) * kTE, false, Y + (int64_t)j * kTE, false, gsm);
  } else {
    for (int j = k; j < nt; ++j)
      tile_mma(acc, L + tslot(j, k) * kTE, true, Y + (int64_t)j * kTE, false, gsm);
  }
  acc_store(acc, out + (int64_t)k * kTE, 0);
}

// Y = E_P (identity columns of tile P; padding included, like the packed
// identity padding of the factors)
__global__ void gp_identity_kernel(double* __restrict__ Y, int P, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / kTE;
    const int c = (int)((e % kTE) / kTT), r = (int)(e % kTT);
    Y[e] = (t == P && r == c) ? 1.0 : 0.0;
  }
}

// panel element (i, c), i = global row, c = panel column
__device__ __forceinline__ int64_t pidx(int64_t i, int c) {
  return (i / kTT) * kTE + (int64_t)c * kTT + (i % kTT);
}

// G2*s2 = Kinv - Ainv - w w^T -> Kinv buffer;  H2 = 2 Kinv - Ainv - KAK - w w^T -> KAK buffer
__global__ void gp_combine_kernel(double* __restrict__ kinv, const double* __restrict__ ainv,
                                  double* __restrict__ kak, const double* __restrict__ w, int P,
                                  int64_t M, int64_t M_pad) {
  const int64_t n = M_pad * kTT;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / kTE;
    const int c = (int)((e % kTE) / kTT), r = (int)(e % kTT);
    const int64_t i = t * kTT + r, j = (int64_t)P * kTT + c;
    const double ww = (i < M && j < M) ? w[i] * w[j] : 0.0;
    const double k1 = kinv[e], a1 = ainv[e];
    kinv[e] = k1 - a1 - ww;
    kak[e] = 2.0 * k1 - a1 - kak[e] - ww;
  }
}

// part[P] = sum over the valid columns c of T(P*128 + c, c)  (trace block)
__global__ void gp_diag_trace_kernel(const double* __restrict__ T, int P, int64_t M,
                                     double* __restrict__ part) {
  double s = 0.0;
  for (int c = threadIdx.x; c < kTT; c += 32)
    if ((int64_t)P * kTT + c < M) s += T[(int64_t)P * kTE + (int64_t)c * kTT + c];
  s = warp_sum(s);
  if (threadIdx.x == 0) part[P] = s;
}

// Per block b: part[b] = (sum_ic Kuu(i, Pc) Ainv(i, c), sum_ic Kuu(i, Pc) w_i w_Pc)
// over the valid entries; Kuu generated on the fly (no panel)
__global__ void __launch_bounds__(256)
gp_kuu_dot_kernel(const double* __restrict__ Zs, const double* __restrict__ ainv,
                  const double* __restrict__ w, int P, int64_t M, KernParams p, double jitter,
                  double* __restrict__ part) {
  __shared__ double red[2][8];
  double s1 = 0.0, s2 = 0.0;
  const int64_t n = M * kTT;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / kTT;
    const int c = (int)(e % kTT);
    const int64_t j = (int64_t)P * kTT + c;
    if (j >= M) continue;
    double r2 = 0.0;
    for (int d = 0; d < p.dim; ++d) {
      const double df = Zs[i * p.dim + d] - Zs[j * p.dim + d];
      r2 = fma(df, df, r2);
    }
    const double k = kern_from_r2(p, r2) + (i == j ? jitter : 0.0);
    s1 = fma(k, ainv[pidx(i, c)], s1);
    s2 = fma(k, w[i] * w[j], s2);
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s1;
    red[1][threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += red[threadIdx.x][q];
    part[2 * blockIdx.x + threadIdx.x] = v;
  }
}

// out1[P] = sum_b part[2b], out2[P] = sum_b part[2b+1] (fixed order, one warp)
__global__ void gp_pair_sum_kernel(const double* __restrict__ part, int nb, int P,
                                   double* __restrict__ out1, double* __restrict__ out2) {
  double a = 0.0, b = 0.0;
  for (int q = threadIdx.x; q < nb; q += 32) {
    a += part[2 * q];
    b += part[2 * q + 1];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (threadIdx.x == 0) {
    out1[P] = a;
    out2[P] = b;
  }
}

// dense row-major [M x nc] copy of panel columns 0..nc-1 (tb_sgpr_kuf_grad's W)
__global__ void gp_to_rowmajor_kernel(const double* __restrict__ Y, int64_t M, int nc,
                                      double* __restrict__ out) {
  const int64_t n = M * nc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = Y[pidx(e / nc, (int)(e % nc))];
}

// Fused data side for panel P: for every block of 128 training points,
//   W(p, n) = (sum_i G2s2(i, P*128+p) Kuf(i, n)) / s2 + (w_p / s2) y_n
// (DMMA over the inducing tiles; Kuf tiles generated in the operand loader),
// then the kernel-derivative contraction of tb_sgpr_kuf_grad in the
// epilogue: dvariance += W k / var, dl_t += W k' (-2 (x_t - z_t)^2 / l_t^3),
// dz_pt += W k' (2 (z_t - x_t) / l_t^2).  Work items (point blocks) are dealt
// round-robin to a fixed grid and every CTA accumulates in a fixed order;
// per-CTA partials are reduced in a fixed order afterwards (deterministic).
template <typename T, int DMAX>
__global__ void __launch_bounds__(256, 1)
gp_data_kernel(const T* __restrict__ X, const T* __restrict__ y, const double* __restrict__ Zs,
               const double* __restrict__ G, const double* __restrict__ w, double inv_s2, int P,
               int nt, int64_t M, int64_t N, KernParams p, double* __restrict__ part_hyp,
               double* __restrict__ part_z) {
  extern __shared__ __align__(16) double gsm[];
  double* mma_sm = gsm;                                   // 2 * 2 * kGKc * kGLd
  double* zt = gsm + 4 * kGKc * kGLd;                     // [128][DMAX] inducing tile (scaled)
  double* zp = zt + kTT * DMAX;                           // [128][DMAX] panel rows
  double* xb = zp + kTT * DMAX;                           // [128][DMAX] point block
  double* yb = xb + kTT * DMAX;                           // [128]
  double* gp_s = yb + kTT;                                // [128] w_p / s2
  double* zacc = gp_s + kTT;                              // [128][DMAX] dz accumulators
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, tg = lane & 3;
  const int dim = p.dim;
  for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
    const int r = e / DMAX, t = e % DMAX;
    const int64_t i = (int64_t)P * kTT + r;
    zp[e] = (t < dim && i < M) ? Zs[i * dim + t] : 0.0;
    zacc[e] = 0.0;
  }
  for (int r = tid; r < kTT; r += blockDim.x) {
    const int64_t i = (int64_t)P * kTT + r;
    gp_s[r] = i < M ? w[i] * inv_s2 : 0.0;
  }
  double gv = 0.0, gl[DMAX];
#pragma unroll
  for (int t = 0; t < DMAX; ++t) gl[t] = 0.0;
  const int64_t nblk = (N + kTT - 1) / kTT;
  const int cr = tid & 127;
  double xr[DMAX];
  for (int64_t nb = blockIdx.x; nb < nblk; nb += gridDim.x) {
    __syncthreads();
    for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
      const int r = e / DMAX, t = e % DMAX;
      const int64_t n = nb * kTT + r;
      xb[e] = (t < dim && n < N) ? (double)X[n * dim + t] * p.inv_ls[t] : 0.0;
    }
    for (int r = tid; r < kTT; r += blockDim.x) {
      const int64_t n = nb * kTT + r;
      yb[r] = n < N ? (double)y[n] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < DMAX; ++t) xr[t] = xb[cr * DMAX + t];     // this thread's loader point
    const bool pvalid = nb * kTT + cr < N;
    double acc[8][4][2];
    acc_zero(acc);
    for (int kt = 0; kt < nt; ++kt) {
      for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
        const int r = e / DMAX, t = e % DMAX;
        const int64_t i = (int64_t)kt * kTT + r;
        zt[e] = (t < dim && i < M) ? Zs[i * dim + t] : 0.0;
      }
      __syncthreads();
      const int64_t ibase = (int64_t)kt * kTT;
      auto gen = [&](int k, int c) -> double {      // Kuf(inducing ibase + k, point c = cr)
        if (!pvalid || ibase + k >= M) return 0.0;
        double r2 = 0.0;
#pragma unroll
        for (int t = 0; t < DMAX; ++t)
          if (t < dim) {
            const double df = zt[k * DMAX + t] - xr[t];
            r2 = fma(df, df, r2);
          }
        return kern_from_r2(p, r2);
      };
      tile_mma_impl(acc, G + (int64_t)kt * kTE, true, nullptr, true, mma_sm, gen, true);
    }
    // epilogue: W and the kernel-derivative contraction
    double* red = mma_sm;                                  // [4 wc][128][DMAX] (reuse)
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int r = wr * 64 + a * 8 + g;
      double gz[DMAX];
#pragma unroll
      for (int t = 0; t < DMAX; ++t) gz[t] = 0.0;
      const bool rvalid = (int64_t)P * kTT + r < M;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = wc * 32 + b * 8 + 2 * tg + e;
          if (!rvalid || nb * kTT + c >= N) continue;
          const double W = acc[a][b][e] * inv_s2 + gp_s[r] * yb[c];
          double r2 = 0.0;
#pragma unroll
          for (int t = 0; t < DMAX; ++t)
            if (t < dim) {
              const double df = zp[r * DMAX + t] - xb[c * DMAX + t];
              r2 = fma(df, df, r2);
            }
          const double k = kern_from_r2(p, r2);
          double dk;
          if (p.kernel == TB_KERNEL_RBF) {
            dk = -0.5 * k;
          } else {
            const double rr = sqrt(fmax(r2, 1e-36));
            dk = -1.5 * p.variance * exp(-1.7320508075688772 * rr);
          }
          const double wd = W * dk;
          gv = fma(W, k, gv);
#pragma unroll
          for (int t = 0; t < DMAX; ++t)
            if (t < dim) {
              const double df = zp[r * DMAX + t] - xb[c * DMAX + t];
              gl[t] = fma(wd * df * df, -2.0 * p.inv_ls[t], gl[t]);
              gz[t] = fma(wd * df, 2.0 * p.inv_ls[t], gz[t]);
            }
        }
      // sum over the 4 lanes sharing row r (tg), then stage per wc
#pragma unroll
      for (int t = 0; t < DMAX; ++t) {
        double v = gz[t];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (tg == 0) red[((int64_t)wc * kTT + r) * DMAX + t] = v;
      }
    }
    __syncthreads();
    for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
      const int r = e / DMAX, t = e % DMAX;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) v += red[((int64_t)q * kTT + r) * DMAX + t];
      zacc[e] += v;
    }
  }
  __syncthreads();
  // per-CTA partials: dz rows of panel P, then (variance, lengthscales)
  for (int e = tid; e < kTT * DMAX; e += blockDim.x) part_z[(int64_t)blockIdx.x * kTT * DMAX + e] = zacc[e];
  double* hred = mma_sm;                                  // [8 warps][1 + DMAX]
  __syncthreads();
  gv = warp_sum(gv);
  if (lane == 0) hred[warp * (1 + DMAX)] = gv;
#pragma unroll
  for (int t = 0; t < DMAX; ++t) {
    const double v = warp_sum(gl[t]);
    if (lane == 0) hred[warp * (1 + DMAX) + 1 + t] = v;
  }
  __syncthreads();
  if (tid < 1 + DMAX) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += hred[q * (1 + DMAX) + tid];
    part_hyp[(int64_t)blockIdx.x * (1 + DMAX) + tid] = tid == 0 ? v / p.variance : v;
  }
}

// Same contract as gp_data_kernel, d <= 12: each inducing tile's Kuf block
// (128 x 128) is generated once into shared memory by all 256 threads with
// 4 independent exps in flight per thread, then the DMMA loop reads it
// there (the loader-side generation of gp_data_kernel serialises every
// exp with the MMA issue of its warp).
constexpr int kBld = kTT + 4;
template <typename T>
__global__ void __launch_bounds__(256, 1)
gp_data12_kernel(const T* __restrict__ X, const T* __restrict__ y, const double* __restrict__ Zs,
                 const double* __restrict__ G, const double* __restrict__ w, double inv_s2, int P,
                 int nt, int64_t M, int64_t N, KernParams p, double* __restrict__ part_hyp,
                 double* __restrict__ part_z) {
  constexpr int DMAX = 12;
  extern __shared__ __align__(16) double gsm[];
  double* Bf = gsm;                                       // [128][kBld] Kuf block
  double* As = Bf + kTT * kBld;                           // 2 * kGKc * kGLd staging
  double* zt = As + 2 * kGKc * kGLd;                      // [128][DMAX]
  double* zp = zt + kTT * DMAX;
  double* xb = zp + kTT * DMAX;
  double* yb = xb + kTT * DMAX;                           // [128]
  double* gp_s = yb + kTT;                                // [128]
  double* zacc = gp_s + kTT;                              // [128][DMAX]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3, g = lane >> 2, tg = lane & 3;
  const int dim = p.dim;
  for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
    const int r = e / DMAX, t = e % DMAX;
    const int64_t i = (int64_t)P * kTT + r;
    zp[e] = (t < dim && i < M) ? Zs[i * dim + t] : 0.0;
    zacc[e] = 0.0;
  }
  for (int r = tid; r < kTT; r += blockDim.x) {
    const int64_t i = (int64_t)P * kTT + r;
    gp_s[r] = i < M ? w[i] * inv_s2 : 0.0;
  }
  double gv = 0.0, gl[DMAX];
#pragma unroll
  for (int t = 0; t < DMAX; ++t) gl[t] = 0.0;
  const int64_t nblk = (N + kTT - 1) / kTT;
  const int cpt = tid & 127, kh = tid >> 7;               // generation: point, row parity
  const int rr = tid >> 1, rk = (tid & 1) * 8;            // A loader ("row" pattern, ta)
  for (int64_t nb = blockIdx.x; nb < nblk; nb += gridDim.x) {
    __syncthreads();
    for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
      const int r = e / DMAX, t = e % DMAX;
      const int64_t n = nb * kTT + r;
      xb[e] = (t < dim && n < N) ? (double)X[n * dim + t] * p.inv_ls[t] : 0.0;
    }
    for (int r = tid; r < kTT; r += blockDim.x) {
      const int64_t n = nb * kTT + r;
      yb[r] = n < N ? (double)y[n] : 0.0;
    }
    __syncthreads();
    double xr[DMAX];
#pragma unroll
    for (int t = 0; t < DMAX; ++t) xr[t] = xb[cpt * DMAX + t];
    const bool pvalid = nb * kTT + cpt < N;
    double acc[8][4][2];
    acc_zero(acc);
    for (int kt = 0; kt < nt; ++kt) {
      const int64_t ibase = (int64_t)kt * kTT;
      for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
        const int r = e / DMAX, t = e % DMAX;
        zt[e] = (t < dim && ibase + r < M) ? Zs[(ibase + r) * dim + t] : 0.0;
      }
      __syncthreads();                                    // zt ready; Bf free (prev. MMAs done)
      // generate Kuf(ibase + k, point cpt) for k = kh, kh + 2, ...: 4 in flight
      for (int k0 = kh; k0 < kTT; k0 += 8) {
        double r2[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r2[u] = 0.0;
#pragma unroll
        for (int t = 0; t < DMAX; ++t)
          if (t < dim) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double df = zt[(k0 + 2 * u) * DMAX + t] - xr[t];
              r2[u] = fma(df, df, r2[u]);
            }
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + 2 * u;
          Bf[k * kBld + cpt] = (pvalid && ibase + k < M) ? kern_from_r2(p, r2[u]) : 0.0;
        }
      }
      // acc(r, c) += sum_k G(ibase + k, r) Bf(k, c): A = G tile (transposed)
      const double* A = G + (int64_t)kt * kTE;
      double ra[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) ra[q] = A[(int64_t)rr * kTT + rk + q];
      int stage = 0;
      for (int k0 = 0; k0 < kTT; k0 += kGKc) {
        double* as = As + stage * kGKc * kGLd;
#pragma unroll
        for (int q = 0; q < 8; ++q) as[(rk + q) * kGLd + rr] = ra[q];
        __syncthreads();                                  // also: Bf generated (first pass)
        if (k0 + kGKc < kTT) {
#pragma unroll
          for (int q = 0; q < 8; ++q) ra[q] = A[(int64_t)rr * kTT + k0 + kGKc + rk + q];
        }
#pragma unroll
        for (int ks = 0; ks < kGKc / 4; ++ks) {
          double af[8], bf[4];
          const double* ak = as + (ks * 4 + tg) * kGLd + wr * 64 + g;
          const double* bk2 = Bf + (k0 + ks * 4 + tg) * kBld + wc * 32 + g;
#pragma unroll
          for (int a = 0; a < 8; ++a) af[a] = ak[a * 8];
#pragma unroll
          for (int b = 0; b < 4; ++b) bf[b] = bk2[b * 8];
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        stage ^= 1;
      }
      __syncthreads();                                    // Bf, zt consumed
    }
    // epilogue: W and the kernel-derivative contraction (as gp_data_kernel)
    double* red = Bf;                                     // [4 wc][128][DMAX]
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int r = wr * 64 + a * 8 + g;
      double gz[DMAX];
#pragma unroll
      for (int t = 0; t < DMAX; ++t) gz[t] = 0.0;
      const bool rvalid = (int64_t)P * kTT + r < M;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = wc * 32 + b * 8 + 2 * tg + e;
          if (!rvalid || nb * kTT + c >= N) continue;
          const double W = acc[a][b][e] * inv_s2 + gp_s[r] * yb[c];
          double r2 = 0.0;
#pragma unroll
          for (int t = 0; t < DMAX; ++t)
            if (t < dim) {
              const double df = zp[r * DMAX + t] - xb[c * DMAX + t];
              r2 = fma(df, df, r2);
            }
          const double k = kern_from_r2(p, r2);
          double dk;
          if (p.kernel == TB_KERNEL_RBF) {
            dk = -0.5 * k;
          } else {
            const double rq = sqrt(fmax(r2, 1e-36));
            dk = -1.5 * p.variance * exp(-1.7320508075688772 * rq);
          }
          const double wd = W * dk;
          gv = fma(W, k, gv);
#pragma unroll
          for (int t = 0; t < DMAX; ++t)
            if (t < dim) {
              const double df = zp[r * DMAX + t] - xb[c * DMAX + t];
              gl[t] = fma(wd * df * df, -2.0 * p.inv_ls[t], gl[t]);
              gz[t] = fma(wd * df, 2.0 * p.inv_ls[t], gz[t]);
            }
        }
#pragma unroll
      for (int t = 0; t < DMAX; ++t) {
        double v = gz[t];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (tg == 0) red[((int64_t)wc * kTT + r) * DMAX + t] = v;
      }
    }
    __syncthreads();
    for (int e = tid; e < kTT * DMAX; e += blockDim.x) {
      const int r = e / DMAX, t = e % DMAX;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) v += red[((int64_t)q * kTT + r) * DMAX + t];
      zacc[e] += v;
    }
  }
  __syncthreads();
  for (int e = tid; e < kTT * DMAX; e += blockDim.x)
    part_z[(int64_t)blockIdx.x * kTT * DMAX + e] = zacc[e];
  double* hred = Bf;
  __syncthreads();
  gv = warp_sum(gv);
  if (lane == 0) hred[warp * (1 + DMAX)] = gv;
#pragma unroll
  for (int t = 0; t < DMAX; ++t) {
    const double v = warp_sum(gl[t]);
    if (lane == 0) hred[warp * (1 + DMAX) + 1 + t] = v;
  }
  __syncthreads();
  if (tid < 1 + DMAX) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += hred[q * (1 + DMAX) + tid];
    part_hyp[(int64_t)blockIdx.x * (1 + DMAX) + tid] = tid == 0 ? v / p.variance : v;
  }
}
static size_t gp_data12_smem() {
  return (size_t)(kTT * kBld + 2 * kGKc * kGLd + 4 * kTT * 12 + 2 * kTT) * sizeof(double);
}

// grad_hyp[j] += sum_b part_hyp[b][j] (j < 1 + dim); grad_z[(P*128 + r)*dim + t]
// += sum_b part_z[b][r][t]  (fixed order)
__global__ void gp_data_reduce_kernel(const double* __restrict__ part_hyp,
                                      const double* __restrict__ part_z, int nb, int dmax,
                                      int dim, int P, int64_t M, double* __restrict__ grad_hyp,
                                      double* __restrict__ grad_z) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < kTT * dmax) {
    const int r = e / dmax, t = e % dmax;
    const int64_t i = (int64_t)P * kTT + r;
    if (t < dim && i < M) {
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += part_z[((int64_t)b * kTT + r) * dmax + t];
      grad_z[i * dim + t] += s;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x <= dim) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part_hyp[(int64_t)b * (1 + dmax) + threadIdx.x];
    grad_hyp[threadIdx.x] += s;
  }
}

constexpr int kGpGrid = 148;
static size_t gp_data_smem(int dmax) {
  return (size_t)(4 * kGKc * kGLd + 4 * kTT * dmax + 2 * kTT) * sizeof(double);
}

int64_t grad_tail_workspace_bytes(int64_t M, int64_t M_pad, int64_t dim) {
  const int64_t nt = M_pad / kTT, tiles = nt * (nt + 1) / 2;
  const int64_t dmax = dim <= 12 ? 12 : 16;
  return round_up(tiles * kTE * 8, 256)                 // L (packed)
         + round_up(2 * nt * kTE * 8, 256)              // diagonal inverses of L, P
         + 3 * round_up(M_pad * kTT * 8, 256)           // three column panels
         + round_up(M * dim * 8, 256)                   // scaled Z
         + round_up(4 * M_pad * 8, 256)                 // u, w, v copy, solve scratch
         + round_up((tiles + 16 + 3 * nt + 2 * 1024) * 8, 256)   // partials, scalars
         + round_up((int64_t)kGpGrid * (kTT * dmax + 1 + dmax) * 8, 256)   // data partials
         + kuf_grad_bytes(kTT, M, dim) + 1024;
}

static int gp_trsm(const double* L, const double* inv, double* Y, int nt, int i0, int trans,
                   cudaStream_t st) {
  void* args[] = {(void*)&L, (void*)&inv, (void*)&Y, (void*)&nt, (void*)&i0};
  const void* fn = trans ? (const void*)gp_trsm_kernel<1> : (const void*)gp_trsm_kernel<0>;
  TB_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(kGpGrid), dim3(256), args, kGSmem, st));
  return TB_OK;
}

int grad_tail_run(int64_t M, int64_t M_pad, const void* Z, const void* X, const void* y,
                  int64_t N, int dtype, const KernParams& kp, double jitter, double noise,
                  double* sigma, const double* v, double* out8, double* grad_hyp,
                  double* grad_z, void* workspace, cudaStream_t st) {
  const int nt = (int)(M_pad / kTT);
  const int tiles = nt * (nt + 1) / 2;
  const int dim = kp.dim;
  // data kernel: d <= 12 -> gp_data12_kernel (12-wide), else the 16-wide loader version
  const int dmax = dim <= 12 ? 12 : 16;
  char* ws = (char*)workspace;
  auto take = [&](int64_t bytes) { char* q = ws; ws += round_up(bytes, 256); return q; };
  double* L = (double*)take((int64_t)tiles * kTE * 8);
  double* invL = (double*)take(2 * (int64_t)nt * kTE * 8);
  double* invP = invL + (int64_t)nt * kTE;
  double* B0 = (double*)take(M_pad * kTT * 8);
  double* B1 = (double*)take(M_pad * kTT * 8);
  double* B2 = (double*)take(M_pad * kTT * 8);
  double* Zs = (double*)take(M * dim * 8);
  double* vec = (double*)take(4 * M_pad * 8);
  double* u = vec;
  double* w = u + M_pad;
  double* vv = w + M_pad;
  double* scratch = vv + M_pad;
  double* part = (double*)take((int64_t)(tiles + 16 + 3 * nt + 2 * 1024) * 8);
  double* scal = part + tiles;            // [0] logdet L [1] logdet P [2] |u|^2 [3..5] traces
                                          // [6] min diag(L)^2 [7] max diag(L)^2
  int* info = (int*)(scal + 8);
  double* tr_part = scal + 16;            // [nt] trace blocks of A Kuu^-1
  double* ak_part = tr_part + nt;         // [nt] blocks of tr(A^-1 Kuu)
  double* wk_part = ak_part + nt;         // [nt] blocks of w^T Kuu w
  double* kd_part = wk_part + nt;         // [1024][2] per-CTA Kuu dots
  double* ph = (double*)take((int64_t)kGpGrid * (kTT * dmax + 1 + dmax) * 8);
  double* pz = ph + (int64_t)kGpGrid * (1 + dmax);
  void* kg_ws = ws;
  const double s2 = noise;
  TB_CUDA_TRY(cudaFuncSetAttribute(tail_potrf_inv_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((size_t)kTT * kTLd * 8)));
  TB_CUDA_TRY(cudaFuncSetAttribute(tail_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kGSmem));
  for (const void* f : {(const void*)gp_trsm_kernel<0>, (const void*)gp_trsm_kernel<1>,
                        (const void*)gp_trmm_kernel<0>, (const void*)gp_trmm_kernel<1>})
    TB_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem));
  TB_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int), st));
  const unsigned zb = (unsigned)ceil_div(std::max<int64_t>(M * dim, 1), 256);
  if (dtype == TB_F32)
    scale_z_kernel<float><<<zb, 256, 0, st>>>((const float*)Z, M, kp, Zs);
  else
    scale_z_kernel<double><<<zb, 256, 0, st>>>((const double*)Z, M, kp, Zs);
  TB_LAUNCH_CHECK("scale_z");
  cudaStream_t side = nullptr;
  cudaEvent_t e_col = nullptr, e_diag = nullptr;
  int lo_p = 0, hi_p = 0;
  TB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
  TB_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi_p));
  TB_CUDA_TRY(cudaEventCreateWithFlags(&e_col, cudaEventDisableTiming));
  TB_CUDA_TRY(cudaEventCreateWithFlags(&e_diag, cudaEventDisableTiming));
  struct Cleanup {
    cudaStream_t s;
    cudaEvent_t a, b;
    ~Cleanup() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaStreamDestroy(s);
    }
  } cleanup{side, e_col, e_diag};
  // L = chol(Kuu), P = chol(Kuu + Sigma / s2) in place over Sigma
  tail_kuu_kernel<<<tiles, 256, 0, st>>>(Zs, M, kp, jitter, 0.0, L);
  TB_LAUNCH_CHECK("tail_kuu");
  int rc = tail_cholesky(L, invL, nt, info, st, side, e_col, e_diag);
  if (rc) return rc;
  tail_kuu_kernel<<<tiles, 256, 0, st>>>(Zs, M, kp, jitter, 1.0 / s2, sigma);
  TB_LAUNCH_CHECK("tail_kuu_add");
  if ((rc = tail_cholesky(sigma, invP, nt, info, st, side, e_col, e_diag))) return rc;
  double* Pf = sigma;
  tail_reduce_kernel<<<tiles, 256, 0, st>>>(L, 0, part);
  sum_kernel<<<1, 32, 0, st>>>(part, tiles, scal + 0);
  tail_diag_range_kernel<<<1, kTT, 0, st>>>(L, nt, M, scal + 6);   // cond(Kuu) lower bound
  tail_reduce_kernel<<<tiles, 256, 0, st>>>(Pf, 0, part);
  sum_kernel<<<1, 32, 0, st>>>(part, tiles, scal + 1);
  TB_LAUNCH_CHECK("grad_logdet");
  // u = P^-1 v, |u|^2, w = P^-T u / s2
  scale_copy_kernel<<<(unsigned)ceil_div(M_pad, 256), 256, 0, st>>>(v, M, M_pad, 1.0, vv);
  if ((rc = tail_solve(Pf, invP, nt, vv, scratch, u, 0, st))) return rc;
  dot_kernel<<<1, 256, 0, st>>>(u, M_pad, scal + 2);
  if ((rc = tail_solve(Pf, invP, nt, u, scratch, w, 1, st))) return rc;
  scale_copy_kernel<<<(unsigned)ceil_div(M_pad, 256), 256, 0, st>>>(w, M, M_pad, 1.0 / s2, w);
  TB_LAUNCH_CHECK("grad_vec");
  TB_CUDA_TRY(cudaFuncSetAttribute((const void*)gp_data12_kernel<float>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gp_data12_smem()));
  TB_CUDA_TRY(cudaFuncSetAttribute((const void*)gp_data12_kernel<double>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gp_data12_smem()));
  TB_CUDA_TRY(cudaFuncSetAttribute((const void*)gp_data_kernel<float, 16>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gp_data_smem(16)));
  TB_CUDA_TRY(cudaFuncSetAttribute((const void*)gp_data_kernel<double, 16>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gp_data_smem(16)));
  const int64_t pn = M_pad * kTT;
  const unsigned eb = (unsigned)std::min<int64_t>(ceil_div(pn, 256), 4096);
  const int kd_blocks = 256;
  for (int P = 0; P < nt; ++P) {
    // B0 = Kuu^-1[:, P]
    gp_identity_kernel<<<eb, 256, 0, st>>>(B0, P, pn);
    if ((rc = gp_trsm(L, invL, B0, nt, P, 0, st))) return rc;
    if ((rc = gp_trsm(L, invL, B0, nt, 0, 1, st))) return rc;
    // B2 = A Kuu^-1[:, P] = P (P^T B0)  (its block P gives tr(Kuu^-1 A)),
    // then B2 = Kuu^-1 A Kuu^-1[:, P]
    gp_trmm_kernel<1><<<nt, 256, kGSmem, st>>>(Pf, B0, B1, nt);
    gp_trmm_kernel<0><<<nt, 256, kGSmem, st>>>(Pf, B1, B2, nt);
    TB_LAUNCH_CHECK("grad_trmm");
    gp_diag_trace_kernel<<<1, 32, 0, st>>>(B2, P, M, tr_part);
    if ((rc = gp_trsm(L, invL, B2, nt, 0, 0, st))) return rc;
    if ((rc = gp_trsm(L, invL, B2, nt, 0, 1, st))) return rc;
    // B1 = A^-1[:, P]
    gp_identity_kernel<<<eb, 256, 0, st>>>(B1, P, pn);
    if ((rc = gp_trsm(Pf, invP, B1, nt, P, 0, st))) return rc;
    if ((rc = gp_trsm(Pf, invP, B1, nt, 0, 1, st))) return rc;
    // tr(A^-1 Kuu) and w^T Kuu w, block P (Kuu generated on the fly)
    gp_kuu_dot_kernel<<<kd_blocks, 256, 0, st>>>(Zs, B1, w, P, M, kp, jitter, kd_part);
    gp_pair_sum_kernel<<<1, 32, 0, st>>>(kd_part, kd_blocks, P, ak_part, wk_part);
    TB_LAUNCH_CHECK("grad_kuu_dot");
    // B0 = G2 s2, B2 = H2
    gp_combine_kernel<<<eb, 256, 0, st>>>(B0, B1, B2, w, P, M, M_pad);
    TB_LAUNCH_CHECK("grad_combine");
    // Kuu side: sum_{i, c in P} H2(i, c) dk(z_i, z_c) (tb_sgpr_kuf_grad, K recomputed)
    const int nc = (int)std::min<int64_t>(kTT, M - (int64_t)P * kTT);
    if (nc > 0) {
      gp_to_rowmajor_kernel<<<eb, 256, 0, st>>>(B2, M, nc, B1);
      TB_LAUNCH_CHECK("grad_rowmajor");
      const char* zp = (const char*)Z + (int64_t)P * kTT * dim * (dtype == TB_F32 ? 4 : 8);
      if ((rc = launch_kuf_grad(zp, Z, B1, nullptr, nc, M, dtype, kp, grad_hyp + 1 + dim,
                                grad_z + M * dim, kg_ws, st)))
        return rc;
    }
    // data side: all N points against G2[:, P]
    if (dtype == TB_F32) {
      if (dmax == 12)
        gp_data12_kernel<float><<<kGpGrid, 256, gp_data12_smem(), st>>>(
            (const float*)X, (const float*)y, Zs, B0, w, 1.0 / s2, P, nt, M, N, kp, ph, pz);
      else
        gp_data_kernel<float, 16><<<kGpGrid, 256, gp_data_smem(16), st>>>(
            (const float*)X, (const float*)y, Zs, B0, w, 1.0 / s2, P, nt, M, N, kp, ph, pz);
    } else {
      if (dmax == 12)
        gp_data12_kernel<double><<<kGpGrid, 256, gp_data12_smem(), st>>>(
            (const double*)X, (const double*)y, Zs, B0, w, 1.0 / s2, P, nt, M, N, kp, ph, pz);
      else
        gp_data_kernel<double, 16><<<kGpGrid, 256, gp_data_smem(16), st>>>(
            (const double*)X, (const double*)y, Zs, B0, w, 1.0 / s2, P, nt, M, N, kp, ph, pz);
    }
    TB_LAUNCH_CHECK("grad_data");
    gp_data_reduce_kernel<<<(unsigned)ceil_div(kTT * dmax, 256), 256, 0, st>>>(
        ph, pz, kGpGrid, dmax, dim, P, M, grad_hyp, grad_z);
    TB_LAUNCH_CHECK("grad_data_reduce");
  }
  // scalars: [0] sum log diag L, [1] sum log diag P, [2] |u|^2, [3] tr(Kuu^-1 A),
  // [4] tr(A^-1 Kuu), [5] w^T Kuu w  (valid entries only)
  sum_kernel<<<1, 32, 0, st>>>(tr_part, nt, scal + 3);
  sum_kernel<<<1, 32, 0, st>>>(ak_part, nt, scal + 4);
  sum_kernel<<<1, 32, 0, st>>>(wk_part, nt, scal + 5);
  TB_LAUNCH_CHECK("grad_scalars");
  TB_CUDA_TRY(cudaMemcpyAsync(out8, scal, 8 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int h_info = 0;
  TB_CUDA_TRY(cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  TB_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_info)
    return fail(TB_ERR_ARG, "sgpr grad tail: Cholesky failed at row " + std::to_string(h_info - 1) +
                                " (matrix not positive definite)");
  return TB_OK;
}

}  // namespace tb
