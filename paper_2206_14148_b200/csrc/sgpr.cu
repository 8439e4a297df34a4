// sgpr.cu — SGPR sufficient statistics (Sigma = Kuf Kuf^T, v = Kuf y,
// yy = y^T y) and the kernel matrix-vector product (predictive mean,
// paper §5.1 MVM).
//
// Statistics, v1 ("exact Gram"): the training axis N
// is streamed in chunks of Nc points sized by the planner under
// memory_limit.  Per chunk:
//   kuf_gen   K[i, n] = k(Z_i, X_n) in fp64 from direct differences
//             (RBF: s2 exp(-r2/2); Matern-3/2: s2 (1+sqrt3 r) exp(-sqrt3 r)),
//             written [M_pad, Nc] (n contiguous);
//   kuf_gemv  v[i] += sum_n K[i,n] y[n]   (one warp per row, deterministic);
//   syrk      Sigma[a-tile, b-tile] += K_a K_b^T for lower tiles a >= b,
//             fp64 FMA on 128x128 register-blocked tiles (exact products of
//             the fp64 kernel values, fp64 accumulation, ascending n).
// The reference cannot split Kuf Kuf^T at all (split.py:210-214); the
// contracted-dim running add it uses for Kuf y (split.py:322-324) is what
// kuf_gemv does per chunk.  The O(M^3) tail runs in fp64 on cuSOLVER via
// torch.linalg (paper_2206_14148_b200/sgpr.py).
#include <cmath>
#include <cstring>
#include <cstdlib>

#include "sgpr_internal.h"

namespace tb {

constexpr int kSyrkTile = 128;
constexpr int kSyrkKc = 8;

// ------------------------------------------------------------- kuf_gen --
// Block: 32 inducing rows x 128 data points; Z rows (scaled) staged in smem.
template <typename T>
__global__ void __launch_bounds__(256)
kuf_gen_kernel(const T* __restrict__ X, const T* __restrict__ Z, int64_t n0, int64_t nc,
               int64_t N, int64_t M, int64_t M_pad, KernParams p, double* __restrict__ K) {
  __shared__ double zs[32][kMaxDim + 1];
  const int i0 = blockIdx.y * 32;
  const int64_t c0 = (int64_t)blockIdx.x * 128;
  for (int e = threadIdx.x; e < 32 * p.dim; e += blockDim.x) {
    const int r = e / p.dim, t = e % p.dim;
    zs[r][t] = (i0 + r < M) ? (double)Z[(int64_t)(i0 + r) * p.dim + t] * p.inv_ls[t] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 127, ty = threadIdx.x >> 7;   // 2 row groups of 16
  const int64_t c = c0 + tx;
  const bool valid = c < nc && n0 + c < N;
  double xs[kMaxDim];
#pragma unroll
  for (int t = 0; t < kMaxDim; ++t)
    if (t < p.dim) xs[t] = valid ? (double)X[(n0 + c) * p.dim + t] * p.inv_ls[t] : 0.0;
  for (int r = ty; r < 32; r += 2) {
    const int i = i0 + r;
    if (i >= M_pad || c >= nc) continue;
    double r2 = 0.0;
#pragma unroll
    for (int t = 0; t < kMaxDim; ++t)
      if (t < p.dim) {
        const double df = zs[r][t] - xs[t];
        r2 = fma(df, df, r2);
      }
    K[(int64_t)i * nc + c] = (valid && i < M) ? kern_from_r2(p, r2) : 0.0;
  }
}

// v[i] += sum_n K[i, n] y[n]  (one warp per inducing row)
template <typename T>
__global__ void kuf_gemv_kernel(const double* __restrict__ K, const T* __restrict__ y,
                                int64_t n0, int64_t nc, int64_t N, int64_t M,
                                double* __restrict__ v) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= M) return;
  double acc = 0.0;
  for (int64_t c = lane; c < nc && n0 + c < N; c += 32) acc = fma(K[i * nc + c], (double)y[n0 + c], acc);
  acc = warp_sum(acc);
  if (lane == 0) v[i] += acc;
}

// yy += sum y^2 over the chunk (single block, fixed order -> deterministic)
template <typename T>
__global__ void sumsq_kernel(const T* __restrict__ y, int64_t n0, int64_t n1,
                             double* __restrict__ out) {
  __shared__ double part[32];
  double acc = 0.0;
  for (int64_t k = n0 + threadIdx.x; k < n1; k += blockDim.x) {
    const double v = (double)y[k];
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out += v;
  }
}

static int launch_sumsq(const void* y, int dtype, int64_t n0, int64_t n1, double* yy,
                        cudaStream_t st) {
  if (dtype == TB_F32)
    sumsq_kernel<float><<<1, 1024, 0, st>>>((const float*)y, n0, n1, yy);
  else
    sumsq_kernel<double><<<1, 1024, 0, st>>>((const double*)y, n0, n1, yy);
  TB_LAUNCH_CHECK("sumsq");
  return TB_OK;
}

// ---------------------------------------------------------------- syrk --
// Sigma[a, b] += sum_n K[a, n] K[b, n] on lower tile pairs (ta >= tb).
// 256 threads, 8x8 fp64 micro-tile per thread over a 128x128 tile.
__global__ void __launch_bounds__(256)
syrk_f64_kernel(const double* __restrict__ K, int64_t nc, int64_t M, int ntiles,
                double* __restrict__ Sigma) {
  __shared__ __align__(16) double As[2][kSyrkKc][kSyrkTile];
  __shared__ __align__(16) double Bs[2][kSyrkKc][kSyrkTile];
  // blockIdx.x -> (ta, tb) with ta >= tb
  int ta = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
  while ((ta + 1) * (ta + 2) / 2 <= (int)blockIdx.x) ++ta;
  while (ta * (ta + 1) / 2 > (int)blockIdx.x) --ta;
  const int tb = blockIdx.x - ta * (ta + 1) / 2;
  const int a0 = ta * kSyrkTile, b0 = tb * kSyrkTile;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  // loader: 128 rows x 8 k per operand; thread -> row tid/2, k (tid&1)*4..+3
  const int lr = tid >> 1, lk = (tid & 1) * 4;
  const double* arow = K + (int64_t)(a0 + lr) * nc;
  const double* brow = K + (int64_t)(b0 + lr) * nc;
  double ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = k0 + lk + j;
      ra[j] = k < nc ? arow[k] : 0.0;
      rb[j] = k < nc ? brow[k] : 0.0;
    }
  };
  load(0);
  int stage = 0;
  for (int64_t k0 = 0; k0 < nc; k0 += kSyrkKc) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      As[stage][lk + j][lr] = ra[j];
      Bs[stage][lk + j][lr] = rb[j];
    }
    __syncthreads();
    if (k0 + kSyrkKc < nc) load(k0 + kSyrkKc);
#pragma unroll
    for (int kk = 0; kk < kSyrkKc; ++kk) {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[stage][kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b[j] = Bs[stage][kk][tx * 4 + j];
        b[4 + j] = Bs[stage][kk][64 + tx * 4 + j];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    stage ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = a0 + ty * 8 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = b0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (c < M && c <= r) Sigma[(int64_t)r * M + c] += acc[i][j];
    }
  }
}

// Same contract on the FP64 tensor cores: DMMA mma.sync m8n8k4 (fp64
// products and accumulation, i.e. the same exact-Gram numerics).  128x128
// CTA tile, 8 warps as 2 (rows) x 4 (cols), 64x32 per warp = 8x4 m8n8 tiles;
// K staged 16 deep, double buffered, k-major with a 4-double pad.
constexpr int kDmKc = 16;
constexpr int kDmLd = kSyrkTile + 4;
constexpr size_t kDmSmem = 2 * 2 * kDmKc * kDmLd * sizeof(double);

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 1)
syrk_dmma_kernel(const double* __restrict__ K, int64_t nc, int64_t M, int ntiles,
                 double* __restrict__ Sigma) {
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                              // [2][kDmKc][kDmLd]
  double* Bs = dsm + 2 * kDmKc * kDmLd;
  int ta = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
  while ((ta + 1) * (ta + 2) / 2 <= (int)blockIdx.x) ++ta;
  while (ta * (ta + 1) / 2 > (int)blockIdx.x) --ta;
  const int tb = blockIdx.x - ta * (ta + 1) / 2;
  const int a0 = ta * kSyrkTile, b0 = tb * kSyrkTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 2, wc = warp & 3;       // 2 x 4 warps
  const int g = lane >> 2, tg = lane & 3;        // fragment coordinates
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // loader: 128 rows x 16 k per operand; thread -> row tid/2, k (tid&1)*8..+7
  const int lr = tid >> 1, lk = (tid & 1) * 8;
  const double* arow = K + (int64_t)(a0 + lr) * nc;
  const double* brow = K + (int64_t)(b0 + lr) * nc;
  double ra[8], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t k = k0 + lk + j;
      ra[j] = k < nc ? arow[k] : 0.0;
      rb[j] = k < nc ? brow[k] : 0.0;
    }
  };
  load(0);
  int stage = 0;
  for (int64_t k0 = 0; k0 < nc; k0 += kDmKc) {
    double* as = As + stage * kDmKc * kDmLd;
    double* bs = Bs + stage * kDmKc * kDmLd;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      as[(lk + j) * kDmLd + lr] = ra[j];
      bs[(lk + j) * kDmLd + lr] = rb[j];
    }
    __syncthreads();
    if (k0 + kDmKc < nc) load(k0 + kDmKc);
#pragma unroll
    for (int ks = 0; ks < kDmKc / 4; ++ks) {
      double af[8], bf[4];
      const double* ak = as + (ks * 4 + tg) * kDmLd + wr * 64 + g;
      const double* bk = bs + (ks * 4 + tg) * kDmLd + wc * 32 + g;
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = ak[i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bk[j * 8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    stage ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = a0 + wr * 64 + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = b0 + wc * 32 + j * 8 + 2 * tg + e;
        if (c < M && c <= r) Sigma[(int64_t)r * M + c] += acc[i][j][e];
      }
    }
  }
}

// copy the lower triangle to the upper one
__global__ void symmetrize_kernel(double* __restrict__ S, int64_t M) {
  const int64_t r = blockIdx.y * 32 + threadIdx.y;
  const int64_t c = blockIdx.x * 32 + threadIdx.x;
  if (r < M && c < M && c > r) S[r * M + c] = S[c * M + r];
}

// ---------------------------------------------------------- kernel MVM --
// out[i] = sum_j k(X_i, Z_j) w_j; one thread per X row, Z tiles staged in
// shared memory (scaled by 1/l), fp64 throughout.
template <typename T>
__global__ void __launch_bounds__(256)
kernel_mvm_kernel(const T* __restrict__ X, const T* __restrict__ Z,
                  const double* __restrict__ w, int64_t n, int64_t M, KernParams p,
                  double* __restrict__ out) {
  constexpr int TZ = 64;
  __shared__ double zs[TZ][kMaxDim + 1];
  __shared__ double ws[TZ];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double xs[kMaxDim];
#pragma unroll
  for (int t = 0; t < kMaxDim; ++t)
    if (t < p.dim) xs[t] = i < n ? (double)X[i * p.dim + t] * p.inv_ls[t] : 0.0;
  double acc = 0.0;
  for (int64_t z0 = 0; z0 < M; z0 += TZ) {
    __syncthreads();
    for (int e = threadIdx.x; e < TZ * p.dim; e += blockDim.x) {
      const int r = e / p.dim, t = e % p.dim;
      zs[r][t] = z0 + r < M ? (double)Z[(z0 + r) * p.dim + t] * p.inv_ls[t] : 0.0;
    }
    for (int e = threadIdx.x; e < TZ; e += blockDim.x) ws[e] = z0 + e < M ? w[z0 + e] : 0.0;
    __syncthreads();
    const int lim = (int)((M - z0) < TZ ? (M - z0) : TZ);
    for (int r = 0; r < lim; ++r) {
      double r2 = 0.0;
#pragma unroll
      for (int t = 0; t < kMaxDim; ++t)
        if (t < p.dim) {
          const double df = xs[t] - zs[r][t];
          r2 = fma(df, df, r2);
        }
      acc = fma(kern_from_r2(p, r2), ws[r], acc);
    }
  }
  if (i < n) out[i] = acc;
}

// Compile-time dimension D and kernel KERN: inputs held in registers (no
// 64-entry local array), Z tiles of 128 rows in shared memory read as
// broadcasts, R rows per thread so R independent exp chains overlap.  The
// paper's §5.1 workload is D = 1 (frontend.py:34-54); the SGPR predictive
// mean uses the data dimension (3, 11 in BASELINE configs).
template <typename T, int D, int KERN, int R>
__global__ void __launch_bounds__(256)
kernel_mvm_fixed_kernel(const T* __restrict__ X, const T* __restrict__ Z,
                        const double* __restrict__ w, int64_t n, int64_t M, KernParams p,
                        double* __restrict__ out) {
  constexpr int TZ = 128;
  __shared__ double zs[TZ * D];
  __shared__ double ws[TZ];
  // RBF: inputs pre-scaled by sqrt(1/2)/l so r2 is already -log of the
  // kernel, and the variance multiplies the finished sum (17 fp64
  // instructions per kernel evaluation instead of 19)
  const double pre = KERN == TB_KERNEL_RBF ? 0.70710678118654752440 : 1.0;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x * R + threadIdx.x;
  double xs[R][D], acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + (int64_t)r * blockDim.x;
    acc[r] = 0.0;
#pragma unroll
    for (int t = 0; t < D; ++t)
      xs[r][t] = i < n ? (double)X[i * D + t] * (p.inv_ls[t] * pre) : 0.0;
  }
  for (int64_t z0 = 0; z0 < M; z0 += TZ) {
    __syncthreads();
    for (int e = threadIdx.x; e < TZ * D; e += blockDim.x)
      zs[e] = z0 + e / D < M ? (double)Z[z0 * D + e] * (p.inv_ls[e % D] * pre) : 0.0;
    for (int e = threadIdx.x; e < TZ; e += blockDim.x) ws[e] = z0 + e < M ? w[z0 + e] : 0.0;
    __syncthreads();
    const int lim = (int)((M - z0) < TZ ? (M - z0) : TZ);
    for (int j = 0; j < lim; ++j) {
      double zj[D];
#pragma unroll
      for (int t = 0; t < D; ++t) zj[t] = zs[j * D + t];
      const double wj = ws[j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double r2 = 0.0;
#pragma unroll
        for (int t = 0; t < D; ++t) {
          const double df = xs[r][t] - zj[t];
          r2 = fma(df, df, r2);
        }
        double k;
        if (KERN == TB_KERNEL_RBF) {
          k = exp(-r2);
        } else {
          const double rr = sqrt(fmax(r2, 1e-36));
          const double s3 = 1.7320508075688772 * rr;
          k = p.variance * (1.0 + s3) * exp(-s3);
        }
        acc[r] = fma(k, wj, acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + (int64_t)r * blockDim.x;
    if (i < n) out[i] = KERN == TB_KERNEL_RBF ? p.variance * acc[r] : acc[r];
  }
}

template <typename T, int D>
static bool launch_mvm_fixed(const void* X, const void* Z, const double* w, int64_t n, int64_t M,
                             const KernParams& kp, double* out, cudaStream_t st) {
  constexpr int R = D <= 4 ? 4 : 2;
  const unsigned blocks = (unsigned)ceil_div(n, 256 * R);
  if (kp.kernel == TB_KERNEL_RBF)
    kernel_mvm_fixed_kernel<T, D, TB_KERNEL_RBF, R><<<blocks, 256, 0, st>>>(
        (const T*)X, (const T*)Z, w, n, M, kp, out);
  else
    kernel_mvm_fixed_kernel<T, D, TB_KERNEL_MATERN32, R><<<blocks, 256, 0, st>>>(
        (const T*)X, (const T*)Z, w, n, M, kp, out);
  return true;
}

template <typename T>
static bool dispatch_mvm_fixed(int dim, const void* X, const void* Z, const double* w, int64_t n,
                               int64_t M, const KernParams& kp, double* out, cudaStream_t st) {
  switch (dim) {
    case 1: return launch_mvm_fixed<T, 1>(X, Z, w, n, M, kp, out, st);
    case 2: return launch_mvm_fixed<T, 2>(X, Z, w, n, M, kp, out, st);
    case 3: return launch_mvm_fixed<T, 3>(X, Z, w, n, M, kp, out, st);
    case 4: return launch_mvm_fixed<T, 4>(X, Z, w, n, M, kp, out, st);
    case 8: return launch_mvm_fixed<T, 8>(X, Z, w, n, M, kp, out, st);
    case 11: return launch_mvm_fixed<T, 11>(X, Z, w, n, M, kp, out, st);
    case 16: return launch_mvm_fixed<T, 16>(X, Z, w, n, M, kp, out, st);
    default: return false;
  }
}

static int make_params(int32_t kernel, int64_t dim, double variance,
                       const double* lengthscales, KernParams* p) {
  if (kernel != TB_KERNEL_RBF && kernel != TB_KERNEL_MATERN32)
    return fail(TB_ERR_ARG, "kernel must be rbf or matern32");
  if (dim < 1 || dim > kMaxDim)
    return fail(TB_ERR_UNSUPPORTED, "input dimension must be in [1, 64]");
  if (!(variance > 0)) return fail(TB_ERR_ARG, "variance must be strictly positive");
  if (!lengthscales) return fail(TB_ERR_ARG, "lengthscales pointer is null");
  p->kernel = kernel;
  p->dim = (int)dim;
  p->variance = variance;
  for (int t = 0; t < kMaxDim; ++t) p->inv_ls[t] = 0.0;
  for (int64_t t = 0; t < dim; ++t) {
    if (!(lengthscales[t] > 0)) return fail(TB_ERR_ARG, "lengthscales must be strictly positive");
    p->inv_ls[t] = 1.0 / lengthscales[t];
  }
  return TB_OK;
}

static bool sm100(std::string* why) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    *why = "no CUDA device visible";
    return false;
  }
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    *why = "this library is built for sm_100a (B200)";
    return false;
  }
  return true;
}

}  // namespace tb

using namespace tb;

extern "C" {

int tb_sgpr_plan_create(int64_t N, int64_t M, int64_t dim, int32_t kernel, int32_t dtype,
                        int32_t engine, int64_t memory_limit, int64_t resident_bytes,
                        tb_sgpr_plan* plan) {
  if (!plan) return fail(TB_ERR_ARG, "plan pointer is null");
  std::memset(plan, 0, sizeof(*plan));
  if (N < 1 || M < 1 || dim < 1) return fail(TB_ERR_ARG, "N, M and dim must be at least 1");
  if (dim > kMaxDim) return fail(TB_ERR_UNSUPPORTED, "input dimension must be <= 64");
  if (kernel != TB_KERNEL_RBF && kernel != TB_KERNEL_MATERN32)
    return fail(TB_ERR_ARG, "kernel must be rbf or matern32");
  if (dtype != TB_F32 && dtype != TB_F64) return fail(TB_ERR_ARG, "dtype must be f32 or f64");
  if (engine < TB_SGPR_ENGINE_AUTO || engine > TB_SGPR_ENGINE_F64_SIMT)
    return fail(TB_ERR_ARG, "unknown SGPR engine");
  if (M >= (1 << 20)) return fail(TB_ERR_UNSUPPORTED, "M must be < 2^20");
  if (engine == TB_SGPR_ENGINE_AUTO) engine = TB_SGPR_ENGINE_I8;
  plan->N = N; plan->M = M; plan->dim = dim; plan->kernel = kernel; plan->dtype = dtype;
  plan->memory_limit = memory_limit; plan->resident_bytes = resident_bytes;
  plan->engine = engine;
  const bool i8 = engine == TB_SGPR_ENGINE_I8;
  // TB_I8_PAIR=1 (opt-in CTA-pair Gram) needs 256-row pair tiles
  const char* pair_env = std::getenv("TB_I8_PAIR");
  const bool pair = i8 && pair_env && pair_env[0] == '1';
  const int64_t M_pad = round_up(M, pair ? 2 * kI8Tile : kSyrkTile);
  plan->M_pad = M_pad;
  plan->sigma_layout = i8 ? TB_SIGMA_TILES : TB_SIGMA_FULL;
  plan->sigma_bytes = i8 ? i8_tiles(M_pad) * kI8Tile * kI8Tile * 8 : M * M * 8;
  plan->output_bytes = plan->sigma_bytes + M * 8 + 8;
  const int64_t limit = memory_limit > 0 ? memory_limit : INT64_MAX;
  // outputs as the caller's allocator charges them (Sigma, v, yy buffers)
  const int64_t fixed = resident_bytes + alloc_bytes(plan->sigma_bytes) + alloc_bytes(M * 8) +
                        alloc_bytes(8);
  auto budget_fail = [&](int64_t ws) {
    return fail(TB_ERR_BUDGET, "sgpr: allocating " + std::to_string(plan->output_bytes + ws) +
                                   " bytes would exceed the budget (live=" +
                                   std::to_string(resident_bytes) + ", limit=" +
                                   std::to_string(memory_limit) + ")");
  };
  if (i8) {
    // chunk buffer = 3 digit planes + v partials; two buffers let chunk c+1's
    // Kuf generation overlap chunk c's Gram.  Largest chunk (multiple of 128,
    // <= kI8MaxChunk: s32 range) that fits, double-buffered unless that
    // would more than halve the chunk.
    auto buf_bytes = [&](int64_t nc) {
      return round_up(i8_planes_bytes(M_pad, nc), 256) + round_up(i8_vpart_bytes(M_pad, nc), 256);
    };
    const int64_t cap = std::min<int64_t>(kI8MaxChunk, round_up(N, 128));
    auto largest = [&](int nbuf) -> int64_t {
      for (int64_t nc = cap; nc >= 128; nc -= 128)
        if (fixed + alloc_bytes(nbuf * buf_bytes(nc)) <= limit) return nc;
      return 0;
    };
    // the packed O(M^3) tail (tb_sgpr_tail_run) runs after the chunk buffers
    // are released: Sigma + v + packed factor + inverses + w must fit too
    const int64_t tail_ws = tail_workspace_bytes(M, M_pad, dim);
    const int64_t tail_peak = fixed + alloc_bytes(tail_ws) + alloc_bytes(M * 8) + alloc_bytes(32);
    if (tail_peak > limit)
      return fail(TB_ERR_BUDGET, "sgpr: the O(M^3) tail needs " + std::to_string(tail_peak) +
                                     " bytes on the device (limit " + std::to_string(memory_limit) +
                                     ")");
    plan->off[5] = tail_ws;
    plan->off[6] = tail_peak;
    const int64_t n1 = largest(1), n2 = N > cap ? largest(2) : 0;
    if (!n1) return budget_fail(buf_bytes(128));
    const int nbuf = (n2 && 2 * n2 >= n1) ? 2 : 1;
    const int64_t nc = nbuf == 2 ? n2 : n1;
    plan->chunk_n = nc;
    plan->off[0] = 0;
    plan->off[1] = round_up(i8_planes_bytes(M_pad, nc), 256);
    plan->off[2] = nbuf == 2 ? buf_bytes(nc) : 0;
    plan->off[3] = plan->off[2] + plan->off[1];
    plan->off[4] = nbuf;
    plan->workspace_bytes = nbuf * buf_bytes(nc);
    plan->peak_bytes = std::max(fixed + alloc_bytes(plan->workspace_bytes), tail_peak);
    return TB_OK;
  }
  // fp64 engines: one fp64 Kuf chunk [M_pad, nc]; as large as the budget
  // allows (amortises the per-chunk Sigma tile read-modify-write), <= 8192
  int64_t nc = std::min<int64_t>(8192, round_up(N, 128));
  for (;;) {
    const int64_t ws = round_up(M_pad * nc * 8, 256);
    if (fixed + alloc_bytes(ws) <= limit) {
      plan->chunk_n = nc;
      plan->workspace_bytes = ws;
      plan->peak_bytes = fixed + alloc_bytes(ws);
      return TB_OK;
    }
    if (nc <= 128) return budget_fail(ws);
    nc = std::max<int64_t>(128, round_up(nc / 2, 128));
  }
}

int tb_sgpr_stats_run(const tb_sgpr_plan* p, const void* X, const void* y, const void* Z,
                      double variance, const double* lengthscales, double* Sigma, double* v,
                      double* yy, int32_t accumulate, void* workspace,
                      int64_t workspace_bytes, void* stream) {
  if (!p) return fail(TB_ERR_ARG, "plan pointer is null");
  if (!X || !y || !Z || !Sigma || !v || !yy || !workspace)
    return fail(TB_ERR_ARG, "null buffer passed to tb_sgpr_stats_run");
  if (workspace_bytes < p->workspace_bytes)
    return fail(TB_ERR_ARG, "workspace smaller than plan->workspace_bytes");
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  KernParams kp;
  int rc = make_params(p->kernel, p->dim, variance, lengthscales, &kp);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t M = p->M, N = p->N, nc = p->chunk_n;
  const int64_t M_pad = p->M_pad;
  if (!accumulate) {
    TB_CUDA_TRY(cudaMemsetAsync(Sigma, 0, p->sigma_bytes, st));
    TB_CUDA_TRY(cudaMemsetAsync(v, 0, M * 8, st));
    TB_CUDA_TRY(cudaMemsetAsync(yy, 0, 8, st));
  }
  if (p->engine == TB_SGPR_ENGINE_I8) {
    // Two chunk buffers: chunk c+1's Kuf generation (fp64 CUDA cores, side
    // stream) runs while chunk c's Gram (INT8 tensor cores) runs on `st`.
    const int nbuf = (int)p->off[4];
    uint8_t* planes[2] = {(uint8_t*)workspace + p->off[0], (uint8_t*)workspace + p->off[2]};
    double* vpart[2] = {(double*)((uint8_t*)workspace + p->off[1]),
                        (double*)((uint8_t*)workspace + p->off[3])};
    cudaStream_t gen = st, user = st;
    cudaEvent_t ev[5] = {};   // start, gen done (buf 0/1), gram done (buf 0/1)
    if (nbuf == 2) {
      // the Grams run on a HIGH-priority internal stream: when a Gram and the
      // next chunk's generation become ready together, the block scheduler
      // places the Gram's persistent CTAs first and the generator's blocks
      // fill the room left beside them, instead of the generator flooding
      // every SM and the two phases serialising
      int lo = 0, hi = 0;
      TB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      TB_CUDA_TRY(cudaStreamCreateWithFlags(&gen, cudaStreamNonBlocking));
      TB_CUDA_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
      for (auto& e : ev) TB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TB_CUDA_TRY(cudaEventRecord(ev[0], user));
      TB_CUDA_TRY(cudaStreamWaitEvent(gen, ev[0], 0));
      TB_CUDA_TRY(cudaStreamWaitEvent(st, ev[0], 0));
    }
    int64_t c = 0;
    for (int64_t n0 = 0; n0 < N && rc == TB_OK; n0 += nc, ++c) {
      const int64_t cur = std::min(nc, N - n0);
      const int b = nbuf == 2 ? (int)(c & 1) : 0;
      if (nbuf == 2 && c >= 2) TB_CUDA_TRY(cudaStreamWaitEvent(gen, ev[3 + b], 0));
      rc = i8_gen_chunk(X, y, Z, p->dtype, n0, cur, M, M_pad, nc, kp, planes[b], vpart[b], v, gen);
      if (rc) break;
      rc = launch_sumsq(y, p->dtype, n0, n0 + cur, yy, gen);
      if (rc) break;
      if (nbuf == 2) {
        TB_CUDA_TRY(cudaEventRecord(ev[1 + b], gen));
        TB_CUDA_TRY(cudaStreamWaitEvent(st, ev[1 + b], 0));
      }
      rc = i8_gram_chunk(cur, M_pad, nc, kp.variance, planes[b], Sigma, st);
      if (nbuf == 2 && rc == TB_OK) TB_CUDA_TRY(cudaEventRecord(ev[3 + b], st));
    }
    if (nbuf == 2) {
      // v / yy (side stream) and the Grams complete before anything later on
      // the caller's stream
      cudaEventRecord(ev[0], gen);
      cudaStreamWaitEvent(user, ev[0], 0);
      cudaEventRecord(ev[1], st);
      cudaStreamWaitEvent(user, ev[1], 0);
      for (auto& e : ev) cudaEventDestroy(e);
      cudaStreamDestroy(gen);
      cudaStreamDestroy(st);
    }
    return rc;
  }
  double* K = (double*)workspace;
  const int ntiles = (int)(M_pad / kSyrkTile);
  const unsigned pairs = (unsigned)(ntiles * (ntiles + 1) / 2);
  // fp64 Gram: FP64 tensor cores (DMMA), or the CUDA-core SYRK (same
  // numerics, kept as an independent cross-check)
  const bool use_dmma = p->engine == TB_SGPR_ENGINE_F64;
  if (use_dmma)
    TB_CUDA_TRY(cudaFuncSetAttribute(syrk_dmma_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDmSmem));
  for (int64_t n0 = 0; n0 < N; n0 += nc) {
    const int64_t cur = std::min(nc, N - n0);
    dim3 g1((unsigned)ceil_div(cur, 128), (unsigned)(M_pad / 32));
    if (p->dtype == TB_F32)
      kuf_gen_kernel<float><<<g1, 256, 0, st>>>((const float*)X, (const float*)Z, n0, cur, N, M,
                                                M_pad, kp, K);
    else
      kuf_gen_kernel<double><<<g1, 256, 0, st>>>((const double*)X, (const double*)Z, n0, cur, N,
                                                 M, M_pad, kp, K);
    TB_LAUNCH_CHECK("kuf_gen");
    const unsigned gb = (unsigned)ceil_div(M, 8);
    if (p->dtype == TB_F32) {
      kuf_gemv_kernel<float><<<gb, 256, 0, st>>>(K, (const float*)y, n0, cur, N, M, v);
      sumsq_kernel<float><<<1, 1024, 0, st>>>((const float*)y, n0, n0 + cur, yy);
    } else {
      kuf_gemv_kernel<double><<<gb, 256, 0, st>>>(K, (const double*)y, n0, cur, N, M, v);
      sumsq_kernel<double><<<1, 1024, 0, st>>>((const double*)y, n0, n0 + cur, yy);
    }
    TB_LAUNCH_CHECK("kuf_gemv");
    if (use_dmma) {
      syrk_dmma_kernel<<<pairs, 256, kDmSmem, st>>>(K, cur, M, ntiles, Sigma);
      TB_LAUNCH_CHECK("syrk_dmma");
    } else {
      syrk_f64_kernel<<<pairs, 256, 0, st>>>(K, cur, M, ntiles, Sigma);
      TB_LAUNCH_CHECK("syrk_f64");
    }
  }
  dim3 gs((unsigned)ceil_div(M, 32), (unsigned)ceil_div(M, 32));
  symmetrize_kernel<<<gs, dim3(32, 32), 0, st>>>(Sigma, M);
  TB_LAUNCH_CHECK("symmetrize");
  return TB_OK;
}

int tb_sgpr_sigma_unpack(const tb_sgpr_plan* p, const double* Sigma, double* full,
                         void* stream) {
  if (!p || !Sigma || !full) return fail(TB_ERR_ARG, "null argument to tb_sgpr_sigma_unpack");
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  cudaStream_t st = (cudaStream_t)stream;
  if (p->sigma_layout == TB_SIGMA_FULL) {
    if (full != Sigma)
      TB_CUDA_TRY(cudaMemcpyAsync(full, Sigma, p->M * p->M * 8, cudaMemcpyDeviceToDevice, st));
    return TB_OK;
  }
  return i8_unpack(Sigma, p->M, p->M_pad, full, st);
}

int64_t tb_sgpr_tail_workspace(const tb_sgpr_plan* p) {
  if (!p || p->sigma_layout != TB_SIGMA_TILES) return -1;
  return tail_workspace_bytes(p->M, p->M_pad, p->dim);
}

int tb_sgpr_tail_run(const tb_sgpr_plan* p, const void* Z, double variance,
                     const double* lengthscales, double jitter, double noise_variance,
                     double* Sigma, const double* v, double* w_out, double* out4,
                     void* workspace, int64_t workspace_bytes, void* stream) {
  if (!p) return fail(TB_ERR_ARG, "plan pointer is null");
  if (p->sigma_layout != TB_SIGMA_TILES)
    return fail(TB_ERR_ARG, "tb_sgpr_tail_run needs the packed-tile Sigma (TB_SIGMA_TILES)");
  if (!Z || !Sigma || !v || !w_out || !out4 || !workspace)
    return fail(TB_ERR_ARG, "null buffer passed to tb_sgpr_tail_run");
  if (!(noise_variance > 0) || !(jitter >= 0))
    return fail(TB_ERR_ARG, "noise_variance must be > 0 and jitter >= 0");
  if (workspace_bytes < tail_workspace_bytes(p->M, p->M_pad, p->dim))
    return fail(TB_ERR_ARG, "workspace smaller than tb_sgpr_tail_workspace()");
  KernParams kp;
  int rc = make_params(p->kernel, p->dim, variance, lengthscales, &kp);
  if (rc) return rc;
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  return tail_run(p->M, p->M_pad, Z, p->dtype, kp, jitter, noise_variance, Sigma, v, w_out, out4,
                  workspace, (cudaStream_t)stream);
}

int64_t tb_sgpr_grad_workspace(const tb_sgpr_plan* p) {
  if (!p || p->sigma_layout != TB_SIGMA_TILES) return -1;
  return grad_tail_workspace_bytes(p->M, p->M_pad, p->dim);
}

int tb_sgpr_grad_run(const tb_sgpr_plan* p, const void* X, const void* y, const void* Z,
                     double variance, const double* lengthscales, double jitter,
                     double noise_variance, double* Sigma, const double* v, double* out8,
                     double* grad_hyp, double* grad_Z, void* workspace, int64_t workspace_bytes,
                     void* stream) {
  if (!p) return fail(TB_ERR_ARG, "plan pointer is null");
  if (p->sigma_layout != TB_SIGMA_TILES)
    return fail(TB_ERR_ARG, "tb_sgpr_grad_run needs the packed-tile Sigma (TB_SIGMA_TILES)");
  if (!X || !y || !Z || !Sigma || !v || !out8 || !grad_hyp || !grad_Z || !workspace)
    return fail(TB_ERR_ARG, "null buffer passed to tb_sgpr_grad_run");
  if (!(noise_variance > 0) || !(jitter >= 0))
    return fail(TB_ERR_ARG, "noise_variance must be > 0 and jitter >= 0");
  if (workspace_bytes < grad_tail_workspace_bytes(p->M, p->M_pad, p->dim))
    return fail(TB_ERR_ARG, "workspace smaller than tb_sgpr_grad_workspace()");
  if (p->dim > 16) return fail(TB_ERR_UNSUPPORTED, "tb_sgpr_grad_run supports dim <= 16");
  KernParams kp;
  int rc = make_params(p->kernel, p->dim, variance, lengthscales, &kp);
  if (rc) return rc;
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  return grad_tail_run(p->M, p->M_pad, Z, X, y, p->N, p->dtype, kp, jitter, noise_variance,
                       Sigma, v, out8, grad_hyp, grad_Z, workspace, (cudaStream_t)stream);
}

int64_t tb_sgpr_kuf_grad_workspace(int64_t nc, int64_t M, int64_t dim) {
  if (nc < 0 || M < 1 || dim < 1 || dim > kMaxDim) return -1;
  return kuf_grad_bytes(nc, M, dim);
}

int tb_sgpr_kuf_grad(const void* Xc, const void* Z, const double* W, const double* K,
                     int64_t nc, int64_t M, int64_t dim, int32_t kernel, int32_t dtype,
                     double variance, const double* lengthscales, double* grad_hyp,
                     double* grad_Z, void* workspace, int64_t workspace_bytes, void* stream) {
  if (nc < 0 || M < 1) return fail(TB_ERR_ARG, "bad kuf_grad extents");
  if (!Xc || !Z || !W || !K || !grad_hyp || !grad_Z || !workspace)
    return fail(TB_ERR_ARG, "null buffer passed to tb_sgpr_kuf_grad");
  if (dtype != TB_F32 && dtype != TB_F64) return fail(TB_ERR_ARG, "dtype must be f32 or f64");
  KernParams kp;
  int rc = make_params(kernel, dim, variance, lengthscales, &kp);
  if (rc) return rc;
  if (workspace_bytes < kuf_grad_bytes(nc, M, dim))
    return fail(TB_ERR_ARG, "workspace smaller than tb_sgpr_kuf_grad_workspace()");
  if (nc == 0) return TB_OK;
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  return launch_kuf_grad(Xc, Z, W, K, nc, M, dtype, kp, grad_hyp, grad_Z, workspace,
                         (cudaStream_t)stream);
}

int tb_kernel_matrix(const void* A, const void* B, int64_t na, int64_t nb, int64_t dim,
                     int32_t kernel, int32_t dtype, double variance,
                     const double* lengthscales, double* out, void* stream) {
  if (na < 0 || nb < 0) return fail(TB_ERR_ARG, "bad kernel_matrix extents");
  if (!A || !B || !out) return fail(TB_ERR_ARG, "null buffer passed to tb_kernel_matrix");
  if (dtype != TB_F32 && dtype != TB_F64) return fail(TB_ERR_ARG, "dtype must be f32 or f64");
  KernParams kp;
  int rc = make_params(kernel, dim, variance, lengthscales, &kp);
  if (rc) return rc;
  if (na == 0 || nb == 0) return TB_OK;
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  cudaStream_t st = (cudaStream_t)stream;
  dim3 g((unsigned)ceil_div(nb, 128), (unsigned)ceil_div(na, 32));
  // rows = A (the "inducing" role), columns = B, out[na, nb] (no padding rows)
  if (dtype == TB_F32)
    kuf_gen_kernel<float><<<g, 256, 0, st>>>((const float*)B, (const float*)A, 0, nb, nb, na,
                                             na, kp, out);
  else
    kuf_gen_kernel<double><<<g, 256, 0, st>>>((const double*)B, (const double*)A, 0, nb, nb,
                                              na, na, kp, out);
  TB_LAUNCH_CHECK("kernel_matrix");
  return TB_OK;
}

int tb_kernel_mvm(const void* X, const void* Z, const double* w, int64_t n, int64_t M,
                  int64_t dim, int32_t kernel, int32_t dtype, double variance,
                  const double* lengthscales, double* out, void* stream) {
  if (n < 0 || M < 1) return fail(TB_ERR_ARG, "bad kernel_mvm extents");
  if (!X || !Z || !w || !out) return fail(TB_ERR_ARG, "null buffer passed to tb_kernel_mvm");
  if (dtype != TB_F32 && dtype != TB_F64) return fail(TB_ERR_ARG, "dtype must be f32 or f64");
  KernParams kp;
  int rc = make_params(kernel, dim, variance, lengthscales, &kp);
  if (rc) return rc;
  if (n == 0) return TB_OK;
  std::string why;
  if (!sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  cudaStream_t st = (cudaStream_t)stream;
  const bool fixed = dtype == TB_F32 ? dispatch_mvm_fixed<float>(kp.dim, X, Z, w, n, M, kp, out, st)
                                     : dispatch_mvm_fixed<double>(kp.dim, X, Z, w, n, M, kp, out, st);
  if (!fixed) {                       // other dimensions: runtime-dim kernel
    const unsigned blocks = (unsigned)ceil_div(n, 256);
    if (dtype == TB_F32)
      kernel_mvm_kernel<float><<<blocks, 256, 0, st>>>((const float*)X, (const float*)Z, w, n, M,
                                                       kp, out);
    else
      kernel_mvm_kernel<double><<<blocks, 256, 0, st>>>((const double*)X, (const double*)Z, w, n,
                                                        M, kp, out);
  }
  TB_LAUNCH_CHECK("kernel_mvm");
  return TB_OK;
}

}  // extern "C"
