// sgpr_grad.cu — the N-streaming half of the SGPR ELBO gradient (GPflow
// 2.3.1 SGPR training loss, paper §5.3 Table 2 workload).
//
// The ELBO depends on the training data only through Sigma = Kuf Kuf^T,
// v = Kuf y (and y^T y), so with G = dELBO/dSigma (symmetric) and
// g = dELBO/dv from the O(M^3) tail (torch autograd on cuSOLVER/cuBLAS):
//     dELBO|_Kuf = sum_{i,n} W_in dK_in,   W = 2 G Kuf + g y^T.
// Per streamed chunk the host forms W with one fp64 GEMM (cuBLAS) and this
// kernel reduces it against the kernel derivatives, with r^2 = |(x-z)/l|^2
// recomputed from the inputs (same formula as the statistics):
//     dk/d(r^2): RBF -k/2;  Matern-3/2 -(3/2) s2 exp(-sqrt3 r)
//     d/d variance   += W k / s2
//     d/d l_t        += W k' (-2 (x_t - z_t)^2 / l_t^3)
//     d/d z_it       += W k' ( 2 (z_t - x_t)   / l_t^2)
// Reductions are fixed-order (per-block partials, then ordered sums), so the
// gradient is deterministic.
#include "sgpr_internal.h"

namespace tb {

constexpr int kGradRows = 32, kGradCols = 128;

__device__ __forceinline__ double dk_dr2(const KernParams& p, double r2, double k) {
  if (p.kernel == TB_KERNEL_RBF) return -0.5 * k;
  const double r = sqrt(fmax(r2, 1e-36));
  return -1.5 * p.variance * exp(-1.7320508075688772 * r);
}

// Block: 32 inducing rows x 128 points; thread = one point, all 32 rows.
template <typename T, int DMAX>
__global__ void __launch_bounds__(kGradCols)
sgpr_kuf_grad_kernel(const T* __restrict__ Xc, const T* __restrict__ Z,
                     const double* __restrict__ W, const double* __restrict__ K, int64_t nc,
                     int64_t M, KernParams p, double* __restrict__ part_hyp,
                     double* __restrict__ part_z) {
  __shared__ double zs[kGradRows][DMAX + 1];
  __shared__ double red[kGradCols / 32][DMAX + 1];
  const int i0 = blockIdx.y * kGradRows;
  const int64_t c = (int64_t)blockIdx.x * kGradCols + threadIdx.x;
  const bool valid = c < nc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kGradRows * p.dim; e += blockDim.x) {
    const int r = e / p.dim, t = e % p.dim;
    zs[r][t] = (i0 + r < M) ? (double)Z[(int64_t)(i0 + r) * p.dim + t] * p.inv_ls[t] : 0.0;
  }
  __syncthreads();
  double xs[DMAX];
#pragma unroll
  for (int t = 0; t < DMAX; ++t)
    if (t < p.dim) xs[t] = valid ? (double)Xc[c * p.dim + t] * p.inv_ls[t] : 0.0;
  double gv = 0.0, gl[DMAX];
#pragma unroll
  for (int t = 0; t < DMAX; ++t) gl[t] = 0.0;
  for (int r = 0; r < kGradRows; ++r) {
    const int64_t i = i0 + r;
    double gz[DMAX];
    const bool on = valid && i < M;
    const double w = on ? W[i * nc + c] : 0.0;
    double r2 = 0.0;
#pragma unroll
    for (int t = 0; t < DMAX; ++t)
      if (t < p.dim) {
        const double df = zs[r][t] - xs[t];
        r2 = fma(df, df, r2);
      }
    // K == nullptr: the kernel value is recomputed from r^2 (no M x nc panel)
    const double k = !on ? 0.0 : (K ? K[i * nc + c] : kern_from_r2(p, r2));
    const double wd = on ? w * dk_dr2(p, r2, k) : 0.0;
    gv = fma(w, k, gv);
#pragma unroll
    for (int t = 0; t < DMAX; ++t)
      if (t < p.dim) {
        const double df = zs[r][t] - xs[t];                     // (z - x) / l
        gl[t] = fma(wd * df * df, -2.0 * p.inv_ls[t], gl[t]);  // -2 (x-z)^2 / l^3
        gz[t] = wd * df * (2.0 * p.inv_ls[t]);                 //  2 (z-x) / l^2
      }
    // d/dz_i: sum over this block's 128 points (warp sums, then the warps)
#pragma unroll
    for (int t = 0; t < DMAX; ++t) {
      if (t >= p.dim) break;
      const double s = warp_sum(gz[t]);
      if (lane == 0) red[warp][t] = s;
    }
    __syncthreads();
    if (threadIdx.x < p.dim) {
      double s = 0.0;
      for (int w2 = 0; w2 < kGradCols / 32; ++w2) s += red[w2][threadIdx.x];
      if (i < M) part_z[((int64_t)blockIdx.x * M + i) * p.dim + threadIdx.x] = s;
    }
    __syncthreads();
  }
  // hyperparameters: this block's partial (variance, lengthscales)
  gv = warp_sum(gv);
  if (lane == 0) red[warp][0] = gv;
  __syncthreads();
  const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w2 = 0; w2 < kGradCols / 32; ++w2) s += red[w2][0];
    part_hyp[blk * (1 + p.dim)] = s / p.variance;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < DMAX; ++t) {
    if (t >= p.dim) break;
    const double s = warp_sum(gl[t]);
    if (lane == 0) red[warp][t] = s;
  }
  __syncthreads();
  if (threadIdx.x < p.dim) {
    double s = 0.0;
    for (int w2 = 0; w2 < kGradCols / 32; ++w2) s += red[w2][threadIdx.x];
    part_hyp[blk * (1 + p.dim) + 1 + threadIdx.x] = s;
  }
}

// grad_hyp[j] += sum_b part_hyp[b][j]; grad_z[i][t] += sum_bx part_z[bx][i][t]
__global__ void grad_reduce_kernel(const double* __restrict__ part_hyp, int64_t nblk,
                                   const double* __restrict__ part_z, int nbx, int64_t Md,
                                   int nh, double* __restrict__ grad_hyp,
                                   double* __restrict__ grad_z) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < Md) {
    double s = 0.0;
    for (int b = 0; b < nbx; ++b) s += part_z[(int64_t)b * Md + e];
    grad_z[e] += s;
  }
  if (blockIdx.x == 0 && threadIdx.x < nh) {
    double s = 0.0;
    for (int64_t b = 0; b < nblk; ++b) s += part_hyp[b * nh + threadIdx.x];
    grad_hyp[threadIdx.x] += s;
  }
}

int64_t kuf_grad_bytes(int64_t nc, int64_t M, int64_t dim) {
  const int64_t nbx = ceil_div(std::max<int64_t>(nc, 1), kGradCols);
  const int64_t nby = ceil_div(M, kGradRows);
  return round_up(nbx * nby * (1 + dim) * 8, 256) + round_up(nbx * M * dim * 8, 256);
}

int launch_kuf_grad(const void* Xc, const void* Z, const double* W, const double* K,
                    int64_t nc, int64_t M, int dtype, const KernParams& kp, double* grad_hyp,
                    double* grad_z, void* workspace, cudaStream_t st) {
  if (nc <= 0) return TB_OK;
  const int64_t nbx = ceil_div(nc, kGradCols), nby = ceil_div(M, kGradRows);
  double* part_hyp = (double*)workspace;
  double* part_z = (double*)((char*)workspace + round_up(nbx * nby * (1 + kp.dim) * 8, 256));
  dim3 g((unsigned)nbx, (unsigned)nby);
#define TB_KG(T, D)                                                                       \
  sgpr_kuf_grad_kernel<T, D><<<g, kGradCols, 0, st>>>((const T*)Xc, (const T*)Z, W, K, nc, M, \
                                                      kp, part_hyp, part_z)
#define TB_KG_DIM(T)                   \
  if (kp.dim <= 4) TB_KG(T, 4);        \
  else if (kp.dim <= 16) TB_KG(T, 16); \
  else TB_KG(T, 64)
  if (dtype == TB_F32) {
    TB_KG_DIM(float);
  } else {
    TB_KG_DIM(double);
  }
#undef TB_KG_DIM
#undef TB_KG
  TB_LAUNCH_CHECK("sgpr_kuf_grad");
  const int64_t Md = M * kp.dim;
  grad_reduce_kernel<<<(unsigned)ceil_div(std::max<int64_t>(Md, 1), 256), 256, 0, st>>>(
      part_hyp, nbx * nby, part_z, (int)nbx, Md, 1 + kp.dim, grad_hyp, grad_z);
  TB_LAUNCH_CHECK("sgpr_grad_reduce");
  return TB_OK;
}

}  // namespace tb
