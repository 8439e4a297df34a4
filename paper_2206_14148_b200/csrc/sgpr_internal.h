// sgpr_internal.h — pieces shared by the SGPR statistics engines
// (sgpr.cu: fp64 Gram engines + kernel MVM; sgpr_i8.cu: exact fixed-point
// Gram on the INT8 tensor cores).
#pragma once
#include "tb_common.cuh"

namespace tb {

constexpr int kMaxDim = 64;

struct KernParams {
  int kernel;   // TB_KERNEL_RBF / TB_KERNEL_MATERN32
  int dim;
  double variance;
  double inv_ls[kMaxDim];
};

// k(r^2) with r^2 = ||(x - z) / l||^2 (GPflow 2.3.1 SquaredExponential /
// Matern32; the SE op order of the reference's build_kernel_mvm,
// frontend.py:49-53, is variance * exp(-0.5 r^2)).
__device__ __forceinline__ double kern_from_r2(const KernParams& p, double r2) {
  if (p.kernel == TB_KERNEL_RBF) return p.variance * exp(-0.5 * r2);
  const double r = sqrt(fmax(r2, 1e-36));
  const double s3 = 1.7320508075688772 * r;
  return p.variance * (1.0 + s3) * exp(-s3);
}

// ---- exact fixed-point Gram engine (sgpr_i8.cu) -------------------------
constexpr int kI8Tile = 128;        // Sigma tile (rows = cols)
constexpr int kI8KB = 64;           // training points per k-block (64-B rows)
constexpr int kI8FracBits = 24;     // Kuf / variance quantised to 2^-24
// int32 accumulators: the widest level (3 products of u8 x u8) must not
// overflow over one chunk: 3 * 255^2 * chunk < 2^31.
constexpr int64_t kI8MaxChunk = 10880;

inline int64_t i8_tiles(int64_t M_pad) {
  const int64_t nt = M_pad / kI8Tile;
  return nt * (nt + 1) / 2;
}
// workspace layout of one chunk: 3 digit planes [3][M_pad][chunk] u8, then
// per-128-point-segment partial v sums [chunk/128][M_pad] fp64
inline int64_t i8_planes_bytes(int64_t M_pad, int64_t nc) { return 3 * M_pad * nc; }
inline int64_t i8_vpart_bytes(int64_t M_pad, int64_t nc) { return (nc / 128) * M_pad * 8; }

// Kuf chunk -> digit planes + v partials (+ v update), on `st`
int i8_gen_chunk(const void* X, const void* y, const void* Z, int dtype, int64_t n0,
                 int64_t cur, int64_t M, int64_t M_pad, int64_t nc, const KernParams& kp,
                 uint8_t* planes, double* vpart, double* v, cudaStream_t st);
// Sigma tiles += Gram of the chunk's planes, on `st`
int i8_gram_chunk(int64_t cur, int64_t M_pad, int64_t nc, double variance, const uint8_t* planes,
                  double* Sigma_tiles, cudaStream_t st);
// packed-tile O(M^3) tail (sgpr_tail.cu)
int64_t tail_workspace_bytes(int64_t M, int64_t M_pad, int64_t dim);
int tail_run(int64_t M, int64_t M_pad, const void* Z, int dtype, const KernParams& kp,
             double jitter, double noise, double* sigma, const double* v, double* w_out,
             double* out4, void* workspace, cudaStream_t st);
// in-budget ELBO gradient on the packed factors (sgpr_tail.cu)
int64_t grad_tail_workspace_bytes(int64_t M, int64_t M_pad, int64_t dim);
int grad_tail_run(int64_t M, int64_t M_pad, const void* Z, const void* X, const void* y,
                  int64_t N, int dtype, const KernParams& kp, double jitter, double noise,
                  double* sigma, const double* v, double* out8, double* grad_hyp,
                  double* grad_z, void* workspace, cudaStream_t st);
// ELBO gradient, N-streaming half (sgpr_grad.cu)
int64_t kuf_grad_bytes(int64_t nc, int64_t M, int64_t dim);
int launch_kuf_grad(const void* Xc, const void* Z, const double* W, const double* K,
                    int64_t nc, int64_t M, int dtype, const KernParams& kp, double* grad_hyp,
                    double* grad_z, void* workspace, cudaStream_t st);
int i8_unpack(const double* tiles, int64_t M, int64_t M_pad, double* full, cudaStream_t st);

}  // namespace tb
