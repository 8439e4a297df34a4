// mma_probe5.cu — tcgen05.mma.cta_group::2 kind::i8 throughput (CTA pairs),
// smem-resident operands, the gram phase-A issue pattern; M256 with N=128
// (4 accumulators) and N=256 (2 accumulators).
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t kA = 128 * 64, kB = (N / 2) * 64, kStage = 3 * (kA + kB);
  constexpr int NS = 4;
  for (int i = threadIdx.x; i < NS * kStage / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x7f7f7f7fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc_2sm(&slot, 512);
  tc_fence_before(); __syncthreads(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = idesc_u8_s32(256, N);
    const uint64_t d0 = desc_k_sw64(smem_u32(smem));
    const uint32_t acc0 = tmem, acc1 = tmem + N, acc2 = tmem + (N == 128 ? 256 : 0),
                   acc3 = tmem + (N == 128 ? 384 : N);
    int s = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint64_t a2 = d0 + (uint64_t)s * (kStage >> 4), b2 = a2 + (kA >> 4);
      const uint64_t a1 = a2 + ((kA + kB) >> 4), b1 = a1 + (kA >> 4);
      const uint64_t a0 = a1 + ((kA + kB) >> 4), b0 = a0 + (kA >> 4);
      if (++s == NS) s = 0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int o = 2 * ks;
        mma_i8_2sm(acc0, a2 + o, b2 + o, idesc, 1);
        mma_i8_2sm(acc1, a2 + o, b1 + o, idesc, 1);
        mma_i8_2sm(acc1, a1 + o, b2 + o, idesc, 1);
        mma_i8_2sm(acc2, a2 + o, b0 + o, idesc, 1);
        mma_i8_2sm(acc2, a1 + o, b1 + o, idesc, 1);
        mma_i8_2sm(acc2, a0 + o, b2 + o, idesc, 1);
        mma_i8_2sm(acc3, a1 + o, b0 + o, idesc, 1);
        mma_i8_2sm(acc3, a0 + o, b1 + o, idesc, 1);
      }
    }
    mma_commit_2sm(&bar, 1);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { cyc[0] = (unsigned long long)(t1 - t0); cyc[1] = (unsigned long long)iters * 16; }
  }
  tc_fence_before(); __syncthreads(); cluster_sync(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc_2sm(tmem, 512);
}

template <int N>
void run(unsigned long long* d, int sms) {
  constexpr int smem = 1024 + 4 * 3 * (128 * 64 + (N / 2) * 64);
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) probe<N><<<sms, 128, smem>>>(4000, d);
  cudaDeviceSynchronize();
  unsigned long long h[2] = {0, 1};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double cpm = (double)h[0] / h[1];
  printf("cta_group::2 M256 N%d K32 i8: %.1f cyc/MMA, per-SM %.0f MAC/clk (%s)\n", N, cpm,
         128.0 * N * 32 / cpm, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128>(d, sms);
  run<256>(d, sms);
  return 0;
}
