// mma_probe4.cu — the gram kernel's phase-A issue sequence (precomputed
// descriptors, 3 ring stages per k-block, ring of NS stages) without TMA or
// barriers: is ~64 cyc/MMA reachable when operands change every k-block?
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

template <int NS, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t kTile = 128 * 64, kB = N * 64, kStage = kTile + kB;
  for (int i = threadIdx.x; i < NS * kStage / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x7f7f7f7fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_u8_s32(128, N);
    const uint64_t d0 = desc_k_sw64(smem_u32(smem));
    const uint32_t acc0 = tmem, acc1 = tmem + N, acc2 = tmem + 2 * N, acc3 = tmem + 3 * N;
    int s = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint64_t a[3];
      for (int p = 2; p >= 0; --p) { a[p] = d0 + (uint64_t)s * (kStage >> 4); if (++s == NS) s = 0; }
      const uint64_t a2 = a[2], a1 = a[1], a0 = a[0];
      const uint64_t b2 = a2 + (kTile >> 4), b1 = a1 + (kTile >> 4), b0 = a0 + (kTile >> 4);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int o = 2 * ks;
        mma_i8(acc0, a2 + o, b2 + o, idesc, 1);
        if (N <= 128) {
          mma_i8(acc1, a2 + o, b1 + o, idesc, 1);
          mma_i8(acc1, a1 + o, b2 + o, idesc, 1);
          mma_i8(acc2, a2 + o, b0 + o, idesc, 1);
          mma_i8(acc2, a1 + o, b1 + o, idesc, 1);
          mma_i8(acc2, a0 + o, b2 + o, idesc, 1);
          mma_i8(acc3, a1 + o, b0 + o, idesc, 1);
          mma_i8(acc3, a0 + o, b1 + o, idesc, 1);
        } else {
          mma_i8(acc1, a2 + o, b1 + o, idesc, 1);
          mma_i8(acc1, a1 + o, b2 + o, idesc, 1);
          mma_i8(acc0, a2 + o, b0 + o, idesc, 1);
          mma_i8(acc0, a1 + o, b1 + o, idesc, 1);
          mma_i8(acc0, a0 + o, b2 + o, idesc, 1);
          mma_i8(acc1, a1 + o, b0 + o, idesc, 1);
          mma_i8(acc1, a0 + o, b1 + o, idesc, 1);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { cyc[0] = (unsigned long long)(t1 - t0); cyc[1] = (unsigned long long)iters * 16; }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int NS, int N>
void run(unsigned long long* d, int sms) {
  constexpr int smem = 1024 + NS * (128 * 64 + N * 64);
  cudaFuncSetAttribute(probe<NS, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) probe<NS, N><<<sms, 128, smem>>>(4000, d);
  cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double cpm = (double)h[0] / h[1];
  printf("ring %2d stages, N=%3d: %.1f cyc/MMA = %.0f%% of the %d-cycle floor (%s)\n", NS, N, cpm,
         100.0 * (N / 2) / cpm, N / 2, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<3, 128>(d, sms);
  run<6, 128>(d, sms);
  run<14, 128>(d, sms);
  run<3, 256>(d, sms);
  run<9, 256>(d, sms);
  return 0;
}
