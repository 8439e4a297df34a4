// mma_issue_probe.cu — cost of the barrier/fence operations the tc1 MMA issuer
// interleaves with its tcgen05.mma (kind::f16 M128.N256.K16, 128-cycle
// floor): after every GROUP MMAs the thread runs variant V:
//   0 nothing, 1 tcgen05.commit, 2 mbarrier wait on a completed phase,
//   3 tcgen05.fence::after_thread_sync, 4 = 2 + 3, 5 = 1 + 2 + 3.
// If the tensor pipe only queues ~1 MMA, every such operation is exposed.
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

template <int V, int GROUP>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, done, dummy;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x3bff3bffu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    mbar_init(&dummy, 1);
    fence_mbar_init();
    mbar_arrive(&done);            // phase 0 of `done` completes now
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, 256);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it & 1) * 256);
      if (V >= 6)    // the tc1 tile's K=16 -||x||^2 block: no-swizzle core matrices
        mma_bf16(d, desc_k_inter(a + 40960, 128, 256), desc_k_inter(b + 16384, 128, 256), idesc,
                 it >= 2);
#pragma unroll
      for (int kk = 0; kk < GROUP; ++kk)
        mma_bf16(d, desc_k_sw128(a + (kk & 3) * 32), desc_k_sw128(b + (kk & 3) * 32), idesc,
                 it >= 2 || kk || V >= 6);
      if (V == 1 || V == 5) mma_commit(&dummy);
      if (V == 2 || V == 4 || V == 5) mbar_wait(&done, 0);
      if (V == 3 || V == 4 || V == 5) tc_fence_after();
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int V, int GROUP>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 1024 + 49152, iters = 8000;
  cudaFuncSetAttribute(probe<V, GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<V, GROUP><<<148, 128, smem>>>(100, d);
  probe<V, GROUP><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const int nm = GROUP + (V >= 6);
  printf("variant %d group %d: %.1f cyc/MMA  (%.1f cyc per group overhead)  %s\n", V, GROUP,
         (double)c / (iters * (double)nm), (double)c / iters - 128.0 * nm,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 9>(); run<6, 8>(); run<0, 8>();
  run<0, 4>(); run<1, 4>(); run<2, 4>(); run<3, 4>(); run<4, 4>(); run<5, 4>();
  run<0, 1>(); run<1, 1>(); run<2, 1>(); run<3, 1>(); run<4, 1>(); run<5, 1>();
  return 0;
}
