// mma_probe.cu — microbenchmark: tcgen05.mma issue throughput per shape
// (smem-resident operands, no TMA), 1 CTA per SM on every SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2206_14148_b200/csrc mma_probe.cu -o mma_probe -lcuda
#include <cstdio>
#include <vector>
#include "sm100.cuh"
using namespace tb::sm100;

template <int KIND>  // 0 = i8 (K=32), 1 = bf16 (K=16)
__global__ void __launch_bounds__(128, 1) probe(int N, int nacc, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* A = smem;              // 128 x 128 B
  uint8_t* B = smem + 16384;      // 256 x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x3f3f3f3fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND == 0 ? idesc_u8_s32(128, N) : idesc_bf16_f32(128, N);
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it % nacc) * N);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (KIND == 0) mma_i8(d, desc_k_sw128(a + kk * 32), desc_k_sw128(b + kk * 32), idesc, it >= nacc || kk);
        else mma_bf16(d, desc_k_sw128(a + kk * 32), desc_k_sw128(b + kk * 32), idesc, it >= nacc || kk);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 1024 + 16384 + 32768;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct S { int kind, N, nacc; } shapes[] = {{0, 64, 8}, {0, 96, 5}, {0, 128, 4}, {0, 256, 2}, {1, 128, 4}, {1, 256, 2}};
  const int iters = 20000;
  for (auto s : shapes) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (s.kind == 0) probe<0><<<sms, 128, smem>>>(s.N, s.nacc, iters, d);
      else probe<1><<<sms, 128, smem>>>(s.N, s.nacc, iters, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const int K = s.kind == 0 ? 32 : 16;
    const double macs = (double)iters * 4 * 128 * s.N * K;
    printf("%s M128 N%3d: %.1f cyc/MMA  %.0f MAC/clk/SM  %.1f T(MAC*2)/s chip  err=%s\n",
           s.kind == 0 ? "i8  " : "bf16", s.N, (double)cyc / (iters * 4.0), macs / cyc,
           2 * macs * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
