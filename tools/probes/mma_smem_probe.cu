// mma_smem_probe.cu — what limits the kNN tc1 MMA pipeline?  One CTA per SM
// on every SM; thread 0 issues tcgen05.mma kind::f16 M128.N256.K16 (SS,
// 128-B swizzle, the tc1 engine's instruction) back to back into two
// accumulators, optionally while
//   COPY: warp 1 streams cp.async.bulk global->smem into a separate 4 x 32 KB
//         ring as fast as it can (the TMA fill of the database stages), and
//   DRAIN: 8 warps read TMEM (tcgen05.ld.32x32b.x32) continuously (the
//         epilogue's accumulator drain; reads race the MMA writes: timing only).
// Reports cycles per MMA (floor 128 = 4096 MAC/clk/SM) and copy bytes/cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2206_14148_b200/csrc \
//        mma_smem_probe.cu -o mma_smem_probe
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

constexpr int kRing = 4;
constexpr uint32_t kStage = 32768;

template <bool COPY, bool DRAIN>
__global__ void __launch_bounds__(320, 1)
probe(int iters, const uint8_t* __restrict__ src, size_t src_bytes, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* A = smem;                 // 128 x 64 fp16 (16 KB) x 2 k-blocks
  uint8_t* B = smem + 32768;         // 256 x 64 fp16 (32 KB) x 2 k-blocks
  uint8_t* ring = smem + 98304;      // 4 x 32 KB
  __shared__ uint64_t bar, full[kRing];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x3bff3bffu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int s = 0; s < kRing; ++s) mbar_init(&full[s], 1);
    stop = 0;
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, 256);
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it & 1) * 256);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(d, desc_k_sw128(a + kb * 16384 + kk * 32), desc_k_sw128(b + kb * 32768 + kk * 32),
                   idesc, it >= 2 || kb || kk);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    stop = 1;
    out[blockIdx.x * 3] = (unsigned long long)(t1 - t0);
  } else if (COPY && warp == 1) {
    if (lane == 0) {
      long long t0 = clock64();
      unsigned long long bytes = 0;
      size_t off = ((size_t)blockIdx.x * 7919 * kStage) % (src_bytes - kStage);
      uint32_t ph[kRing] = {0, 0, 0, 0};
      for (int s = 0; s < kRing; ++s) {
        mbar_expect_tx(&full[s], kStage);
        bulk_load(ring + s * kStage, src + off, kStage, &full[s]);
        off = (off + kStage) % (src_bytes - kStage);
      }
      int s = 0;
      while (!stop) {
        mbar_wait(&full[s], ph[s]);
        ph[s] ^= 1;
        bytes += kStage;
        mbar_expect_tx(&full[s], kStage);
        bulk_load(ring + s * kStage, src + off, kStage, &full[s]);
        off = (off + kStage) % (src_bytes - kStage);
        s = (s + 1) % kRing;
      }
      for (int r = 0; r < kRing; ++r) {
        mbar_wait(&full[s], ph[s]);
        ph[s] ^= 1;
        s = (s + 1) % kRing;
      }
      out[blockIdx.x * 3 + 1] = bytes;
      out[blockIdx.x * 3 + 2] = (unsigned long long)(clock64() - t0);
    }
  } else if (DRAIN && warp >= 2) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp - 2) >> 2) * 128;
    uint32_t acc = 0;
    int c = 0;
    while (!stop) {
      uint32_t r[32];
      tmem_ld32(base + (c & 3) * 32, r);
      tmem_ld_wait();
      acc ^= r[0] ^ r[31];
      ++c;
    }
    if (acc == 0x12345) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <bool COPY, bool DRAIN>
void run(const char* name, const uint8_t* src, size_t src_bytes) {
  const int grid = 148, iters = 20000;
  const int smem = 1024 + 98304 + kRing * kStage;
  cudaFuncSetAttribute(probe<COPY, DRAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, grid * 3 * 8);
  cudaMemset(d, 0, grid * 3 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<COPY, DRAIN><<<grid, 320, smem>>>(100, src, src_bytes, d);
  cudaEventRecord(e0);
  probe<COPY, DRAIN><<<grid, 320, smem>>>(iters, src, src_bytes, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148 * 3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0, ccyc = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += (double)h[3 * i] / grid;
    bytes += (double)h[3 * i + 1] / grid;
    ccyc += (double)h[3 * i + 2] / grid;
  }
  const double macs = (double)iters * 8 * 128 * 256 * 16;
  printf("%-26s %.1f cyc/MMA  %.0f MAC/clk/SM  %.0f TF/s chip (%.3f ms)  copy %.1f B/cyc/SM  %s\n",
         name, cyc / (iters * 8.0), macs / cyc, 2 * macs * grid / (ms * 1e-3) / 1e12, ms,
         ccyc > 0 ? bytes / ccyc : 0.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  const size_t src_bytes = 48u << 20;      // L2-resident source, like the engine's tiles
  uint8_t* src;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 0x3b, src_bytes);
  for (int rep = 0; rep < 2; ++rep) {
    run<false, false>("mma only", src, src_bytes);
    run<true, false>("mma + bulk copy", src, src_bytes);
    run<false, true>("mma + tmem drain", src, src_bytes);
    run<true, true>("mma + copy + drain", src, src_bytes);
  }
  return 0;
}
