// i8_peak_probe.cu — measured tcgen05 kind::i8 peak on this B200: every SM
// issues the SGPR Gram's instruction (M128.N128.K32 u8 x u8 -> s32, SS
// operands, 64-byte swizzle, four accumulators, the phase-A pattern of 16
// MMAs per k-block with an elected issuing lane) back to back with
// smem-resident operands.  One short launch (burst) and one launch of
// ~`seconds` (sustained, the clock under the power cap); prints JSON.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_2206_14148_b200/csrc i8_peak_probe.cu -o i8_peak_probe
#include <cstdio>
#include <cstdlib>
#include "sm100.cuh"
using namespace tb::sm100;

__global__ void __launch_bounds__(128, 1) probe(long long iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t kTile = 128 * 64, kStage = 6 * kTile;
  for (int i = threadIdx.x; i < kStage / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x7f7f7f7fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = idesc_u8_s32(128, 128);
    const uint32_t acc0 = tmem, acc1 = tmem + 128, acc2 = tmem + 256, acc3 = tmem + 384;
    const uint64_t a2 = desc_k_sw64(smem_u32(smem)), b2 = a2 + (kTile >> 4);
    const uint64_t a1 = a2 + 2 * (kTile >> 4), b1 = a2 + 3 * (kTile >> 4);
    const uint64_t a0 = a2 + 4 * (kTile >> 4), b0 = a2 + 5 * (kTile >> 4);
    long long t0 = clock64();
    for (long long it = 0; it < iters; ++it) {
      if (elect_one_sync()) {
#pragma unroll
        for (int o = 0; o < 4; o += 2) {
          const uint32_t acc = it || o ? 1u : 0u;
          mma_i8(acc0, a2 + o, b2 + o, idesc, acc);
          mma_i8(acc1, a2 + o, b1 + o, idesc, acc);
          mma_i8(acc1, a1 + o, b2 + o, idesc, 1);
          mma_i8(acc2, a2 + o, b0 + o, idesc, acc);
          mma_i8(acc2, a1 + o, b1 + o, idesc, 1);
          mma_i8(acc2, a0 + o, b2 + o, idesc, 1);
          mma_i8(acc3, a1 + o, b0 + o, idesc, acc);
          mma_i8(acc3, a0 + o, b1 + o, idesc, 1);
        }
      }
      __syncwarp();
    }
    if (elect_one_sync()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

static double run(long long iters, int sms, unsigned long long* d, double* cyc_per_mma) {
  const int smem = 1024 + 6 * 128 * 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += (double)h[i] / sms;
  *cyc_per_mma = c / (iters * 16.0);
  const double ops = 2.0 * 128 * 128 * 32 * 16 * (double)iters * sms;
  return ops / (ms * 1e-3) / 1e12;   // TOPS
}

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 5.0;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 256 * 8);
  double cpm;
  run(1000, sms, d, &cpm);                              // warm-up
  double burst = 0, bcpm = 0;
  for (int r = 0; r < 5; ++r) {
    const double t = run(20000, sms, d, &cpm);          // ~20 ms
    if (t > burst) { burst = t; bcpm = cpm; }
  }
  // iterations for ~`seconds` at the burst rate
  const long long iters = (long long)(seconds * burst * 1e12 / (2.0 * 128 * 128 * 32 * 16 * sms));
  double scpm;
  const double sus = run(iters, sms, d, &scpm);
  printf("{\"i8_tops_burst\": %.1f, \"burst_cyc_per_mma\": %.2f, \"i8_tops_sustained\": %.1f, "
         "\"sustained_cyc_per_mma\": %.2f, \"sustained_seconds\": %.2f, \"sms\": %d, "
         "\"instruction\": \"tcgen05.mma.cta_group::1.kind::i8 M128.N128.K32 SS sw64, 16 per "
         "k-block over 4 accumulators (the SGPR Gram's phase A)\", \"err\": \"%s\"}\n",
         burst, bcpm, sus, scpm, seconds, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
