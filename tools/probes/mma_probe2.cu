// mma_probe2.cu — i8 M128 N128 MMA throughput vs operand layout / issue
// pattern (smem-resident operands, no TMA, every SM).
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

// pattern 0: 4 consecutive MMAs into one acc (rotating accs), SW128, same A/B
// pattern 1: same as 0 with SW64 descriptors
// pattern 2: the gram phase-A sequence: 8 products x 2 k-steps, 6 tiles, SW64
// pattern 3: pattern 2 with SW128 (k-step offset 32 B inside a 128-B row)
__global__ void __launch_bounds__(128, 1) probe(int pattern, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[3];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 6 * 16384 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x7f7f7f7fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 3; ++i) mbar_init(&bar2[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_u8_s32(128, 128);
    const uint32_t base = smem_u32(smem);
    uint32_t a[3], b[3];
    for (int p = 0; p < 3; ++p) { a[p] = base + p * 32768; b[p] = a[p] + 16384; }
    const bool sw64 = pattern != 0 && pattern != 3;
    auto D = [&](uint32_t x) { return sw64 ? desc_k_sw64(x) : desc_k_sw128(x); };
    const uint32_t acc0 = tmem, acc1 = tmem + 128, acc2 = tmem + 256, acc3 = tmem + 384;
    long long t0 = clock64();
    int n = 0;
    for (int it = 0; it < iters; ++it) {
      if (pattern <= 1) {
        const uint32_t d = tmem + (uint32_t)((it & 3) * 128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(d, D(a[0] + (kk & 1) * 32), D(b[0] + (kk & 1) * 32), idesc, 1);
        n += 4;
      } else {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t o = ks * 32;
          mma_i8(acc0, D(a[2] + o), D(b[2] + o), idesc, 1);
          mma_i8(acc1, D(a[2] + o), D(b[1] + o), idesc, 1);
          mma_i8(acc1, D(a[1] + o), D(b[2] + o), idesc, 1);
          mma_i8(acc2, D(a[2] + o), D(b[0] + o), idesc, 1);
          mma_i8(acc2, D(a[1] + o), D(b[1] + o), idesc, 1);
          mma_i8(acc2, D(a[0] + o), D(b[2] + o), idesc, 1);
          mma_i8(acc3, D(a[1] + o), D(b[0] + o), idesc, 1);
          mma_i8(acc3, D(a[0] + o), D(b[1] + o), idesc, 1);
        }
        n += 16;
        if (pattern == 4 || pattern == 6) tc_fence_after();
        if (pattern == 5 || pattern == 6) { mma_commit(&bar2[0]); mma_commit(&bar2[1]); mma_commit(&bar2[2]); }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { cyc[0] = (unsigned long long)(t1 - t0); cyc[1] = n; }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 1024 + 6 * 16384 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"4x same acc, SW128", "4x same acc, SW64", "gram phase A, SW64", "gram phase A, SW128",
                         "A + fence/16", "A + 3 commits/16", "A + fence + commits"};
  for (int p = 0; p < 7; ++p) {
    for (int rep = 0; rep < 2; ++rep) probe<<<sms, 128, smem>>>(p, p <= 1 ? 20000 : 5000, d);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-22s %.1f cyc/MMA (%s)\n", names[p], (double)h[0] / h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
