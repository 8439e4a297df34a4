// mma_probe3.cu — i8 M128 N128 SW64 MMA throughput on FRESH operands: the
// gram phase-A k-block (3 stages of A/B tiles, 16 MMAs into 4 accs) cycling
// through a 14-stage smem ring like the real kernel, in 3 product orders.
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

__global__ void __launch_bounds__(128, 1) probe(int order, int nstage, int iters, unsigned long long* cyc, int a_stride, int b_off, int b_stride) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 225 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x7f7f7f7fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_u8_s32(128, 128);
    const uint32_t base = smem_u32(smem);
    const uint32_t acc[4] = {tmem, tmem + 128, tmem + 256, tmem + 384};
    // products (s, t, level-acc): original order / grouped by A / grouped by B
    const int P[3][8][3] = {
        {{2,2,0},{2,1,1},{1,2,1},{2,0,2},{1,1,2},{0,2,2},{1,0,3},{0,1,3}},
        {{2,2,0},{2,1,1},{2,0,2},{1,2,1},{1,1,2},{1,0,3},{0,2,2},{0,1,3}},
        {{2,2,0},{1,2,1},{0,2,2},{2,1,1},{1,1,2},{0,1,3},{2,0,2},{1,0,3}}};
    int st = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t a[3], b[3];
      for (int p = 2; p >= 0; --p) {
        a[p] = base + st * a_stride; b[p] = base + b_off + st * b_stride;
        if (++st == nstage) st = 0;
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int* q = P[order][j];
          mma_i8(acc[q[2]], desc_k_sw64(a[q[0]] + ks * 32), desc_k_sw64(b[q[1]] + ks * 32), idesc, 1);
        }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { cyc[0] = (unsigned long long)(t1 - t0); cyc[1] = iters * 16; }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 1024 + 225 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int K = 1024;
  struct C { int ns, as, bo, bs; const char* what; } cs[] = {
    {3, 16*K, 8*K, 16*K, "interleaved A|B 8K, stage 16K (kernel)"},
    {14, 16*K, 8*K, 16*K, "same, 14 stages"},
    {3, 32*K, 16*K, 32*K, "interleaved A|B 16K, stage 32K (probe2)"},
    {3, 8*K, 24*K, 8*K, "A region, B region at +24K"},
    {3, 8*K, 32*K, 8*K, "A region, B region at +32K"},
    {3, 8*K, 64*K, 8*K, "A region, B region at +64K"},
    {3, 8*K, 112*K, 8*K, "A region, B region at +112K"},
    {14, 8*K, 112*K, 8*K, "14 stages, B region at +112K"},
    {3, 16*K, 64*K, 16*K, "A stride 16K, B at +64K stride 16K"},
  };
  for (auto c : cs) {
    for (int rep = 0; rep < 2; ++rep) probe<<<sms, 128, smem>>>(0, c.ns, 4000, d, c.as, c.bo, c.bs);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-45s %.1f cyc/MMA (%s)\n", c.what, (double)h[0] / h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
