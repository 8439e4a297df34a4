// tmem_ld_probe.cu — TMEM read throughput on sm_100a: how many bytes per
// cycle per SM can tcgen05.ld.32x32b deliver, as a function of the number of
// reading warps, loads in flight per warp and the ALU work between loads?
// (The kNN tc1 epilogue reads 4 B of fp32 accumulator per (query, row)
// pair; if TMEM reads are the limiter, the drain sets the engine's floor.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2206_14148_b200/csrc \
//        tmem_ld_probe.cu -o tmem_ld_probe && ./tmem_ld_probe
#include <cstdio>
#include "sm100.cuh"
using namespace tb::sm100;

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <int WARPS, int DEPTH, int WORK>
__global__ void __launch_bounds__(32 * WARPS, 1) probe(int iters, unsigned long long* cyc,
                                                        float* sink) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  const int quad = warp & 3;
  const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[DEPTH][32];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d)
      tmem_ld32(base + (uint32_t)(((it * DEPTH + d) * 32 + (warp >> 2) * 64) & 511), r[d]);
    tmem_ld_wait();
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (WORK) {
        float m = -INFINITY;
#pragma unroll
        for (int i = 0; i < 30; i += 3)
          m = max3f(m, max3f(__uint_as_float(r[d][i]), __uint_as_float(r[d][i + 1]),
                             __uint_as_float(r[d][i + 2])), -INFINITY);
        acc += m;
      } else {
        acc += __uint_as_float(r[d][0] ^ r[d][31]);
      }
    }
  }
  long long t1 = clock64();
  if (acc == 1.2345f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int WARPS, int DEPTH, int WORK>
void run(const char* name) {
  const int iters = 4096, grid = 148;
  unsigned long long* d_cyc;
  float* sink;
  cudaMalloc(&d_cyc, grid * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  probe<WARPS, DEPTH, WORK><<<grid, 32 * WARPS>>>(16, d_cyc, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<WARPS, DEPTH, WORK><<<grid, 32 * WARPS>>>(iters, d_cyc, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += (double)h[i] / grid;
  const double bytes_per_sm = (double)WARPS * iters * DEPTH * 32 * 32 * 4;
  printf("%-28s warps %2d depth %d work %d: %7.1f B/cyc/SM  (%.3f ms, %.2f TB/s chip) %s\n",
         name, WARPS, DEPTH, WORK, bytes_per_sm / avg, ms, bytes_per_sm * grid / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d_cyc);
  cudaFree(sink);
}

int main() {
  run<4, 1, 0>("1 warp/SMSP");
  run<4, 2, 0>("1 warp/SMSP");
  run<4, 4, 0>("1 warp/SMSP");
  run<8, 1, 0>("2 warps/SMSP");
  run<8, 2, 0>("2 warps/SMSP");
  run<8, 2, 1>("2 warps/SMSP + max tree");
  run<8, 4, 0>("2 warps/SMSP");
  run<16, 1, 0>("4 warps/SMSP");
  run<16, 2, 0>("4 warps/SMSP");
  run<16, 2, 1>("4 warps/SMSP + max tree");
  run<16, 1, 1>("4 warps/SMSP + max tree");
  run<32, 1, 0>("8 warps/SMSP");
  run<32, 1, 1>("8 warps/SMSP + max tree");
  return 0;
}
