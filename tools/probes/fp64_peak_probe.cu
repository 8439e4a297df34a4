// fp64_peak_probe.cu — measured FP64 FMA throughput of this B200 (the
// denominator of the kernel-MVM roofline): 148 x 8 resident blocks of 256
// threads, 8 independent DFMA chains per thread; prints JSON.
#include <cstdio>
__global__ void __launch_bounds__(256) dfma_loop(long long iters, double* out) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-9 + j;
  const double b = 0.999999, c = 1e-7;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0) out[0] = s;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256;
  dfma_loop<<<blocks, threads>>>(1000, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long iters = 200000;
  cudaEventRecord(e0);
  dfma_loop<<<blocks, threads>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * iters * (double)blocks * threads;
  printf("{\"fp64_tflops\": %.2f, \"ms\": %.1f, \"how\": \"DFMA loop, %d blocks x 256 threads x 8 chains\", \"err\": \"%s\"}\n",
         flops / (ms * 1e-3) / 1e12, ms, blocks, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
