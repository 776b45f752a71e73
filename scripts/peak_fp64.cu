// Micro-benchmark: sustained DFMA and FFMA throughput (independent chains).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k_fma(T *out, int iters) {
  T a[16];
  for (int i = 0; i < 16; ++i) a[i] = (T)(threadIdx.x + i) * (T)1e-3;
  const T b = (T)0.999, c = (T)1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  T s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == (T)12345) out[0] = s;
}
template <typename T>
double run(const char *name) {
  T *out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  k_fma<T><<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_fma<T><<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double fmas = (double)blocks * threads * iters * 16;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s: %.2f T fma/s  (%.1f fma/clk/SM at %.0f MHz nominal)\n", name, fmas / ms / 1e9,
         fmas / ms / 1e3 / sms / (clk / 1e3), clk / 1e3);
  return fmas / ms;
}
int main() {
  run<double>("DFMA");
  run<float>("FFMA");
  return 0;
}
