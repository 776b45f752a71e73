// Micro-benchmark: FP64 tensor-core (DMMA) throughput on sm_100a for the
// mma.sync f64 shapes, independent accumulator chains, operands in registers.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void k_dmma(double *out, int iters) {
  // 4 independent accumulators per warp
  double acc[4][4];
  for (int c = 0; c < 4; ++c)
    for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (SHAPE == 0) {  // m8n8k4: a 1 reg, b 1 reg, c 2 regs
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a[c]), "d"(b[c]));
      } else if (SHAPE == 1) {  // m16n8k4: a 2, b 1, c 4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[c]), "d"(a[c + 4]), "d"(b[c]));
      } else if (SHAPE == 2) {  // m16n8k8: a 4, b 2, c 4
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[c & 1]), "d"(b[2 + (c & 1)]));
      } else {  // m16n8k16: a 8, b 4, c 4
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int c = 0; c < 4; ++c)
    for (int i = 0; i < 4; ++i) s += acc[c][i];
  if (s == 12345.0) out[0] = s;
}

template <int SHAPE>
void run(const char *name, double fma_per_mma, int warps) {
  double *out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048, threads = 32 * warps, blocks = sms * 2;
  k_dmma<SHAPE><<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_dmma<SHAPE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double fmas = (double)blocks * warps * iters * 4 * fma_per_mma;
  printf("%-10s warps/CTA=%2d: %.2f T fma/s (%.1f TFLOP/s)  err=%s\n", name, warps,
         fmas / ms / 1e9, 2 * fmas / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int w : {4, 8, 16}) {
    run<0>("m8n8k4", 8 * 8 * 4, w);
    run<1>("m16n8k4", 16 * 8 * 4, w);
    run<2>("m16n8k8", 16 * 8 * 8, w);
    run<3>("m16n8k16", 16 * 8 * 16, w);
  }
  return 0;
}
