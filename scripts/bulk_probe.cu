// Probe (diagnostic): per-SM throughput of 1-D bulk copies (cp.async.bulk,
// the TMA path the contraction / W-statistics producers use) from an
// L2-resident source, all 148 SMs at once, for copy size x copies in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 bulk_probe.cu -o bulk_probe
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__global__ void probe(const uint8_t *src, int64_t src_bytes, int bytes, int depth, int iters,
                      long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 16; ++s) tc::mbar_init(&bar[s], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t off = (int64_t)blockIdx.x * 7919 * 1024 % (src_bytes - bytes);
  off &= ~(int64_t)1023;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % depth, ph = (it / depth) & 1;
    if (it >= depth) tc::mbar_wait(&bar[s], ph ^ 1);
    tc::mbar_arrive_expect_tx(&bar[s], (uint32_t)bytes);
    tc::bulk_g2s(sm + (size_t)s * bytes, src + off, (uint32_t)bytes, &bar[s]);
    off += bytes;
    if (off + bytes > src_bytes) off = 0;
  }
  for (int it = iters; it < iters + depth; ++it) {
    const int s = it % depth, ph = (it / depth) & 1;
    tc::mbar_wait(&bar[s], ph ^ 1);
  }
  cyc[blockIdx.x] = clock64() - c0;
}

int main() {
  const int64_t src_bytes = 64ll << 20;  // L2-resident
  uint8_t *src;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  long long *d, h[148];
  cudaMalloc(&d, sizeof h);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int bytes : {4096, 8192, 16384, 24576, 49152})
    for (int depth : {1, 2, 4, 8}) {
      if ((size_t)bytes * depth > 200 * 1024) continue;
      const int iters = 2000;
      probe<<<148, 32, (size_t)bytes * depth>>>(src, src_bytes, bytes, depth, 8, d);  // warm
      probe<<<148, 32, (size_t)bytes * depth>>>(src, src_bytes, bytes, depth, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("copy %6d B x %d in flight: %6.1f B/clk/SM  %s\n", bytes, depth,
             (double)bytes * iters / avg, cudaGetErrorString(e));
    }
  return 0;
}
