// Probe: per-SM bulk-copy (cp.async.bulk) throughput, global -> shared, with a
// ring of S stages of C bytes, 148 CTAs; source L2-resident (32 MB) or not (2 GB).
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__global__ void probe(const uint8_t *src, size_t span, int chunk, int stages, int iters, int ncopies,
                      long long *out, int nowait) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) tc::mbar_init(&full[s], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  size_t off = (size_t)blockIdx.x * 7919 * 1024 % span;
  const int piece = chunk / ncopies;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages && !nowait) tc::mbar_wait(&full[s], ((it / stages) - 1) & 1);
    tc::mbar_arrive_expect_tx(&full[s], chunk);
    for (int c = 0; c < ncopies; ++c) {
      tc::bulk_g2s(sm + (size_t)s * chunk + c * piece, src + off + c * piece, piece, &full[s]);
    }
    off = (off + (size_t)chunk * 148 + 4096) & (span - 1);  // span is a power of two
    if (off + chunk > span) off = 0;
  }
  if (!nowait) {
    for (int it = iters; it < iters + stages; ++it) {
      const int s = it % stages;
      tc::mbar_wait(&full[s], ((it / stages) - 1) & 1);
    }
  } else {
    // all copies signalled the same (single-stage) barrier; wait for its last phase
    tc::mbar_wait(&full[0], (iters - 1) & 1);
  }
  out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t *buf;
  const size_t big = 2ull << 30;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  long long *d, h[148];
  cudaMalloc(&d, sizeof h);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int nowait : {0, 1})
  for (size_t span : {(size_t)32 << 20, big})
    for (int chunk : {4096, 8192, 32768})
      for (int stages : {1, 4})
        for (int nc : {1}) {
          if (nowait && stages != 1) continue;
          if (!nowait && stages == 1) continue;
          const int iters = 400;
          probe<<<148, 32, chunk * stages>>>(buf, span, chunk, stages, iters, nc, d, nowait);
          cudaError_t e = cudaDeviceSynchronize();
          cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
          double avg = 0;
          for (int i = 0; i < 148; ++i) avg += h[i];
          avg /= 148;
          const double bytes_per_cyc = (double)chunk * iters / avg;
          printf("nowait %d span %4zu MB chunk %6d stages %d: %6.1f B/clk/SM  %.0f cyc/copy (chip %.2f TB/s) %s\n",
                 nowait, span >> 20, chunk, stages, bytes_per_cyc, avg / iters,
                 bytes_per_cyc * 1.965 * 148 / 1000, cudaGetErrorString(e));
        }
  return 0;
}
