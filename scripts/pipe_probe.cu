// Probe (diagnostic): tcgen05 MMA pipeline with accumulator hand-off to
// epilogue warps that do no work. One CTA per SM; the MMA warp issues
// `nmma` bf16 SS MMAs (M=128, N) per chunk into a ring of `slots`
// accumulators; EW epilogue warps wait for each chunk's commit and release
// its slot. Reports ns per chunk (globaltimer) and the ideal N/2-cycle rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 pipe_probe.cu -o pipe_probe
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__device__ __forceinline__ long long now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(b)) : "memory");
}

__global__ void __launch_bounds__(576, 1) probe(int N, int nmma, int slots, int chunks, int ew, int ldtm, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t cf[8], ce[8];
  __shared__ uint32_t tb;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < (128 + 256) * 48 * 4 / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
  if (w == 1) tc::tmem_alloc(&tb, 512);
  if (t == 0) {
    for (int s = 0; s < 8; ++s) {
      tc::mbar_init(&cf[s], 1);
      tc::mbar_init(&ce[s], ew);
    }
    tc::mbar_fence_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tb;
  const int stride = 512 / slots;
  long long t0 = now(), c0 = clock64();
  if (w == 1) {
    const uint64_t ad = tc::smem_desc(tc::smem_u32(sm), 128 * 16, 128);
    const uint64_t bd = tc::smem_desc(tc::smem_u32(sm) + 128 * 48 * 4, N * 16, 128);
    const uint32_t id = tc::idesc_bf16(128, N);
    int s = 0, ph = 0;
    for (int c = 0; c < chunks; ++c) {
      tc::mbar_wait(&ce[s], ph ^ 1);
      tc::fence_after();
      if (tc::elect_one()) {
        const uint32_t d = tm + (uint32_t)(s * stride);
        for (int k = 0; k < nmma; ++k) tc::mma_bf16(d, ad + 2 * (k % 3), bd + 2 * (k % 3), id, k > 0);
        tc::mma_commit(&cf[s]);
      }
      __syncwarp();
      if (++s == slots) { s = 0; ph ^= 1; }
    }
  } else if (w >= 2 && w < 2 + ew) {
    const uint32_t lane_off = (uint32_t)(32 * (w & 3)) << 16;
    int s = 0, ph = 0;
    float acc = 0.f;
    for (int c = 0; c < chunks; ++c) {
      tc::mbar_wait(&cf[s], ph);
      tc::fence_after();
      for (int u = 0; u < ldtm; u += 32) {
        float v[32];
        tc::tmem_ld32(tm + lane_off + (uint32_t)(s * stride + u), v);
        tc::tmem_wait_ld();
        for (int i = 0; i < 32; ++i) acc += v[i];
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) arrive(&ce[s]);
      if (++s == slots) { s = 0; ph ^= 1; }
    }
    if (acc == 1234.f) out[1000] = 1;
    if (w == 2 && lane == 0) { out[blockIdx.x] = now() - t0; out[200 + blockIdx.x] = clock64() - c0; }
  }
  tc::fence_before();
  __syncthreads();
  long long t1 = now(), c1 = clock64();
  (void)t1; (void)c1;
  if (w == 1) tc::tmem_dealloc(tm, 512);
}

int main() {
  long long *d, h[400];
  cudaMalloc(&d, 1001 * sizeof(long long));
  cudaMemset(d, 0, 1001 * sizeof(long long));
  const int smem = (128 + 256) * 48 * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int chunks = 2000;
  struct Cfg { int N, nmma, slots, ew, ldtm; };
  Cfg cfgs[] = {{240, 9, 2, 12, 0}, {240, 9, 2, 4, 0}, {240, 9, 2, 1, 0}, {256, 9, 2, 12, 0},
                {120, 9, 4, 12, 0}, {240, 18, 2, 12, 0}, {240, 9, 2, 12, 64}, {240, 9, 2, 12, 160},
                {240, 9, 2, 12, 240}, {240, 9, 2, 8, 240}, {128, 9, 4, 12, 0}, {64, 9, 8, 12, 0}};
  for (const Cfg &c : cfgs) {
    probe<<<148, 64 + 32 * 16, smem>>>(c.N, c.nmma, c.slots, chunks, c.ew, c.ldtm, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("raw ns %lld cyc %lld | ", h[0], h[200]);
    printf("N=%3d nmma=%2d slots=%d ew=%2d ldtm_cols=%3d: %7.1f ns/chunk (ideal %6.1f ns at 1.9 GHz, N/2 cyc/mma) %s\n",
           c.N, c.nmma, c.slots, c.ew, c.ldtm, avg / chunks, c.nmma * c.N / 2 / 1.9, cudaGetErrorString(e));
  }
  return 0;
}
