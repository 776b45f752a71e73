// Probe: issue cost of back-to-back tcgen05.mma (cta_group::1, M=128) per
// instruction for kind::tf32 / kind::f16 (bf16 in, fp32 acc), A from shared
// memory (SS) or tensor memory (TS), over N. One CTA per SM, 4096 MMAs each.
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(int N, int kind, int ts, int iters, long long *cyc, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int t = threadIdx.x;
  for (int i = t; i < (128 + 256) * 32 / 4; i += blockDim.x) ((float *)sm)[i] = 0.001f * (i % 7);
  if (t < 32) tc::tmem_alloc(&tb, 512);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::fence_async_smem(); tc::fence_before(); __syncthreads(); tc::fence_after();
  if (t == 0) {
    const uint32_t sa = tc::smem_u32(sm), sb = sa + 128 * 32;
    const uint64_t ad = tc::smem_desc(sa, 128 * 16, 128), bd = tc::smem_desc(sb, N * 16, 128);
    const uint32_t id = kind ? idesc_bf16(128, N) : tc::idesc_tf32(128, N);
    const uint32_t ta = tb + 256;  // A in TMEM columns 256.. (8 cols)
    long long c0 = clock64();
    if (kind == 0 && ts == 0) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          tc::mma_tf32(tb + (uint32_t)((u % nacc) * (256 / nacc) / 16 * 16), ad, bd, id, 1u);
      }
    } else if (kind == 0) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          tc::mma_tf32_ts(tb + (uint32_t)((u % nacc) * (256 / nacc) / 16 * 16), ta, bd, id, 1u);
      }
    } else if (ts == 0) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          mma_f16_ss(tb + (uint32_t)((u % nacc) * (256 / nacc) / 16 * 16), ad, bd, id, 1u);
      }
    } else {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          mma_f16_ts(tb + (uint32_t)((u % nacc) * (256 / nacc) / 16 * 16), ta, bd, id, 1u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long c1 = clock64();
    cyc[blockIdx.x] = c1 - c0;
  }
  tc::fence_before(); __syncthreads();
  if (t < 32) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d; cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  for (int nacc : {1, 2, 4})
  for (int kind = 0; kind < 2; ++kind)
    for (int ts = 0; ts < 2; ++ts)
      for (int N : {16, 48, 64, 128, 240, 256}) {
        if (N * nacc > 256 && N != 16 && N != 48 && N != 64) continue;
        probe<<<148, 128, 64 * 1024>>>(N, kind, ts, iters, d, nacc);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
        const double k = kind ? 16 : 8;
        printf("nacc=%d %s %s N=%3d: %7.1f cyc/mma  floor %5.1f  MAC/clk/SM %7.1f  %s\n", nacc,
               kind ? "bf16" : "tf32", ts ? "TS" : "SS", N, avg / iters, 128.0 * N / 256,
               128.0 * N * k / (avg / iters), cudaGetErrorString(e));
      }
  return 0;
}
