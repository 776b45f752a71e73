// Probe (diagnostic): issue cost of back-to-back tcgen05.mma with A from TMEM
// (the W-statistics shape: M = 128 (i,j) rows per SM, N = K_out, K = 16
// samples) for cta_group::1 (one SM, M = 128) and cta_group::2 (a 2-CTA
// cluster, M = 256 over the pair, issued by the even CTA). Reports cycles per
// MMA instruction and MACs per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma2sm_probe.cu -o mma2sm_probe
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CG>
__global__ void __launch_bounds__(128, 1) probe(int N, int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 256 * 16 * 2 / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  if (w == 0) {
    if (CG == 2)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       tc::smem_u32(&tb)), "r"(512));
    else
      tc::tmem_alloc(&tb, 512);
  }
  if (t == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  if (CG == 2) cooperative_groups::this_cluster().sync();
  else __syncthreads();
  tc::fence_after();
  const uint32_t tm = tb;
  long long c0 = clock64();
  if (w == 0 && rank == 0) {
    const uint64_t bd = tc::smem_desc(tc::smem_u32(sm), (uint32_t)((CG == 2 ? N / 2 : N) * 16), 128);
    const uint32_t M = CG == 2 ? 256 : 128;
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                        ((M >> 4) << 24);
    const uint32_t ta = tm + 256;
    for (int i = 0; i < iters; i += 8) {
      if (tc::elect_one()) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t d = tm + (uint32_t)((u & 1) * 128);
          if (CG == 2)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                "r"(ta + 8 * (u & 3)), "l"(bd), "r"(id), "r"(1u));
          else
            tc::mma_bf16_ts(d, ta + 8 * (u & 3), bd, id, 1u);
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) {
      if (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                tc::smem_u32(&bar)), "h"((uint16_t)3)
            : "memory");
      else
        tc::mma_commit(&bar);
    }
    __syncwarp();
  }
  if (t == 0) tc::mbar_wait(&bar, 0);
  long long c1 = clock64();
  if (t == 0) cyc[blockIdx.x] = c1 - c0;
  tc::fence_before();
  if (CG == 2) cooperative_groups::this_cluster().sync();
  else __syncthreads();
  if (w == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
    } else {
      tc::tmem_dealloc(tm, 512);
    }
  }
}

int main() {
  long long *d, h[148];
  cudaMalloc(&d, sizeof h);
  const int smem = 256 * 16 * 2 * 2;
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 4096;
  for (int N : {32, 48, 64, 96, 128, 256}) {
    for (int cg : {1, 2}) {
      if (cg == 2 && N % 32) continue;
      cudaMemset(d, 0, sizeof h);
      cudaError_t e;
      if (cg == 1) {
        probe<1><<<148, 128, smem>>>(N, iters, d);
        e = cudaGetLastError();
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, probe<2>, N, iters, d);
      }
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      int n = 0;
      for (int i = 0; i < 148; i += cg) {
        avg += h[i];
        ++n;
      }
      avg /= n;
      const double cpm = avg / iters;
      const double macs_per_sm = 128.0 * N * 16 / cpm;  // per SM (each SM: 128 rows)
      printf("cta_group::%d N=%3d: %6.1f cyc/mma  %7.0f MAC/clk/SM  %s\n", cg, N, cpm, macs_per_sm,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
