// Tensor-core (tcgen05, 3xTF32) EinsumLayer kernels.
//
// fp32 operands are split x = hi + lo (hi = tf32(x)); each product uses
// hi*hi + hi*lo + lo*hi MMAs accumulated in TMEM (fp32), which keeps the EM
// statistics at fp32-equivalent accuracy.
#include <climits>
#include <cmath>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

// ---------------------------------------------------------------------------
// self test: D[128 x N] = A[128 x K] B[N x K]^T with one CTA (validation of the
// descriptors, instruction descriptor and TMEM lane mapping)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_selftest_gemm(const float *__restrict__ A,
                                                       const float *__restrict__ B,
                                                       float *__restrict__ D, int N, int K,
                                                       uint32_t tcols) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float *ahi = (float *)sm;
  float *alo = ahi + 128 * K;
  float *bhi = alo + 128 * K;
  float *blo = bhi + N * K;
  const int t = threadIdx.x;
  if (t < 32) tc::tmem_alloc(&tbase, tcols);
  if (t == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  for (int k = 0; k < K; ++k) {
    float h, l;
    tc::split_tf32(A[t * K + k], h, l);
    ahi[tc::kmaj_off(t, k, 128) / 4] = h;
    alo[tc::kmaj_off(t, k, 128) / 4] = l;
  }
  for (int n = t; n < N; n += 128)
    for (int k = 0; k < K; ++k) {
      float h, l;
      tc::split_tf32(B[n * K + k], h, l);
      bhi[tc::kmaj_off(n, k, N) / 4] = h;
      blo[tc::kmaj_off(n, k, N) / 4] = l;
    }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t id = tc::idesc_tf32(128, N);
    const uint32_t sa = tc::smem_u32(ahi), sl = tc::smem_u32(alo);
    const uint32_t sb = tc::smem_u32(bhi), sbl = tc::smem_u32(blo);
    for (int s = 0; s < K / 8; ++s) {
      tc::mma_tf32(tm, tc::kstep_desc(sa, 128, s), tc::kstep_desc(sb, N, s), id, s > 0);
      tc::mma_tf32(tm, tc::kstep_desc(sa, 128, s), tc::kstep_desc(sbl, N, s), id, 1);
      tc::mma_tf32(tm, tc::kstep_desc(sl, 128, s), tc::kstep_desc(sb, N, s), id, 1);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  const int w = t >> 5;
  const uint32_t ta = tm + ((uint32_t)(32 * w) << 16);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(ta + c, v);
    tc::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (c + i < N) D[t * N + c + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (t < 32) tc::tmem_dealloc(tm, tcols);
}

int launch_selftest_gemm(const float *A, const float *B, float *D, int N, int K,
                         cudaStream_t st) {
  if (N < 16 || N > 256 || N % 16 || K < 8 || K % 8)
    return fail(EINET_ERR_USAGE, "selftest gemm: N in [16,256] multiple of 16, K multiple of 8");
  uint32_t cols = 32;
  while (cols < (uint32_t)N) cols *= 2;
  const size_t smem = sizeof(float) * 2 * (128 + N) * K;
  cudaFuncSetAttribute(k_selftest_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_selftest_gemm<<<1, 128, smem, st>>>(A, B, D, N, K, cols);
  count_launch();
  return check_cuda(cudaGetLastError(), "selftest gemm");
}

}  // namespace einet
