// Probe: how does tcgen05.mma kind::tf32 treat the 13 low mantissa bits of an
// fp32 operand (truncate, round, or keep)? One CTA, A = 128 x 8, B = 16 x 8,
// B = e_0 (column k=0 is 1), so D[m][0] = A[m][0] as the tensor core sees it.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__global__ void probe(const float *A, float *D) {
  __shared__ __align__(128) float a[128 * 8];
  __shared__ __align__(128) float b[16 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int t = threadIdx.x;
  if (t < 32) tc::tmem_alloc(&tb, 32);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  for (int k = 0; k < 8; ++k) a[tc::kmaj_off(t, k, 128) / 4] = A[t * 8 + k];
  if (t < 16) for (int k = 0; k < 8; ++k) b[tc::kmaj_off(t, k, 16) / 4] = (t == 0 && k == 0) ? 1.f : 0.f;
  tc::fence_async_smem(); tc::fence_before(); __syncthreads(); tc::fence_after();
  if (t == 0) {
    tc::mma_tf32(tb, tc::kstep_desc(tc::smem_u32(a), 128, 0), tc::kstep_desc(tc::smem_u32(b), 16, 0),
                 tc::idesc_tf32(128, 16), 0u);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  float v[8];
  tc::tmem_ld8(tb + ((uint32_t)(32 * (t >> 5)) << 16), v);
  tc::tmem_wait_ld();
  D[t] = v[0];
  tc::fence_before(); __syncthreads();
  if (t < 32) tc::tmem_dealloc(tb, 32);
}

int main() {
  float hA[128 * 8] = {0};
  // row m: 1 + m * 2^-13 (m < 64: sweeps the dropped bits), rows 64+: negatives
  for (int m = 0; m < 128; ++m) {
    float v = 1.0f + (float)(m % 64) * ldexpf(1.f, -16);
    hA[m * 8] = m < 64 ? v : -v;
  }
  float *dA, *dD, hD[128];
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  int trunc = 0, keep = 0, other = 0;
  for (int m = 0; m < 128; ++m) {
    uint32_t ai = *(uint32_t *)&hA[m * 8];
    float tr = *(float *)&(ai &= 0xFFFFE000u, ai);
    if (hD[m] == hA[m * 8]) ++keep;
    else if (hD[m] == tr) ++trunc;
    else ++other;
    if (m % 16 == 5) printf("m=%d in=%.9g out=%.9g trunc=%.9g\n", m, hA[m * 8], hD[m], tr);
  }
  printf("keep=%d trunc=%d other=%d (rows whose dropped bits are 0 count as keep)\n", keep, trunc, other);
  return 0;
}
