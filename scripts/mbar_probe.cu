// Hand-off latency probe (diagnostic): producer / consumer warps ping-pong
// through an mbarrier ring of S stages, N iterations; reports cycles per
// iteration for plain arrive, cp.async noinc arrive and tcgen05.commit.
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

__device__ __forceinline__ void arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(b)) : "memory");
}
template <int MODE, int S>
__global__ void k(int n, long long *out) {
  __shared__ uint64_t full[S], empty[S];
  __shared__ uint32_t tb;
  const int w = threadIdx.x >> 5;
  if (w == 1) tc::tmem_alloc(&tb, 32);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], MODE == 1 ? 32 : 1); tc::mbar_init(&empty[s], 1); }
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  long long t0 = clock64();
  if (w == 0) {  // producer
    for (int i = 0; i < n; ++i) {
      const int s = i % S, ph = (i / S) & 1;
      tc::mbar_wait(&empty[s], ph ^ 1);
      if (MODE == 1) {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[s])) : "memory");
      } else if ((threadIdx.x & 31) == 0) arrive(&full[s]);
    }
  } else if (w == 1) {  // consumer
    for (int i = 0; i < n; ++i) {
      const int s = i % S, ph = (i / S) & 1;
      tc::mbar_wait(&full[s], ph);
      tc::fence_after();
      if (MODE == 2) {
        if (tc::elect_one()) tc::mma_commit(&empty[s]);
        __syncwarp();
      } else if ((threadIdx.x & 31) == 0) arrive(&empty[s]);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  if (w == 1) tc::tmem_dealloc(tb, 32);
}
template <int MODE, int S>
void run(const char *name) {
  long long *d, h;
  cudaMalloc(&d, 8 * 148);
  const int n = 20000;
  k<MODE, S><<<148, 64>>>(n, d);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s S=%d: %.1f cycles / iteration (%s)\n", name, S, (double)h / n, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0, 1>("arrive/try_wait");
  run<0, 4>("arrive/try_wait");
  run<1, 1>("cp.async noinc");
  run<1, 4>("cp.async noinc");
  run<2, 1>("tcgen05.commit");
  run<2, 4>("tcgen05.commit");
  return 0;
}
