// Probe: tcgen05.ld (32x32b) throughput per SM for 4..16 warps and .x8/.x16/.x32
// shapes: each warp reads its lane quarter, 128 columns per round, many rounds.
#include <cstdio>
#include <cstdint>
#include "../paper_2004_06231_b200/csrc/tc_common.cuh"
using namespace einet;

template <int X>
__device__ __forceinline__ void ldx(uint32_t addr, float *v);
template <> __device__ __forceinline__ void ldx<8>(uint32_t a, float *v) {
  float t[8]; tc::tmem_ld8(a, *(float(*)[8])t); for (int i = 0; i < 8; ++i) v[i] += t[i]; }
template <> __device__ __forceinline__ void ldx<16>(uint32_t a, float *v) {
  float t[16]; tc::tmem_ld16(a, *(float(*)[16])t); for (int i = 0; i < 16; ++i) v[i] += t[i]; }
template <> __device__ __forceinline__ void ldx<32>(uint32_t a, float *v) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
      : "r"(a));
  for (int i = 0; i < 32; ++i) v[i % 16] += __uint_as_float(r[i]); }

template <int X>
__global__ void probe(int rounds, int batch, long long *out, float *sink) {
  __shared__ uint32_t tb;
  const int w = threadIdx.x >> 5;
  if (w == 0) tc::tmem_alloc(&tb, 512);
  tc::fence_before(); __syncthreads(); tc::fence_after();
  float v[16] = {0};
  const uint32_t base = tb + ((uint32_t)(32 * (w & 3)) << 16);
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    // batch loads of X columns, then one wait
    for (int c = 0; c < 128; c += X * batch) {
      for (int b = 0; b < batch; ++b) ldx<X>(base + ((c + b * X + 128 * (w >> 2)) & 511), v);
      tc::tmem_wait_ld();
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 123.f) sink[0] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc::fence_before(); __syncthreads();
  if (w == 0) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d, h[148]; float *sink;
  cudaMalloc(&d, sizeof h); cudaMalloc(&sink, 4);
  const int rounds = 200;
  for (int warps : {4, 8, 16})
    for (int X : {8, 16, 32})
      for (int batch : {1, 2, 4}) {
        if (X * batch > 128) continue;
        if (X == 8) probe<8><<<148, 32 * warps>>>(rounds, batch, d, sink);
        if (X == 16) probe<16><<<148, 32 * warps>>>(rounds, batch, d, sink);
        if (X == 32) probe<32><<<148, 32 * warps>>>(rounds, batch, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
        const double bytes = (double)warps * 32 * 128 * 4 * rounds;
        printf("warps %2d x%-2d batch %d: %6.1f B/clk/SM  %s\n", warps, X, batch, bytes / avg,
               cudaGetErrorString(e));
      }
  return 0;
}
