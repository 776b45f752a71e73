// Data formats on either side of the EM path.
//
// Dataset payloads (reference modelio.py:145-166): an EIND1 u8 payload is
// converted to float64 and, by default, divided by 255. The engine consumes
// fp32 batches, so the device decode writes (float)((double)v / divisor) --
// bit-identical to staging the reference's float64 array as fp32 on the host
// -- and the host->device copy moves one byte per variable instead of four.
#include <cmath>

#include "einet_internal.h"

namespace einet {

// HBM-bound: 1 byte read + 4 bytes written per value. A 256-entry table in
// shared memory, 16-byte loads, four 16-byte stores per thread and step,
// grid-stride over whole 16-value groups, scalar tail.
__global__ void __launch_bounds__(256) k_decode_u8(const uint8_t *__restrict__ src, int64_t count,
                                                   double divisor, float *__restrict__ dst,
                                                   int vec) {
  EINET_KERNEL_PROLOGUE();
  __shared__ float lut[256];
  lut[threadIdx.x] = (float)((double)threadIdx.x / divisor);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t done = 0;
  if (vec) {
    const int64_t groups = count >> 4;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (int64_t g = t0; g < groups; g += stride) {
      const uint4 v = __ldcs(s4 + g);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        __stcs(d4 + 4 * g + q, make_float4(lut[w[q] & 0xFF], lut[(w[q] >> 8) & 0xFF],
                                           lut[(w[q] >> 16) & 0xFF], lut[w[q] >> 24]));
    }
    done = groups << 4;
  }
  for (int64_t i = done + t0; i < count; i += stride) dst[i] = lut[src[i]];
}

int launch_decode_u8(const uint8_t *src, int64_t count, double divisor, float *dst,
                     cudaStream_t st) {
  if (count <= 0) return EINET_OK;
  const int vec = ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = vec ? (count >> 4) + 1 : count;
  // two CTAs per SM: the pipelined EM steps decode batch i+1 on the copy stream
  // while step i runs; a narrow grid leaves the step its SMs (measured: 1.139
  // vs 1.157 ms per pipelined step with eight per SM)
  const int blocks = (int)std::min<int64_t>((int64_t)sms * 2, (work + 255) / 256);
  launch_k(k_decode_u8, blocks, 256, 0, st, src, count, divisor, dst, vec);
  count_launch();
  return check_cuda(cudaGetLastError(), "decode_u8");
}

}  // namespace einet

namespace einet {

// ---------------------------------------------------------------------------
// EINM1 model files (reference modelio.py:55-134): after the JSON header the
// file holds one blob per tensor (u32 ndim, u32 dims, little-endian f64
// payload) closed by the zlib CRC32 of the blob section. The host parses the
// header; the blob section moves to the device in one copy and these kernels
// check its CRC32, check every embedded shape against the header and scatter
// the payloads into the flat parameter buffer (or, for saving, gather the
// parameters into a blob and checksum it).
// ---------------------------------------------------------------------------

// CRC32 (zlib: reflected polynomial 0xEDB88320, init and final xor ~0) as
// GF(2) polynomial arithmetic. The blob is cut into CRC_SEG-byte segments, one
// per thread; each computes its segment's raw CRC (zero init), multiplies it
// by x^(8 * bytes after the segment) mod P and XOR-reduces it into the result
// (the CRC is linear in the message). The init term is x^(8 len) * ~0 mod P.
constexpr int CRC_SEG = 1024;
constexpr uint32_t CRC_POLY = 0xEDB88320u;

struct CrcTables {
  uint32_t byte[256];  // raw CRC of each byte value
  uint32_t x2n[64];    // x^(2^k) mod P (no wrap-around for n < 2^60)
};

__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  // a * b mod P, bit 31 = x^0 (reflected)
  uint32_t p = 0;
  for (uint32_t m = 1u << 31; m; m >>= 1) {
    if (a & m) p ^= b;
    b = (b & 1) ? (b >> 1) ^ CRC_POLY : b >> 1;
  }
  return p;
}

// x^(n * 2^k) mod P
__host__ __device__ inline uint32_t crc_x2nmodp(const uint32_t *x2n, uint64_t n, int k) {
  uint32_t p = 1u << 31;
  while (n) {
    if (n & 1) p = crc_multmodp(x2n[k & 63], p);
    n >>= 1;
    ++k;
  }
  return p;
}

static const CrcTables &crc_tables() {
  static CrcTables t = [] {
    CrcTables c;
    for (uint32_t v = 0; v < 256; ++v) {
      uint32_t r = v;
      for (int b = 0; b < 8; ++b) r = (r & 1) ? (r >> 1) ^ CRC_POLY : r >> 1;
      c.byte[v] = r;
    }
    uint32_t p = 1u << 30;  // x^1
    for (int k = 0; k < 64; ++k) {
      c.x2n[k] = p;
      p = crc_multmodp(p, p);
    }
    return c;
  }();
  return t;
}

__global__ void __launch_bounds__(256) k_crc32_segments(const uint8_t *__restrict__ data,
                                                        int64_t len, CrcTables tabs,
                                                        uint32_t *acc) {
  EINET_KERNEL_PROLOGUE();
  __shared__ uint32_t tab[256];
  __shared__ uint32_t x2n[64];
  tab[threadIdx.x] = tabs.byte[threadIdx.x];
  if (threadIdx.x < 64) x2n[threadIdx.x] = tabs.x2n[threadIdx.x];
  __syncthreads();
  const int64_t seg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lo = seg * CRC_SEG;
  uint32_t contrib = 0;
  if (lo < len) {
    const int64_t hi = lo + CRC_SEG < len ? lo + CRC_SEG : len;
    uint32_t c = 0;
    int64_t i = lo;
    if (((uintptr_t)data & 15) == 0) {
      for (; i + 16 <= hi; i += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(data + i));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int b = 0; b < 4; ++b) c = tab[(c ^ (w[q] >> (8 * b))) & 0xFF] ^ (c >> 8);
      }
    }
    for (; i < hi; ++i) c = tab[(c ^ data[i]) & 0xFF] ^ (c >> 8);
    contrib = c ? crc_multmodp(crc_x2nmodp(x2n, (uint64_t)(len - hi), 3), c) : 0u;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) contrib ^= __shfl_xor_sync(0xffffffffu, contrib, o);
  if ((threadIdx.x & 31) == 0 && contrib) atomicXor(acc, contrib);
}

__global__ void k_crc32_final(int64_t len, CrcTables tabs, uint32_t *acc) {
  EINET_KERNEL_PROLOGUE();
  *acc = ~(crc_multmodp(crc_x2nmodp(tabs.x2n, (uint64_t)len, 3), 0xFFFFFFFFu) ^ *acc);
}

int launch_crc32(const uint8_t *data, int64_t len, uint32_t *crc, cudaStream_t st) {
  const CrcTables &t = crc_tables();
  int rc = check_cuda(cudaMemsetAsync(crc, 0, sizeof(uint32_t), st), "crc32 init");
  if (rc) return rc;
  if (len > 0) {
    const int64_t segs = (len + CRC_SEG - 1) / CRC_SEG;
    launch_k(k_crc32_segments, (int)((segs + 255) / 256), 256, 0, st, data, len, t, crc);
    count_launch();
  }
  launch_k(k_crc32_final, 1, 1, 0, st, len, t, crc);
  count_launch();
  return check_cuda(cudaGetLastError(), "crc32");
}

// Blob tables: per tensor {blob offset of its u32 ndim, ndim, d0, d1, d2, d3,
// parameter offset, element count} (int64, device memory).
constexpr int BLOB_COLS = 8;
constexpr int BLOB_MAX_NDIM = 4;

__device__ inline uint32_t load_u32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// one block per tensor: check the embedded ndim and dims, then copy the
// payload (4-byte aligned in the blob: two u32 loads per value)
__global__ void k_blob_to_params(const uint8_t *__restrict__ blob, int64_t blob_len,
                                 const int64_t *__restrict__ table, double *__restrict__ params,
                                 int32_t *bad) {
  EINET_KERNEL_PROLOGUE();
  const int64_t *e = table + (int64_t)blockIdx.x * BLOB_COLS;
  const int64_t off = e[0], ndim = e[1], dst = e[6], count = e[7];
  const int64_t pay = off + 4 + 4 * ndim;
  if (pay + 8 * count > blob_len || ndim > BLOB_MAX_NDIM) {
    if (threadIdx.x == 0) atomicMin(bad, (int32_t)blockIdx.x);
    return;
  }
  bool ok = load_u32(blob + off) == (uint32_t)ndim;
  for (int d = 0; d < ndim && ok; ++d) ok = load_u32(blob + off + 4 + 4 * d) == (uint32_t)e[2 + d];
  if (!ok) {
    if (threadIdx.x == 0) atomicMin(bad, (int32_t)blockIdx.x);
    return;
  }
  if (dst < 0) return;  // a manifest entry the circuit does not use: checked, not copied
  const uint32_t *src = reinterpret_cast<const uint32_t *>(blob + pay);
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.y * blockDim.x; i < count;
       i += (int64_t)blockDim.x * gridDim.y) {
    const uint64_t v = (uint64_t)src[2 * i] | ((uint64_t)src[2 * i + 1] << 32);
    params[dst + i] = __longlong_as_double((long long)v);
  }
}

__global__ void k_params_to_blob(const double *__restrict__ params,
                                 const int64_t *__restrict__ table, uint8_t *__restrict__ blob) {
  EINET_KERNEL_PROLOGUE();
  const int64_t *e = table + (int64_t)blockIdx.x * BLOB_COLS;
  const int64_t off = e[0], ndim = e[1], src = e[6], count = e[7];
  uint32_t *hdr = reinterpret_cast<uint32_t *>(blob + off);
  if (blockIdx.y == 0 && threadIdx.x <= ndim)
    hdr[threadIdx.x] = threadIdx.x == 0 ? (uint32_t)ndim : (uint32_t)e[1 + threadIdx.x];
  uint32_t *dst = reinterpret_cast<uint32_t *>(blob + off + 4 + 4 * ndim);
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.y * blockDim.x; i < count;
       i += (int64_t)blockDim.x * gridDim.y) {
    const uint64_t v = (uint64_t)__double_as_longlong(params[src + i]);
    dst[2 * i] = (uint32_t)v;
    dst[2 * i + 1] = (uint32_t)(v >> 32);
  }
}

static int blob_grid_y(int64_t max_count) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(64, (max_count + 1023) / 1024));
}

int launch_blob_to_params(const uint8_t *blob, int64_t blob_len, const int64_t *table,
                          int n_tensors, int64_t max_count, double *params, int32_t *bad,
                          cudaStream_t st) {
  if (n_tensors < 1) return EINET_OK;
  launch_k(k_blob_to_params, dim3(n_tensors, blob_grid_y(max_count)), 256, 0, st, blob, blob_len, table,
                                                                          params, bad);
  count_launch();
  return check_cuda(cudaGetLastError(), "blob_to_params");
}

int launch_params_to_blob(const double *params, const int64_t *table, int n_tensors,
                          int64_t max_count, uint8_t *blob, cudaStream_t st) {
  if (n_tensors < 1) return EINET_OK;
  launch_k(k_params_to_blob, dim3(n_tensors, blob_grid_y(max_count)), 256, 0, st, params, table, blob);
  count_launch();
  return check_cuda(cudaGetLastError(), "params_to_blob");
}


}  // namespace einet
