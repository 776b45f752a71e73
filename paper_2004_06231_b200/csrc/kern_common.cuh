// Device-side views of the compute and workspace buffers plus shared helpers.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math_constants.h>
#include <stdint.h>

#include "einet_internal.h"
#include "tc_common.cuh"

namespace einet {

constexpr double kLog2Pi = 1.8378770664093453;  // log(2*pi)
constexpr double kEpsCount = 1e-12;             // trainer.py:23

struct CompView {
  float *w32;
  float *mix32;
  void *leafp;     // gaussian/binomial: float2 [R][D][K]; categorical: float [R][D][K][S]
  float *center;   // gaussian: fp32 mean [R][D][K] (centre of the leaf statistics)
  double *cnst;    // [n_leaf][K] fp64 scope constant
  uint8_t *active; // [D] 1 = not marginalised
  double *logh;    // binomial log base measure per count
  double *leafimg; // DMMA leaf forward: B-fragment image [kstep][K/8][32] (padded scopes)
  double *cm2;     // DMMA leaf forward: [n_leaf][K] sum of squared centred offsets
};

struct WsView {
  float *off;      // [slab][Bc/32][KS][32] (32-sample transposed blocks, tb_idx)
  double *shift;   // [slab][Bc]
  float *slots;    // [slot][Bc/32][KS][32]
  double *leafpart;
  float *ea, *eb;  // [row][Bc][K]
  float *rt;       // [row][Bc/32][KS][32]
  float *ebm;      // tcgen05 A operand EB: [einsum row][Bc/128][hi|lo][128 x kp] bf16 (K-major core matrices)
  float *rhob;     // tcgen05 B operand rho^T of the leaf statistics: [leaf][Bc/32][hi|lo][nn x 32]
  float *rtb;      // tcgen05 B operand RT^T of the W statistics: [row][Bc/32][hi|lo][nn x 32]
  float *eam;      // tcgen05 A operand EA (direct child-rho of K_out == 1 rows), as ebm
  float *rtm;      // tcgen05 A operand RT: [row][Bc/128][hi|lo][128 x kob] bf16
  double *wpart;
  float *rho;      // [leaf][Bc][K]
  double *lspart;
  double *ppart;
  double *mixpart;
  double *llpart;
  int64_t bc;
  int ks;
};

inline CompView comp_view(const Plan &p, const uint8_t *c) {
  CompView v;
  uint8_t *b = const_cast<uint8_t *>(c);
  v.w32 = (float *)(b + p.c_w32);
  v.mix32 = (float *)(b + p.c_mix32);
  v.leafp = (void *)(b + p.c_leafp);
  v.center = (float *)(b + p.c_center);
  v.cnst = (double *)(b + p.c_const);
  v.active = (uint8_t *)(b + p.c_active);
  v.logh = (double *)(b + p.c_logh);
  v.leafimg = (double *)(b + p.c_leafimg);
  v.cm2 = (double *)(b + p.c_cm2);
  return v;
}

inline WsView ws_view(const Plan &p, const uint8_t *w) {
  WsView v;
  uint8_t *b = const_cast<uint8_t *>(w);
  v.off = (float *)(b + p.w_off);
  v.shift = (double *)(b + p.w_shift);
  v.slots = (float *)(b + p.w_slots);
  v.leafpart = (double *)(b + p.w_leafpart);
  v.ea = (float *)(b + p.w_ea);
  v.eb = (float *)(b + p.w_eb);
  v.rt = (float *)(b + p.w_rt);
  v.ebm = (float *)(b + p.w_ebm);
  v.rtm = (float *)(b + p.w_rtm);
  v.eam = (float *)(b + p.w_eam);
  v.rtb = (float *)(b + p.w_rtb);
  v.rhob = (float *)(b + p.w_rhob);
  v.wpart = (double *)(b + p.w_wpart);
  v.rho = (float *)(b + p.w_rho);
  v.lspart = (double *)(b + p.w_lspart);
  v.ppart = (double *)(b + p.w_ppart);
  v.mixpart = (double *)(b + p.w_mixpart);
  v.llpart = (double *)(b + p.w_llpart);
  v.bc = p.bc;
  v.ks = p.ks;
  return v;
}

// Per-sample vectors EA, EB, RT and the leaf responsibilities live in 32-sample
// transposed blocks: entry i of sample b in row l of a width-W array is at
//   (l*bc + b - b%32)*W + i*32 + b%32      (bc is a multiple of 32)
// so one block is a contiguous [W][32] tile (a batch-reduction GEMM stages it
// with 16-byte copies) and per-sample loops read coalesced across a warp.
__device__ __forceinline__ int64_t tb_idx(int64_t l, int64_t b, int i, int64_t bc, int W) {
  return (l * bc + (b & ~31LL)) * W + (int64_t)i * 32 + (b & 31);
}

// The normalised child exponentials EA / EB use the same 32-sample blocks with
// each entry row padded to EV_ROW floats: a block [K][EV_ROW] is contiguous, so
// one bulk copy lands it in shared memory where 32 threads reading one 16-byte
// chunk of 32 consecutive rows hit 8 distinct bank groups.
__device__ __host__ __forceinline__ int64_t ev_idx(int64_t l, int64_t b, int i, int64_t bc, int K) {
  return (l * (bc >> 5) + (b >> 5)) * ((int64_t)K * EV_ROW) + (int64_t)i * EV_ROW + (b & 31);
}

// One sample's entries of a slab or slot: entry k of sample b lives at
// tb_idx(slab, b, k, bc, ks), i.e. stride 32 floats, so a warp of consecutive
// samples touching entry k reads or writes one contiguous 128-byte line.
struct Col32 {
  float *p;
  __device__ __forceinline__ float &operator[](int k) const { return p[(int64_t)k * 32]; }
};
__device__ __forceinline__ Col32 slab_off(const WsView &w, int slab, int64_t b) {
  return Col32{w.off + tb_idx(slab, b, 0, w.bc, w.ks)};
}
__device__ __forceinline__ double *slab_shift(const WsView &w, int slab) {
  return w.shift + (int64_t)slab * w.bc;
}
__device__ __forceinline__ Col32 slot_ptr(const WsView &w, int slot, int64_t b) {
  return Col32{w.slots + tb_idx(slot, b, 0, w.bc, w.ks)};
}

// Responsibility of slab `slab` for sample b, entry k: ordered sum of its
// contribution slots (deterministic stand-in for np.add.at), or 1 at the root.
__device__ __forceinline__ float gather_rho(const WsView &w, const int *csr_off,
                                            const int *csr_slot, const uint8_t *ones,
                                            int slab, int64_t b, int k) {
  if (ones[slab]) return 1.0f;
  float acc = 0.0f;
  const int e = csr_off[slab + 1];
  for (int q = csr_off[slab]; q < e; ++q) acc += slot_ptr(w, csr_slot[q], b)[k];
  return acc;
}

__device__ __forceinline__ bool is_nan_f(float v) { return v != v; }

// tcgen05 A-operand tiles of per-sample vectors (width W, multiple of 4):
// 128-sample tile t holds the truncated-TF32 part then the fp32 remainder,
// each 128 x W in the K-major no-swizzle core-matrix layout (8 samples x 4
// entries = 128 contiguous bytes). Float index of (sample b, entries 4q..4q+3)
// in the hi part; the lo part is + 128 * W.
__device__ __forceinline__ int64_t mt_idx(int64_t row, int64_t b, int q, int64_t ntl, int W) {
  const int r = (int)(b & 127);
  return ((row * ntl + (b >> 7)) * 2) * (128LL * W) + q * 512 + (r >> 3) * 32 + (r & 7) * 4;
}
// hi = tf32(x) rounded to nearest (cvt.rna), lo = x - hi (exact in fp32; the
// tensor core truncates it to TF32). Round-to-nearest keeps the sign of lo
// random, so the truncation errors of the lo products do not accumulate with
// one sign over long batch reductions (a truncated hi would make every lo
// positive: a 2^-20 relative bias that the leaf statistics' un-centring
// exposes as an absolute error, profiles/r01_s2_profile.md).
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}
__device__ __forceinline__ void store_hilo4_at(float *hi, int64_t lo_off, float4 v) {
  float4 h, l;
  h.x = tf32_rn(v.x);
  h.y = tf32_rn(v.y);
  h.z = tf32_rn(v.z);
  h.w = tf32_rn(v.w);
  l.x = v.x - h.x;
  l.y = v.y - h.y;
  l.z = v.z - h.z;
  l.w = v.w - h.w;
  *(float4 *)hi = h;
  *(float4 *)(hi + lo_off) = l;
}
__device__ __forceinline__ void store_hilo4(float *hi, int W, float4 v) {
  store_hilo4_at(hi, 128LL * W, v);
}

// A 32-sample block [n][32] (rows n < nvalid, written by this CTA before a
// __syncthreads) as a tcgen05 B operand: rows n < nn, K = 32 samples, hi | lo,
// K-major core matrices. Rows n >= nvalid are zero.
__device__ __forceinline__ void bt_tile(const float *src, float *dst, int nvalid, int nn) {
  for (int e = threadIdx.x; e < nn * 8; e += blockDim.x) {
    const int n = e >> 3, q = e & 7;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n < nvalid) v = *(const float4 *)(src + n * 32 + 4 * q);
    store_hilo4_at(dst + q * (nn * 4) + (n >> 3) * 32 + (n & 7) * 4, nn * 32, v);
  }
}

// bf16 A-operand tiles of per-sample vectors (3xBF16 contraction kernels):
// 128-sample tile t of row `row` holds the bf16 hi part then the lo part, each
// 128 x W (W a multiple of 16) in K-major core matrices (tc::kmaj_off16).
// Stores entries 4q..4q+3 of sample b (8 bytes per part).
__device__ __forceinline__ void store_bf16_quad(void *base, int64_t row, int64_t b, int q,
                                                int64_t ntl, int W, float4 v) {
  uint8_t *tile = (uint8_t *)base + ((row * ntl + (b >> 7)) * 4) * (128LL * W);
  const int r = (int)(b & 127), k = 4 * q;
  const uint32_t off = (uint32_t)((k >> 3) * (128 * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
  const __nv_bfloat162 h01 = __floats2bfloat162_rn(v.x, v.y), h23 = __floats2bfloat162_rn(v.z, v.w);
  const __nv_bfloat162 l01 = __floats2bfloat162_rn(v.x - __low2float(h01), v.y - __high2float(h01));
  const __nv_bfloat162 l23 = __floats2bfloat162_rn(v.z - __low2float(h23), v.w - __high2float(h23));
  uint2 hv, lv;
  hv.x = *(const uint32_t *)&h01;
  hv.y = *(const uint32_t *)&h23;
  lv.x = *(const uint32_t *)&l01;
  lv.y = *(const uint32_t *)&l23;
  *(uint2 *)(tile + off) = hv;
  *(uint2 *)(tile + 2LL * 128 * W + off) = lv;
}

// bf16 variant of bt_tile (the W-statistics B operand RT^T): rows n < nn,
// K = 32 samples, bf16 hi | lo (tc::kmaj_off16 layout, 8 samples per 16-byte
// core-matrix row); rows n >= nvalid are zero.
__device__ __forceinline__ void bt_tile16(const float *src, uint8_t *dst, int nvalid, int nn) {
  for (int e = threadIdx.x; e < nn * 4; e += blockDim.x) {
    const int n = e >> 2, q = e & 3;  // samples 8q .. 8q+7
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (n < nvalid) {
      const float4 a = *(const float4 *)(src + n * 32 + 8 * q);
      const float4 b = *(const float4 *)(src + n * 32 + 8 * q + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) tc::split_bf16x2(v[2 * u], v[2 * u + 1], h[u], l[u]);
    const uint32_t off = (uint32_t)(q * (nn * 16) + (n >> 3) * 128 + (n & 7) * 16);
    *(uint4 *)(dst + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *(uint4 *)(dst + nn * 64 + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

// cp.async (LDGSTS) helpers shared by the staged kernels
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// INT8 leaf forward (leaf_i8.cu): the three coefficients of (variable d,
// component k) from lp = (sa, -mu sa), and the column scale 2^(E-8) with
// max |G| * 2^(8-E) <= 127 (1 when the column is empty).
__device__ __forceinline__ void i8_coefs(double2 q, double &gu, double &gh, double &gl) {
  const double a = q.x * q.x;
  gu = 2.0 * q.x * q.y / 255.0;
  gh = a * (256.0 / 65025.0);
  gl = a / 65025.0;
}
__device__ __forceinline__ double i8_scale(double m) {
  double scale = 1.0;
  if (m > 0.0 && isfinite(m)) {
    int e;
    frexp(m * (256.0 / 127.0), &e);
    while (m * ldexp(1.0, 8 - e) > 127.0) ++e;
    scale = ldexp(1.0, e - 8);
  }
  return scale;
}

}  // namespace einet
