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
                                                       uint32_t tcols, int a_in_tmem) {
  EINET_KERNEL_PROLOGUE();
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
  if (a_in_tmem) {
    // A_hi at columns [256, 256+K), A_lo at [256+K, 256+2K) (lane = row)
    const uint32_t ta = tm + 256 + ((uint32_t)(32 * (t >> 5)) << 16);
    for (int c = 0; c < K; c += 16) {
      float h[16], l[16];
      for (int u = 0; u < 16; ++u) {
        const float v = c + u < K ? A[t * K + c + u] : 0.f;
        tc::split_tf32(v, h[u], l[u]);
      }
      tc::tmem_st16(ta + c, h);
      tc::tmem_st16(ta + K + c, l);
    }
    tc::tmem_wait_st();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
      const uint32_t id = tc::idesc_tf32(128, N);
      const uint32_t sb = tc::smem_u32(bhi), sbl = tc::smem_u32(blo);
      for (int s = 0; s < K / 8; ++s) {
        const uint32_t ah = tm + 256 + 8 * s, al = tm + 256 + K + 8 * s;
        tc::mma_tf32_ts(tm, ah, tc::kstep_desc(sb, N, s), id, s > 0);
        tc::mma_tf32_ts(tm, ah, tc::kstep_desc(sbl, N, s), id, 1);
        tc::mma_tf32_ts(tm, al, tc::kstep_desc(sb, N, s), id, 1);
      }
      tc::mma_commit(&bar);
    }
  } else if (t == 0) {
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
  const int a_tmem = N < 0;
  if (a_tmem) N = -N;
  if (N < 16 || N > 256 || N % 16 || K < 8 || K % 8 || (a_tmem && 2 * K > 256))
    return fail(EINET_ERR_USAGE, "selftest gemm: N in [16,256] multiple of 16, K multiple of 8");
  uint32_t cols = a_tmem ? 512 : 32;
  while (cols < (uint32_t)N) cols *= 2;
  const size_t smem = sizeof(float) * 2 * (128 + N) * K;
  cudaFuncSetAttribute(k_selftest_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(k_selftest_gemm, 1, 128, smem, st, A, B, D, N, K, cols, a_tmem);
  count_launch();
  return check_cuda(cudaGetLastError(), "selftest gemm");
}

// ===========================================================================
// production EinsumLayer kernels
// ===========================================================================

constexpr int TC_M = 128;                    // batch (or (i,j)) rows per MMA tile
constexpr int64_t TC_SMEM_MAX = 220 * 1024;  // dynamic smem budget per CTA

static inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// contraction kernel (contract_tc.cu, 3xBF16): resident weight chunk (bf16
// hi | lo), at least two A stages and two contraction-vector stages
static int64_t fwd_smem(int rows_tile, int K, int kp) {
  return 4LL * rows_tile * kp + 2LL * 4 * TC_M * kp + 2LL * 4 * K * EV_ROW * 4 + 1024;
}
static int64_t cr_smem(int rows_tile, int kob, int K) {
  return 4LL * rows_tile * kob + 2LL * 4 * TC_M * kob + 2LL * 4 * K * EV_ROW * 4 + 1024;
}
size_t wstats_smem(int K, int nn);  // wstats_tc.cu
static int64_t ws_smem(int K, int nn) { return (int64_t)wstats_smem(K, nn); }

size_t contract_big_smem(int K, int ka, int64_t tile_bytes);  // contract_big.cu

void plan_tc_tiling(Plan &p) {
  const int K = p.k;
  p.kp = round_up(K, 16);
  const int kp = p.kp;
  // large K (96, 128): one output per weight chunk, tile-stationary kernel
  // (contract_big.cu) streaming the chunks
  const bool big = K == 96 || K == 128;
  for (auto &L : p.layers) {
    L.tc = 0;
    if (L.kind != EINET_LAYER_EINSUM) continue;
    // K multiple of 8 up to 64, and K = 10, 20 (BASELINE configs C1, C2, C5):
    // the MMA K dimension is padded to 16 with zero operand entries
    if (!((K % 8 == 0 && K >= 8 && K <= 64) || K == 10 || K == 20 || big)) continue;
    const int Ko = L.k_out;
    int kg = big ? 1 : std::max(1, std::min(Ko, 256 / K));
    while (kg > 1 && fwd_smem(round_up(kg * K, 16), K, kp) > TC_SMEM_MAX) --kg;
    L.kg = kg;
    L.ng = ceil_div(Ko, kg);
    L.fw_rows = round_up(kg * K, 16);
    L.fw_tile = 4LL * L.fw_rows * kp;
    L.kob = round_up(Ko, 16);
    int ig = big ? 1 : std::max(1, std::min(K, 256 / K));
    while (ig > 1 && cr_smem(round_up(ig * K, 16), L.kob, K) > TC_SMEM_MAX) --ig;
    L.ig = ig;
    L.ni = ceil_div(K, ig);
    L.uw_rows = round_up(ig * K, 16);
    L.uw_tile = 4LL * L.uw_rows * L.kob;
    L.nn = round_up(Ko, 16);
    L.direct = Ko == 1;
    L.rw_rows = round_up(K, 16);
    L.rw_tile = 4LL * L.rw_rows * kp;
    if (L.fw_rows > 256 || L.uw_rows > 256 || L.nn > 128 || L.kob > 256) continue;
    if (big) {
      if (kp % 32 || (!L.direct && L.kob % 32) ||
          (int64_t)contract_big_smem(K, kp, L.fw_tile) > TC_SMEM_MAX ||
          (!L.direct && (int64_t)contract_big_smem(K, L.kob, L.uw_tile) > TC_SMEM_MAX) ||
          ws_smem(K, L.nn) > TC_SMEM_MAX)
        continue;
    } else if (L.nn > 64 || fwd_smem(L.fw_rows, K, kp) > TC_SMEM_MAX ||
               cr_smem(L.uw_rows, L.kob, K) > TC_SMEM_MAX || ws_smem(K, L.nn) > TC_SMEM_MAX) {
      continue;
    }
    L.tc = 1;
  }
}

// --- pre-tiled weight images (built by prepare after every parameter change) ---
// bf16 hi | lo, K-major core matrices (kmaj_off16), K dims padded to 16 with zeros.
// forward tile g of row l: rows n = kl*K + i (k = g*kg + kl), K dim = j (kp)
// child-rho tile h of row l: rows n = il*K + j (i = h*ig + il), K dim = k (kob)
// right child-rho tile h of row l: rows n = jl*K + i (j = h*ig + jl), K dim = k
// direct right tile of a K_out == 1 row: rows n = j, K dim = i (kp)
//
// Every tensor-core weight image of every layer from the fp32 weights, in
// tile order: one thread per (tile, K chunk of 8, row) writes the chunk's 8
// bf16 hi and 8 lo values as two 16-byte stores (consecutive threads:
// consecutive rows = consecutive 16-byte slots of a core-matrix column), zero
// padding included; one launch for all layers (item ranges in the tile descriptors).
__global__ void __launch_bounds__(256) k_build_tiles_all(const float *__restrict__ w32,
                                                         const int64_t *__restrict__ td, int ntd,
                                                         int64_t n_items, uint8_t *compute,
                                                         int K, int kp) {
  EINET_KERNEL_PROLOGUE();
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < ntd && td[(q + 1) * TD_WORDS + TD_IT0] <= it) ++q;
    const int64_t *d = td + (int64_t)q * TD_WORDS;
    const float *W = w32 + d[TD_WOFF];
    const int Ko = (int)d[TD_KO];
    int64_t r = it - d[TD_IT0];
    const int64_t nfw = d[TD_NFW], nuw = d[TD_NUW];
    float v[8];
    uint8_t *tile;
    int rows, kdim, row, kc;
    if (r < nfw) {  // forward: rows kl*K + i, K dim j
      rows = (int)d[TD_FW_ROWS];
      kdim = kp;
      row = (int)(r % rows);
      r /= rows;
      kc = (int)(r % (kdim / 8));
      const int64_t t = r / (kdim / 8);  // l * ng + g
      const int ng = (int)d[TD_NG], kg = (int)d[TD_KG];
      const int l = (int)(t / ng), g = (int)(t % ng);
      const int kl = row / K, i = row % K, k = g * kg + kl;
      tile = compute + d[TD_FW_OFF] + t * d[TD_FW_TILE];
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const int j = kc * 8 + z;
        v[z] = (kl < kg && k < Ko && j < K) ? W[(((int64_t)l * Ko + k) * K + i) * K + j] : 0.f;
      }
    } else if (r < nfw + 2 * nuw) {  // child-rho: left rows il*K + j, right jl*K + i; K dim k
      const bool right = r >= nfw + nuw;
      r -= right ? nfw + nuw : nfw;
      rows = (int)d[TD_UW_ROWS];
      kdim = (int)d[TD_KOB];
      row = (int)(r % rows);
      r /= rows;
      kc = (int)(r % (kdim / 8));
      const int64_t t = r / (kdim / 8);  // l * ni + h
      const int ni = (int)d[TD_NI], ig = (int)d[TD_IG];
      const int l = (int)(t / ni), h = (int)(t % ni);
      const int ol = row / K, in = row % K, o = h * ig + ol;
      const int i = right ? in : o, j = right ? o : in;
      tile = compute + (right ? d[TD_VW_OFF] : d[TD_UW_OFF]) + t * d[TD_UW_TILE];
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const int kk = kc * 8 + z;
        v[z] = (ol < ig && o < K && kk < Ko) ? W[(((int64_t)l * Ko + kk) * K + i) * K + j] : 0.f;
      }
    } else {  // K_out == 1: right tile rows j, K dim i
      r -= nfw + 2 * nuw;
      rows = (int)d[TD_RW_ROWS];
      kdim = kp;
      row = (int)(r % rows);
      r /= rows;
      kc = (int)(r % (kdim / 8));
      const int64_t l = r / (kdim / 8);
      tile = compute + d[TD_VW_OFF] + l * d[TD_RW_TILE];
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const int i = kc * 8 + z;
        v[z] = (row < K && i < K) ? W[((int64_t)l * K + i) * K + row] : 0.f;
      }
    }
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) tc::split_bf16x2(v[2 * z], v[2 * z + 1], hv[z], lv[z]);
    const uint32_t off = tc::kmaj_off16(row, kc * 8, rows);
    *(uint4 *)(tile + off) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    *(uint4 *)(tile + 2LL * rows * kdim + off) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
  }
}

int launch_build_tiles_all(Plan &p, uint8_t *compute, cudaStream_t st) {
  if (p.n_tile_items == 0) return 0;
  CompView c = comp_view(p, compute);
  launch_k(k_build_tiles_all, (int)std::min<int64_t>((p.n_tile_items + 255) / 256, 4 * p.num_sms),
           256, 0, st, (const float *)c.w32, (const int64_t *)p.d_tiledesc, p.n_tiledesc,
           p.n_tile_items, compute, p.k, p.kp);
  count_launch();
  return check_cuda(cudaGetLastError(), "build tc tiles");
}

int launch_prepare_tc_tiles(Plan &p, uint8_t *compute, cudaStream_t st) {
  return launch_build_tiles_all(p, compute, st);
}

__device__ __forceinline__ void store_split4(float *hi, float *lo, float4 v) {
  float4 h, l;
  tc::split_tf32(v.x, h.x, l.x);
  tc::split_tf32(v.y, h.y, l.y);
  tc::split_tf32(v.z, h.z, l.z);
  tc::split_tf32(v.w, h.w, l.w);
  *(float4 *)hi = h;
  *(float4 *)lo = l;
}

// Issue the 3xTF32 MMAs of one (M=128) x N tile over ksteps K-steps.
__device__ __forceinline__ void mma_3xtf32(uint32_t d, uint32_t a_hi, uint32_t a_lo, int a_rows,
                                           uint32_t b_hi, uint32_t b_lo, int b_rows, int N,
                                           int ksteps, bool accumulate_first) {
  const uint32_t id = tc::idesc_tf32(TC_M, N);
  for (int s = 0; s < ksteps; ++s) {
    const uint64_t ah = tc::kstep_desc(a_hi, a_rows, s), al = tc::kstep_desc(a_lo, a_rows, s);
    const uint64_t bh = tc::kstep_desc(b_hi, b_rows, s), bl = tc::kstep_desc(b_lo, b_rows, s);
    tc::mma_tf32(d, ah, bh, id, (s > 0 || accumulate_first) ? 1u : 0u);
    tc::mma_tf32(d, ah, bl, id, 1u);
    tc::mma_tf32(d, al, bh, id, 1u);
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

#define EINET_TC_DISPATCH(FN, ...)                         \
  switch (p.k) {                                           \
    case 8: return FN<8>(__VA_ARGS__);                     \
    case 16: return FN<16>(__VA_ARGS__);                   \
    case 24: return FN<24>(__VA_ARGS__);                   \
    case 32: return FN<32>(__VA_ARGS__);                   \
    case 40: return FN<40>(__VA_ARGS__);                   \
    case 48: return FN<48>(__VA_ARGS__);                   \
    case 56: return FN<56>(__VA_ARGS__);                   \
    case 64: return FN<64>(__VA_ARGS__);                   \
    default: return fail(EINET_ERR_USAGE, "tc path: unsupported k"); \
  }

}  // namespace einet
