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
  k_selftest_gemm<<<1, 128, smem, st>>>(A, B, D, N, K, cols, a_tmem);
  count_launch();
  return check_cuda(cudaGetLastError(), "selftest gemm");
}

// ===========================================================================
// production EinsumLayer kernels
// ===========================================================================

constexpr int TC_M = 128;                    // batch (or (i,j)) rows per MMA tile
constexpr int64_t TC_SMEM_MAX = 200 * 1024;  // dynamic smem budget per CTA
constexpr int WS_STAGE = 32;                 // samples per W-statistics MMA stage
constexpr int WS_DRAIN = 8;                  // stages accumulated in TMEM before fp64 drain

static inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

static int64_t fwd_smem(int rows_tile, int K) {
  return 2LL * rows_tile * K * 4 + 2LL * 2 * TC_M * K * 4;
}
static int64_t cr_smem(int rows_tile, int ko8) {
  return 2LL * TC_M * ko8 * 4 + 2LL * (2LL * rows_tile * ko8 * 4);
}
static int64_t ws_smem(int K, int nn) {  // W-statistics kernel (staging + B tile)
  return 2LL * (2 * K + nn) * WS_STAGE * 4 + 2LL * nn * WS_STAGE * 4;
}

void plan_tc_tiling(Plan &p) {
  const int K = p.k;
  for (auto &L : p.layers) {
    L.tc = 0;
    if (L.kind != EINET_LAYER_EINSUM) continue;
    if (K % 8 != 0 || K < 8 || K > 64 || p.ks % 4 != 0) continue;
    const int Ko = L.k_out;
    int kg = std::max(1, std::min(Ko, 256 / K));
    while (kg > 1 && fwd_smem(round_up(kg * K, 16), K) > TC_SMEM_MAX) --kg;
    L.kg = kg;
    L.ng = ceil_div(Ko, kg);
    L.fw_rows = round_up(kg * K, 16);
    L.fw_tile = 2LL * L.fw_rows * K * 4;
    L.ko8 = round_up(Ko, 8);
    int ig = std::max(1, std::min(K, 256 / K));
    while (ig > 1 && cr_smem(round_up(ig * K, 16), L.ko8) > TC_SMEM_MAX) --ig;
    L.ig = ig;
    L.ni = ceil_div(K, ig);
    L.uw_rows = round_up(ig * K, 16);
    L.uw_tile = 2LL * L.uw_rows * L.ko8 * 4;
    L.nn = round_up(Ko, 16);
    if (L.fw_rows > 256 || L.uw_rows > 256 || L.nn > 64 || L.ko8 > 256) continue;
    if (fwd_smem(L.fw_rows, K) > TC_SMEM_MAX || cr_smem(L.uw_rows, L.ko8) > TC_SMEM_MAX ||
        ws_smem(K, L.nn) > TC_SMEM_MAX)
      continue;
    L.tc = 1;
  }
}

// --- pre-tiled weight images (built by prepare after every parameter change) ---
// forward tile g of row l: rows n = kl*K + i (k = g*kg + kl), K dim = j
// child-rho tile h of row l: rows n = il*K + j (i = h*ig + il), K dim = k
__global__ void k_build_tiles(const float *__restrict__ W, uint8_t *fw, uint8_t *uw, int L,
                              int Ko, int K, int kg, int ng, int fw_rows, int ig, int ni,
                              int uw_rows, int ko8) {
  const int64_t n_fw = (int64_t)L * ng * fw_rows * K;
  const int64_t n_uw = (int64_t)L * ni * uw_rows * ko8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_fw + n_uw;
       e += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    float *hi, *lo;
    if (e < n_fw) {
      const int kk = (int)(e % K);
      const int n = (int)((e / K) % fw_rows);
      const int64_t tile = e / ((int64_t)K * fw_rows);  // l * ng + g
      const int l = (int)(tile / ng), g = (int)(tile % ng);
      const int kl = n / K, i = n % K, k = g * kg + kl;
      if (kl < kg && k < Ko) v = W[(((int64_t)l * Ko + k) * K + i) * K + kk];
      float *base = (float *)(fw + tile * (2LL * fw_rows * K * 4));
      hi = base + tc::kmaj_off(n, kk, fw_rows) / 4;
      lo = hi + fw_rows * K;
    } else {
      const int64_t q = e - n_fw;
      const int kk = (int)(q % ko8);
      const int n = (int)((q / ko8) % uw_rows);
      const int64_t tile = q / ((int64_t)ko8 * uw_rows);  // l * ni + h
      const int l = (int)(tile / ni), h = (int)(tile % ni);
      const int il = n / K, j = n % K, i = h * ig + il;
      if (il < ig && i < K && kk < Ko) v = W[(((int64_t)l * Ko + kk) * K + i) * K + j];
      float *base = (float *)(uw + tile * (2LL * uw_rows * ko8 * 4));
      hi = base + tc::kmaj_off(n, kk, uw_rows) / 4;
      lo = hi + uw_rows * ko8;
    }
    float h, l2;
    tc::split_tf32(v, h, l2);
    *hi = h;
    *lo = l2;
  }
}

int launch_prepare_tc_tiles(Plan &p, uint8_t *compute, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  for (auto &L : p.layers) {
    if (!L.tc) continue;
    const int64_t n = (int64_t)L.rows * (L.ng * L.fw_rows * p.k + L.ni * L.uw_rows * L.ko8);
    k_build_tiles<<<(int)std::min<int64_t>((n + 255) / 256, 8192), 256, 0, st>>>(
        c.w32 + L.w_off, compute + L.fw_off, compute + L.uw_off, L.rows, L.k_out, p.k, L.kg,
        L.ng, L.fw_rows, L.ig, L.ni, L.uw_rows, L.ko8);
    count_launch();
  }
  return check_cuda(cudaGetLastError(), "build tc tiles");
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

// ---- forward: T[b,(kl,i)] = sum_j EB[b,j] W[k,i,j]; out[b,k] = log sum_i EA[b,i] T ----
// grid (ng, L, bsplit), block 128; weights of (l, g) arrive by one bulk copy.
template <int K>
__global__ void __launch_bounds__(128, 1) k_einsum_fwd_tc(
    const float *__restrict__ EA, const float *__restrict__ EB, WsView ws,
    const int *__restrict__ out_slab, const uint8_t *__restrict__ tiles, int64_t tile_bytes,
    int ng, int kg, int rows_tile, int Ko, int64_t B, int tiles_per_split) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[3];
  __shared__ uint32_t tbase;
  const int g = blockIdx.x, l = blockIdx.y;
  const int t = threadIdx.x, w = t >> 5;
  float *wt = (float *)sm;
  float *abuf = (float *)(sm + tile_bytes);
  const int nk = min(kg, Ko - g * kg);
  const int nmma = (nk * K + 15) / 16 * 16;
  const int64_t nbt = (B + TC_M - 1) / TC_M;
  const int64_t j0 = (int64_t)blockIdx.z * tiles_per_split;
  const int64_t j1 = min(nbt, j0 + tiles_per_split);
  if (w == 0) tc::tmem_alloc(&tbase, 512);
  if (t == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::mbar_init(&bars[2], 1);
    tc::mbar_fence_init();
    tc::mbar_arrive_expect_tx(&bars[0], (uint32_t)tile_bytes);
    tc::bulk_g2s(wt, tiles + ((int64_t)l * ng + g) * tile_bytes, (uint32_t)tile_bytes, &bars[0]);
  }
  auto build = [&](int buf, int64_t jt) {
    const int64_t b = jt * TC_M + t;
    const bool ok = b < B;
    const float *src = EB + tb_idx(l, ok ? b : 0, 0, ws.bc, K);
    float *ahi = abuf + buf * 2 * TC_M * K;
    float *alo = ahi + TC_M * K;
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) v = make_float4(src[(4 * q) * 32], src[(4 * q + 1) * 32], src[(4 * q + 2) * 32],
                              src[(4 * q + 3) * 32]);
      const uint32_t o = tc::kmaj_off(t, 4 * q, TC_M) / 4;
      store_split4(ahi + o, alo + o, v);
    }
  };
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  if (j0 < j1) build(0, j0);
  int it = 0;
  for (int64_t jt = j0; jt < j1; ++jt, ++it) {
    const int buf = it & 1;
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
      if (it == 0) tc::mbar_wait(&bars[0], 0);
      const uint32_t ah = tc::smem_u32(abuf + buf * 2 * TC_M * K);
      const uint32_t bh = tc::smem_u32(wt);
      mma_3xtf32(tm + buf * 256, ah, ah + TC_M * K * 4, TC_M, bh, bh + rows_tile * K * 4,
                 rows_tile, nmma, K / 8, false);
      tc::mma_commit(&bars[1 + buf]);
    }
    if (jt + 1 < j1) build(buf ^ 1, jt + 1);
    tc::mbar_wait(&bars[1 + buf], (it >> 1) & 1);
    tc::fence_after();
    const int64_t b = jt * TC_M + t;
    const bool live = b < B;
    float ea[K];
    {
      const float *src = EA + tb_idx(l, live ? b : 0, 0, ws.bc, K);
#pragma unroll
      for (int i = 0; i < K; ++i) ea[i] = live ? src[i * 32] : 0.f;
    }
    const uint32_t ta = tm + buf * 256 + ((uint32_t)(32 * w) << 16);
    const Col32 o = slab_off(ws, out_slab[l], live ? b : 0);
    for (int kl = 0; kl < nk; ++kl) {
      float v[K];
#pragma unroll
      for (int q = 0; q < K / 8; ++q) {
        float c8[8];
        tc::tmem_ld8(ta + kl * K + 8 * q, c8);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[8 * q + u] = c8[u];
      }
      tc::tmem_wait_ld();
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < K; ++i) a4[i & 3] = fmaf(v[i], ea[i], a4[i & 3]);
      const float acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      if (live) o[g * kg + kl] = acc > 0.f ? logf(acc) : -CUDART_INF_F;
    }
  }
  if (t == 0 && it == 0) tc::mbar_wait(&bars[0], 0);  // never exit with the copy in flight
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 512);
}

// ---- child responsibilities: U[b,(il,j)] = sum_k RT[b,k] W[k,i,j];
//      left[b,i] = EA_i sum_j U EB_j, right[b,j] = EB_j sum_i U EA_i
// grid (ceil(B/128), L), block 128; weight tiles double-buffered by bulk copies.
template <int K>
__global__ void __launch_bounds__(128, 1) k_einsum_childrho_tc(
    const float *__restrict__ EA, const float *__restrict__ EB, const float *__restrict__ RT,
    WsView ws, const int *__restrict__ slot_left, const int *__restrict__ slot_right,
    const uint8_t *__restrict__ tiles, int64_t tile_bytes, int ni, int ig, int rows_tile,
    int ko8, int Ko, int64_t B) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t wbar[2], mbar[2];
  __shared__ uint32_t tbase;
  const int l = blockIdx.y;
  const int t = threadIdx.x, w = t >> 5;
  float *ahi = (float *)sm;
  float *alo = ahi + TC_M * ko8;
  uint8_t *wbuf = sm + 2LL * TC_M * ko8 * 4;
  const int64_t b = (int64_t)blockIdx.x * TC_M + t;
  const bool live = b < B;
  const int64_t bsafe = live ? b : 0;
  const uint8_t *ltiles = tiles + (int64_t)l * ni * tile_bytes;
  if (w == 0) tc::tmem_alloc(&tbase, 512);
  if (t == 0) {
    for (int q = 0; q < 2; ++q) {
      tc::mbar_init(&wbar[q], 1);
      tc::mbar_init(&mbar[q], 1);
    }
    tc::mbar_fence_init();
    for (int h = 0; h < min(2, ni); ++h) {
      tc::mbar_arrive_expect_tx(&wbar[h], (uint32_t)tile_bytes);
      tc::bulk_g2s(wbuf + h * tile_bytes, ltiles + h * tile_bytes, (uint32_t)tile_bytes,
                   &wbar[h]);
    }
  }
  // A operand: the sample's rho/r row (K dim = k, padded to ko8)
  for (int q = 0; q < ko8 / 4; ++q) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      const float *src = RT + tb_idx(l, b, 4 * q, ws.bc, ws.ks);
      v.x = 4 * q + 0 < Ko ? src[0] : 0.f;
      v.y = 4 * q + 1 < Ko ? src[32] : 0.f;
      v.z = 4 * q + 2 < Ko ? src[64] : 0.f;
      v.w = 4 * q + 3 < Ko ? src[96] : 0.f;
    }
    const uint32_t o = tc::kmaj_off(t, 4 * q, TC_M) / 4;
    store_split4(ahi + o, alo + o, v);
  }
  float eb[K], right[K];
  {
    const float *src = EB + tb_idx(l, bsafe, 0, ws.bc, K);
#pragma unroll
    for (int j = 0; j < K; ++j) eb[j] = live ? src[j * 32] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < K; ++j) right[j] = 0.f;
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t a_hi = tc::smem_u32(ahi), a_lo = tc::smem_u32(alo);
  auto issue = [&](int h) {
    const int hb = h & 1;
    const int nil = min(ig, K - h * ig);
    const int nmma = (nil * K + 15) / 16 * 16;
    tc::mbar_wait(&wbar[hb], (h >> 1) & 1);
    const uint32_t bh = tc::smem_u32(wbuf + hb * tile_bytes);
    mma_3xtf32(tm + hb * 256, a_hi, a_lo, TC_M, bh, bh + rows_tile * ko8 * 4, rows_tile, nmma,
               ko8 / 8, false);
    tc::mma_commit(&mbar[hb]);
  };
  if (t == 0) issue(0);
  const Col32 dl = slot_ptr(ws, slot_left[l], live ? b : 0);
  const float *earow = EA + tb_idx(l, bsafe, 0, ws.bc, K);
  for (int h = 0; h < ni; ++h) {
    const int hb = h & 1;
    tc::mbar_wait(&mbar[hb], (h >> 1) & 1);
    if (t == 0) {
      if (h + 2 < ni) {
        tc::mbar_arrive_expect_tx(&wbar[hb], (uint32_t)tile_bytes);
        tc::bulk_g2s(wbuf + hb * tile_bytes, ltiles + (h + 2) * tile_bytes,
                     (uint32_t)tile_bytes, &wbar[hb]);
      }
      if (h + 1 < ni) issue(h + 1);
    }
    tc::fence_after();
    const int nil = min(ig, K - h * ig);
    const uint32_t ta = tm + hb * 256 + ((uint32_t)(32 * w) << 16);
    for (int il = 0; il < nil; ++il) {
      const int i = h * ig + il;
      float v[K];
#pragma unroll
      for (int q = 0; q < K / 8; ++q) {
        float c8[8];
        tc::tmem_ld8(ta + il * K + 8 * q, c8);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[8 * q + u] = c8[u];
      }
      tc::tmem_wait_ld();
      const float eai = live ? earow[i * 32] : 0.f;
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < K; ++j) {
        l4[j & 3] = fmaf(v[j], eb[j], l4[j & 3]);
        right[j] = fmaf(v[j], eai, right[j]);
      }
      if (live) dl[i] = eai * ((l4[0] + l4[1]) + (l4[2] + l4[3]));
    }
    tc::fence_before();
    __syncthreads();
  }
  if (live) {
    const Col32 dr = slot_ptr(ws, slot_right[l], b);
#pragma unroll
    for (int j = 0; j < K; ++j) dr[j] = eb[j] * right[j];
  }
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 512);
}

// ---- W statistics: S[(i,j), k] = sum_b EA[b,i] EB[b,j] RT[b,k] (M = (i,j) rows) ----
// Per 32-sample block: EA/EB/RT blocks are prefetched with cp.async, the
// outer-product A operand (128 (i,j) rows x 32 samples, hi/lo) is generated in
// registers and written to TMEM with tcgen05.st, the RT^T B tile goes to smem;
// 12 MMAs (4 K-steps x 3xTF32) accumulate in TMEM, drained to fp64 registers
// every WS_DRAIN blocks. 8 warps: warp w and w+4 share TMEM lanes and split the
// 32 samples / accumulator columns. grid (ceil(K^2/128), L, bsplit).
__device__ __forceinline__ void cpa16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int WS_ROW = WS_STAGE + 4;  // padded staging row (floats)

static int64_t ws_smem_v3(int K, int nn, int ko4) {
  return 2LL * (2 * K + ko4) * WS_ROW * 4 + 2LL * nn * WS_STAGE * 4;
}

// hi = x with the low 13 mantissa bits cleared (exact TF32 value), lo = x - hi
// (exact in fp32, |lo| < 2^-10 |x|, truncated to TF32 by the tensor core).
__device__ __forceinline__ void split_trunc(float x, float &hi, float &lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

constexpr int WS_MAX_SAMPLES = 4096;  // per CTA: fp32 TMEM accumulation, one drain

// grid (ceil(ceil(K^2/128)/2), L, bsplit), block 256: warpgroup g (warps 4g..4g+3)
// owns (i,j)-tile 2*blockIdx.x + g; both share the staged block and the B tile.
template <int K>
__global__ void __launch_bounds__(256, 2) k_einsum_wstats_tc(
    const float *__restrict__ EA, const float *__restrict__ EB, const float *__restrict__ RT,
    int64_t Bc, int ks, int Ko, int nn, int64_t B, int bsplit, double *wpart, int L) {
  constexpr int KK = K * K;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int l = blockIdx.y, split = blockIdx.z;
  const int t = threadIdx.x, w = t >> 5, g = t >> 7, r = t & 127;
  const int m = (2 * blockIdx.x + g) * TC_M + r;
  const bool mvalid = m < KK;
  const int mi = mvalid ? m / K : 0, mj = mvalid ? m % K : 0;
  const int ko4 = (Ko + 3) / 4 * 4;
  const int sw = (2 * K + ko4) * WS_ROW;
  float *stg = (float *)sm;                   // [2][EA | EB | RT rows][WS_ROW]
  float *bhi = stg + 2 * sw, *blo = bhi + nn * WS_STAGE;
  const int64_t nblk = (B + WS_STAGE - 1) / WS_STAGE;
  const int64_t per = (nblk + bsplit - 1) / bsplit;
  const int64_t blk0 = split * per, blk1 = min(nblk, blk0 + per);
  const int nstages = (int)max((int64_t)0, blk1 - blk0);
  // TMEM columns: acc tile g at [g*nn, (g+1)*nn), A(hi|lo) of warpgroup g at 128 + 64 g
  if (w == 0) tc::tmem_alloc(&tbase, 256);
  if (t == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  auto prefetch = [&](int q) {
    float *sb = stg + (q & 1) * sw;
    const int64_t b0 = (blk0 + q) * WS_STAGE;
    const float *ga = EA + ((int64_t)l * Bc + b0) * K;
    const float *gb = EB + ((int64_t)l * Bc + b0) * K;
    const float *gr = RT + ((int64_t)l * Bc + b0) * ks;
    const int nchunks = (2 * K + ko4) * (WS_STAGE / 4);
    for (int e = t; e < nchunks; e += 256) {
      const int row = e >> 3, c = (e & 7) * 4;
      const float *src = row < K ? ga + row * 32 + c
                         : row < 2 * K ? gb + (row - K) * 32 + c
                                       : gr + (row - 2 * K) * 32 + c;
      cpa16(sb + row * WS_ROW + c, src);
    }
    cpa_commit();
  };
  if (nstages > 0) prefetch(0);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * (w & 3)) << 16;
  const uint32_t acol = 128 + 64 * g;
  for (int q = 0; q < nstages; ++q) {
    const int qb = q & 1;
    const int nb = (int)min((int64_t)WS_STAGE, B - (blk0 + q) * WS_STAGE);
    if (q + 1 < nstages) {
      prefetch(q + 1);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    float *sb = stg + qb * sw;
    if (nb < WS_STAGE) {  // tail block: samples past the batch contribute exactly 0
      __syncthreads();
      for (int e = t; e < (2 * K + ko4) * WS_STAGE; e += 256)
        if ((e & 31) >= nb) sb[(e >> 5) * WS_ROW + (e & 31)] = 0.f;
    }
    __syncthreads();
    // B tile (RT^T, n = k) shared by both (i,j) tiles; the previous stage's MMAs
    // (which read B and the A columns) must have completed
    if (q >= 1) tc::mbar_wait(&mbar, (q - 1) & 1);
    tc::fence_after();
    for (int e = t; e < nn * (WS_STAGE / 4); e += 256) {
      const int n = e >> 3, c = (e & 7) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < Ko) v = *(const float4 *)(sb + (2 * K + n) * WS_ROW + c);
      float4 h4, l4;
      split_trunc(v.x, h4.x, l4.x);
      split_trunc(v.y, h4.y, l4.y);
      split_trunc(v.z, h4.z, l4.z);
      split_trunc(v.w, h4.w, l4.w);
      const uint32_t o = tc::kmaj_off(n, c, nn) / 4;
      *(float4 *)(bhi + o) = h4;
      *(float4 *)(blo + o) = l4;
    }
    // A: row m's 32 outer products -> TMEM (two 16-column halves, hi and lo)
    {
      const float *ea = sb + mi * WS_ROW, *eb = sb + (K + mj) * WS_ROW;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float hv[16], lv[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 a4 = *(const float4 *)(ea + 16 * half + 4 * u);
          const float4 e4 = *(const float4 *)(eb + 16 * half + 4 * u);
          split_trunc(a4.x * e4.x, hv[4 * u + 0], lv[4 * u + 0]);
          split_trunc(a4.y * e4.y, hv[4 * u + 1], lv[4 * u + 1]);
          split_trunc(a4.z * e4.z, hv[4 * u + 2], lv[4 * u + 2]);
          split_trunc(a4.w * e4.w, hv[4 * u + 3], lv[4 * u + 3]);
        }
        tc::tmem_st16(tm + lane_base + acol + 16 * half, hv);
        tc::tmem_st16(tm + lane_base + acol + 32 + 16 * half, lv);
      }
    }
    tc::tmem_wait_st();
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
      const uint32_t id = tc::idesc_tf32(TC_M, nn);
      const uint32_t bh = tc::smem_u32(bhi), bl = tc::smem_u32(blo);
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
        const uint32_t d = tm + gg * nn, ah = tm + 128 + 64 * gg;
#pragma unroll
        for (int s = 0; s < WS_STAGE / 8; ++s) {
          tc::mma_tf32_ts(d, ah + 8 * s, tc::kstep_desc(bh, nn, s), id, (s > 0 || q > 0) ? 1u : 0u);
          tc::mma_tf32_ts(d, ah + 8 * s, tc::kstep_desc(bl, nn, s), id, 1u);
          tc::mma_tf32_ts(d, ah + 32 + 8 * s, tc::kstep_desc(bh, nn, s), id, 1u);
        }
      }
      tc::mma_commit(&mbar);
    }
  }
  if (nstages > 0) tc::mbar_wait(&mbar, (nstages - 1) & 1);
  tc::fence_after();
  // drain: warpgroup g reads its tile's accumulator rows (lane = row m)
  for (int c = 0; c < nn; c += 8) {
    float v[8];
    tc::tmem_ld8(tm + lane_base + g * nn + c, v);
    tc::tmem_wait_ld();
    if (mvalid && nstages > 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = c + u;
        if (k < Ko) wpart[(((int64_t)split * L + l) * Ko + k) * KK + m] = (double)v[u];
      }
    }
  }
  if (mvalid && nstages == 0)
    for (int k = 0; k < Ko; ++k) wpart[(((int64_t)split * L + l) * Ko + k) * KK + m] = 0.0;
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 256);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <int K>
static int fwd_tc(Plan &p, const LayerPlan &L, const uint8_t *compute, const float *EA,
                  const float *EB, WsView &w, int64_t B, cudaStream_t st) {
  const int64_t smem = fwd_smem(L.fw_rows, K);
  cudaFuncSetAttribute(k_einsum_fwd_tc<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  const int64_t nbt = (B + TC_M - 1) / TC_M;
  const int64_t ctas = (int64_t)L.ng * L.rows;
  int bs = pick_split(ctas, device_slots((const void *)k_einsum_fwd_tc<K>, 128, smem, p.num_sms), 1,
                      (int)std::min<int64_t>(nbt, 1024));
  const int per = (int)((nbt + bs - 1) / bs);
  bs = (int)((nbt + per - 1) / per);
  dim3 grid(L.ng, L.rows, bs);
  k_einsum_fwd_tc<K><<<grid, 128, smem, st>>>(EA, EB, w, L.d_out_slab, compute + L.fw_off,
                                              L.fw_tile, L.ng, L.kg, L.fw_rows, L.k_out, B, per);
  return check_cuda(cudaGetLastError(), "einsum fwd tc");
}

template <int K>
static int cr_tc(Plan &p, const LayerPlan &L, const uint8_t *compute, const float *EA,
                 const float *EB, WsView &w, int64_t B, cudaStream_t st) {
  (void)p;
  const int64_t smem = cr_smem(L.uw_rows, L.ko8);
  cudaFuncSetAttribute(k_einsum_childrho_tc<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  dim3 grid(ceil_div(B, TC_M), L.rows);
  k_einsum_childrho_tc<K><<<grid, 128, smem, st>>>(
      EA, EB, w.rt, w, L.d_slot_left, L.d_slot_right, compute + L.uw_off, L.uw_tile, L.ni,
      L.ig, L.uw_rows, L.ko8, L.k_out, B);
  return check_cuda(cudaGetLastError(), "einsum child-rho tc");
}

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

int launch_einsum_fwd_tc(Plan &p, const LayerPlan &L, const uint8_t *compute, const float *EA,
                         const float *EB, WsView &w, int64_t B, cudaStream_t st) {
  EINET_TC_DISPATCH(fwd_tc, p, L, compute, EA, EB, w, B, st)
}

int launch_einsum_childrho_tc(Plan &p, const LayerPlan &L, const uint8_t *compute,
                              const float *EA, const float *EB, WsView &w, int64_t B,
                              cudaStream_t st) {
  EINET_TC_DISPATCH(cr_tc, p, L, compute, EA, EB, w, B, st)
}

// Batch splits of the W-statistics kernel for a batch of B samples: at most
// WS_MAX_SAMPLES per CTA (one fp32 TMEM accumulation), full waves on the
// resident slots (2 CTAs per SM). With upper_bound the cap of the search is
// returned; it is monotone in B, so the plan sizes the partial buffer with it.
int wstats_tc_bsplit(const Plan &p, const LayerPlan &L, int64_t B, bool upper_bound) {
  const int mpairs = ceil_div(ceil_div((int64_t)p.k * p.k, TC_M), 2);
  const int64_t nblk = (B + WS_STAGE - 1) / WS_STAGE;
  const int64_t ctas = (int64_t)mpairs * L.rows;
  const int64_t slots = 2LL * p.num_sms;
  const int lo = (int)std::min<int64_t>(kMaxBSplit, (nblk + WS_MAX_SAMPLES / WS_STAGE - 1) /
                                                        (WS_MAX_SAMPLES / WS_STAGE));
  const int hi = (int)std::max<int64_t>(
      lo, std::min<int64_t>(std::min<int64_t>(nblk, kMaxBSplit),
                            std::max<int64_t>(4, (8 * slots + ctas - 1) / ctas)));
  if (upper_bound) return hi;
  int bs = pick_split(ctas, slots, lo, hi);
  const int64_t per = (nblk + bs - 1) / bs;
  return (int)((nblk + per - 1) / per);
}

template <int K>
static int ws_tc(Plan &p, const LayerPlan &L, const float *EA, const float *EB, WsView &w,
                 int64_t B, int *bsplit, cudaStream_t st) {
  const int mpairs = ceil_div(ceil_div((int64_t)K * K, TC_M), 2);
  const int bs = wstats_tc_bsplit(p, L, B, false);
  const int64_t smem = ws_smem_v3(K, L.nn, (L.k_out + 3) / 4 * 4);
  cudaFuncSetAttribute(k_einsum_wstats_tc<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  dim3 grid(mpairs, L.rows, bs);
  k_einsum_wstats_tc<K><<<grid, 256, smem, st>>>(EA, EB, w.rt, w.bc, w.ks, L.k_out, L.nn, B, bs,
                                                 w.wpart, L.rows);
  *bsplit = bs;
  return check_cuda(cudaGetLastError(), "einsum wstats tc");
}

int launch_einsum_wstats_tc(Plan &p, const LayerPlan &L, const float *EA, const float *EB,
                            WsView &w, int64_t B, int *bsplit, cudaStream_t st) {
  EINET_TC_DISPATCH(ws_tc, p, L, EA, EB, w, B, bsplit, st)
}

}  // namespace einet
