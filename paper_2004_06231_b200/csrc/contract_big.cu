// tcgen05 EinsumLayer contraction for large K (96, 128; BASELINE configs[4]
// sweeps K up to 128): the same three contractions as contract_tc.cu
// (forward, left / right child responsibilities, 3xBF16 on round-to-nearest
// bf16 hi/lo splits, fp32 accumulation), with one output per chunk (N = K
// accumulator columns) and the roles of the operands swapped:
//
//   * tile-stationary: a job is one (einsum row, 128-sample tile); its A tile
//     (the K-wide bf16 hi | lo operand, 2 x 32 KB at K = 128) and its
//     contraction-vector tile (EA or EB, [4][K][EV_ROW] fp32, 73.7 KB) are
//     loaded once and stay resident while the CTA runs every output chunk;
//   * the weights stream: each chunk's image (N = K rows x K, bf16 hi | lo,
//     64 KB) arrives as two K-halves through a 2-stage ring, one bulk copy per
//     half (hi and lo), so a chunk's first half of MMAs overlaps the copy of
//     its second half. Consecutive CTAs work on tiles of the same row, so a
//     row's weights (8 MB at K = 128) are shared through L2.
//
// The weight-stationary layout of contract_tc.cu would need the A tile, the
// contraction vector and a weight chunk resident at once (266 KB at K = 128).
//
// Roles (320 threads): warp 0 = bulk-copy producer, warp 1 = TMEM owner and
// single-thread MMA issuer (4 accumulator slots of K columns), warps 2..9 =
// epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (one sample per thread);
// the two warps of a lane quarter split the K accumulator columns (i-halves)
// and hold their half of the sample's contraction vector in registers; the
// half sums meet in shared memory (named barrier per warp pair) and are added
// in a fixed order, so results are deterministic.
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

constexpr int CB_THREADS = 320;
constexpr int CB_SLOTS = 4;  // TMEM accumulator slots (K <= 128 columns each)

struct BigArgs {
  const uint8_t *a_ops;   // A operand tiles of the layer's first row ([row][tile][hi|lo][128 x ka])
  int64_t a_row_stride;   // bytes per row
  int ka;                 // MMA K dimension (multiple of 32)
  const float *e1;        // contraction vector (EV blocks, width K)
  const float *sv;        // per-output scale (EV blocks) or rt (direct); null = forward
  const uint8_t *tiles;   // weight chunk images [row][chunk] (rows x ka, bf16 hi | lo)
  int64_t tile_bytes;
  int rows_tile, nchunk, n_out;
  const int *dst;         // per row: output slab (forward) or slot (left/right)
  int64_t B, ntl;
  int L;
  int direct;             // K_out == 1 child-rho: out[o] = e1[o] * rt * acc[o]
  int sv_w;
};

__device__ __forceinline__ void cb_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

template <int K>
__device__ __forceinline__ float cb_dot(const float (&v)[K / 2], const float (&e)[K / 2]) {
  uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
  for (int i = 0; i < K / 2; i += 2) {
    uint64_t vp, ep;
    asm("mov.b64 %0, {%1, %2};" : "=l"(vp) : "f"(v[i]), "f"(v[i + 1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ep) : "f"(e[i]), "f"(e[i + 1]));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[(i >> 1) & 1]) : "l"(vp), "l"(ep));
  }
  float a0, a1, a2, a3;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc[0]));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a2), "=f"(a3) : "l"(acc[1]));
  return (a0 + a2) + (a1 + a3);
}

template <int K, bool FWD>
__global__ void __launch_bounds__(CB_THREADS, 1) k_contract_big(BigArgs a, WsView ws) {
  EINET_KERNEL_PROLOGUE();
  constexpr int KH = K / 2;                       // accumulator columns per epilogue warp
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar_af, bar_ae, bar_ef, bar_ee, bar_wf[2], bar_we[2], bar_cf[CB_SLOTS],
      bar_ce[CB_SLOTS];
  __shared__ uint32_t tbase;
  __shared__ float xbuf[2][4][32];               // i-half partial sums (chunk parity, quarter)
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int64_t J = (int64_t)a.L * a.ntl;
  const int64_t j0 = (int64_t)blockIdx.x * J / gridDim.x;
  const int64_t j1 = (int64_t)(blockIdx.x + 1) * J / gridDim.x;
  const uint32_t abytes = (uint32_t)(128 * a.ka * 4);  // A tile: hi | lo
  const uint32_t ebytes = (uint32_t)(4 * K * EV_ROW * 4);
  const uint32_t whalf = (uint32_t)(a.tile_bytes / 4);  // one K-half of hi (or lo)
  uint8_t *abuf = sm;
  float *ebuf = (float *)(sm + abytes);
  uint8_t *wbuf = sm + abytes + ((ebytes + 1023) / 1024) * 1024;  // [2][hi half | lo half]
  if (w == 1) tc::tmem_alloc(&tbase, 512);
  if (t == 0) {
    tc::mbar_init(&bar_af, 1);
    tc::mbar_init(&bar_ae, 1);
    tc::mbar_init(&bar_ef, 1);
    tc::mbar_init(&bar_ee, 8);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&bar_wf[s], 1);
      tc::mbar_init(&bar_we[s], 1);
    }
    for (int s = 0; s < CB_SLOTS; ++s) {
      tc::mbar_init(&bar_cf[s], 1);
      tc::mbar_init(&bar_ce[s], 8);
    }
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const int nchunk = a.direct ? 1 : a.nchunk;

  if (w == 0) {
    // ---- producer ----
    if (lane == 0) {
      int it = 0, wn = 0;
      for (int64_t j = j0; j < j1; ++j, ++it) {
        const int l = (int)(j / a.ntl), jt = (int)(j % a.ntl);
        tc::mbar_wait(&bar_ae, (it & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&bar_af, abytes);
        tc::bulk_g2s(abuf, a.a_ops + l * a.a_row_stride + (int64_t)jt * abytes, abytes, &bar_af);
        tc::mbar_wait(&bar_ee, (it & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&bar_ef, ebytes);
        tc::bulk_g2s(ebuf, a.e1 + ev_idx(l, (int64_t)jt * 128, 0, ws.bc, K), ebytes, &bar_ef);
        for (int c = 0; c < nchunk; ++c) {
          const uint8_t *img = a.tiles + ((int64_t)l * a.nchunk + c) * a.tile_bytes;
          for (int h = 0; h < 2; ++h, ++wn) {
            const int s = wn & 1, ph = (wn >> 1) & 1;
            tc::mbar_wait(&bar_we[s], ph ^ 1);
            tc::mbar_arrive_expect_tx(&bar_wf[s], 2 * whalf);
            uint8_t *dst = wbuf + s * 2 * whalf;
            tc::bulk_g2s(dst, img + h * whalf, whalf, &bar_wf[s]);                  // hi half
            tc::bulk_g2s(dst + whalf, img + 2 * whalf + h * whalf, whalf, &bar_wf[s]);  // lo half
          }
        }
      }
    }
  } else if (w == 1) {
    // ---- MMA issuer (whole warp in the loop, one elected lane issues) ----
    const uint32_t nmma = (uint32_t)a.rows_tile;
    const uint32_t id = tc::idesc_bf16(128, nmma);
    const uint64_t a_desc0 = tc::smem_desc(tc::smem_u32(abuf), 128 * 16, 128u);
    const uint64_t b_desc0 = tc::smem_desc(tc::smem_u32(wbuf), (uint32_t)(a.rows_tile * 16), 128u);
    const uint32_t a_lo_units = abytes / 2 / 16;  // lo part of the A tile
    const uint32_t a_half_units = abytes / 4 / 16;  // first K-half of hi
    const uint32_t b_lo_units = whalf / 16, b_stage_units = 2 * whalf / 16;
    const uint32_t a_ks_units = 2 * 128, b_ks_units = 2 * a.rows_tile;
    const int ks_half = a.ka / 32;  // MMA K-steps (16) per K-half
    int it = 0, wn = 0, cn = 0;
    for (int64_t j = j0; j < j1; ++j, ++it) {
      tc::mbar_wait(&bar_af, it & 1);
      tc::fence_after();
      for (int c = 0; c < nchunk; ++c, ++cn) {
        const int q = cn % CB_SLOTS, qph = (cn / CB_SLOTS) & 1;
        tc::mbar_wait(&bar_ce[q], qph ^ 1);
        tc::fence_after();
        for (int h = 0; h < 2; ++h, ++wn) {
          const int s = wn & 1, ph = (wn >> 1) & 1;
          tc::mbar_wait(&bar_wf[s], ph);
          tc::fence_after();
          if (tc::elect_one()) {
            const uint32_t d = tm + (uint32_t)(q * 128);
            uint64_t ah = a_desc0 + (uint64_t)(h * a_half_units);
            uint64_t al = ah + a_lo_units;
            uint64_t bh = b_desc0 + (uint64_t)(s * b_stage_units), bl = bh + b_lo_units;
            for (int ks = 0; ks < ks_half; ++ks) {
              tc::mma_bf16(d, ah, bh, id, (h > 0 || ks > 0) ? 1u : 0u);
              tc::mma_bf16(d, ah, bl, id, 1u);
              tc::mma_bf16(d, al, bh, id, 1u);
              ah += a_ks_units;
              al += a_ks_units;
              bh += b_ks_units;
              bl += b_ks_units;
            }
            tc::mma_commit(&bar_we[s]);
            if (h == 1) tc::mma_commit(&bar_cf[q]);
            if (h == 1 && c == nchunk - 1) tc::mma_commit(&bar_ae);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---- epilogue ----
    const int quarter = w & 3, half = (w - 2) >> 2;
    const int r = 32 * quarter + lane;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    const uint32_t bar_id = 1 + quarter;  // named barrier of the quarter's warp pair
    int it = 0, cn = 0;
    for (int64_t j = j0; j < j1; ++j, ++it) {
      const int l = (int)(j / a.ntl), jt = (int)(j % a.ntl);
      const int64_t b = (int64_t)jt * 128 + r;
      const bool live = b < a.B;
      const int64_t bs = live ? b : 0;
      tc::mbar_wait(&bar_ef, it & 1);
      float e1[KH];
      {
        const float *src = ebuf + (r >> 5) * (K * EV_ROW) + half * KH * EV_ROW + lane;
#pragma unroll
        for (int i = 0; i < KH; ++i) e1[i] = src[i * EV_ROW];
      }
      __syncwarp();
      if (lane == 0) cb_arrive(&bar_ee);  // the tile's vector is in registers
      float *out = (FWD ? ws.off : ws.slots) + tb_idx(a.dst[l], bs, 0, ws.bc, ws.ks);
      float rt = 0.f;
      if (!FWD && a.direct) rt = a.sv[tb_idx(l, bs, 0, ws.bc, a.sv_w)];
      // per-output scale of the next chunk (left / right), loaded a chunk ahead
      float sv_next = 0.f;
      if (!FWD && !a.direct && half == 0) sv_next = a.sv[ev_idx(l, bs, 0, ws.bc, K)];
      for (int c = 0; c < nchunk; ++c, ++cn) {
        const int q = cn % CB_SLOTS, qph = (cn / CB_SLOTS) & 1;
        const float sv = sv_next;
        if (!FWD && !a.direct && half == 0 && c + 1 < nchunk)
          sv_next = a.sv[ev_idx(l, bs, c + 1, ws.bc, K)];
        tc::mbar_wait(&bar_cf[q], qph);
        tc::fence_after();
        float v[KH];
        tc::tmem_ld_cols<KH>(tm + lane_off + (uint32_t)(q * 128 + half * KH), v);
        tc::tmem_wait_ld();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) cb_arrive(&bar_ce[q]);  // accumulator slot free for the next chunk
        if (a.direct) {
          if (live) {
#pragma unroll
            for (int i = 0; i < KH; ++i) out[(half * KH + i) * 32] = e1[i] * (rt * v[i]);
          }
          continue;
        }
        const float p = cb_dot<K>(v, e1);
        const int pb = cn & 1;
        if (half == 1) xbuf[pb][quarter][lane] = p;
        asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        if (half == 0) {
          const float acc = p + xbuf[pb][quarter][lane];
          float res;
          if (FWD) res = acc > 0.f ? __log2f(acc) * 0.69314718055994531f : -CUDART_INF_F;
          else res = sv * acc;
          if (live) out[c * 32] = res;
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (w == 1) tc::tmem_dealloc(tm, 512);
}

size_t contract_big_smem(int K, int ka, int64_t tile_bytes) {
  const size_t ebytes = (size_t)4 * K * EV_ROW * 4;
  return (size_t)128 * ka * 4 + (ebytes + 1023) / 1024 * 1024 + (size_t)tile_bytes;
}

template <int K, bool FWD>
static int contract_big_t(Plan &p, BigArgs &a, const WsView &w, cudaStream_t st) {
  const size_t smem = contract_big_smem(K, a.ka, a.tile_bytes);
  if (smem > 220 * 1024) return fail(EINET_ERR_UNSUPPORTED, "large-K contraction exceeds shared memory");
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_contract_big<K, FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = smem;
  }
  const int64_t J = (int64_t)a.L * a.ntl;
  const int grid = (int)std::min<int64_t>(J, p.num_sms);
  launch_k(k_contract_big<K, FWD>, grid, CB_THREADS, smem, st, a, w);
  count_launch();
  return check_cuda(cudaGetLastError(), "einsum contraction, large K (tcgen05)");
}

// mode 0: forward, 1: left child responsibilities, 2: right (contract_tc.cu)
int launch_contract_big(Plan &p, const LayerPlan &L, int mode, const uint8_t *compute,
                        const float *EA, const float *EB, const WsView &w, int64_t B,
                        cudaStream_t st) {
  BigArgs a;
  const int K = p.k;
  a.B = B;
  a.ntl = (B + 127) / 128;
  a.L = L.rows;
  a.direct = 0;
  a.sv_w = K;
  if (mode != 0 && L.direct) {
    a.direct = 1;
    a.a_ops = (const uint8_t *)((mode == 1 ? w.ebm : w.eam) + (int64_t)L.erow_base * w.bc * p.kp);
    a.a_row_stride = w.bc * p.kp * 4;
    a.ka = p.kp;
    a.e1 = mode == 1 ? EA : EB;
    a.sv = w.rt;
    a.sv_w = w.ks;
    a.tiles = compute + (mode == 1 ? L.fw_off : L.vw_off);
    a.tile_bytes = mode == 1 ? L.fw_tile : L.rw_tile;
    a.rows_tile = mode == 1 ? L.fw_rows : L.rw_rows;
    a.nchunk = 1;
    a.n_out = K;
    a.dst = mode == 1 ? L.d_slot_left : L.d_slot_right;
  } else if (mode == 0) {
    a.a_ops = (const uint8_t *)(w.ebm + (int64_t)L.erow_base * w.bc * p.kp);
    a.a_row_stride = w.bc * p.kp * 4;
    a.ka = p.kp;
    a.e1 = EA;
    a.sv = nullptr;
    a.tiles = compute + L.fw_off;
    a.tile_bytes = L.fw_tile;
    a.rows_tile = L.fw_rows;
    a.nchunk = L.ng;
    a.n_out = L.k_out;
    a.dst = L.d_out_slab;
  } else {
    a.a_ops = (const uint8_t *)w.rtm;
    a.a_row_stride = w.bc * L.kob * 4;
    a.ka = L.kob;
    a.e1 = mode == 1 ? EB : EA;
    a.sv = mode == 1 ? EA : EB;
    a.tiles = compute + (mode == 1 ? L.uw_off : L.vw_off);
    a.tile_bytes = L.uw_tile;
    a.rows_tile = L.uw_rows;
    a.nchunk = L.ni;
    a.n_out = K;
    a.dst = mode == 1 ? L.d_slot_left : L.d_slot_right;
  }
  if (a.ka % 32 != 0 || a.rows_tile != K)
    return fail(EINET_ERR_UNSUPPORTED, "large-K contraction: tile geometry");
  switch (K) {
    case 96: return mode == 0 ? contract_big_t<96, true>(p, a, w, st) : contract_big_t<96, false>(p, a, w, st);
    case 128: return mode == 0 ? contract_big_t<128, true>(p, a, w, st) : contract_big_t<128, false>(p, a, w, st);
    default: return fail(EINET_ERR_USAGE, "large-K contraction: unsupported k");
  }
}

}  // namespace einet
