// Warp-specialised tcgen05 contraction kernel shared by the EinsumLayer
// forward and the two child-responsibility passes (3xBF16: hi*hi + hi*lo +
// lo*hi of round-to-nearest bf16 splits, fp32 accumulation; ~2^-17 relative
// per product with random signs).
//
// All three are, per einsum row l and 128-sample tile, a GEMM against a
// stationary chunk of that row's weights followed by a per-sample contraction
// of the accumulator with one of the layer's normalised child vectors:
//
//   forward (engine.py:91-109):  T[b,(kl,i)] = sum_j EB[b,j] W[k,i,j]
//                                out[b,k]    = log sum_i EA[b,i] T        -> slab offsets
//   left    (engine.py:312-313): U[b,(il,j)] = sum_k RT[b,k] W[k,i,j]
//                                left[b,i]   = EA[b,i] sum_j EB[b,j] U    -> left slot
//   right   (engine.py:314-315): V[b,(jl,i)] = sum_k RT[b,k] W[k,i,j]
//                                right[b,j]  = EB[b,j] sum_i EA[b,i] V    -> right slot
//
// The A operand (EB or RT = rho / r) is written by its producer kernel in the
// K-major core-matrix layout of a 128-sample tile as bf16 hi and lo parts, so
// it reaches shared memory with one bulk copy.
// The weight chunks (<= 256 accumulator columns each: `og` outputs x K) are
// pre-tiled images (einsum_tc.cu, k_build_tiles). A CTA walks a contiguous
// run of (row, chunk group, 128-sample tile) jobs; the group's G (<= 2)
// consecutive chunks stay resident in shared memory, and every job loads its
// A tile and contraction-vector tile once for G chunk GEMMs. The per-SM
// bulk-copy traffic (A + contraction vector, 47.6 KB per job at K = 40) was
// what bounded the one-chunk-per-job kernel.
//
// Roles (320 threads): warp 0 = bulk-copy producer, warp 1 = TMEM owner and
// single-thread MMA issuer, warps 2..9 = epilogue (warp w reads TMEM lanes
// 32*(w%4)..+31, one sample per thread; the two warps of a lane quarter take
// alternate outputs). Pipelines: A stages (full/empty), contraction-vector
// stages (bulk copies of four [K][EV_ROW] blocks; a stage is released as soon
// as the epilogue holds it in registers), two TMEM accumulators of 256
// columns, one per chunk GEMM (full/empty), and the weight group
// (full/empty). The epilogue's dot products use packed fp32x2 FMAs (FFMA2);
// the per-output scales (left/right) are loaded from global memory one job
// ahead. Per-job timelines: EINET_CT_TRACE; profiles/r02_contract.md.
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

constexpr int CT_STAGES = 4;      // max A-operand / contraction-vector ring depth
constexpr int CT_GMAX = 2;        // max weight chunks resident per (row, group)
constexpr int CT_EPI_WARPS = 8;                 // two per TMEM lane quarter
constexpr int CT_THREADS = 64 + 32 * CT_EPI_WARPS;

// Per side (forward: one side; child responsibilities: left and right in one
// launch, the job space being side-major): operand and output pointers.
struct ContractArgs {
  const float *a_ops[2];  // A operand tiles of the layer's first row
  int64_t a_row_stride;   // bytes per row (ntl * 128 * ka * 4: bf16 hi | lo)
  int ka;                 // MMA K dimension (multiple of 16)
  const float *e1[2];     // contraction vector, 32-sample transposed, width K
  const float *sv[2];     // per-output scale vector (left/right), width K; null = forward
  const uint8_t *tiles[2];  // weight chunk images [row][chunk]
  int64_t tile_bytes;
  int nchunk, og, rows_tile, n_out;
  int G, ngroup;          // weight chunks resident per (row, group) run, groups per row
  const int *dst[2];      // per row: output slab (forward) or slot (left/right)
  int nside;              // 1 (forward) or 2 (left and right child responsibilities)
  int64_t B, ntl;
  int L;
  int stages;             // A-operand ring depth (2..4, by shared-memory fit)
  int se;                 // contraction-vector ring depth (2..4)
  int direct;             // K_out == 1 child-rho: out[o] = e1[o] * rt * acc[o] (no contraction)
  int sv_w;               // transposed-block width of sv
  int debug;              // EINET_CT_DEBUG (timing experiments only): 1 no epilogue math, 2 no MMA
  int terms;              // 3: 3xBF16 (default); 1: hi*hi only (EINET_CONTRACT_TERMS=1, forward:
                          // reduced-precision variant, ~2^-8 relative per layer, own tolerance)
  long long *trace;       // EINET_CT_TRACE (diagnostics): per-job timestamps of CTA 0
};

__device__ __forceinline__ long long ct_now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// (side, row, chunk group, 128-sample tile) of consecutive jobs, advanced
// incrementally (64-bit division costs hundreds of cycles in the issue loops)
struct JobCursor {
  int jt, l, c, side;
  __device__ __forceinline__ void init(int64_t j, int64_t ntl, int ngroup, int L) {
    const int pair = (int)(j / ntl);
    jt = (int)(j % ntl);
    c = pair % ngroup;
    l = (pair / ngroup) % L;
    side = pair / ngroup / L;
  }
  // returns true when the next job starts a new (side, row, group)
  __device__ __forceinline__ bool next(int ntl, int ngroup, int L) {
    if (++jt < ntl) return false;
    jt = 0;
    if (++c == ngroup) {
      c = 0;
      if (++l == L) {
        l = 0;
        ++side;
      }
    }
    return true;
  }
};

#define CT_TRACE(slot, it)                                                      \
  do {                                                                          \
    if (a.trace && blockIdx.x == 0 && (it) < 64) a.trace[(it) * 8 + (slot)] = ct_now(); \
  } while (0)

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// sum_i v[i] * e[i] with packed fp32x2 FMAs (two independent pair chains)
__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
template <int K>
__device__ __forceinline__ float dot_f32x2(const float (&v)[K], const float (&e)[K]) {
  uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
  for (int i = 0; i + 1 < K; i += 2)
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(acc[(i >> 1) & 1])
        : "l"(pack_f32x2(v[i], v[i + 1])), "l"(pack_f32x2(e[i], e[i + 1])));
  float a0, a1, a2, a3;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc[0]));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a2), "=f"(a3) : "l"(acc[1]));
  if (K & 1) a0 = fmaf(v[K - 1], e[K - 1], a0);
  return (a0 + a2) + (a1 + a3);
}

template <int K, bool FWD>
__global__ void __launch_bounds__(CT_THREADS, 1) k_contract_tc(ContractArgs a, WsView ws) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar_wf, bar_we, bar_af[CT_STAGES], bar_ae[CT_STAGES], bar_cf[2], bar_ce[2],
      bar_ef[CT_STAGES], bar_ee[CT_STAGES];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int64_t J = (int64_t)a.nside * a.L * a.ngroup * a.ntl;
  const int64_t j0 = (int64_t)blockIdx.x * J / gridDim.x;
  const int64_t j1 = (int64_t)(blockIdx.x + 1) * J / gridDim.x;
  const int64_t wbytes = (a.tile_bytes + 1023) / 1024 * 1024;
  const uint32_t abytes = (uint32_t)(128 * a.ka * 4);  // bf16 hi | lo
  const uint32_t ebytes = (uint32_t)(4 * K * EV_ROW * 4);
  uint8_t *wsm = sm;
  uint8_t *abuf = sm + (int64_t)a.G * wbytes;
  float *ebuf = (float *)(abuf + (int64_t)a.stages * abytes);  // [se][128 x K] contraction vector
  if (w == 1) tc::tmem_alloc(&tbase, 512);
  if (t == 0) {
    tc::mbar_init(&bar_wf, 1);
    tc::mbar_init(&bar_we, 1);
    for (int s = 0; s < CT_STAGES; ++s) {
      tc::mbar_init(&bar_af[s], 1);
      tc::mbar_init(&bar_ae[s], 1);
      tc::mbar_init(&bar_ef[s], 1);
      tc::mbar_init(&bar_ee[s], CT_EPI_WARPS);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&bar_cf[s], 1);
      tc::mbar_init(&bar_ce[s], CT_EPI_WARPS);
    }
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;

  if (w == 0) {
    // ---- producer ----
    if (lane == 0) {
      const int ntl = (int)a.ntl;
      JobCursor cur;
      cur.init(j0, a.ntl, a.ngroup, a.L);
      bool fresh = true;
      int q = -1, it = 0, s = 0, ph = 0;
      for (int64_t j = j0; j < j1; ++j, ++it) {
        const int jt = cur.jt, l = cur.l, sd = cur.side;
        if (fresh) {
          // the group's chunks are consecutive images: one copy
          ++q;
          if (q > 0) tc::mbar_wait(&bar_we, (q - 1) & 1);
          const int gc = min(a.G, a.nchunk - cur.c * a.G);
          const uint32_t bytes = (uint32_t)(gc * a.tile_bytes);
          tc::mbar_arrive_expect_tx(&bar_wf, bytes);
          tc::bulk_g2s(wsm, a.tiles[sd] + ((int64_t)l * a.nchunk + cur.c * a.G) * a.tile_bytes, bytes,
                       &bar_wf);
        }
        tc::mbar_wait(&bar_ae[s], ph ^ 1);
        CT_TRACE(0, it);
        // (single-term variant: the hi half of the tile only)
        const uint32_t acopy = a.terms == 1 ? abytes / 2 : abytes;
        tc::mbar_arrive_expect_tx(&bar_af[s], acopy);
        tc::bulk_g2s(abuf + (int64_t)s * abytes,
                     (const uint8_t *)a.a_ops[sd] + l * a.a_row_stride + (int64_t)jt * abytes, acopy,
                     &bar_af[s]);
        if (++s == a.stages) {
          s = 0;
          ph ^= 1;
        }
        // the tile's contraction vector: 4 contiguous [K][EV_ROW] blocks
        const int se = it % a.se, eph = (it / a.se) & 1;
        tc::mbar_wait(&bar_ee[se], eph ^ 1);
        tc::mbar_arrive_expect_tx(&bar_ef[se], ebytes);
        tc::bulk_g2s(ebuf + se * 4 * K * EV_ROW, a.e1[sd] + ev_idx(l, (int64_t)jt * 128, 0, ws.bc, K),
                     ebytes, &bar_ef[se]);
        fresh = cur.next(ntl, a.ngroup, a.L);
      }
    }
  } else if (w == 1) {
    // ---- MMA issuer: the whole warp runs the loop (uniform registers), one
    // elected lane issues; descriptors advance by adding to their 14-bit
    // start-address field (16-byte units) ----
    const uint64_t a_desc0 = tc::smem_desc(tc::smem_u32(abuf), 128 * 16, 128u);
    const uint64_t b_desc0 = tc::smem_desc(tc::smem_u32(wsm), (uint32_t)(a.rows_tile * 16), 128u);
    const uint32_t a_lo_units = 128 * a.ka * 2 / 16, b_lo_units = a.rows_tile * a.ka * 2 / 16;
    const uint32_t a_ks_units = 2 * 128, b_ks_units = 2 * a.rows_tile;
    const int nks = (a.debug & 2) ? 0 : a.ka / 16;
    const int ntl = (int)a.ntl;
    const uint32_t w_units = (uint32_t)(wbytes >> 4);
    JobCursor cur;
    cur.init(j0, a.ntl, a.ngroup, a.L);
    int q = 0, it = 0, s = 0, ph = 0, acc_n = 0;
    if (j0 < j1) tc::mbar_wait(&bar_wf, 0);
    for (int64_t j = j0; j < j1; ++j, ++it) {
      const int g = cur.c, jt = cur.jt;
      const int gc = min(a.G, a.nchunk - g * a.G);
      tc::mbar_wait(&bar_af[s], ph);
      if (lane == 0) CT_TRACE(1, it);
      const bool last_of_pair = j + 1 == j1 || jt + 1 == ntl;
      for (int c = 0; c < gc; ++c, ++acc_n) {
        const int chunk = g * a.G + c;
        const int nol = min(a.og, a.n_out - chunk * a.og);
        const int nmma = a.direct ? (K + 15) / 16 * 16 : (nol * K + 15) / 16 * 16;
        const int buf = acc_n & 1, bph = (acc_n >> 1) & 1;
        tc::mbar_wait(&bar_ce[buf], bph ^ 1);
        tc::fence_after();
        if (lane == 0 && c == 0) CT_TRACE(2, it);
        if (tc::elect_one()) {
          const uint32_t id = tc::idesc_bf16(128, nmma);
          const uint32_t d = tm + (uint32_t)(buf * 256);
          uint64_t ah = a_desc0 + (uint64_t)(s * (abytes >> 4));
          uint64_t al = ah + a_lo_units;
          uint64_t bh = b_desc0 + (uint64_t)c * w_units, bl = bh + b_lo_units;
          for (int ks = 0; ks < nks; ++ks) {
            tc::mma_bf16(d, ah, bh, id, ks > 0 ? 1u : 0u);
            if (a.terms == 3) {
              tc::mma_bf16(d, ah, bl, id, 1u);
              tc::mma_bf16(d, al, bh, id, 1u);
            }
            ah += a_ks_units;
            al += a_ks_units;
            bh += b_ks_units;
            bl += b_ks_units;
          }
          tc::mma_commit(&bar_cf[buf]);
          if (c == gc - 1) {
            tc::mma_commit(&bar_ae[s]);
            if (last_of_pair) tc::mma_commit(&bar_we);
          }
        }
        __syncwarp();
      }
      if (++s == a.stages) {
        s = 0;
        ph ^= 1;
      }
      if (cur.next(ntl, a.ngroup, a.L) && j + 1 < j1) tc::mbar_wait(&bar_wf, (++q) & 1);
    }
  } else {
    // ---- epilogue: one sample per thread. The two warps of a lane quarter
    // take alternate outputs (ol = half, half + 2, ...); every output is a
    // K-long dot product of accumulator columns with the contraction vector,
    // done with packed fp32x2 FMAs (FFMA2) on register pairs ----
    constexpr int OGM = 256 / K;          // outputs per chunk (accumulator columns / K)
    constexpr int NPW = (OGM + 1) / 2;    // outputs per warp per job
    constexpr int OPW = (96 / K) < 1 ? 1 : ((96 / K) < NPW ? (96 / K) : NPW);  // per tcgen05.wait
    constexpr int NSV = FWD ? 1 : CT_GMAX * NPW;
    const int quarter = w & 3, half = (w - 2) >> 2;
    const int r = 32 * quarter + lane;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    // per-output scales (left/right) of this warp's outputs in the next job's
    // chunks ([c][u] -> c * NPW + u)
    float sv_next[NSV];
    const int ntl = (int)a.ntl;
    JobCursor cur, nxt;
    cur.init(j0, a.ntl, a.ngroup, a.L);
    nxt = cur;
    auto load_next = [&](int64_t j) {
      if (FWD || j >= j1) return;
      const int l = nxt.l, g = nxt.c;
      const float *svs = a.sv[nxt.side];
      const int64_t b = min((int64_t)nxt.jt * 128 + r, a.B - 1);
      if (a.direct) {
        sv_next[0] = svs[tb_idx(l, b, 0, ws.bc, a.sv_w)];
        return;
      }
      const int gc = min(a.G, a.nchunk - g * a.G);
#pragma unroll
      for (int c = 0; c < CT_GMAX; ++c) {
        if (c >= gc) break;
        const int chunk = g * a.G + c;
        const int nol = min(a.og, a.n_out - chunk * a.og);
        const float *svp = svs + ev_idx(l, b, chunk * a.og, ws.bc, K);
#pragma unroll
        for (int u = 0; u < NPW; ++u)
          if (half + 2 * u < nol) sv_next[c * NPW + u] = svp[(half + 2 * u) * EV_ROW];
      }
    };
    load_next(j0);
    nxt.next(ntl, a.ngroup, a.L);
    int it = 0, acc_n = 0;
    for (int64_t j = j0; j < j1; ++j, ++it) {
      const int l = cur.l, g = cur.c, sd = cur.side;
      const int gc = min(a.G, a.nchunk - g * a.G);
      const int64_t b = (int64_t)cur.jt * 128 + r;
      const bool live = b < a.B;
      const int64_t bs = live ? b : 0;
      float sv[NSV];
#pragma unroll
      for (int u = 0; u < NSV; ++u) sv[u] = sv_next[u];
      load_next(j + 1);
      nxt.next(ntl, a.ngroup, a.L);
      cur.next(ntl, a.ngroup, a.L);
      const int se = it % a.se, eph = (it / a.se) & 1;
      if (w == 2 && lane == 0) CT_TRACE(6, it);
      tc::mbar_wait(&bar_ef[se], eph);
      float e1[K];
      {
        const float *src = ebuf + se * 4 * K * EV_ROW + (r >> 5) * (K * EV_ROW) + lane;
#pragma unroll
        for (int i = 0; i < K; ++i) e1[i] = src[i * EV_ROW];
      }
      // e1 is in registers: release the stage to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_ee[se]);
      if (w == 2 && lane == 0) CT_TRACE(3, it);
      float *out = (FWD ? ws.off : ws.slots) + tb_idx(a.dst[sd][l], bs, 0, ws.bc, ws.ks);
#pragma unroll 1
      for (int c = 0; c < gc; ++c, ++acc_n) {
        const int chunk = g * a.G + c;
        const int nol = min(a.og, a.n_out - chunk * a.og);
        const int buf = acc_n & 1, bph = (acc_n >> 1) & 1;
        tc::mbar_wait(&bar_cf[buf], bph);
        if (w == 2 && lane == 0 && c == 0) CT_TRACE(4, it);
        tc::fence_after();
        const uint32_t ta = tm + lane_off + (uint32_t)(buf * 256);
        if (a.direct) {
          float v[K];
          tc::tmem_ld_cols<K>(ta, v);
          tc::tmem_wait_ld();
          const float rt = sv[0];
          if (live) {
#pragma unroll
            for (int o = 0; o < K; ++o)
              if ((o & 1) == half) out[o * 32] = e1[o] * (rt * v[o]);
          }
        } else if (!(a.debug & 1)) {
#pragma unroll
          for (int g0 = 0; g0 < NPW; g0 += OPW) {
            if (half + 2 * g0 >= nol) break;
            float v[OPW][K];
#pragma unroll
            for (int gi = 0; gi < OPW; ++gi) {
              const int ol = half + 2 * (g0 + gi);
              if (g0 + gi < NPW && ol < nol) tc::tmem_ld_cols<K>(ta + ol * K, v[gi]);
            }
            tc::tmem_wait_ld();
#pragma unroll
            for (int gi = 0; gi < OPW; ++gi) {
              const int ol = half + 2 * (g0 + gi);
              if (g0 + gi < NPW && ol < nol) {
                const float acc = dot_f32x2<K>(v[gi], e1);
                const int o = chunk * a.og + ol;
                float res;
                if (FWD) {
                  res = acc > 0.f ? __log2f(acc) * 0.69314718055994531f : -CUDART_INF_F;
                } else {
                  float scale = 0.f;
#pragma unroll
                  for (int cc = 0; cc < CT_GMAX; ++cc)
                    if (cc == c) scale = sv[(FWD ? 0 : cc * NPW) + g0 + gi];
                  res = scale * acc;
                }
                if (live) out[o * 32] = res;
              }
            }
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_ce[buf]);
      }
      if (w == 2 && lane == 0) CT_TRACE(5, it);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (w == 1) tc::tmem_dealloc(tm, 512);
}

constexpr size_t CT_SMEM_MAX = 220 * 1024;

size_t contract_smem(int64_t tile_bytes, int ka, int G, int stages, int se, int K) {
  return (size_t)G * tile_bytes + (size_t)stages * 128 * ka * 4 + (size_t)se * 4 * K * EV_ROW * 4;
}

template <int K, bool FWD>
static int contract_t(Plan &p, ContractArgs &a, const WsView &w, cudaStream_t st) {
  // Weight chunks resident per job: every job's A tile and contraction
  // vector serve G chunk GEMMs, which divides the per-SM bulk-copy traffic
  // (the limit at G = 1) by G; small batches keep G = 1 for more jobs. Then
  // the contraction-vector ring, then the A ring, as deep as shared memory
  // allows.
  int G = 1;
  if ((int64_t)a.L * a.nchunk * a.ntl >= 4LL * p.num_sms)
    while (G < std::min(CT_GMAX, a.nchunk) &&
           contract_smem(a.tile_bytes, a.ka, G + 1, 2, 2, K) <= CT_SMEM_MAX)
      ++G;
  if (const char *env = getenv("EINET_CT_G")) G = std::max(1, std::min(atoi(env), G));
  a.G = G;
  a.ngroup = ceil_div(a.nchunk, G);

  a.stages = 2;
  a.se = 2;
  while (a.se < 3 && contract_smem(a.tile_bytes, a.ka, G, a.stages, a.se + 1, K) <= CT_SMEM_MAX) ++a.se;
  while (a.stages < CT_STAGES &&
         contract_smem(a.tile_bytes, a.ka, G, a.stages + 1, a.se, K) <= CT_SMEM_MAX)
    ++a.stages;
  while (a.se < CT_STAGES && contract_smem(a.tile_bytes, a.ka, G, a.stages, a.se + 1, K) <= CT_SMEM_MAX)
    ++a.se;
  const size_t smem = contract_smem(a.tile_bytes, a.ka, G, a.stages, a.se, K);
  if (smem > CT_SMEM_MAX) return fail(EINET_ERR_UNSUPPORTED, "contraction tile exceeds shared memory");
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_contract_tc<K, FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = smem;
  }
  const int64_t J = (int64_t)a.nside * a.L * a.ngroup * a.ntl;
  const int grid = (int)std::min<int64_t>(J, p.num_sms);
  static long long *trace_buf = nullptr;
  a.trace = nullptr;
  const bool tracing = getenv("EINET_CT_TRACE") != nullptr;
  if (tracing) {
    if (!trace_buf) cudaMalloc(&trace_buf, 64 * 8 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 64 * 8 * sizeof(long long), st);
    a.trace = trace_buf;
  }
  launch_k(k_contract_tc<K, FWD>, grid, CT_THREADS, smem, st, a, w);
  if (tracing) {
    long long h[64 * 8];
    cudaMemcpyAsync(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "contract trace L=%d nchunk=%d G=%d ka=%d direct=%d stages=%d se=%d\n", a.L,
            a.nchunk, a.G, a.ka, a.direct, a.stages, a.se);
    for (int i = 0; i < 12; ++i)
      fprintf(stderr, "  it %2d prod %6lld a_full %6lld acc_free %6lld | e_wait %6lld e_ok %6lld acc_full %6lld epi_done %6lld\n",
              i, h[i * 8] - h[0], h[i * 8 + 1] - h[0], h[i * 8 + 2] - h[0], h[i * 8 + 6] - h[0],
              h[i * 8 + 3] - h[0], h[i * 8 + 4] - h[0], h[i * 8 + 5] - h[0]);
  }
  count_launch();
  return check_cuda(cudaGetLastError(), "einsum contraction (tcgen05)");
}

int launch_contract_big(Plan &p, const LayerPlan &L, int mode, const uint8_t *compute,
                        const float *EA, const float *EB, const WsView &w, int64_t B,
                        cudaStream_t st);

// mode 0: forward, 1: left child responsibilities, 2: right, 3: both sides in one launch
int launch_contract_tc(Plan &p, const LayerPlan &L, int mode, const uint8_t *compute,
                       const float *EA, const float *EB, const WsView &w, int64_t B,
                       cudaStream_t st) {
  ContractArgs a;
  const int K = p.k;
  if (K > 64) {
    if (mode != 3) return launch_contract_big(p, L, mode, compute, EA, EB, w, B, st);
    const int rc = launch_contract_big(p, L, 1, compute, EA, EB, w, B, st);
    return rc ? rc : launch_contract_big(p, L, 2, compute, EA, EB, w, B, st);
  }
  a.B = B;
  a.ntl = (B + 127) / 128;
  a.L = L.rows;
  a.direct = 0;
  a.sv_w = K;
  {
    const char *env = getenv("EINET_CT_DEBUG");
    a.debug = env ? atoi(env) : 0;
    static const int terms = getenv("EINET_CONTRACT_TERMS") ? atoi(getenv("EINET_CONTRACT_TERMS")) : 3;
    a.terms = (mode == 0 && terms == 1) ? 1 : 3;
  }
  // mode 3: both child-responsibility sides (left = side 0, right = side 1)
  a.nside = mode == 3 ? 2 : 1;
  const int m0 = mode == 3 ? 1 : mode;
  for (int sd = 0; sd < a.nside; ++sd) {
    const int md = m0 + sd;  // 0 forward, 1 left, 2 right
    if (md != 0 && L.direct) {
      a.direct = 1;
      a.a_ops[sd] = (md == 1 ? w.ebm : w.eam) + (int64_t)L.erow_base * w.bc * p.kp;
      a.a_row_stride = w.bc * p.kp * 4;
      a.ka = p.kp;
      a.e1[sd] = md == 1 ? EA : EB;
      a.sv[sd] = w.rt;
      a.sv_w = w.ks;
      a.tiles[sd] = compute + (md == 1 ? L.fw_off : L.vw_off);
      a.tile_bytes = md == 1 ? L.fw_tile : L.rw_tile;  // equal: fw_rows == rw_rows at K_out = 1
      a.nchunk = 1;
      a.og = K;
      a.rows_tile = md == 1 ? L.fw_rows : L.rw_rows;
      a.n_out = K;
      a.dst[sd] = md == 1 ? L.d_slot_left : L.d_slot_right;
    } else if (md == 0) {
      a.a_ops[sd] = w.ebm + (int64_t)L.erow_base * w.bc * p.kp;
      a.a_row_stride = w.bc * p.kp * 4;
      a.ka = p.kp;
      a.e1[sd] = EA;
      a.sv[sd] = nullptr;
      a.tiles[sd] = compute + L.fw_off;
      a.tile_bytes = L.fw_tile;
      a.nchunk = L.ng;
      a.og = L.kg;
      a.rows_tile = L.fw_rows;
      a.n_out = L.k_out;
      a.dst[sd] = L.d_out_slab;
    } else {
      a.a_ops[sd] = w.rtm;
      a.a_row_stride = w.bc * L.kob * 4;
      a.ka = L.kob;
      a.e1[sd] = md == 1 ? EB : EA;
      a.sv[sd] = md == 1 ? EA : EB;
      a.tiles[sd] = compute + (md == 1 ? L.uw_off : L.vw_off);
      a.tile_bytes = L.uw_tile;
      a.nchunk = L.ni;
      a.og = L.ig;
      a.rows_tile = L.uw_rows;
      a.n_out = K;
      a.dst[sd] = md == 1 ? L.d_slot_left : L.d_slot_right;
    }
  }
  if (a.nside == 1) {
    a.a_ops[1] = a.a_ops[0];
    a.e1[1] = a.e1[0];
    a.sv[1] = a.sv[0];
    a.tiles[1] = a.tiles[0];
    a.dst[1] = a.dst[0];
  }
  switch (K) {
    case 8: return mode == 0 ? contract_t<8, true>(p, a, w, st) : contract_t<8, false>(p, a, w, st);
    case 10: return mode == 0 ? contract_t<10, true>(p, a, w, st) : contract_t<10, false>(p, a, w, st);
    case 16: return mode == 0 ? contract_t<16, true>(p, a, w, st) : contract_t<16, false>(p, a, w, st);
    case 20: return mode == 0 ? contract_t<20, true>(p, a, w, st) : contract_t<20, false>(p, a, w, st);
    case 24: return mode == 0 ? contract_t<24, true>(p, a, w, st) : contract_t<24, false>(p, a, w, st);
    case 32: return mode == 0 ? contract_t<32, true>(p, a, w, st) : contract_t<32, false>(p, a, w, st);
    case 40: return mode == 0 ? contract_t<40, true>(p, a, w, st) : contract_t<40, false>(p, a, w, st);
    case 48: return mode == 0 ? contract_t<48, true>(p, a, w, st) : contract_t<48, false>(p, a, w, st);
    case 56: return mode == 0 ? contract_t<56, true>(p, a, w, st) : contract_t<56, false>(p, a, w, st);
    case 64: return mode == 0 ? contract_t<64, true>(p, a, w, st) : contract_t<64, false>(p, a, w, st);
    default: return fail(EINET_ERR_USAGE, "tc path: unsupported k");
  }
}

}  // namespace einet
