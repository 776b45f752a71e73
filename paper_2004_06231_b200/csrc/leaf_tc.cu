// Gaussian leaf statistics on tcgen05 (engine.py:318-327):
//
//   S[(v, t), k] = sum_b y_bv^(t+1) rho[b,l,k],   y = x - c_v  (c = stats centre)
//
// as a batch-reduction GEMM per leaf region: M = 128 scope variables per
// segment (two TMEM tiles of 64 variables x {y, y^2}), N = K (padded to 16),
// reduction over 32-sample blocks. Warp-specialised, like wstats_tc.cu:
//   * warps 0..3 gather the segment's x values for a unit of LS_QB blocks
//     with cp.async (16-byte groups of four consecutive, aligned variables when
//     the scope allows it -- image leaves do -- else 4-byte), zero-filling
//     samples past the batch; warp 0 also bulk-copies the unit's rho^T B tiles
//     (hi | lo, written by k_leaf_rho);
//   * warp 4 owns TMEM and issues the 3xTF32 MMAs (A from TMEM);
//   * warps 5..20 generate the A operand (y or y^2: round-to-nearest TF32 part
//     and fp32 remainder) straight into TMEM, one (tile, TMEM lane quarter,
//     16-sample half of each block) per warp (8 warps, one per (tile,
//     quarter) walking both halves, left the generation on the critical path:
//     two warps per scheduler); the half-0 warps drain the accumulators.
// A CTA runs over <= 4096 samples of one or two segments (fp32 accumulation
// runs); partials go to per-(segment, slot) fp32 buffers, summed in slot
// order and un-centred in fp64 by k_leaf_stats_finish:
//   sum rho x = S_y + c P,  sum rho x^2 = S_y2 + 2 c S_y + c^2 P.
#include <climits>
#include <cmath>
#include <cstdlib>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

constexpr int LS_QB = 2;          // 32-sample blocks per unit
constexpr int LS_STAGES = 3;
constexpr int LS_ASTAGES = 3;     // TMEM A ring (2 tiles x 64 columns per block)
constexpr int LS_MAX_RUN = 64;    // units per CTA run (<= 4096 samples)
constexpr int LS_GATHER_WARPS = 4;
constexpr int LS_GEN_WARPS = 16;  // 2 tiles x 2 sample halves x 4 TMEM lane quarters
constexpr int LS_THREADS = 32 * (LS_GATHER_WARPS + 1 + LS_GEN_WARPS);
constexpr int LS_SEGV = 128;      // scope variables per segment

struct LeafStatsArgs {
  const float *x;
  const float *rhob;        // [leaf][Bc/32][hi | lo][nn x 32]
  const float *center;      // [R][D]
  const uint8_t *active;    // [D]
  const int *scope_off, *scope_vars, *leaf_rep;
  const int *seg_leaf, *seg_v0;  // per segment: leaf, first scope position
  const uint8_t *seg_vec;        // per segment: 16-byte gathers allowed
  float *part;              // [slot][n_phi] fp32
  int64_t B, bc, n_phi;
  int D, K, R, nn;
  int nblk, nq;
  int64_t units;
  int grid;
  int debug;                // EINET_LS_DEBUG (diagnostics): 1 scalar gathers
};

__device__ __forceinline__ void ls_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cpa16_zfill(void *smem, const void *gmem, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(tc::smem_u32(smem)),
               "l"(gmem), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cpa4_zfill(void *smem, const void *gmem, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(tc::smem_u32(smem)),
               "l"(gmem), "r"(ok ? 4 : 0));
}

__host__ __device__ inline int64_t ls_u0(int64_t c, int64_t U, int64_t G) { return c * U / G; }
__host__ __device__ inline int64_t ls_cta_of(int64_t u, int64_t U, int64_t G) {
  int64_t c = u * G / U;
  while (c + 1 < G && ls_u0(c + 1, U, G) <= u) ++c;
  while (c > 0 && ls_u0(c, U, G) > u) --c;
  return c;
}

__global__ void __launch_bounds__(LS_THREADS, 1) k_leaf_stats_tc(LeafStatsArgs a) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t s_full[LS_STAGES], s_empty[LS_STAGES], a_full[LS_ASTAGES],
      a_empty[LS_ASTAGES], c_full, c_empty;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int nn = a.nn, nq = a.nq, nblk = a.nblk, K = a.K, D = a.D;
  const uint32_t xs_floats = 32 * LS_SEGV, rb_floats = 2 * nn * 32;
  const uint32_t stage_floats = LS_QB * (xs_floats + rb_floats);
  float *ring = (float *)sm;
  const int64_t u0 = ls_u0(blockIdx.x, a.units, a.grid);
  const int64_t u1 = ls_u0(blockIdx.x + 1, a.units, a.grid);
  constexpr int MMA_WARP = LS_GATHER_WARPS;
  if (w == MMA_WARP) tc::tmem_alloc(&tbase, 512);
  if (t == 0) {
    for (int s = 0; s < LS_STAGES; ++s) {
      tc::mbar_init(&s_full[s], 32 * LS_GATHER_WARPS + 1);
      tc::mbar_init(&s_empty[s], LS_GEN_WARPS + 1);
    }
    for (int s = 0; s < LS_ASTAGES; ++s) {
      tc::mbar_init(&a_full[s], LS_GEN_WARPS);
      tc::mbar_init(&a_empty[s], 1);
    }
    tc::mbar_init(&c_full, 1);
    tc::mbar_init(&c_empty, LS_GEN_WARPS);
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const int seg0 = (int)(u0 / nq), q0 = (int)(u0 % nq);

  if (w < LS_GATHER_WARPS) {
    // ---- gather x (and the rho^T tiles) ----
    const int gt = t;  // 0 .. 32*LS_GATHER_WARPS-1
    int seg = seg0, q = q0, it = 0;
    int cur_seg = -1, leaf = 0, sbeg = 0, nv = 0;
    bool vec = false;
    int dgrp = 0;  // this thread's fixed variable group (vector path)
    for (int64_t u = u0; u < u1; ++u, ++it) {
      if (seg != cur_seg) {
        cur_seg = seg;
        leaf = a.seg_leaf[seg];
        sbeg = a.scope_off[leaf] + a.seg_v0[seg];
        nv = min(LS_SEGV, a.scope_off[leaf + 1] - sbeg);
        vec = a.seg_vec[seg] != 0 && !(a.debug & 1);
        const int g = gt & 31;  // group of 4 variables
        dgrp = 4 * g < nv ? a.scope_vars[sbeg + 4 * g] : -1;
      }
      const int s = it % LS_STAGES, ph = (it / LS_STAGES) & 1;
      const int b0 = q * LS_QB, nb = min(LS_QB, nblk - b0);
      tc::mbar_wait(&s_empty[s], ph ^ 1);
      float *dst = ring + (int64_t)s * stage_floats;
      if (w == 0 && tc::elect_one()) {
        const uint32_t rbb = (uint32_t)(nb * rb_floats * 4);
        tc::mbar_arrive_expect_tx(&s_full[s], rbb);
        tc::bulk_g2s(dst + LS_QB * xs_floats,
                     a.rhob + ((int64_t)leaf * (a.bc / 32) + b0) * rb_floats, rbb, &s_full[s]);
      }
      const int64_t bbase = (int64_t)b0 * 32;
      if (vec) {
        // thread gt: variable group (gt & 31), samples (gt >> 5) + 4 i
        const int g = gt & 31;
        for (int sidx = gt >> 5; sidx < nb * 32; sidx += LS_GATHER_WARPS) {
          const int64_t b = bbase + sidx;
          const bool ok = b < a.B && dgrp >= 0;
          const float *src = a.x + (ok ? b * D + dgrp : 0);
          cpa16_zfill(dst + sidx * LS_SEGV + 4 * g, src, ok);
        }
      } else {
        for (int e = gt; e < nb * 32 * LS_SEGV; e += 32 * LS_GATHER_WARPS) {
          const int v = e & (LS_SEGV - 1), sidx = e >> 7;
          const int64_t b = bbase + sidx;
          const bool ok = b < a.B && v < nv;
          const float *src = a.x + (ok ? b * D + a.scope_vars[sbeg + v] : 0);
          cpa4_zfill(dst + sidx * LS_SEGV + v, src, ok);
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                       tc::smem_u32(&s_full[s]))
                   : "memory");
      if (++q == nq) {
        q = 0;
        ++seg;
      }
    }
  } else if (w == MMA_WARP) {
    // ---- MMA issuer ----
    const uint32_t id = tc::idesc_tf32(128, nn);
    const uint64_t bdesc0 =
        tc::smem_desc(tc::smem_u32(ring + LS_QB * xs_floats), (uint32_t)(nn * 16), 128u);
    const uint32_t stage_units = stage_floats * 4 / 16, blk_units = rb_floats * 4 / 16;
    const uint32_t kstep_units = 2 * nn, lo_units = nn * 8;
    int seg = seg0, q = q0, it = 0, ab = 0, nrun = 0;
    bool first = true;
    for (int64_t u = u0; u < u1; ++u, ++it) {
      const int s = it % LS_STAGES, ph = (it / LS_STAGES) & 1;
      const int nb = min(LS_QB, nblk - q * LS_QB);
      const bool last = u + 1 == u1 || q + 1 == nq;
      if (first) tc::mbar_wait(&c_empty, (nrun & 1) ^ 1);
      tc::mbar_wait(&s_full[s], ph);
      for (int sb = 0; sb < nb; ++sb, ++ab) {
        const int as = ab % LS_ASTAGES, aph = (ab / LS_ASTAGES) & 1;
        tc::mbar_wait(&a_full[as], aph);
        tc::fence_after();
        if (tc::elect_one()) {
          const uint64_t bh = bdesc0 + (uint64_t)(s * stage_units + sb * blk_units);
          const uint64_t bl = bh + lo_units;
          const uint32_t acc0 = (first && sb == 0) ? 0u : 1u;
          const uint32_t ah0 = tm + 128 + (uint32_t)(as * 128);
          // 3xTF32 per K-step (hi*hi, hi*lo, lo*hi), the two tiles' MMAs
          // alternating so consecutive instructions accumulate into different
          // TMEM accumulators (a chain into one accumulator stalls at N = K:
          // profiles/r02_probes.md)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t kh = bh + ks * kstep_units, kl = bl + ks * kstep_units;
#pragma unroll
            for (int term = 0; term < 3; ++term) {
#pragma unroll
              for (int g = 0; g < 2; ++g) {
                const uint32_t d = tm + (uint32_t)(g * nn), ah = ah0 + g * 64;
                tc::mma_tf32_ts(d, ah + (term == 2 ? 32 : 0) + 8 * ks, term == 1 ? kl : kh, id,
                                (ks == 0 && term == 0) ? acc0 : 1u);
              }
            }
          }
          tc::mma_commit(&a_empty[as]);
          if (sb + 1 == nb) {
            tc::mma_commit(&s_empty[s]);
            if (last) tc::mma_commit(&c_full);
          }
        }
        __syncwarp();
      }
      first = last;
      if (last) ++nrun;
      if (++q == nq) {
        q = 0;
        ++seg;
      }
    }
  } else {
    // ---- generators / drainers: tile g (64 variables), TMEM lane quarter,
    // sample half (16 of each 32-sample block); the half-0 warps drain ----
    const int gw = w - MMA_WARP - 1;  // 0..15
    const int g = (gw >> 2) & 1, shalf = gw >> 3, quarter = w & 3;
    const int r = 32 * quarter + lane;            // TMEM lane = A row
    const int vloc = 64 * g + (r & 63), tsel = r >> 6;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    int seg = seg0, q = q0, it = 0, ab = 0, nrun = 0;
    int cur_seg = -1, d = -1, rep = 0;
    float cen = 0.f;
    bool act = false;
    for (int64_t u = u0; u < u1; ++u, ++it) {
      if (seg != cur_seg) {
        cur_seg = seg;
        const int leaf = a.seg_leaf[seg];
        const int sbeg = a.scope_off[leaf] + a.seg_v0[seg];
        const int nv = min(LS_SEGV, a.scope_off[leaf + 1] - sbeg);
        rep = a.leaf_rep[leaf];
        d = vloc < nv ? a.scope_vars[sbeg + vloc] : -1;
        act = d >= 0 && a.active[d];
        cen = d >= 0 ? a.center[(int64_t)rep * D + d] : 0.f;
      }
      const int s = it % LS_STAGES, ph = (it / LS_STAGES) & 1;
      const int nb = min(LS_QB, nblk - q * LS_QB);
      const bool last = u + 1 == u1 || q + 1 == nq;
      tc::mbar_wait(&s_full[s], ph);
      const float *st = ring + (int64_t)s * stage_floats;
      for (int sb = 0; sb < nb; ++sb, ++ab) {
        const int as = ab % LS_ASTAGES, aph = (ab / LS_ASTAGES) & 1;
        tc::mbar_wait(&a_empty[as], aph ^ 1);
        tc::fence_after();
        const float *xv = st + sb * xs_floats + vloc;
        const uint32_t acol = tm + lane_off + 128 + (uint32_t)(as * 128 + g * 64);
        {
          float hv[16], lv[16];
#pragma unroll
          for (int z = 0; z < 16; ++z) {
            const float y = act ? xv[(16 * shalf + z) * LS_SEGV] - cen : 0.f;
            const float p = tsel ? y * y : y;
            tc::split_tf32(p, hv[z], lv[z]);  // round-to-nearest hi (kern_common.cuh)
          }
          tc::tmem_st16(acol + 16 * shalf, hv);
          tc::tmem_st16(acol + 32 + 16 * shalf, lv);
        }
        tc::tmem_wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) ls_arrive(&a_full[as]);
      }
      if (lane == 0) ls_arrive(&s_empty[s]);
      if (last) {
        tc::mbar_wait(&c_full, nrun & 1);
        tc::fence_after();
        const int64_t slot = blockIdx.x - ls_cta_of((int64_t)seg * nq, a.units, a.grid);
        float *dst = a.part + slot * a.n_phi;
        for (int c = 0; shalf == 0 && c < nn; c += 8) {
          float v[8];
          tc::tmem_ld8(tm + lane_off + (uint32_t)(g * nn + c), v);
          tc::tmem_wait_ld();
          if (d >= 0) {
#pragma unroll
            for (int z = 0; z < 8; ++z) {
              const int k = c + z;
              if (k < K) dst[((((int64_t)d * K + k) * a.R + rep) * 2 + tsel)] = v[z];
            }
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) ls_arrive(&c_empty);
        ++nrun;
      }
      if (++q == nq) {
        q = 0;
        ++seg;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (w == MMA_WARP) tc::tmem_dealloc(tm, 512);
}

// acc_pt[d,k,r,:] += un-centred (sum over the segment's slots of S_y, S_y2)
// for covered, unmasked (d, r); one thread per (d, k, r).
__global__ void k_leaf_stats_finish(const float *__restrict__ part, const double *__restrict__ P,
                                    const float *__restrict__ center,
                                    const int *__restrict__ leaf_of,
                                    const int *__restrict__ phi_seg,
                                    const uint8_t *__restrict__ active, double *acc_pt, int D,
                                    int K, int R, int64_t n_phi, int64_t nq, int64_t units,
                                    int grid) {
  EINET_KERNEL_PROLOGUE();
  const int64_t n = (int64_t)D * K * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int rr = (int)(e % R);
    const int k = (int)((e / R) % K);
    const int d = (int)(e / ((int64_t)R * K));
    const int l = leaf_of[(int64_t)rr * D + d];
    if (l < 0 || !active[d]) continue;
    const int64_t seg = phi_seg[(int64_t)rr * D + d];
    const int64_t c0 = ls_cta_of(seg * nq, units, grid);
    const int64_t c1 = ls_cta_of((seg + 1) * nq - 1, units, grid);
    double s0 = 0.0, s1 = 0.0;
    for (int64_t q = 0; q <= c1 - c0; ++q) {
      s0 += (double)part[q * n_phi + e * 2];
      s1 += (double)part[q * n_phi + e * 2 + 1];
    }
    const double c = (double)center[(int64_t)rr * D + d];
    const double p = P[(int64_t)l * K + k];
    acc_pt[e * 2] += s0 + c * p;
    acc_pt[e * 2 + 1] += s1 + 2.0 * c * s0 + c * c * p;
  }
}

static size_t leaf_tc_smem(int nn) {
  return (size_t)LS_STAGES * LS_QB * (32 * LS_SEGV + 2 * nn * 32) * 4;
}

bool leaf_tc_supported(const Plan &p) {
  const int nn = (p.k + 15) / 16 * 16;
  return p.use_tc && p.family == EINET_FAMILY_GAUSSIAN && p.k <= 64 && p.n_lseg > 0 &&
         leaf_tc_smem(nn) <= 220 * 1024;
}

// One CTA per SM, or the largest multiple of the segment count below it:
// then every segment is cut at the same sample blocks, so the CTAs of the
// segments covering the same image rows of neighbouring leaves walk the same
// samples at the same time -- x pieces of 96 bytes per image row and strip
// share 64-byte DRAM blocks with the next strip, which are then fetched once
// (L2) instead of once per strip (the x traffic was 1.25x the batch).
// EINET_LS_ALIGN=0 restores one CTA per SM (A/B).
static int leaf_stats_grid(const Plan &p, int64_t units) {
  int64_t g = std::min<int64_t>(units, p.num_sms);
  static const bool align = [] {
    const char *e = getenv("EINET_LS_ALIGN");
    return !(e && e[0] == '0');
  }();
  const int64_t nseg = std::max(1, p.n_lseg);
  if (align && units >= p.num_sms && nseg <= p.num_sms && units % nseg == 0)
    g = (p.num_sms / nseg) * nseg;
  g = std::max<int64_t>(g, (units + LS_MAX_RUN - 1) / LS_MAX_RUN);
  return (int)g;
}

// Upper bound of the partial slots any segment needs for batches <= B.
int64_t leaf_stats_slots(const Plan &p, int64_t B) {
  const int64_t nq = ((B + 31) / 32 + LS_QB - 1) / LS_QB;
  const int64_t nseg = std::max(1, p.n_lseg);
  int64_t best = 1;
  for (int64_t n : {nq, std::min<int64_t>(nq, (int64_t)p.num_sms)}) {
    const int64_t units = nseg * n;
    const int64_t G = leaf_stats_grid(p, units);
    const int64_t per = std::max<int64_t>(1, units / G);
    best = std::max(best, std::min<int64_t>(n, n / per + 2));
  }
  return std::max<int64_t>(best, std::min<int64_t>(nq, p.num_sms / nseg + 2));
}

int launch_leaf_stats_tc(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                         uint8_t *wsb, double *stats, const double *Pcall, cudaStream_t st,
                         cudaEvent_t p_ready) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  LeafStatsArgs a;
  a.x = x;
  a.rhob = w.rhob;
  a.center = c.center;
  a.active = c.active;
  a.scope_off = p.d_scope_off;
  a.scope_vars = p.d_scope_vars;
  a.leaf_rep = p.d_leaf_rep;
  a.seg_leaf = p.d_lseg_leaf;
  a.seg_v0 = p.d_lseg_v0;
  a.seg_vec = p.d_lseg_vec;
  a.part = (float *)w.lspart;
  a.B = B;
  a.bc = w.bc;
  a.n_phi = p.n_phi;
  a.D = p.d_vars;
  a.K = p.k;
  a.R = p.num_replicas;
  a.nn = (p.k + 15) / 16 * 16;
  a.nblk = (int)((B + 31) / 32);
  a.nq = (a.nblk + LS_QB - 1) / LS_QB;
  a.units = (int64_t)p.n_lseg * a.nq;
  a.grid = leaf_stats_grid(p, a.units);
  {
    const char *env = getenv("EINET_LS_DEBUG");
    a.debug = env ? atoi(env) : 0;
  }
  const size_t smem = leaf_tc_smem(a.nn);
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_leaf_stats_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  launch_k(k_leaf_stats_tc, a.grid, LS_THREADS, smem, st, a);
  if (p_ready) {  // P (Pcall) reduced on the reduction stream
    const int rc = check_cuda(cudaStreamWaitEvent(st, p_ready, 0), "leaf P join");
    if (rc) return rc;
  }
  const int64_t n = (int64_t)p.d_vars * p.k * p.num_replicas;
  launch_k(k_leaf_stats_finish, (int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st, 
      a.part, Pcall, c.center, p.d_leaf_of, p.d_phi_seg, c.active,
      stats + p.sizes.stats_acc_pt_offset, p.d_vars, p.k, p.num_replicas, p.n_phi, a.nq,
      a.units, a.grid);
  count_launch(2);
  return check_cuda(cudaGetLastError(), "leaf stats tc");
}

}  // namespace einet
