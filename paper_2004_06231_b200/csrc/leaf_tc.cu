// Gaussian leaf statistics on tcgen05 (engine.py:318-327):
//   S[(v, t), k] = sum_b y_bv^(t+1) rho[b,l,k],  y = x - c_d  (c = stats centre)
// as a batch-reduction GEMM: M = 64 scope variables x {y, y^2}, N = K (padded
// to 16), reduction over samples in 32-sample blocks. The A operand is built in
// registers from a cp.async-gathered x block and stored to TMEM (tcgen05.st);
// the rho block (32-sample transposed layout) is the B operand in smem; 3xTF32
// MMAs accumulate in TMEM and drain to fp64 every 8 blocks. The centred sums of
// all batch splits are reduced and un-centred once per call:
//   sum rho x = S_y + c P,  sum rho x^2 = S_y2 + 2 c S_y + c^2 P.
#include <climits>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

namespace {

constexpr int LT_BLK = 32;    // samples per block (MMA K of 4 steps)
constexpr int LT_VARS = 64;   // scope variables per CTA (128 rows: y and y^2)
constexpr int LT_DRAIN = 8;

__device__ __forceinline__ void cpa4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(tc::smem_u32(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cpa16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int XROW = 36;  // padded x row (16-byte aligned, spreads the gather's banks)

int64_t leaf_tc_smem(int K, int nn) {
  return 2LL * LT_VARS * XROW * 4 + 2LL * K * LT_BLK * 4 + 2LL * 2 * nn * LT_BLK * 4;
}

}  // namespace

// grid (ceil(max_scope/64), n_leaf, lsplit), block 256
__global__ void __launch_bounds__(256, 1) k_leaf_stats_tc(
    const float *__restrict__ x, int64_t B, int D, int K, int R, int nn,
    const int *__restrict__ scope_off, const int *__restrict__ scope_vars,
    const int *__restrict__ leaf_rep, const float *__restrict__ rho, int64_t Bc,
    const float *__restrict__ center, const uint8_t *__restrict__ active, double *lspart,
    int64_t n_phi, int lsplit) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tbase;
  __shared__ int dv[LT_VARS];
  const int leaf = blockIdx.y, split = blockIdx.z;
  const int t = threadIdx.x, w = t >> 5, h = t >> 7, r = t & 127;
  const int v = r & (LT_VARS - 1), tsel = r >> 6;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int v0 = blockIdx.x * LT_VARS;
  if (v0 >= slen) return;
  const int nv = min(LT_VARS, slen - v0);
  const int rep = leaf_rep[leaf];
  float *xs = (float *)sm;                              // [2][64][XROW]
  float *rs = xs + 2 * LT_VARS * XROW;                  // [2][K][32]
  float *bbuf = rs + 2 * K * LT_BLK;                    // [2][hi|lo][nn x 32]
  const int64_t nblk = (B + LT_BLK - 1) / LT_BLK;
  const int64_t per = (nblk + lsplit - 1) / lsplit;
  const int64_t blk0 = split * per, blk1 = min(nblk, blk0 + per);
  const int nstages = (int)max((int64_t)0, blk1 - blk0);
  const int half = nn / 2;
  if (t < LT_VARS) dv[t] = t < nv ? scope_vars[sbeg + v0 + t] : -1;
  if (w == 0) tc::tmem_alloc(&tbase, 256);
  if (t == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::mbar_fence_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const int d_mine = dv[v];
  const bool act = d_mine >= 0 && active[d_mine];
  const float cmine = d_mine >= 0 ? center[(int64_t)rep * D + d_mine] : 0.f;
  const float *rl = rho + (int64_t)leaf * Bc * K;
  auto prefetch = [&](int q) {
    const int qb = q & 1;
    const int64_t b0 = (blk0 + q) * LT_BLK;
    const int nb = (int)min((int64_t)LT_BLK, B - b0);
    float *xb = xs + qb * LT_VARS * XROW;
    for (int e = t; e < LT_VARS * LT_BLK; e += 256) {
      const int vv = e & (LT_VARS - 1), s = e >> 6;
      const int d = dv[vv];
      if (d >= 0 && s < nb) cpa4(xb + vv * XROW + s, x + (b0 + s) * D + d);
      else xb[vv * XROW + s] = 0.f;
    }
    float *rb = rs + qb * K * LT_BLK;
    const float *src = rl + b0 * K;  // block of K rows x 32 samples
    for (int e = t; e < K * (LT_BLK / 4); e += 256) cpa16(rb + 4 * e, src + 4 * e);
    cpa_commit();
  };
  if (nstages > 0) prefetch(0);
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * (w & 3)) << 16;
  double red[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) red[c] = 0.0;
  for (int q = 0; q < nstages; ++q) {
    const int qb = q & 1;
    const int nb = (int)min((int64_t)LT_BLK, B - (blk0 + q) * LT_BLK);
    if (q + 1 < nstages) {
      prefetch(q + 1);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    if (q >= 2) tc::mbar_wait(&mbar[qb], ((q - 2) >> 1) & 1);
    tc::fence_after();
    {
      const float *xrow = xs + qb * LT_VARS * XROW + v * XROW + 16 * h;
      float hv[16], lv[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 x4 = *(const float4 *)(xrow + 4 * u);
        const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const float y = (act && 16 * h + 4 * u + z < nb) ? xv[z] - cmine : 0.f;
          tc::split_tf32(tsel ? y * y : y, hv[4 * u + z], lv[4 * u + z]);
        }
      }
      const uint32_t acol = 64 + qb * 64 + 16 * h;
      tc::tmem_st16(tm + lane_base + acol, hv);
      tc::tmem_st16(tm + lane_base + acol + 32, lv);
    }
    const float *rb = rs + qb * K * LT_BLK;
    float *bhi = bbuf + qb * 2 * nn * LT_BLK, *blo = bhi + nn * LT_BLK;
    for (int e = t; e < nn * (LT_BLK / 4); e += 256) {
      const int n = e >> 3, c = (e & 7) * 4;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < K) {
        val = *(const float4 *)(rb + n * LT_BLK + c);
        if (c + 0 >= nb) val.x = 0.f;
        if (c + 1 >= nb) val.y = 0.f;
        if (c + 2 >= nb) val.z = 0.f;
        if (c + 3 >= nb) val.w = 0.f;
      }
      float4 hh, ll;
      tc::split_tf32(val.x, hh.x, ll.x);
      tc::split_tf32(val.y, hh.y, ll.y);
      tc::split_tf32(val.z, hh.z, ll.z);
      tc::split_tf32(val.w, hh.w, ll.w);
      const uint32_t o = tc::kmaj_off(n, c, nn) / 4;
      *(float4 *)(bhi + o) = hh;
      *(float4 *)(blo + o) = ll;
    }
    tc::tmem_wait_st();
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
      const uint32_t id = tc::idesc_tf32(128, nn);
      const uint32_t bh = tc::smem_u32(bhi), bl = tc::smem_u32(blo);
      const uint32_t ah = tm + 64 + qb * 64;
      const bool acc0 = (q % LT_DRAIN) != 0;
#pragma unroll
      for (int s = 0; s < LT_BLK / 8; ++s) {
        tc::mma_tf32_ts(tm, ah + 8 * s, tc::kstep_desc(bh, nn, s), id, (s > 0 || acc0) ? 1u : 0u);
        tc::mma_tf32_ts(tm, ah + 8 * s, tc::kstep_desc(bl, nn, s), id, 1u);
        tc::mma_tf32_ts(tm, ah + 32 + 8 * s, tc::kstep_desc(bh, nn, s), id, 1u);
      }
      tc::mma_commit(&mbar[qb]);
    }
    if ((q % LT_DRAIN) == LT_DRAIN - 1 || q == nstages - 1) {
      tc::mbar_wait(&mbar[qb], (q >> 1) & 1);
      tc::fence_after();
      for (int c = 0; c < half; c += 8) {
        float vv[8];
        tc::tmem_ld8(tm + lane_base + h * half + c, vv);
        tc::tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) red[c + u] += (double)vv[u];
      }
      tc::fence_before();
    }
  }
  if (v < nv) {
    for (int c = 0; c < half; ++c) {
      const int k = h * half + c;
      if (k < K)
        lspart[(int64_t)split * n_phi + ((((int64_t)d_mine * K + k) * R + rep) * 2 + tsel)] =
            red[c];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tm, 256);
}

// acc_pt[d,k,r,:] += un-centred (S_y, S_y2) for covered, unmasked (d, r).
__global__ void k_leaf_uncenter(const double *__restrict__ S, const double *__restrict__ P,
                                const float *__restrict__ center, const int *__restrict__ leaf_of,
                                const uint8_t *__restrict__ active, double *acc_pt, int D, int K,
                                int R) {
  const int64_t n = (int64_t)D * K * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int rr = (int)(e % R);
    const int k = (int)((e / R) % K);
    const int d = (int)(e / ((int64_t)R * K));
    const int l = leaf_of[(int64_t)rr * D + d];
    if (l < 0 || !active[d]) continue;
    const double c = (double)center[(int64_t)rr * D + d];
    const double p = P[(int64_t)l * K + k];
    const double s0 = S[e * 2], s1 = S[e * 2 + 1];
    acc_pt[e * 2] += s0 + c * p;
    acc_pt[e * 2 + 1] += s1 + 2.0 * c * s0 + c * c * p;
  }
}

bool leaf_tc_supported(const Plan &p) {
  return p.use_tc && p.family == EINET_FAMILY_GAUSSIAN && p.k <= 64 &&
         leaf_tc_smem(p.k, (p.k + 15) / 16 * 16) <= 200 * 1024;
}

int launch_leaf_stats_tc(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                         uint8_t *wsb, double *stats, const double *Pcall, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  const int K = p.k, nn = (K + 15) / 16 * 16;
  const int vchunks = ceil_div(p.max_scope, LT_VARS);
  const int64_t ctas = (int64_t)vchunks * p.n_leaf;
  const int64_t nblk = (B + LT_BLK - 1) / LT_BLK;
  const int64_t smem = leaf_tc_smem(K, nn);
  cudaFuncSetAttribute(k_leaf_stats_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int ls = pick_split(ctas, device_slots((const void *)k_leaf_stats_tc, 256, smem, p.num_sms), 1,
                      (int)std::min<int64_t>(nblk, p.max_lsplit));
  const int64_t per = (nblk + ls - 1) / ls;
  ls = (int)((nblk + per - 1) / per);
  dim3 grid(vchunks, p.n_leaf, ls);
  k_leaf_stats_tc<<<grid, 256, smem, st>>>(x, B, p.d_vars, K, p.num_replicas, nn, p.d_scope_off,
                                           p.d_scope_vars, p.d_leaf_rep, w.rho, w.bc, c.center,
                                           c.active, w.lspart, p.n_phi, ls);
  double *S = (double *)(wsb + p.w_tmp_s);
  launch_reduce_partials_store(S, w.lspart, ls, p.n_phi, p.n_phi, st);
  const int64_t n = (int64_t)p.d_vars * K * p.num_replicas;
  k_leaf_uncenter<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(
      S, Pcall, c.center, p.d_leaf_of, c.active, stats + p.sizes.stats_acc_pt_offset, p.d_vars,
      K, p.num_replicas);
  count_launch(2);
  return check_cuda(cudaGetLastError(), "leaf stats tc");
}

}  // namespace einet
