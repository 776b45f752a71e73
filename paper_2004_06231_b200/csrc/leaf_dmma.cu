// Gaussian leaf forward on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Reference semantics: expfam.py:153-163 (Gaussian log density) summed over a
// leaf region's scope (engine.py:154-160, log_prob on the region's variables).
//
// With y = x - c (c = per-(replica, variable) centre of the component means,
// the same centre the leaf statistics use) and m = (mu - c) * sa,
// sa = sqrt(1 / (2 var)):
//     sum_d (x sa - mu sa)^2 = sum_d  y^2 * sa^2  +  y * (-2 sa m)  +  m^2
// i.e. a GEMM  Q[b, k] = F[b, :] . G[:, k] + C[k]  with per-sample features
// F = (y_d^2, y_d) over the scope and per-component coefficients
// G = (sa^2, -2 sa m). Everything is fp64: the expanded terms are summed to
// ~1e-16 relative, far below the ~1e-12 the reference's float64 leaf rows
// carry at |log p| ~ 1e4, and the per-row constant C = sum_d m^2 (fp64,
// k_prepare_cm2) restores the direct form.
//
// B200's FP64 pipe issues DFMA and DMMA at the same peak (~18.5 T fma/s
// measured, scripts/peak_dmma.cu), but one DMMA carries 256 FMAs, so the
// tensor-core form is bounded by the FP64 pipe instead of by issue slots,
// register pressure and the fp32->fp64 converts of the SIMT kernel.
//
// Layout: G is pre-tiled in prepare into the exact B-fragment order of
// m8n8k4 (one 256-byte fragment per (k-step of 2 variables, n-tile of 8
// components)); leaf scopes are padded to 32 variables with zero coefficients,
// so one scope chunk of 32 variables is one contiguous 16*K*32-byte block.
#include <climits>
#include <cmath>

#include "kern_common.cuh"

namespace einet {

constexpr int LD_VC = 32;          // scope variables per chunk (16 k-steps)
constexpr int LD_VP = LD_VC + 2;   // padded x row (floats): conflict-free both ways

// B-fragment image: element (kstep, nt, lane) holds G[feature q][component n]
// with q = lane % 4 (variable 2*kstep + q/2 of the padded scope, feature
// q%2: 0 -> y^2 coefficient sa^2, 1 -> y coefficient -2 sa m) and
// n = 8*nt + lane/4.
__global__ void k_prepare_leaf_img(const double2 *__restrict__ lp, const float *__restrict__ center,
                                   const int *__restrict__ scope_off,
                                   const int *__restrict__ scope_vars, const int *leaf_rep,
                                   const int *__restrict__ pvo, int n_leaf, int D, int K,
                                   double *__restrict__ img, int64_t n_img) {
  EINET_KERNEL_PROLOGUE();
  const int NT = K / 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_img;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31);
    const int nt = (int)((e >> 5) % NT);
    const int64_t kstep = (e >> 5) / NT;
    const int pv = (int)(2 * kstep) + ((lane & 3) >> 1);
    int lo = 0, hi = n_leaf;  // leaf with pvo[leaf] <= pv < pvo[leaf + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pvo[mid] <= pv) lo = mid;
      else hi = mid;
    }
    const int leaf = lo, v = pv - pvo[leaf];
    double val = 0.0;
    if (v < scope_off[leaf + 1] - scope_off[leaf]) {
      const int d = scope_vars[scope_off[leaf] + v], r = leaf_rep[leaf];
      const int k = nt * 8 + (lane >> 2);
      const double2 q = lp[((int64_t)r * D + d) * K + k];
      const double sa = q.x, m = -fma((double)center[(int64_t)r * D + d], sa, q.y);
      val = (lane & 1) ? -2.0 * sa * m : sa * sa;
    }
    img[e] = val;
  }
}

// C[leaf, k] = sum over the scope of m^2 (fixed-order tree), grid (n_leaf, K).
__global__ void __launch_bounds__(256) k_prepare_cm2(const double2 *__restrict__ lp,
                                                     const float *__restrict__ center,
                                                     const int *scope_off, const int *scope_vars,
                                                     const int *leaf_rep, int D, int K,
                                                     double *cm2) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[8];
  const int leaf = blockIdx.x, k = blockIdx.y, r = leaf_rep[leaf];
  double acc = 0.0;
  for (int q = scope_off[leaf] + threadIdx.x; q < scope_off[leaf + 1]; q += 256) {
    const int d = scope_vars[q];
    const double2 p = lp[((int64_t)r * D + d) * K + k];
    const double m = -fma((double)center[(int64_t)r * D + d], p.x, p.y);
    acc += __dmul_rn(m, m);  // rounded square: the fused M-step's order (mstep.cu)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    cm2[leaf * K + k] = s;
  }
}

int launch_prepare_leaf_dmma(Plan &p, uint8_t *compute, cudaStream_t st) {
  if (!p.leaf_dmma) return 0;
  CompView c = comp_view(p, compute);
  const int64_t n_img = (int64_t)p.h_leaf_pvo.back() * 2 * p.k;
  launch_k(k_prepare_leaf_img, (int)std::min<int64_t>((n_img + 255) / 256, 8192), 256, 0, st, 
      (const double2 *)c.leafp, c.center, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep,
      p.d_leaf_pvo, p.n_leaf, p.d_vars, p.k, c.leafimg, n_img);
  launch_k(k_prepare_cm2, dim3(p.n_leaf, p.k), 256, 0, st, (const double2 *)c.leafp, c.center,
                                                      p.d_scope_off, p.d_scope_vars,
                                                      p.d_leaf_rep, p.d_vars, p.k, c.cm2);
  count_launch(2);
  return check_cuda(cudaGetLastError(), "leaf DMMA image");
}

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Q[b, leaf, k] partial over one split of the scope -> part[split][leaf][b][k].
// grid (ceil(B/TBS), n_leaf, dsplit), block 32*WARPS (warps x 8*MT samples each).
// Per chunk of 32 variables: x gathered with cp.async ([sample][var], padded),
// the 16*K*32-byte image chunk copied with 16-byte cp.async, both double
// buffered; warp tile = 8*MT samples x K components, MT*NT fragments.
template <int NT, int MT, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 8 / WARPS + 1) k_leaf_fwd_dmma(
    const float *__restrict__ x, int64_t B, int D, const int *__restrict__ scope_off,
    const int *__restrict__ scope_vars, const int *__restrict__ leaf_rep,
    const int *__restrict__ pvo, const double *__restrict__ img, const float *__restrict__ center,
    const double *__restrict__ cm2, const uint8_t *__restrict__ active, double *__restrict__ part,
    int64_t Bc, int n_leaf, int dsplit, int32_t *status, const int *gate) {
  EINET_KERNEL_PROLOGUE();
  if (gate && *(volatile const int *)gate == 0) return;  // the INT8 pass covered the batch
  constexpr int K = NT * 8;
  constexpr int TBS = WARPS * 8 * MT;
  constexpr int IS = (LD_VC / 2) * NT * 32;  // doubles per image chunk
  constexpr int XS = TBS * LD_VP;            // floats per x chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *is = (double *)smem_raw;                 // [2][IS]
  float *xs = (float *)(is + 2 * IS);              // [2][TBS][VP]
  float *cs = xs + 2 * XS;                         // [2][VC]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int leaf = blockIdx.y, split = blockIdx.z;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int nch = (slen + LD_VC - 1) / LD_VC;
  const int per = (nch + dsplit - 1) / dsplit;
  const int ch0 = split * per, ch1 = min(nch, ch0 + per);
  const int r = leaf_rep[leaf];
  const int64_t b0 = (int64_t)blockIdx.x * TBS;
  const int nbl = (int)min((int64_t)TBS, B - b0);
  const double *limg = img + (int64_t)(pvo[leaf] / 2) * NT * 32;
  // unmasked compute: x goes straight into the contraction; a non-finite value
  // makes the leaf row non-finite, which k_leaf_finalize flags for k_leaf_check
  const bool masked = active[D] != 0;

  auto stage = [&](int buf, int ch) {
    const int c0 = ch * LD_VC, nv = min(LD_VC, slen - c0);
    float *xb = xs + buf * XS;
    if (lane < nv) {
      const int d = scope_vars[sbeg + c0 + lane];
      const float *src = x + b0 * D + d;
      for (int bl = warp; bl < TBS; bl += WARPS) {
        if (bl < nbl) cp_async4(xb + bl * LD_VP + lane, src + (int64_t)bl * D);
        else xb[bl * LD_VP + lane] = 0.f;
      }
      if (warp == 0) cs[buf * LD_VC + lane] = center[(int64_t)r * D + d];
    } else {
      for (int bl = warp; bl < TBS; bl += WARPS) xb[bl * LD_VP + lane] = 0.f;
      if (warp == 0) cs[buf * LD_VC + lane] = 0.f;
    }
    const double *src = limg + (int64_t)ch * IS;
    double *dst = is + buf * IS;
    for (int e = tid; e < IS / 2; e += 32 * WARPS) cp_async16(dst + 2 * e, src + 2 * e);
    cp_async_commit();
  };
  // masked / non-finite entries -> 0 (their coefficients are 0 for masked
  // variables); an active non-finite value raises the support error.
  auto fixup = [&](int buf, int ch) {
    const int c0 = ch * LD_VC, nv = min(LD_VC, slen - c0);
    if (lane >= nv) return;
    const int d = scope_vars[sbeg + c0 + lane];
    const bool act = active[d] != 0;
    float *xb = xs + buf * XS + lane;
    for (int bl = warp; bl < nbl; bl += WARPS) {
      const float xv = xb[bl * LD_VP];
      if (!act || !isfinite(xv)) {
        if (act) atomicMin(&status[0], d);
        xb[bl * LD_VP] = 0.f;
      }
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    double c0 = 0.0, c1 = 0.0;
    if (split == 0) {
      c0 = cm2[leaf * K + nt * 8 + 2 * q];
      c1 = cm2[leaf * K + nt * 8 + 2 * q + 1];
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      acc[mt][nt][0] = c0;
      acc[mt][nt][1] = c1;
    }
  }

  const int wrow = warp * 8 * MT + g;  // this thread's A-fragment sample rows: wrow + 8*mt
  if (ch0 < ch1) stage(0, ch0);
  int it = 0;
  for (int ch = ch0; ch < ch1; ++ch, ++it) {
    const int buf = it & 1;
    if (ch + 1 < ch1) {
      stage(buf ^ 1, ch + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if (masked) fixup(buf, ch);
    __syncthreads();
    const double *ib = is + buf * IS;
    const float *xb = xs + buf * XS;
    const float *cb = cs + buf * LD_VC;
#pragma unroll 2
    for (int s = 0; s < LD_VC / 2; ++s) {
      double bf[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = ib[(s * NT + nt) * 32 + lane];
      const int vv = 2 * s + (q >> 1);
      const double cc = (double)cb[vv];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double y = (double)xb[(wrow + 8 * mt) * LD_VP + vv] - cc;
        const double a = (q & 1) ? y : y * y;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a, bf[nt]);
      }
    }
    __syncthreads();
  }

  // C fragment: row g (sample), columns 2q, 2q+1 of each n-tile
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int64_t b = b0 + wrow + 8 * mt;
    if (b >= B) continue;
    double *dst = part + (((int64_t)split * n_leaf + leaf) * Bc + b) * K + 2 * q;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      *(double2 *)(dst + nt * 8) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
  }
}

template <int NT, int MT, int WARPS>
static size_t fwd_dmma_smem() {
  return 2 * sizeof(double) * (LD_VC / 2) * NT * 32 +
         2 * sizeof(float) * (WARPS * 8 * MT * LD_VP + LD_VC);
}

// (resident CTAs, split, wave efficiency) of one CTA shape for this batch
template <int NT, int MT, int WARPS>
static double fwd_dmma_shape(const Plan &p, int64_t B, int *ds_out) {
  constexpr int TBS = WARPS * 8 * MT;
  const size_t smem = fwd_dmma_smem<NT, MT, WARPS>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_leaf_fwd_dmma<NT, MT, WARPS>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t tiles = (int64_t)ceil_div(B, TBS) * p.n_leaf;
  const int64_t slots =
      device_slots((const void *)k_leaf_fwd_dmma<NT, MT, WARPS>, 32 * WARPS, smem, p.num_sms);
  // at least 4 chunks of 32 variables per split keep the double buffer busy
  const int cap = std::max(1, std::min(kMaxDSplit, ceil_div(p.max_scope, LD_VC) / 4));
  const int ds = pick_split(tiles, slots, 1, cap, 0.90);
  *ds_out = ds;
  const int64_t n = tiles * ds;
  return (double)n / (double)(ceil_div(n, slots) * slots);
}

template <int NT, int MT, int WARPS>
static void launch_fwd_dmma_t(Plan &p, const CompView &c, const float *x, int64_t B,
                              const WsView &w, int32_t *status, cudaStream_t st, int ds,
                              const int *gate) {
  constexpr int TBS = WARPS * 8 * MT;
  dim3 grid(ceil_div(B, TBS), p.n_leaf, ds);
  launch_k(k_leaf_fwd_dmma<NT, MT, WARPS>, grid, 32 * WARPS, fwd_dmma_smem<NT, MT, WARPS>(), st, 
      x, B, p.d_vars, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep, p.d_leaf_pvo, c.leafimg,
      c.center, c.cm2, c.active, w.leafpart, w.bc, p.n_leaf, ds, status, gate);
}

// 8-warp CTAs reuse each coefficient fragment over more samples; 4-warp CTAs
// quantise the grid more finely. Take the 8-warp shape unless the 4-warp one
// fills the waves clearly better.
template <int NT, int MT>
static int launch_fwd_dmma_nt(Plan &p, const CompView &c, const float *x, int64_t B,
                              const WsView &w, int32_t *status, cudaStream_t st, int *ds_out,
                              const int *gate) {
  int ds8, ds4;
  const double e8 = fwd_dmma_shape<NT, MT, 8>(p, B, &ds8);
  const double e4 = fwd_dmma_shape<NT, MT, 4>(p, B, &ds4);
  if (e4 > e8 + 0.03) {
    launch_fwd_dmma_t<NT, MT, 4>(p, c, x, B, w, status, st, ds4, gate);
    *ds_out = ds4;
  } else {
    launch_fwd_dmma_t<NT, MT, 8>(p, c, x, B, w, status, st, ds8, gate);
    *ds_out = ds8;
  }
  return 0;
}

int launch_leaf_fwd_dmma(Plan &p, const CompView &c, const float *x, int64_t B, const WsView &w,
                         int32_t *status, cudaStream_t st, int *ds_out, const int *gate) {
  switch (p.k / 8) {
    case 1: return launch_fwd_dmma_nt<1, 4>(p, c, x, B, w, status, st, ds_out, gate);
    case 2: return launch_fwd_dmma_nt<2, 4>(p, c, x, B, w, status, st, ds_out, gate);
    case 3: return launch_fwd_dmma_nt<3, 4>(p, c, x, B, w, status, st, ds_out, gate);
    case 4: return launch_fwd_dmma_nt<4, 4>(p, c, x, B, w, status, st, ds_out, gate);
    case 5: return launch_fwd_dmma_nt<5, 4>(p, c, x, B, w, status, st, ds_out, gate);
    case 6: return launch_fwd_dmma_nt<6, 2>(p, c, x, B, w, status, st, ds_out, gate);
    case 7: return launch_fwd_dmma_nt<7, 2>(p, c, x, B, w, status, st, ds_out, gate);
    case 8: return launch_fwd_dmma_nt<8, 2>(p, c, x, B, w, status, st, ds_out, gate);
    default: return fail(EINET_ERR_UNSUPPORTED, "DMMA leaf forward needs K % 8 == 0, K <= 64");
  }
}

}  // namespace einet
