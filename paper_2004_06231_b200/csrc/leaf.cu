// Exponential-family leaf kernels: parameter preparation, leaf-region forward,
// leaf responsibilities and leaf sufficient statistics.
//
// Reference semantics: expfam.py:82-309 (log densities, projections),
// engine.py:318-327 (leaf statistics). The per-variable tensor E of
// ef_log_prob (expfam.py:288) is never materialised on the hot path: the
// leaf-region rows are accumulated straight from x.
//
// Gaussian leaves use the direct form  -(x-mu)^2/(2 var) = -(x*sa + nmsa)^2
// with sa = sqrt(1/(2 var)), nmsa = -mu*sa (two FFMA per (sample, var, k)),
// plus a per-(leaf, k) constant sum_d -0.5(log 2pi + log var) kept in fp64.
// fp32 partial sums over chunks of 32 variables are folded into fp64, so the
// leaf row is accurate to ~1e-5 absolute even at |log p| ~ 1e4.
#include <climits>
#include <cmath>
#include <cstdlib>

#include "kern_common.cuh"

namespace einet {

constexpr int LF_KPT = 8;    // k entries per thread
constexpr int LF_NS = 4;     // samples per thread
constexpr int LF_VC = 32;    // variables per shared-memory chunk
constexpr int LF_TB = 32 * LF_NS;  // samples per CTA

// ---------------------------------------------------------------------------
// parameter preparation (master fp64 -> device compute tensors)
// ---------------------------------------------------------------------------

__global__ void k_to_f32(const double *__restrict__ src, float *__restrict__ dst, int64_t n) {
  EINET_KERNEL_PROLOGUE();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

// active[d] = not marginalised; active[D] = 1 when a mask was given (the DMMA
// leaf forward then zeroes masked / non-finite x before the contraction).
__global__ void k_prepare_active(const uint8_t *mask, uint8_t *active, int D) {
  EINET_KERNEL_PROLOGUE();
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < D) active[d] = mask ? (mask[d] ? 0 : 1) : 1;
  if (d == 0) active[D] = mask ? 1 : 0;
}

// phi (D,K,R,2) = (mean, second moment) -> fp64 (sa, -mu*sa), [r][d][k]
__global__ void k_prepare_gauss(const double *__restrict__ phi, const uint8_t *active,
                                double2 *lp, float *center, int D, int K, int R) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = (int64_t)R * D * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(e % K);
    int d = (int)((e / K) % D);
    int r = (int)(e / ((int64_t)K * D));
    const double *ph = phi + (((int64_t)d * K + k) * R + r) * 2;
    double mu = ph[0];
    double var = ph[1] - mu * mu;
    double sa = sqrt(0.5 / var);
    double2 v = make_double2(0.0, 0.0);
    if (active[d]) v = make_double2(sa, -mu * sa);
    lp[e] = v;
  }
}

// categorical: log phi per state, [r][d][k][s]; masked variables -> 0
__global__ void k_prepare_cat(const double *__restrict__ phi, const uint8_t *active, double *lp,
                              int D, int K, int R, int S) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = (int64_t)R * D * K * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int s = (int)(e % S);
    int64_t q = e / S;
    int k = (int)(q % K);
    int d = (int)((q / K) % D);
    int r = (int)(q / ((int64_t)K * D));
    double p = phi[(((int64_t)d * K + k) * R + r) * S + s];
    lp[e] = active[d] ? log(p) : 0.0;
  }
}

// binomial: (theta, A) with log p(x) = log h(x) + x*theta + A
__global__ void k_prepare_binom(const double *__restrict__ phi, const uint8_t *active,
                                double2 *lp, int D, int K, int R, int n_trials) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = (int64_t)R * D * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(e % K);
    int d = (int)((e / K) % D);
    int r = (int)(e / ((int64_t)K * D));
    double p = phi[((int64_t)d * K + k) * R + r] / (double)n_trials;
    double l1 = log1p(-p);
    double2 v = make_double2(0.0, 0.0);
    if (active[d]) v = make_double2(log(p) - l1, n_trials * l1);
    lp[e] = v;
  }
}

__global__ void k_prepare_logh(double *logh, int n) {
  EINET_KERNEL_PROLOGUE();
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x <= n) logh[x] = lgamma((double)n + 1.0) - lgamma((double)x + 1.0) -
                        lgamma((double)(n - x) + 1.0);
}

// per (leaf, k): sum over the unmasked scope of the k-only terms, in fp64.
// grid (n_leaf, K), block 256: strided partial sums + fixed-order tree.
__global__ void __launch_bounds__(256) k_prepare_const(
    const double *__restrict__ phi, const uint8_t *active, const double *leaf_offset,
    const int *scope_off, const int *scope_vars, const int *leaf_rep, double *cnst, int D,
    int K, int R, int family) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[8];
  const int leaf = blockIdx.x, k = blockIdx.y;
  const int r = leaf_rep[leaf];
  double acc = 0.0;
  for (int q = scope_off[leaf] + threadIdx.x; q < scope_off[leaf + 1]; q += 256) {
    const int d = scope_vars[q];
    if (!active[d]) continue;
    const int64_t base = ((int64_t)d * K + k) * R + r;
    if (family == EINET_FAMILY_GAUSSIAN) {
      const double mu = phi[base * 2], var = phi[base * 2 + 1] - mu * mu;
      acc += -0.5 * (kLog2Pi + log(var));
    }
    if (leaf_offset) acc += leaf_offset[base];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    cnst[leaf * K + k] = s;
  }
}

// Gaussian statistics centre per (r, d): mean over k of the component means.
// Centring the fp32 batch partial sums keeps E[x^2] - E[x]^2 well conditioned.
// Gaussian statistics centre per (r, d): mean over k of the component means.
// Centring the fp32 batch partial sums keeps E[x^2] - E[x]^2 well conditioned.
// One warp per (r, d), lanes over k, xor-butterfly: the summation order of the
// fused M-step (mstep.cu k_mstep_leaf_gauss), so a re-prepared compute buffer
// equals the one the M-step left behind bit for bit.
__global__ void __launch_bounds__(256) k_prepare_center(const double *__restrict__ phi,
                                                        float *center, int D, int K, int R) {
  EINET_KERNEL_PROLOGUE();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)R * D) return;
  const int d = (int)(w % D), r = (int)(w / D);
  double s = 0.0;
  for (int k = lane; k < K; k += 32) s += phi[(((int64_t)d * K + k) * R + r) * 2];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) center[w] = (float)(s / K);
}

int launch_prepare(Plan &p, const double *params, uint8_t *compute, const uint8_t *mask,
                   const double *leaf_offset, cudaStream_t st) {
  ProfScope prof("prepare", st);
  CompView c = comp_view(p, compute);
  const int D = p.d_vars, K = p.k, R = p.num_replicas;
  const double *phi = params + p.sizes.phi_offset;
  auto grid_for = [](int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 4096); };
  if (p.n_w) launch_k(k_to_f32, grid_for(p.n_w), 256, 0, st, params, c.w32, p.n_w);
  if (p.n_mix) launch_k(k_to_f32, grid_for(p.n_mix), 256, 0, st, params + p.n_w, c.mix32, p.n_mix);
  launch_k(k_prepare_active, ceil_div(D, 256), 256, 0, st, mask, c.active, D);
  const int64_t rdk = (int64_t)R * D * K;
  if (p.family == EINET_FAMILY_GAUSSIAN) {
    launch_k(k_prepare_gauss, grid_for(rdk), 256, 0, st, phi, c.active, (double2 *)c.leafp,
                                                   c.center, D, K, R);
  } else if (p.family == EINET_FAMILY_CATEGORICAL) {
    launch_k(k_prepare_cat, grid_for(rdk * p.num_states), 256, 0, st, phi, c.active, (double *)c.leafp,
                                                               D, K, R, p.num_states);
  } else {
    launch_k(k_prepare_binom, grid_for(rdk), 256, 0, st, phi, c.active, (double2 *)c.leafp, D, K, R,
                                                   p.n_trials);
    launch_k(k_prepare_logh, ceil_div(p.n_trials + 1, 256), 256, 0, st, c.logh, p.n_trials);
    count_launch();
  }
  launch_k(k_prepare_const, dim3(p.n_leaf, K), 256, 0, st, phi, c.active, leaf_offset,
                                                     p.d_scope_off, p.d_scope_vars, p.d_leaf_rep,
                                                     c.cnst, D, K, R, p.family);
  if (p.family == EINET_FAMILY_GAUSSIAN) {
    launch_k(k_prepare_center, ceil_div((int64_t)R * D * 32, 256), 256, 0, st, phi, c.center, D, K, R);
    count_launch();
  }
  count_launch((p.n_w ? 1 : 0) + (p.n_mix ? 1 : 0) + 3);
  int rc = launch_prepare_tc_tiles(p, compute, st);
  if (rc) return rc;
  if ((rc = launch_prepare_leaf_dmma(p, compute, st))) return rc;
  if ((rc = launch_prepare_leaf_i8(p, compute, st))) return rc;
  return check_cuda(cudaGetLastError(), "prepare kernels");
}

// Leaf compute tensors only (categorical / binomial families after the
// M-step): the einsum and mixing compute copies are written by the M-step
// kernels themselves, and the training compute is unmasked (c.active stays
// all ones), so only the per-(d, k, r) leaf terms and the per-leaf constants
// are re-derived.
int launch_prepare_leaves(Plan &p, const double *params, uint8_t *compute, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  const int D = p.d_vars, K = p.k, R = p.num_replicas;
  const double *phi = params + p.sizes.phi_offset;
  auto grid_for = [](int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 4096); };
  const int64_t rdk = (int64_t)R * D * K;
  if (p.family == EINET_FAMILY_CATEGORICAL) {
    launch_k(k_prepare_cat, grid_for(rdk * p.num_states), 256, 0, st, phi, c.active,
             (double *)c.leafp, D, K, R, p.num_states);
  } else if (p.family == EINET_FAMILY_BINOMIAL) {
    launch_k(k_prepare_binom, grid_for(rdk), 256, 0, st, phi, c.active, (double2 *)c.leafp, D, K,
             R, p.n_trials);
  } else {
    return fail(EINET_ERR_USAGE, "launch_prepare_leaves: categorical / binomial only");
  }
  launch_k(k_prepare_const, dim3(p.n_leaf, K), 256, 0, st, phi, c.active, (const double *)nullptr,
           p.d_scope_off, p.d_scope_vars, p.d_leaf_rep, c.cnst, D, K, R, p.family);
  count_launch(2);
  return check_cuda(cudaGetLastError(), "prepare leaves");
}

// ---------------------------------------------------------------------------
// leaf forward
// ---------------------------------------------------------------------------

// Gaussian: Q[b,l,k] = sum_{d in scope} (x_bd*sa_dk + nmsa_dk)^2 with two fp64 FMAs
// per term (B200 FP64 runs at half the FP32 rate): the leaf rows, whose
// differences drive every posterior, stay exact to ~1e-12 even at |log p| ~ 1e4.
// grid (ceil(B/128), n_leaf, dsplit*nkc), block 32*KG threads (KG = ceil(K/8) <= 8).
// Chunks of 32 scope variables are gathered with cp.async into a double buffer
// so the next chunk's loads overlap the current chunk's FMAs.
__global__ void __launch_bounds__(256) k_leaf_fwd_gauss(
    const float *__restrict__ x, int64_t B, int D, int K, int R,
    const int *__restrict__ scope_off, const int *__restrict__ scope_vars,
    const int *__restrict__ leaf_rep, const double2 *__restrict__ lp,
    const uint8_t *__restrict__ active, double *__restrict__ part, int64_t Bc, int n_leaf,
    int dsplit, int32_t *status, const int *gate) {
  EINET_KERNEL_PROLOGUE();
  if (gate && *(volatile const int *)gate == 0) return;  // the INT8 pass covered the batch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int KG = blockDim.x / 32;
  const int KP = KG * LF_KPT;
  constexpr int XS = LF_VC * (LF_TB + 1);                      // floats per x buffer
  float *xs = (float *)smem_raw;                               // [2][VC][TB+1]
  double2 *ps = (double2 *)(smem_raw + ((2 * XS * 4 + 15) & ~15));  // [2][VC][KP]
  const int nkc = gridDim.z / dsplit;  // k chunks of KP entries
  const int leaf = blockIdx.y, split = blockIdx.z / nkc;
  const int kbase = (blockIdx.z % nkc) * KP;
  const int lane = threadIdx.x & 31, kq = threadIdx.x >> 5;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int per = (slen + dsplit - 1) / dsplit;
  const int vbeg = split * per, vend = min(slen, vbeg + per);
  const int r = leaf_rep[leaf];
  const int64_t b0 = (int64_t)blockIdx.x * LF_TB;
  const int nbl = (int)min((int64_t)LF_TB, B - b0);

  // thread -> (variable lane, sample rows) of the gather; fixed across chunks
  auto stage = [&](int buf, int c0) {
    const int nv = min(LF_VC, vend - c0);
    float *xb = xs + buf * XS;
    const int v = lane;
    if (v < nv) {
      const int d = scope_vars[sbeg + c0 + v];
      const float *src = x + b0 * D + d;
      for (int bl = kq; bl < LF_TB; bl += KG) {
        if (bl < nbl) cp_async4(xb + v * (LF_TB + 1) + bl, src + (int64_t)bl * D);
        else xb[v * (LF_TB + 1) + bl] = 0.f;
      }
    } else {
      for (int bl = kq; bl < LF_TB; bl += KG) xb[v * (LF_TB + 1) + bl] = 0.f;
    }
    double2 *pb = ps + buf * LF_VC * KP;
    for (int e = threadIdx.x; e < LF_VC * KP; e += blockDim.x) {
      const int vv = e / KP, k = e % KP;
      if (vv < nv && kbase + k < K)
        cp_async16(pb + e, lp + ((int64_t)r * D + scope_vars[sbeg + c0 + vv]) * K + kbase + k);
      else
        pb[e] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
  };
  // masked / non-finite entries -> 0 (and the support error) by the issuing thread
  auto fixup = [&](int buf, int c0) {
    const int nv = min(LF_VC, vend - c0);
    const int v = lane;
    if (v >= nv) return;
    const int d = scope_vars[sbeg + c0 + v];
    const bool act = active[d] != 0;
    float *xb = xs + buf * XS + v * (LF_TB + 1);
    for (int bl = kq; bl < nbl; bl += KG) {
      const float xv = xb[bl];
      if (!act || !isfinite(xv)) {
        if (act) atomicMin(&status[0], d);
        xb[bl] = 0.f;
      }
    }
  };

  double tot[LF_NS][LF_KPT];
#pragma unroll
  for (int s = 0; s < LF_NS; ++s)
#pragma unroll
    for (int j = 0; j < LF_KPT; ++j) tot[s][j] = 0.0;

  if (vbeg < vend) stage(0, vbeg);
  int it = 0;
  for (int c0 = vbeg; c0 < vend; c0 += LF_VC, ++it) {
    const int buf = it & 1;
    const int nv = min(LF_VC, vend - c0);
    if (c0 + LF_VC < vend) {
      stage(buf ^ 1, c0 + LF_VC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fixup(buf, c0);
    __syncthreads();
    const float *xb = xs + buf * XS;
    const double2 *pb = ps + buf * LF_VC * KP;
    for (int v = 0; v < nv; ++v) {
      double xv[LF_NS];
#pragma unroll
      for (int s = 0; s < LF_NS; ++s) xv[s] = (double)xb[v * (LF_TB + 1) + lane + 32 * s];
      const double2 *pp = pb + v * KP + kq * LF_KPT;
#pragma unroll
      for (int j = 0; j < LF_KPT; ++j) {
        const double2 q = pp[j];
#pragma unroll
        for (int s = 0; s < LF_NS; ++s) {
          const double t = fma(xv[s], q.x, q.y);
          tot[s][j] = fma(t, t, tot[s][j]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < LF_NS; ++s) {
    const int64_t b = b0 + lane + 32 * s;
    if (b >= B) continue;
    double *dst = part + (((int64_t)split * n_leaf + leaf) * Bc + b) * K;
#pragma unroll
    for (int j = 0; j < LF_KPT; ++j) {
      const int k = kbase + kq * LF_KPT + j;
      if (k < K) dst[k] = tot[s][j];
    }
  }
}

// Categorical / binomial: S[b,l,k] = sum_d term(x_bd, k). One sample per lane.
// grid (ceil(B/32), n_leaf, dsplit), block 32*KG.
__global__ void __launch_bounds__(1024) k_leaf_fwd_discrete(
    const float *__restrict__ x, int64_t B, int D, int K, int R, const int *scope_off,
    const int *scope_vars, const int *leaf_rep, const void *lpv, const uint8_t *active,
    const double *logh, int family, int S, int n_trials, double *part, int64_t Bc,
    int n_leaf, int dsplit, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  const int leaf = blockIdx.y, split = blockIdx.z;
  const int lane = threadIdx.x & 31, kq = threadIdx.x >> 5;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int per = (slen + dsplit - 1) / dsplit;
  const int vbeg = split * per, vend = min(slen, vbeg + per);
  const int r = leaf_rep[leaf];
  const int64_t b = (int64_t)blockIdx.x * 32 + lane;
  const bool live = b < B;
  const int top = family == EINET_FAMILY_CATEGORICAL ? S - 1 : n_trials;
  double tot[LF_KPT];
#pragma unroll
  for (int j = 0; j < LF_KPT; ++j) tot[j] = 0.0;
  for (int q = vbeg; q < vend; ++q) {
    const int d = scope_vars[sbeg + q];
    if (!active[d] || !live) continue;
    const float xv = x[b * D + d];
    const bool ok = xv >= 0.f && xv <= (float)top && xv == floorf(xv);
    if (!ok) atomicMin(&status[0], d);
    const int xi = ok ? (int)xv : 0;
    const int64_t base = ((int64_t)r * D + d) * K;
    if (family == EINET_FAMILY_CATEGORICAL) {
      const double *lp = (const double *)lpv;
#pragma unroll
      for (int j = 0; j < LF_KPT; ++j) {
        const int k = kq * LF_KPT + j;
        if (k < K) tot[j] += lp[(base + k) * S + xi];
      }
    } else {
      const double2 *lp = (const double2 *)lpv;
      const double h = logh[xi];
      const double xf = (double)xi;
#pragma unroll
      for (int j = 0; j < LF_KPT; ++j) {
        const int k = kq * LF_KPT + j;
        if (k < K) {
          const double2 t = lp[base + k];
          tot[j] += fma(xf, t.x, t.y) + h;
        }
      }
    }
  }
  if (!live) return;
  double *dst = part + (((int64_t)split * n_leaf + leaf) * Bc + b) * K;
#pragma unroll
  for (int j = 0; j < LF_KPT; ++j) {
    const int k = kq * LF_KPT + j;
    if (k < K) dst[k] = tot[j];
  }
}

// leaf row = cnst + sign * sum over splits, then the slab (shift = max_k value,
// offsets = value - shift). grid (ceil(B/32), n_leaf), block 256; smem
// [32][K+1] doubles. The split sums are read coalesced ([b][k] rows are
// contiguous per leaf), one warp per sample takes the max over k, and the
// block's [K][32] slab tile (contiguous in the 32-sample transposed layout) is
// written coalesced.
__global__ void __launch_bounds__(256) k_leaf_finalize(
    const double *__restrict__ part, int dsplit, const double *__restrict__ cnst, int64_t B,
    int K, int n_leaf, const int *leaf_slab, WsView ws, double sign, int32_t *status,
    const int *gate) {
  EINET_KERNEL_PROLOGUE();
  if (gate && *(volatile const int *)gate == 0) return;  // the INT8 pass covered the batch
  extern __shared__ double vals[];  // [32][K+1]
  __shared__ double mxs[32];
  const int leaf = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int nb = (int)min((int64_t)32, B - b0);
  const int slab = leaf_slab[leaf];
  bool bad = false;
  const int64_t qs = (int64_t)n_leaf * ws.bc * K;  // split stride
  const double *base = part + ((int64_t)leaf * ws.bc + b0) * K;
  if ((K & 1) == 0) {
    // two adjacent entries per thread: 16-byte loads, every split's load in
    // flight before the (split-ordered) sums
    for (int e2 = threadIdx.x; e2 < nb * K / 2; e2 += 256) {
      const int e = 2 * e2, bl = e / K, k = e - bl * K;
      double s0 = 0.0, s1 = 0.0;
      for (int q0 = 0; q0 < dsplit; q0 += 8) {
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q0 + q < dsplit) v[q] = __ldcs((const double2 *)(base + (q0 + q) * qs + e));
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q0 + q < dsplit) {
            s0 += v[q].x;
            s1 += v[q].y;
          }
      }
      vals[bl * (K + 1) + k] = cnst[leaf * K + k] + sign * s0;
      vals[bl * (K + 1) + k + 1] = cnst[leaf * K + k + 1] + sign * s1;
      bad |= !isfinite(s0) || !isfinite(s1);
    }
  } else {
    for (int e = threadIdx.x; e < nb * K; e += 256) {
      const int bl = e / K, k = e - bl * K;
      double s = 0.0;
      for (int q = 0; q < dsplit; ++q) s += base[q * qs + e];
      vals[bl * (K + 1) + k] = cnst[leaf * K + k] + sign * s;
      bad |= !isfinite(s);
    }
  }
  if (bad && status) atomicMin(&status[2], 0);  // non-finite x reached a leaf row
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int bl = threadIdx.x >> 5; bl < nb; bl += 8) {
    const double *v = vals + bl * (K + 1);
    double mx = -CUDART_INF;
    for (int k = lane; k < K; k += 32) mx = fmax(mx, v[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      mxs[bl] = mx;
      slab_shift(ws, slab)[b0 + bl] = mx;
    }
  }
  __syncthreads();
  float *tile = ws.off + tb_idx(slab, b0, 0, ws.bc, ws.ks);
  for (int e = threadIdx.x; e < K * 32; e += 256) {
    const int k = e >> 5, bl = e & 31;
    if (bl >= nb) continue;
    const double mx = mxs[bl];
    tile[e] = mx == -CUDART_INF ? 0.f : (float)(vals[bl * (K + 1) + k] - mx);
  }
}

// Reference support check (expfam.py:278-294) for the unmasked DMMA path:
// only when a leaf row came out non-finite, report the lowest active variable
// holding a non-finite value (atomicMin, like the gathering kernels).
__global__ void k_leaf_check(const float *__restrict__ x, int64_t B, int D,
                             const uint8_t *__restrict__ active, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  if (status[2] == INT_MAX) return;
  const int64_t n = B * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    if (active[d] && !isfinite(x[e])) atomicMin(&status[0], d);
  }
}

static int leaf_dsplit(const Plan &p, int64_t B, int tb, int64_t slots, int nkc) {
  const int64_t blocks = (int64_t)ceil_div(B, tb) * p.n_leaf * nkc;
  // at least four 32-variable chunks per split, unless the grid would not
  // fill a wave (small batches): then down to one chunk per split
  const int min_chunks = blocks * ceil_div(p.max_scope, 4 * LF_VC) < slots ? 1 : 4;
  const int cap = std::max(1, std::min(kMaxDSplit, ceil_div(p.max_scope, min_chunks * LF_VC)));
  return pick_split(blocks, slots, 1, cap);
}

// The CUDA-core / FP64 leaf forward + finalize + support check on stream st.
// gate != nullptr: every kernel returns at once unless *gate != 0 (the INT8
// pass flagged the batch).
static int launch_leaf_fallback(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                                uint8_t *wsb, int32_t *status, cudaStream_t st,
                                const int *gate) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  const int KG = ceil_div(p.k, LF_KPT);
  int ds;
  if (p.leaf_dmma && p.use_tc) {
    int rc = launch_leaf_fwd_dmma(p, c, x, B, w, status, st, &ds, gate);
    if (rc) return rc;
  } else if (p.family == EINET_FAMILY_GAUSSIAN) {
    const int kg = std::min(KG, 8);          // <= 64 k entries per CTA
    const int nkc = ceil_div(KG, kg);
    const int threads = 32 * kg;
    const size_t smem = ((2 * LF_VC * (LF_TB + 1) * sizeof(float) + 15) & ~(size_t)15) +
                        2 * sizeof(double2) * LF_VC * kg * LF_KPT;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_leaf_fwd_gauss, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    ds = leaf_dsplit(p, B, LF_TB,
                     device_slots((const void *)k_leaf_fwd_gauss, threads, smem, p.num_sms), nkc);
    dim3 grid(ceil_div(B, LF_TB), p.n_leaf, ds * nkc);
    launch_k(k_leaf_fwd_gauss, grid, threads, smem, st, 
        x, B, p.d_vars, p.k, p.num_replicas, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep,
        (const double2 *)c.leafp, c.active, w.leafpart, w.bc, p.n_leaf, ds, status, gate);
  } else {
    const int threads = 32 * KG;
    if (threads > 1024) return fail(EINET_ERR_USAGE, "k too large for the leaf kernel (k <= 256)");
    ds = leaf_dsplit(p, B, 32, 2LL * p.num_sms, 1);
    dim3 grid(ceil_div(B, 32), p.n_leaf, ds);
    launch_k(k_leaf_fwd_discrete, grid, threads, 0, st, 
        x, B, p.d_vars, p.k, p.num_replicas, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep,
        c.leafp, c.active, c.logh, p.family, p.num_states, p.n_trials, w.leafpart, w.bc,
        p.n_leaf, ds, status);
  }
  dim3 g2(ceil_div(B, 32), p.n_leaf);
  const size_t fsmem = sizeof(double) * 32 * (p.k + 1);
  if (fsmem > 48 * 1024)
    cudaFuncSetAttribute(k_leaf_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fsmem);
  launch_k(k_leaf_finalize, g2, 256, fsmem, st, w.leafpart, ds, c.cnst, B, p.k, p.n_leaf, p.d_leaf_slab,
                                      w, p.family == EINET_FAMILY_GAUSSIAN ? -1.0 : 1.0,
                                      status, gate);
  count_launch(2);
  if (p.leaf_dmma && p.use_tc) {
    launch_k(k_leaf_check, 2 * p.num_sms, 256, 0, st, x, B, p.d_vars, c.active, status);
    count_launch();
  }
  return check_cuda(cudaGetLastError(), "leaf forward kernels");
}

// Leaf slabs from split partials of the INT8 pass (leaf_i8.cu scope split):
// cnst - sum_q part[q] in split order, then the slab shift / offsets.
int launch_leaf_finalize_parts(Plan &p, const uint8_t *compute, const double *part, int nsplit,
                               int64_t B, uint8_t *wsb, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  dim3 g2(ceil_div(B, 32), p.n_leaf);
  const size_t fsmem = sizeof(double) * 32 * (p.k + 1);
  if (fsmem > 48 * 1024)
    cudaFuncSetAttribute(k_leaf_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fsmem);
  launch_k(k_leaf_finalize, g2, 256, fsmem, st, part, nsplit, (const double *)c.cnst, B, p.k,
           p.n_leaf, (const int *)p.d_leaf_slab, w, -1.0, (int32_t *)nullptr, (const int *)nullptr);
  count_launch();
  return check_cuda(cudaGetLastError(), "leaf finalize (INT8 split)");
}

// Image data: the INT8 tensor-core pass (leaf_i8.cu) writes the slabs and
// flags an off-grid batch; only then does the fallback sequence run. Under
// CUDA-graph capture the fallback is the body of a conditional (IF) node whose
// condition the INT8 kernel sets, so a clean batch costs no launches; eagerly
// the fallback kernels are launched gated on the flag (they return at once).
int launch_leaf_forward(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                        uint8_t *wsb, int32_t *status, cudaStream_t st) {
  ProfScope prof("leaf_fwd", st);
  // below ~1024 samples the FP64 path's short per-CTA chains win (the INT8
  // kernel walks a leaf pair's whole scope per CTA); EINET_LEAF_I8_MIN_BATCH
  // overrides (tests force the INT8 path at small sizes)
  const char *mb = getenv("EINET_LEAF_I8_MIN_BATCH");
  const int64_t min_batch = mb ? atoll(mb) : 1024;
  if (!leaf_i8_supported(p) || B < min_batch)
    return launch_leaf_fallback(p, compute, x, B, wsb, status, st, nullptr);
  int *flag = (int *)(wsb + p.w_i8flag);
  int rc = check_cuda(cudaMemsetAsync(flag, 0, sizeof(int), st), "leaf i8 flag");
  if (rc) return rc;
  const char *dbg = getenv("EINET_I8_DEBUG");
  const bool no_fallback = dbg && (atoi(dbg) & 32);  // diagnostics
  // EINET_LEAF_COND=0: gated launches inside captured graphs too (ncu cannot
  // profile kernel nodes of graphs that hold conditional nodes)
  const char *cenv = getenv("EINET_LEAF_COND");
  const bool use_cond = !(cenv && cenv[0] == '0');
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t *deps = nullptr;
  size_t ndeps = 0;
  if ((rc = check_cuda(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &ndeps),
                       "capture info")))
    return rc;
  if (cs != cudaStreamCaptureStatusActive || no_fallback || !use_cond) {
    if ((rc = launch_leaf_fwd_i8(p, compute, x, B, wsb, flag, 0ULL, st))) return rc;
    if (no_fallback) return 0;
    return launch_leaf_fallback(p, compute, x, B, wsb, status, st, flag);
  }
  cudaGraphConditionalHandle cond;
  if ((rc = check_cuda(cudaGraphConditionalHandleCreate(&cond, graph, 0,
                                                        cudaGraphCondAssignDefault),
                       "conditional handle")))
    return rc;
  if ((rc = launch_leaf_fwd_i8(p, compute, x, B, wsb, flag, cond, st))) return rc;
  if ((rc = check_cuda(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &ndeps),
                       "capture info")))
    return rc;
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeIf;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if ((rc = check_cuda(cudaGraphAddNode(&node, graph, deps, ndeps, &np), "conditional node")))
    return rc;
  cudaGraph_t body = np.conditional.phGraph_out[0];
  if ((rc = check_cuda(cudaStreamBeginCaptureToGraph(p.side_stream, body, nullptr, nullptr, 0,
                                                     cudaStreamCaptureModeRelaxed),
                       "capture fallback")))
    return rc;
  rc = launch_leaf_fallback(p, compute, x, B, wsb, status, p.side_stream, nullptr);
  cudaGraph_t got = nullptr;
  const int rc2 = check_cuda(cudaStreamEndCapture(p.side_stream, &got), "end fallback capture");
  if (rc) return rc;
  if (rc2) return rc2;
  return check_cuda(cudaStreamUpdateCaptureDependencies(st, &node, 1,
                                                        cudaStreamSetCaptureDependencies),
                    "capture dependencies");
}

// ---------------------------------------------------------------------------
// leaf responsibilities and statistics (engine.py:318-327)
// ---------------------------------------------------------------------------

// rho_leaf[b,l,k] from the slot CSR (elementwise over a 32-sample block) and
// the block's partial of P[l,k] = sum_b rho: a warp covers one k for the 32
// samples, reduced with a fixed shuffle tree.
// grid (ceil(B/32), n_leaf), block 128.
__global__ void __launch_bounds__(128) k_leaf_rho(WsView ws, const int *csr_off,
                                                  const int *__restrict__ csr_slot,
                                                  const uint8_t *ones, const int *leaf_slab,
                                                  int64_t B, int K, int n_leaf, double *ppart,
                                                  int nn) {
  EINET_KERNEL_PROLOGUE();
  const int leaf = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int slab = leaf_slab[leaf];
  const int q0 = csr_off[slab], q1 = csr_off[slab + 1];
  const bool one = ones[slab] != 0;
  // tensor-core statistics (nn > 0, K <= 64): the block's rho only feeds the
  // rho^T B tile below, so it stays in shared memory (no fp32 round trip)
  __shared__ __align__(16) float srho[64 * 32];
  float *rho = nn > 0 ? srho : ws.rho + tb_idx(leaf, b0, 0, ws.bc, K);
  constexpr int NE = 16;  // entries per thread gathered together (K <= 64)
  const int ne = K * 32;
  if (ne <= 128 * NE) {
    // slot by slot (the per-entry summation order of the loop below), every
    // entry's load of one slot in flight at once
    float acc[NE];
#pragma unroll
    for (int j = 0; j < NE; ++j) acc[j] = one ? 1.f : 0.f;
    for (int q = q0; !one && q < q1; ++q) {
      const float *sp = ws.slots + tb_idx(csr_slot[q], b0, 0, ws.bc, ws.ks);
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const int e = threadIdx.x + 128 * j;
        if (e < ne) acc[j] += sp[e];
      }
    }
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = threadIdx.x + 128 * j;
      if (e >= ne) break;
      float v = b0 + (e & 31) < B ? acc[j] : 0.f;
      rho[e] = v;  // samples past the batch hold 0 (the statistics sum whole blocks)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((e & 31) == 0) ppart[((int64_t)blockIdx.x * n_leaf + leaf) * K + (e >> 5)] = (double)v;
    }
  } else {
    for (int e = threadIdx.x; e < ne; e += 128) {
      float v = 0.f;
      if (b0 + (e & 31) < B) {
        if (one) {
          v = 1.f;
        } else {
          for (int q = q0; q < q1; ++q) v += ws.slots[tb_idx(csr_slot[q], b0, 0, ws.bc, ws.ks) + e];
        }
      }
      rho[e] = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((e & 31) == 0) ppart[((int64_t)blockIdx.x * n_leaf + leaf) * K + (e >> 5)] = (double)v;
    }
  }
  if (nn > 0) {  // tensor-core leaf statistics: the block's rho^T B operand
    __syncthreads();
    bt_tile(rho, ws.rhob + ((int64_t)leaf * (ws.bc / 32) + b0 / 32) * (2 * nn * 32), K, nn);
  }
}

constexpr int LS_VC = 32;   // variables per CTA
constexpr int LS_BT = 32;   // samples per fp32 run before folding into fp64
constexpr int LS_MAXP = 16; // (var,k,t) entries per thread

// Gaussian: acc_pt[d,k,r,:] += sum_b rho*(x, x^2). fp32 runs of 32 samples are
// accumulated centred at c = centre[r][d] (y = x - c) and un-centred in fp64:
//   sum rho x = A + c P,  sum rho x^2 = Q + 2 c A + c^2 P.
// Register tile of 4 variables x 4 k per thread: per sample 3 LDS.128 feed
// 32 FFMA. grid (ceil(max_scope/64) * nkc, n_leaf, lsplit), block 16*KQ.
constexpr int LS_VT = 64;
__global__ void __launch_bounds__(256) k_leaf_stats_gauss(
    const float *__restrict__ x, int64_t B, int D, int K, int R, const int *scope_off,
    const int *scope_vars, const int *leaf_rep, const float *__restrict__ rho_all, int64_t Bc,
    const float *__restrict__ center, const uint8_t *__restrict__ active, double *lspart,
    int64_t n_phi, int lsplit, int nkc) {
  EINET_KERNEL_PROLOGUE();
  __shared__ __align__(16) float ys[LS_BT][LS_VT];
  __shared__ __align__(16) float y2s[LS_BT][LS_VT];
  extern __shared__ __align__(16) float rs[];  // [LS_BT][KPC]
  __shared__ int dv[LS_VT];
  __shared__ float cv[LS_VT];
  const int KQ = blockDim.x / 16;  // k quads in this CTA
  const int KPC = KQ * 4;
  const int leaf = blockIdx.y, split = blockIdx.z;
  const int vchunk = blockIdx.x / nkc;
  const int kbase = (blockIdx.x % nkc) * KPC;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int v0 = vchunk * LS_VT;
  if (v0 >= slen) return;
  const int nv = min(LS_VT, slen - v0);
  const int r = leaf_rep[leaf];
  const int64_t per = (B + lsplit - 1) / lsplit;
  const int64_t bb = split * per, be = min(B, bb + per);
  const int tv = threadIdx.x % 16, tk = threadIdx.x / 16;
  for (int v = threadIdx.x; v < LS_VT; v += blockDim.x) {
    const int d = v < nv ? scope_vars[sbeg + v0 + v] : -1;
    dv[v] = (d >= 0 && active[d]) ? d : -1;
    cv[v] = d >= 0 ? center[(int64_t)r * D + d] : 0.f;
  }
  __syncthreads();
  float c[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) c[u] = cv[4 * tv + u];
  float a1[4][4], a2[4][4], pk[4];
  double t0[4][4], t1[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a1[u][j] = a2[u][j] = 0.f;
      t0[u][j] = t1[u][j] = 0.0;
    }
  for (int64_t t = bb; t < be; t += LS_BT) {
    const int nb = (int)min((int64_t)LS_BT, be - t);
    __syncthreads();
    for (int e = threadIdx.x; e < LS_BT * LS_VT; e += blockDim.x) {
      const int v = e % LS_VT, bl = e / LS_VT;
      const int d = dv[v];
      float y = 0.f;
      if (d >= 0 && bl < nb) {
        const float xv = x[(t + bl) * D + d];
        y = isfinite(xv) ? xv - cv[v] : 0.f;
      }
      ys[bl][v] = y;
      y2s[bl][v] = y * y;
    }
    for (int e = threadIdx.x; e < LS_BT * KPC; e += blockDim.x) {
      const int bl = e / KPC, k = kbase + e % KPC;
      rs[e] = (bl < nb && k < K) ? rho_all[tb_idx(leaf, t + bl, k, Bc, K)] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) pk[j] = 0.f;
    for (int bl = 0; bl < nb; ++bl) {
      const float4 y4 = *(const float4 *)&ys[bl][4 * tv];
      const float4 q4 = *(const float4 *)&y2s[bl][4 * tv];
      const float4 r4 = *(const float4 *)&rs[bl * KPC + 4 * tk];
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
      const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
      const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pk[j] += rv[j];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a1[u][j] = fmaf(rv[j], yv[u], a1[u][j]);
          a2[u][j] = fmaf(rv[j], qv[u], a2[u][j]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double cu = (double)c[u];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double A = a1[u][j], Q = a2[u][j], P = pk[j];
        t0[u][j] += A + cu * P;
        t1[u][j] += Q + 2.0 * cu * A + cu * cu * P;
        a1[u][j] = a2[u][j] = 0.f;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int v = 4 * tv + u;
    if (v >= nv) continue;
    const int d = scope_vars[sbeg + v0 + v];
    const bool act = dv[v] >= 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = kbase + 4 * tk + j;
      if (k >= K) continue;
      double *dst = lspart + (int64_t)split * n_phi + ((((int64_t)d * K + k) * R + r) * 2);
      dst[0] = act ? t0[u][j] : 0.0;
      dst[1] = act ? t1[u][j] : 0.0;
    }
  }
}

// Categorical (T = S one-hot) / binomial (T = 1, x): entries (var, k, t).
__global__ void __launch_bounds__(256) k_leaf_stats_discrete(
    const float *__restrict__ x, int64_t B, int D, int K, int R, int T, int family,
    const int *scope_off, const int *scope_vars, const int *leaf_rep,
    const float *__restrict__ rho_all, int64_t Bc, const uint8_t *__restrict__ active,
    double *lspart, int64_t n_phi, int lsplit) {
  EINET_KERNEL_PROLOGUE();
  const int leaf = blockIdx.y, split = blockIdx.z;
  const int sbeg = scope_off[leaf], slen = scope_off[leaf + 1] - sbeg;
  const int v0 = blockIdx.x * LS_VC;
  if (v0 >= slen) return;
  const int nv = min(LS_VC, slen - v0);
  const int r = leaf_rep[leaf];
  const int64_t per = (B + lsplit - 1) / lsplit;
  const int64_t bb = split * per, be = min(B, bb + per);
  const int64_t n_ent = (int64_t)nv * K * T;
  // one warp per (variable, k, t) entry; lanes stride over the samples (fp32
  // runs of <= LS_BT samples folded into fp64), then a fixed shuffle tree
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t e = wid; e < n_ent; e += blockDim.x >> 5) {
    const int t = (int)(e % T);
    const int k = (int)((e / T) % K);
    const int v = (int)(e / ((int64_t)T * K));
    const int d = scope_vars[sbeg + v0 + v];
    double tot = 0.0;
    if (active[d]) {
      float run = 0.f;
      int cnt = 0;
#pragma unroll 4
      for (int64_t b = bb + lane; b < be; b += 32) {
        const float xv = x[b * D + d];
        const float rr = rho_all[tb_idx(leaf, b, k, Bc, K)];
        if (family == EINET_FAMILY_CATEGORICAL)
          run += ((int)xv == t && xv == floorf(xv)) ? rr : 0.f;
        else
          run = fmaf(rr, xv, run);
        if (++cnt == LS_BT) {
          tot += (double)run;
          run = 0.f;
          cnt = 0;
        }
      }
      tot += (double)run;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
    if (lane == 0) lspart[(int64_t)split * n_phi + ((((int64_t)d * K + k) * R + r) * T + t)] = tot;
  }
}

int leaf_lsplit(const Plan &p, int64_t B) {
  if (p.family == EINET_FAMILY_GAUSSIAN) return (int)std::max<int64_t>(1, std::min<int64_t>(16, (B + 255) / 256));
  int64_t blocks = (int64_t)ceil_div(p.max_scope, LS_VT) * p.n_leaf;
  int want = (int)std::max<int64_t>(1, (2 * p.num_sms + blocks - 1) / blocks);
  int cap = (int)std::max<int64_t>(1, std::min<int64_t>(8, (B + 255) / 256));
  return std::min(want, cap);
}

int launch_leaf_backward(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                         uint8_t *wsb, double *stats, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  const int K = p.k, D = p.d_vars, R = p.num_replicas, T = p.suff;
  const int nb = ceil_div(B, 32);
  double *Pcall = (double *)(wsb + p.w_tmp_p);
  // tensor-core path: the P reductions (read only by k_leaf_stats_finish and
  // the M-step) run beside k_leaf_stats_tc on the fork stream (idle until the
  // M-step) -- not on the reduction stream, where they would queue behind the
  // W-statistics reductions and hold k_leaf_stats_finish until those end
  const bool tcs = leaf_tc_supported(p);
  cudaStream_t rs = tcs && p.fork_stream && !profiling_enabled() ? p.fork_stream : st;
  {
  ProfScope prof("leaf_rho", st);
  launch_k(k_leaf_rho, dim3(nb, p.n_leaf), 128, 0, st, w, p.d_csr_off, p.d_csr_slot, p.d_slab_ones,
                                                 p.d_leaf_slab, B, K, p.n_leaf, w.ppart,
                                                 leaf_tc_supported(p) ? (K + 15) / 16 * 16 : 0);
  if (rs != st) {
    int rc = check_cuda(cudaEventRecord(p.red_fork[3], st), "leaf P fork");
    if (!rc) rc = check_cuda(cudaStreamWaitEvent(rs, p.red_fork[3], 0), "leaf P fork");
    if (rc) return rc;
  }
  launch_reduce_partials_store(Pcall, w.ppart, nb, (int64_t)p.n_leaf * K,
                               (int64_t)p.n_leaf * K, rs);
  launch_reduce_partials(stats + p.sizes.stats_p_offset, Pcall, 1, (int64_t)p.n_leaf * K,
                         (int64_t)p.n_leaf * K, nullptr, rs);
  if (rs != st) {
    int rc = check_cuda(cudaEventRecord(p.red_done[3], rs), "leaf P done");
    if (rc) return rc;
  }
  }
  ProfScope prof("leaf_stats", st);
  if (leaf_tc_supported(p)) {
    int rc = launch_leaf_stats_tc(p, compute, x, B, wsb, stats, Pcall, st,
                                  rs != st ? p.red_done[3] : nullptr);
    count_launch(1);
    return rc;
  }
  const int ls = leaf_lsplit(p, B);
  const int64_t n_phi = p.n_phi;
  cudaMemsetAsync(w.lspart, 0, sizeof(double) * n_phi * ls, st);
  dim3 grid(ceil_div(p.max_scope, LS_VC), p.n_leaf, ls);
  if (p.family == EINET_FAMILY_GAUSSIAN) {
    const int K4 = ceil_div(K, 4);
    const int kq = std::min(K4, 16);
    const int nkc = ceil_div(K4, kq);
    dim3 g(ceil_div(p.max_scope, LS_VT) * nkc, p.n_leaf, ls);
    launch_k(k_leaf_stats_gauss, g, 16 * kq, sizeof(float) * LS_BT * kq * 4, st, 
        x, B, D, K, R, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep, w.rho, w.bc, c.center,
        c.active, w.lspart, n_phi, ls, nkc);
  } else {
    launch_k(k_leaf_stats_discrete, grid, 256, 0, st, x, B, D, K, R, T, p.family, p.d_scope_off,
                                               p.d_scope_vars, p.d_leaf_rep, w.rho, w.bc,
                                               c.active, w.lspart, n_phi, ls);
  }
  launch_reduce_partials(stats + p.sizes.stats_acc_pt_offset, w.lspart, ls, n_phi, n_phi,
                         nullptr, st);
  count_launch(2);
  return check_cuda(cudaGetLastError(), "leaf backward kernels");
}

// ---------------------------------------------------------------------------
// conversions / exports
// ---------------------------------------------------------------------------

__global__ void k_expand_acc_p(const double *P, const int *leaf_of, double *acc_p, int D, int K,
                               int R) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = (int64_t)D * K * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(e % R);
    int k = (int)((e / R) % K);
    int d = (int)(e / ((int64_t)R * K));
    int l = leaf_of[(int64_t)r * D + d];
    acc_p[e] = l >= 0 ? P[(int64_t)l * K + k] : 0.0;
  }
}

int launch_expand_acc_p(Plan &p, const double *stats, double *acc_p, cudaStream_t st) {
  int64_t n = (int64_t)p.d_vars * p.k * p.num_replicas;
  launch_k(k_expand_acc_p, (int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st, 
      stats + p.sizes.stats_p_offset, p.d_leaf_of, acc_p, p.d_vars, p.k, p.num_replicas);
  count_launch();
  return check_cuda(cudaGetLastError(), "expand acc_p");
}

// E[b,d,k,r] in fp64 straight from the master parameters (expfam.py:278-294).
__global__ void k_ef_log_prob(const double *__restrict__ phi, const float *__restrict__ x,
                              int64_t B, int D, int K, int R, int family, int S, int n_trials,
                              const uint8_t *mask, double *out, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = B * D * K * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % R);
    const int k = (int)((e / R) % K);
    const int d = (int)((e / ((int64_t)R * K)) % D);
    const int64_t b = e / ((int64_t)R * K * D);
    if (mask && mask[d]) {
      out[e] = 0.0;
      continue;
    }
    const double xv = (double)x[b * D + d];
    const int64_t base = ((int64_t)d * K + k) * R + r;
    double v;
    if (family == EINET_FAMILY_GAUSSIAN) {
      if (!isfinite(xv)) atomicMin(&status[0], d);
      const double mu = phi[base * 2], var = phi[base * 2 + 1] - mu * mu;
      v = -0.5 * (kLog2Pi + log(var)) - (xv - mu) * (xv - mu) / (2.0 * var);
    } else {
      const int top = family == EINET_FAMILY_CATEGORICAL ? S - 1 : n_trials;
      const bool ok = xv >= 0.0 && xv <= (double)top && xv == floor(xv);
      if (!ok) atomicMin(&status[0], d);
      const int xi = ok ? (int)xv : 0;
      if (family == EINET_FAMILY_CATEGORICAL) {
        v = log(phi[base * S + xi]);
      } else {
        const double pr = phi[base] / (double)n_trials;
        v = lgamma((double)n_trials + 1.0) - lgamma((double)xi + 1.0) -
            lgamma((double)(n_trials - xi) + 1.0) + xi * log(pr) +
            (n_trials - xi) * log1p(-pr);
      }
    }
    out[e] = v;
  }
}

int launch_ef_log_prob(Plan &p, const double *params, const float *x, int64_t B,
                       const uint8_t *mask, double *out, int32_t *status, cudaStream_t st) {
  int64_t n = B * p.d_vars * p.k * p.num_replicas;
  launch_k(k_ef_log_prob, (int)std::min<int64_t>((n + 255) / 256, 8192), 256, 0, st, 
      params + p.sizes.phi_offset, x, B, p.d_vars, p.k, p.num_replicas, p.family, p.num_states,
      p.n_trials, mask, out, status);
  count_launch();
  return check_cuda(cudaGetLastError(), "ef_log_prob");
}

__global__ void k_export_rows(WsView ws, const int *slabs, int nrows, int64_t B, int K,
                              double *out) {
  EINET_KERNEL_PROLOGUE();
  int64_t n = B * nrows * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % K);
    const int row = (int)((e / K) % nrows);
    const int64_t b = e / ((int64_t)K * nrows);
    const int slab = slabs ? slabs[row] : row;
    const double s = slab_shift(ws, slab)[b];
    out[e] = s == -CUDART_INF ? -CUDART_INF : s + (double)slab_off(ws, slab, b)[k];
  }
}

int launch_export_buffer(Plan &p, const uint8_t *wsb, int64_t B, double *out, cudaStream_t st) {
  WsView w = ws_view(p, wsb);
  int64_t n = B * p.nbr * p.k;
  if (n == 0) return EINET_OK;
  launch_k(k_export_rows, (int)std::min<int64_t>((n + 255) / 256, 8192), 256, 0, st, 
      w, nullptr, p.nbr, B, p.k, out);
  count_launch();
  return check_cuda(cudaGetLastError(), "export buffer");
}

int launch_export_leaf_rows(Plan &p, const uint8_t *wsb, int64_t B, double *out,
                            cudaStream_t st) {
  WsView w = ws_view(p, wsb);
  int64_t n = B * p.n_leaf * p.k;
  launch_k(k_export_rows, (int)std::min<int64_t>((n + 255) / 256, 8192), 256, 0, st, 
      w, p.d_leaf_slab, p.n_leaf, B, p.k, out);
  count_launch();
  return check_cuda(cudaGetLastError(), "export leaf rows");
}

}  // namespace einet
