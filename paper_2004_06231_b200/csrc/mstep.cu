// Fused M-step (trainer.py:69-124, engine.py:46-54, expfam project) in fp64,
// the deterministic partial-sum reduction and the standalone fp64
// log_einsum_exp (engine.py:91-109).
#include <climits>
#include <cmath>

#include "kern_common.cuh"
#include "tc_common.cuh"

namespace einet {

// dst[i] (+)= scale[i] * sum_p part[p*stride + i]. Few partials: one thread per
// output, loads unrolled. Many partials over few outputs: one CTA per output,
// threads stride over the partials, fixed shuffle tree. Both fixed-order.
__global__ void k_reduce_partials(double *__restrict__ dst, const double *__restrict__ part,
                                  int nparts, int64_t n, int64_t stride,
                                  const double *__restrict__ scale, int store) {
  EINET_KERNEL_PROLOGUE();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * stride + i];
    if (scale) s *= scale[i];
    dst[i] = store ? s : dst[i] + s;
  }
}

__global__ void __launch_bounds__(256) k_reduce_partials_cta(
    double *__restrict__ dst, const double *__restrict__ part, int nparts, int64_t stride,
    const double *__restrict__ scale, int store) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += 256) s += part[(int64_t)p * stride + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
    if (scale) t *= scale[i];
    dst[i] = store ? t : dst[i] + t;
  }
}

// 32 consecutive outputs per CTA: warp ty sums parts ty, ty + 8, ... of its
// 32 columns (coalesced 256-byte rows), then a fixed tree over the 8 warps.
__global__ void __launch_bounds__(256) k_reduce_partials_tile(
    double *__restrict__ dst, const double *__restrict__ part, int nparts, int64_t n,
    int64_t stride, const double *__restrict__ scale, int store) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + tx;
  double s = 0.0;
  if (i < n) {
#pragma unroll 4
    for (int p = ty; p < nparts; p += 8) s += part[(int64_t)p * stride + i];
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && i < n) {
    double t = ((red[0][tx] + red[1][tx]) + (red[2][tx] + red[3][tx])) +
               ((red[4][tx] + red[5][tx]) + (red[6][tx] + red[7][tx]));
    if (scale) t *= scale[i];
    dst[i] = store ? t : dst[i] + t;
  }
}

static void reduce_partials(double *dst, const double *part, int nparts, int64_t n,
                            int64_t stride, const double *scale, int store, cudaStream_t st) {
  if (n <= 0) return;
  if (nparts >= 64 && n >= 2048 && n <= (1 << 22)) {
    launch_k(k_reduce_partials_tile, (unsigned)((n + 31) / 32), 256, 0, st, dst, part, nparts, n,
             stride, scale, store);
  } else if (nparts >= 64 && n <= 65536) {
    launch_k(k_reduce_partials_cta, (unsigned)n, 256, 0, st, dst, part, nparts, stride, scale, store);
  } else {
    const int grid = (int)std::min<int64_t>((n + kReduceThreads - 1) / kReduceThreads, 8192);
    launch_k(k_reduce_partials, grid, kReduceThreads, 0, st, dst, part, nparts, n, stride, scale,
                                                       store);
  }
  count_launch();
}

void launch_reduce_partials_store(double *dst, const double *part, int nparts, int64_t n,
                                  int64_t stride, cudaStream_t st) {
  reduce_partials(dst, part, nparts, n, stride, nullptr, 1, st);
}

void launch_reduce_partials(double *dst, const double *part, int nparts, int64_t n,
                            int64_t stride, const double *scale, cudaStream_t st) {
  reduce_partials(dst, part, nparts, n, stride, scale, 0, st);
}

__device__ __forceinline__ bool step_failed(const int32_t *status) {
  // word 3 = 0: another rank of the process group failed this step
  return status && (status[0] != INT_MAX || status[1] != INT_MAX || status[3] != INT_MAX);
}

// Deterministic block sum (fixed shuffle tree, fixed warp order). blockDim 256.
__device__ __forceinline__ double block_sum_256(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w];
  __syncthreads();
  return s;
}

// One (l, k) slice of K*K weights per CTA (all einsum layers are contiguous
// in the same order in params and stats). trainer.py:74-77, 110-111,
// engine.py:46-49.
__global__ void __launch_bounds__(256) k_mstep_einsum(double *__restrict__ W,
                                                      float *__restrict__ w32,
                                                      const double *__restrict__ n, int K,
                                                      double lam, double eps,
                                                      const int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  const int KK = K * K;
  __shared__ double red[8];
  if (step_failed(status)) return;
  const int64_t base = (int64_t)blockIdx.x * KK;
  double s = 0.0;
  for (int e = threadIdx.x; e < KK; e += 256) s += n[base + e];
  const double den = block_sum_256(s, red);
  double s2 = 0.0;
  for (int e = threadIdx.x; e < KK; e += 256) {
    const double old = W[base + e];
    const double tgt = den > 0.0 ? n[base + e] / den : old;
    double v = (1.0 - lam) * old + lam * tgt;
    v = fmax(v, eps);
    W[base + e] = v;
    s2 += v;
  }
  const double tot = block_sum_256(s2, red);
  for (int e = threadIdx.x; e < KK; e += 256) {
    const double v = W[base + e] / tot;
    W[base + e] = v;
    w32[base + e] = (float)v;
  }
}

// One mixing row per thread (trainer.py:79-81, 112-113, engine.py:52-54).
__global__ void k_mstep_mixing(double *__restrict__ Wm, float *__restrict__ m32,
                               const double *__restrict__ n, const int *row_off,
                               const int *row_len, const uint8_t *mask, int nrows, double lam,
                               double eps, const int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows || step_failed(status)) return;
  const int o = row_off[r], len = row_len[r];
  double den = 0.0;
  for (int c = 0; c < len; ++c) den += n[o + c];
  double tot = 0.0;
  for (int c = 0; c < len; ++c) {
    const double old = Wm[o + c];
    const double tgt = den > 0.0 ? n[o + c] / den : old;
    double v = (1.0 - lam) * old + lam * tgt;
    v = mask[o + c] ? fmax(v, eps) : 0.0;
    Wm[o + c] = v;
    tot += v;
  }
  for (int c = 0; c < len; ++c) {
    const double v = Wm[o + c] / tot;
    Wm[o + c] = v;
    m32[o + c] = (float)v;
  }
}

// Leaf parameters, one (d, k, r) per thread (trainer.py:82-85, 114, 96).
__global__ void k_mstep_leaf(double *__restrict__ phi, const double *__restrict__ acc_pt,
                             const double *__restrict__ P, const int *__restrict__ leaf_of,
                             int D, int K, int R, int T, int family, double lam,
                             double var_min, double var_max, double p_min, int n_trials,
                             const int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  if (step_failed(status)) return;
  const int64_t n = (int64_t)D * K * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % R);
    const int k = (int)((e / R) % K);
    const int d = (int)(e / ((int64_t)R * K));
    const int l = leaf_of[(int64_t)r * D + d];
    const double p = l >= 0 ? P[(int64_t)l * K + k] : 0.0;
    const bool keep = p <= kEpsCount;
    double *ph = phi + e * T;
    const double *acc = acc_pt + e * T;
    if (family == EINET_FAMILY_GAUSSIAN) {
      const double t0 = keep ? ph[0] : acc[0] / p;
      const double t1 = keep ? ph[1] : acc[1] / p;
      const double m = (1.0 - lam) * ph[0] + lam * t0;
      const double s = (1.0 - lam) * ph[1] + lam * t1;
      const double var = fmin(fmax(s - m * m, var_min), var_max);
      ph[0] = m;
      ph[1] = var + m * m;
    } else if (family == EINET_FAMILY_CATEGORICAL) {
      double tot = 0.0;
      for (int t = 0; t < T; ++t) {
        const double tg = keep ? ph[t] : acc[t] / p;
        const double v = fmax((1.0 - lam) * ph[t] + lam * tg, p_min);
        ph[t] = v;
        tot += v;
      }
      for (int t = 0; t < T; ++t) ph[t] = ph[t] / tot;
    } else {
      const double tg = keep ? ph[0] : acc[0] / p;
      const double v = (1.0 - lam) * ph[0] + lam * tg;
      const double nt = (double)n_trials;
      const double pr = fmin(fmax(v / nt, p_min), 1.0 - p_min);
      ph[0] = pr * nt;
    }
  }
}

// Gaussian leaves, one warp per (r, d), lanes over k: the M-step update
// (trainer.py:82-85, 114, 96; expfam.py GaussianFamily.project) followed by the
// per-variable compute tensors the forward and the statistics read (leaf.cu
// k_prepare_gauss / k_prepare_center, leaf_dmma.cu k_prepare_leaf_img) and the
// per-(variable, k) terms of the leaf constants (reduced by k_leaf_consts).
// Masked variables never reach a cached compute buffer (marginal queries build
// their own), so every covered variable is active here.
__global__ void __launch_bounds__(256) k_mstep_leaf_gauss(
    double *__restrict__ phi, const double *__restrict__ acc_pt, const double *__restrict__ P,
    const int *__restrict__ leaf_of, const int *__restrict__ scope_pos,
    const int *__restrict__ pvo, int D, int K, int R, double lam, double var_min,
    double var_max, const int32_t *status, CompView c, int dmma, double *__restrict__ mtmp) {
  EINET_KERNEL_PROLOGUE();
  if (step_failed(status)) return;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= R * D) return;
  const int r = wid / D, d = wid - r * D;
  const int l = leaf_of[(int64_t)r * D + d];
  double mu[2] = {0.0, 0.0}, var[2] = {1.0, 1.0};
  double csum = 0.0;
  for (int u = 0; u < 2; ++u) {
    const int k = lane + 32 * u;
    if (k >= K) continue;
    const int64_t e = ((int64_t)d * K + k) * R + r;
    double *ph = phi + e * 2;
    double m = ph[0], s2 = ph[1];
    {  // every entry, covered or not (uncovered: acc_p = 0 -> keep), like k_mstep_leaf
      const double p = l >= 0 ? P[(int64_t)l * K + k] : 0.0;
      const bool keep = p <= kEpsCount;
      const double t0 = keep ? m : acc_pt[e * 2] / p;
      const double t1 = keep ? s2 : acc_pt[e * 2 + 1] / p;
      const double mn = (1.0 - lam) * m + lam * t0;
      const double sn = (1.0 - lam) * s2 + lam * t1;
      const double v = fmin(fmax(sn - mn * mn, var_min), var_max);
      m = mn;
      s2 = v + mn * mn;
      ph[0] = m;
      ph[1] = s2;
    }
    mu[u] = m;
    var[u] = s2 - m * m;
    csum += m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  const float cen = (float)(csum / K);
  if (lane == 0) c.center[(int64_t)r * D + d] = cen;
  const int pos = scope_pos[(int64_t)r * D + d];
  double2 *lp = (double2 *)c.leafp;
  for (int u = 0; u < 2; ++u) {
    const int k = lane + 32 * u;
    if (k >= K) continue;
    const double sa = sqrt(0.5 / var[u]);
    const double nmsa = -mu[u] * sa;
    lp[((int64_t)r * D + d) * K + k] = make_double2(sa, nmsa);
    // same roundings as the prepare path (leaf_dmma.cu k_prepare_leaf_img / _cm2)
    const double m = -fma((double)cen, sa, nmsa);
    if (l >= 0) {
      double *t = mtmp + (((int64_t)r * D + d) * K + k) * 2;
      t[0] = -0.5 * (kLog2Pi + log(var[u]));
      t[1] = __dmul_rn(m, m);
      if (dmma) {
        const int pv = pvo[l] + pos;
        double *img = c.leafimg + ((int64_t)(pv >> 1) * (K / 8) + k / 8) * 32 + (k % 8) * 4 +
                      (pv & 1) * 2;
        img[0] = sa * sa;
        img[1] = -2.0 * sa * m;
      }
    }
  }
}

// per (leaf, k): scope sums of the per-variable terms (fixed-order tree):
// cnst = sum -0.5 (log 2 pi + log var), cm2 = sum m^2. grid (n_leaf, K).
// With i8c (INT8 leaf forward): also the column scale and C = sum (mu sa)^2
// of leaf_i8.cu k_i8_colscale, from the freshly written lp (every covered
// variable is active in the cached training compute).
__global__ void __launch_bounds__(256) k_leaf_consts(const double *__restrict__ mtmp,
                                                     const int *scope_off, const int *scope_vars,
                                                     const int *leaf_rep, int D, int K,
                                                     double *cnst, double *cm2,
                                                     const int32_t *status,
                                                     const double2 *__restrict__ lp, int K8,
                                                     double *i8c) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[4][8];
  if (step_failed(status)) return;
  const int leaf = blockIdx.x, k = blockIdx.y, r = leaf_rep[leaf];
  double a = 0.0, b = 0.0, mx = 0.0, cs = 0.0;
  for (int q = scope_off[leaf] + threadIdx.x; q < scope_off[leaf + 1]; q += 256) {
    const int d = scope_vars[q];
    const double *t = mtmp + (((int64_t)r * D + d) * K + k) * 2;
    a += t[0];
    b += t[1];
    if (i8c) {
      const double2 v = lp[((int64_t)r * D + d) * K + k];
      double gu, gh, gl;
      i8_coefs(v, gu, gh, gl);
      mx = fmax(mx, fmax(fabs(gu), fmax(fabs(gh), fabs(gl))));
      cs += v.y * v.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    cs += __shfl_down_sync(0xffffffffu, cs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = b;
    red[2][threadIdx.x >> 5] = mx;
    red[3][threadIdx.x >> 5] = cs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0, m = 0.0, sc = 0.0;
    for (int w = 0; w < 8; ++w) {
      sa += red[0][w];
      sb += red[1][w];
      m = fmax(m, red[2][w]);
      sc += red[3][w];
    }
    cnst[leaf * K + k] = sa;
    if (cm2) cm2[leaf * K + k] = sb;
    if (i8c) {
      i8c[((int64_t)leaf * K8 + k) * 2] = i8_scale(m);
      i8c[((int64_t)leaf * K8 + k) * 2 + 1] = sc;
    }
  }
}

int launch_mstep(Plan &p, double *params, uint8_t *compute, const double *stats, double lam,
                 double eps_w, const int32_t *status, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  const int K = p.k;
  const int KK = K * K;
  ProfScope prof("mstep", st);
  // fused path (Gaussian leaves): the M-step kernels also re-derive every compute
  // tensor of the cached, unmasked training compute (tensor-core weight images
  // for tc-capable layers, DMMA leaf image), replacing launch_prepare
  const bool fused = p.family == EINET_FAMILY_GAUSSIAN && p.k <= 64;
  // categorical / binomial leaves: the weight and mixing compute copies (and
  // tensor-core images) come from the M-step kernels as in the fused path;
  // only the leaf terms are re-derived afterwards (launch_prepare_leaves)
  const bool fused_w = fused || p.family != EINET_FAMILY_GAUSSIAN;
  // The fused leaf branch (Gaussian) is independent of the weight updates:
  // it runs on the fork stream beside them (two branches of the CUDA graph).
  cudaStream_t ls = st;
  if (fused && p.fork_stream) {
    int rc = check_cuda(cudaEventRecord(p.fork_ev, st), "fork");
    if (!rc) rc = check_cuda(cudaStreamWaitEvent(p.fork_stream, p.fork_ev, 0), "fork");
    if (rc) return rc;
    ls = p.fork_stream;
  }
  if (fused) {
    const int64_t warps = (int64_t)p.num_replicas * p.d_vars;
    double *mtmp = (double *)(compute + p.c_mtmp);
    launch_k(k_mstep_leaf_gauss, (int)((warps + 7) / 8), 256, 0, ls, 
        params + p.sizes.phi_offset, stats + p.sizes.stats_acc_pt_offset,
        stats + p.sizes.stats_p_offset, p.d_leaf_of, p.d_scope_pos, p.d_leaf_pvo, p.d_vars, K,
        p.num_replicas, lam, p.var_min, p.var_max, status, c, p.leaf_dmma, mtmp);
    launch_k(k_leaf_consts, dim3(p.n_leaf, K), 256, 0, ls, 
        mtmp, p.d_scope_off, p.d_scope_vars, p.d_leaf_rep, p.d_vars, K, c.cnst,
        p.leaf_dmma ? c.cm2 : nullptr, status, (const double2 *)c.leafp, p.i8_k8,
        p.leaf_i8 ? (double *)(compute + p.c_i8c) : nullptr);
    count_launch(2);
    int rc = launch_i8_img(p, compute, ls);
    if (rc) return rc;
  }
  if (p.n_w) {
    const int nslices = (int)(p.n_w / KK);
    // fp64 update + fp32 copy per (l, k) slice, then the tensor-core images
    // from the fp32 copy in tile order (coalesced 16-byte stores)
    launch_k(k_mstep_einsum, nslices, 256, 0, st, params, c.w32, stats, K, lam, eps_w, status);
    count_launch();
    if (fused_w) {
      int rc = launch_build_tiles_all(p, compute, st);
      if (rc) return rc;
    }
  }
  if (p.n_mixrows) {
    launch_k(k_mstep_mixing, ceil_div(p.n_mixrows, 128), 128, 0, st, 
        params + p.n_w, c.mix32, stats + p.n_w, p.d_mixrow_off, p.d_mixrow_len,
        p.d_mix_mask_all, p.n_mixrows, lam, eps_w, status);
    count_launch();
  }
  if (fused) {
    if (ls != st) {
      int rc = check_cuda(cudaEventRecord(p.join_ev, ls), "join");
      if (!rc) rc = check_cuda(cudaStreamWaitEvent(st, p.join_ev, 0), "join");
      if (rc) return rc;
    }
    return check_cuda(cudaGetLastError(), "fused mstep kernels");
  }
  const int64_t n = (int64_t)p.d_vars * K * p.num_replicas;
  launch_k(k_mstep_leaf, (int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st, 
      params + p.sizes.phi_offset, stats + p.sizes.stats_acc_pt_offset,
      stats + p.sizes.stats_p_offset, p.d_leaf_of, p.d_vars, K, p.num_replicas, p.suff,
      p.family, lam, p.var_min, p.var_max, p.p_min, p.n_trials, status);
  count_launch();
  int rc = check_cuda(cudaGetLastError(), "mstep kernels");
  if (rc) return rc;
  if (fused_w) return launch_prepare_leaves(p, params, compute, st);
  return launch_prepare(p, params, compute, nullptr, nullptr, st);
}

// ---------------------------------------------------------------------------
// standalone fp64 log_einsum_exp (engine.py:91-109)
// ---------------------------------------------------------------------------

__global__ void k_log_einsum_exp(const double *__restrict__ left, const double *__restrict__ right,
                                 const double *__restrict__ w, int64_t B, int L, int K, int Ko,
                                 double *out) {
  EINET_KERNEL_PROLOGUE();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= B * L * Ko) return;
  const int k = (int)(e % Ko);
  const int l = (int)((e / Ko) % L);
  const int64_t b = e / ((int64_t)Ko * L);
  const double *ln = left + (b * L + l) * K, *rn = right + (b * L + l) * K;
  double a = -CUDART_INF, c = -CUDART_INF;
  bool nan = false;
  for (int i = 0; i < K; ++i) {
    nan |= ln[i] != ln[i] || rn[i] != rn[i];
    a = fmax(a, ln[i]);
    c = fmax(c, rn[i]);
  }
  const bool ok = !nan && isfinite(a) && isfinite(c);
  double r = 0.0;
  if (ok) {
    const double *wk = w + ((int64_t)l * Ko + k) * K * K;
    for (int i = 0; i < K; ++i) {
      const double ei = exp(ln[i] - a);
      double t = 0.0;
      for (int j = 0; j < K; ++j) t += wk[i * K + j] * exp(rn[j] - c);
      r += ei * t;
    }
  }
  out[e] = (ok && r > 0.0) ? a + c + log(r) : -CUDART_INF;
}

int launch_log_einsum_exp(const double *left, const double *right, const double *w, int64_t B,
                          int L, int K, int Ko, double *out, cudaStream_t st) {
  const int64_t n = B * L * Ko;
  launch_k(k_log_einsum_exp, ceil_div(n, 128), 128, 0, st, left, right, w, B, L, K, Ko, out);
  count_launch();
  return check_cuda(cudaGetLastError(), "log_einsum_exp");
}

__global__ void k_status_reset(int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  if (threadIdx.x < EINET_STATUS_WORDS) status[threadIdx.x] = INT_MAX;
}

// Cross-rank error protocol (one collective per EM update): the E-step ends by
// writing its own failure flag into the statistics buffer, which the stats
// all-reduce(sum) turns into the number of failing ranks; the M-step starts
// by turning a non-zero count into status word 3, so every rank skips the
// same update (the exact error words travel in a MIN all-reduce only then).
__global__ void k_status_to_stats(const int32_t *status, double *flag) {
  EINET_KERNEL_PROLOGUE();
  if (threadIdx.x == 0)
    *flag = (status[0] != INT_MAX || status[1] != INT_MAX || status[3] != INT_MAX) ? 1.0 : 0.0;
}

__global__ void k_status_from_stats(const double *flag, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  if (threadIdx.x == 0 && *flag > 0.0) status[3] = 0;
}

int launch_status_to_stats(const int32_t *status, double *flag, cudaStream_t st) {
  launch_k(k_status_to_stats, 1, 32, 0, st, status, flag);
  count_launch();
  return check_cuda(cudaGetLastError(), "status to stats");
}

int launch_status_from_stats(const double *flag, int32_t *status, cudaStream_t st) {
  launch_k(k_status_from_stats, 1, 32, 0, st, flag, status);
  count_launch();
  return check_cuda(cudaGetLastError(), "status from stats");
}

// Device log of a pipelined sequence of EM steps (trainer.em_stochastic_steps):
// the step's LL sum and sample count and its status words go to row *cursor of
// log_ll / log_st and the cursor advances -- the last node of the step's CUDA
// graph, so consecutive graph replays need no host-side copies in between.
__global__ void k_log_step(const double *ll2, const int32_t *status, double *log_ll,
                           int32_t *log_st, int64_t *cursor, int64_t cap) {
  EINET_KERNEL_PROLOGUE();
  const int64_t row = *cursor;
  __syncwarp();
  if (row < cap) {
    if (threadIdx.x < 2) log_ll[row * 2 + threadIdx.x] = ll2[threadIdx.x];
    if (threadIdx.x < EINET_STATUS_WORDS)
      log_st[row * EINET_STATUS_WORDS + threadIdx.x] = status[threadIdx.x];
  }
  __syncwarp();
  if (threadIdx.x == 0) *cursor = row + 1;
}

int launch_log_step(const double *ll2, const int32_t *status, double *log_ll, int32_t *log_st,
                    int64_t *cursor, int64_t cap, cudaStream_t st) {
  launch_k(k_log_step, 1, 32, 0, st, ll2, status, log_ll, log_st, cursor, cap);
  count_launch();
  return check_cuda(cudaGetLastError(), "log step");
}

int launch_status_reset(int32_t *status, cudaStream_t st) {
  launch_k(k_status_reset, 1, 32, 0, st, status);
  count_launch();
  return check_cuda(cudaGetLastError(), "status reset");
}

}  // namespace einet
