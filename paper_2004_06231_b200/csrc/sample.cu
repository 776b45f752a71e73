// Batched ancestral and conditional sampling (reference engine.py:331-423).
//
// The reference descends the region graph sample by sample in Python. Here a
// sample is one thread per layer: the chosen component of every slab on the
// sample's induced tree lives in kk[slab][sample] (-1 = not on the tree), the
// layers are processed root-first (one launch per layer), and every decision
// inverts a cumulative weight vector with a uniform from a counter-based
// Philox4x32-10 stream keyed by (seed, sample, decision site) -- the site of a
// sum decision is the slab it expands, the site of a leaf draw is
// num_slabs + variable -- so a sample's value does not depend on n or on the
// launch shape. Einsum decisions use per-(row, k) fp64 cumulative sums of
// W[l,k,:,:] (times the evidence posterior exp(log n_i + log n'_j - log s_k)
// from a forward pass of x_e for conditional sampling, engine.py:389-395),
// built sequentially so they equal numpy's cumsum; mixing decisions use the
// masked weights (times exp(log s_c - log s) conditionally, engine.py:372-379).
#include <climits>
#include <cmath>

#include "kern_common.cuh"

namespace einet {

struct Philox {
  __device__ static uint4 round10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// two uniforms in [0, 1) with 53 random bits each, for (seed, sample, site)
__device__ __forceinline__ void uniforms2(uint64_t seed, int64_t b, int site, double &u0,
                                          double &u1) {
  const uint4 r = Philox::round10(make_uint4((uint32_t)b, (uint32_t)(b >> 32), (uint32_t)site, 0u),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  u0 = ((double)(r.x >> 5) * 67108864.0 + (double)(r.y >> 6)) * (1.0 / 9007199254740992.0);
  u1 = ((double)(r.z >> 5) * 67108864.0 + (double)(r.w >> 6)) * (1.0 / 9007199254740992.0);
}

// np.searchsorted(cdf, t, side="right"): first index with cdf[i] > t
__device__ __forceinline__ int search_right(const double *cdf, int n, double t) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cdf[mid] > t) hi = mid;
    else lo = mid + 1;
  }
  return lo < n ? lo : n - 1;
}

// Cumulative (i,j) weights of every (einsum row, k): one thread per (row, k),
// sequential fp64 sum. Conditional: times exp(log n_i + log n'_j - log s_k) of
// sample 0 of the forward workspace.
__global__ void k_sample_cdf(const double *__restrict__ W, WsView ws, const int *left_slab,
                             const int *right_slab, const int *out_slab, int rows, int Ko, int K,
                             int conditional, double *cdf) {
  EINET_KERNEL_PROLOGUE();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * Ko) return;
  const int l = e / Ko, k = e % Ko;
  const int KK = K * K;
  const double *w = W + (int64_t)e * KK;
  double *c = cdf + (int64_t)e * KK;
  double base = 0.0;
  const Col32 ol = slab_off(ws, left_slab[l], 0), orr = slab_off(ws, right_slab[l], 0);
  if (conditional) {
    const double so = slab_shift(ws, out_slab[l])[0];
    const double sl = slab_shift(ws, left_slab[l])[0], sr = slab_shift(ws, right_slab[l])[0];
    base = (sl + sr) - so - (double)slab_off(ws, out_slab[l], 0)[k];
    if (so == -CUDART_INF || sl == -CUDART_INF || sr == -CUDART_INF) base = -CUDART_INF;
  }
  double acc = 0.0;
  for (int ij = 0; ij < KK; ++ij) {
    double v = w[ij];
    if (conditional) {
      const double ex = base + (double)ol[ij / K] + (double)orr[ij % K];
      v = ex == -CUDART_INF ? 0.0 : v * exp(ex);
    }
    acc += v;
    c[ij] = acc;
  }
}

// one einsum layer: expand every (sample, row) on the tree into its children
__global__ void k_sample_einsum(const double *__restrict__ cdf, int16_t *kk, int64_t n, int K,
                                int Ko, const int *left_slab, const int *right_slab,
                                const int *out_slab, uint64_t seed, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  const int l = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int os = out_slab[l];
  const int k = kk[(int64_t)os * n + b];
  if (k < 0) return;
  const int KK = K * K;
  const double *c = cdf + ((int64_t)l * Ko + k) * KK;
  const double tot = c[KK - 1];
  if (!(tot > 0.0)) {
    atomicMin(&status[3], os);
    return;
  }
  double u0, u1;
  uniforms2(seed, b, os, u0, u1);
  const int idx = search_right(c, KK, u0 * tot);
  kk[(int64_t)left_slab[l] * n + b] = (int16_t)(idx / K);
  kk[(int64_t)right_slab[l] * n + b] = (int16_t)(idx % K);
}

// one mixing layer: choose the child partition of every (sample, row) on the tree
__global__ void k_sample_mixing(const double *__restrict__ wm, WsView ws, int16_t *kk,
                                int64_t n, int dmax, const int *src_slab, const uint8_t *mask,
                                const int *out_slab, int conditional, uint64_t seed,
                                int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  const int m = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int os = out_slab[m];
  const int k = kk[(int64_t)os * n + b];
  if (k < 0) return;
  double s_out = 0.0;
  if (conditional) s_out = slab_shift(ws, os)[0] + (double)slab_off(ws, os, 0)[k];
  double acc = 0.0, target = -1.0, u0, u1;
  uniforms2(seed, b, os, u0, u1);
  double tot = 0.0;
  for (int c = 0; c < dmax; ++c) {  // total first (the draw scales by the last cumsum)
    double v = mask[m * dmax + c] ? wm[m * dmax + c] : 0.0;
    if (conditional && v != 0.0) {
      const int sl = src_slab[m * dmax + c];
      const double d = slab_shift(ws, sl)[0] + (double)slab_off(ws, sl, 0)[k] - s_out;
      v = isfinite(d) ? v * exp(d) : 0.0;
    }
    tot += v;
  }
  if (!(tot > 0.0)) {
    atomicMin(&status[3], os);
    return;
  }
  target = u0 * tot;
  int pick = dmax - 1;
  for (int c = 0; c < dmax; ++c) {
    double v = mask[m * dmax + c] ? wm[m * dmax + c] : 0.0;
    if (conditional && v != 0.0) {
      const int sl = src_slab[m * dmax + c];
      const double d = slab_shift(ws, sl)[0] + (double)slab_off(ws, sl, 0)[k] - s_out;
      v = isfinite(d) ? v * exp(d) : 0.0;
    }
    acc += v;
    if (acc > target) {
      pick = c;
      break;
    }
  }
  kk[(int64_t)src_slab[m * dmax + pick] * n + b] = (int16_t)k;
}

// leaves: one thread per (sample, variable)
__global__ void k_sample_leaves(const double *__restrict__ phi, const int16_t *kk, int64_t n,
                                int D, int K, int R, int family, int S, int n_trials,
                                const int *leaf_of, const int *leaf_slab, int num_slabs,
                                const double *x_e, const uint8_t *evidence, uint64_t seed,
                                double *out) {
  EINET_KERNEL_PROLOGUE();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * D) return;
  const int d = (int)(e % D);
  const int64_t b = e / D;
  if (evidence && evidence[d]) {
    out[e] = x_e[d];
    return;
  }
  int r = -1, k = -1;
  for (int q = 0; q < R && k < 0; ++q) {
    const int l = leaf_of[(int64_t)q * D + d];
    if (l < 0) continue;
    const int kq = kk[(int64_t)leaf_slab[l] * n + b];
    if (kq >= 0) {
      r = q;
      k = kq;
    }
  }
  if (k < 0) {
    out[e] = CUDART_NAN;
    return;
  }
  double u0, u1;
  uniforms2(seed, b, num_slabs + d, u0, u1);
  const int64_t base = ((int64_t)d * K + k) * R + r;
  if (family == EINET_FAMILY_GAUSSIAN) {
    const double mu = phi[base * 2], var = phi[base * 2 + 1] - mu * mu;
    // Box-Muller on (1 - u0) in (0, 1]
    const double z = sqrt(-2.0 * log(1.0 - u0)) * cos(6.283185307179586 * u1);
    out[e] = mu + sqrt(var) * z;
  } else if (family == EINET_FAMILY_CATEGORICAL) {
    const double *p = phi + base * S;
    double tot = 0.0;
    for (int s = 0; s < S; ++s) tot += p[s];
    const double t = u0 * tot;
    double acc = 0.0;
    int pick = S - 1;
    for (int s = 0; s < S; ++s) {
      acc += p[s];
      if (acc > t) {
        pick = s;
        break;
      }
    }
    out[e] = (double)pick;
  } else {
    const double pr = phi[base] / (double)n_trials;
    double acc = 0.0;
    int pick = n_trials;
    for (int x = 0; x <= n_trials; ++x) {
      acc += exp(lgamma((double)n_trials + 1.0) - lgamma((double)x + 1.0) -
                 lgamma((double)(n_trials - x) + 1.0) + x * log(pr) +
                 (n_trials - x) * log1p(-pr));
      if (acc > u0) {
        pick = x;
        break;
      }
    }
    out[e] = (double)pick;
  }
}

int64_t sample_scratch_bytes(const Plan &p, int64_t n) {
  return align_up(8 * p.n_w, 256) + align_up(2 * (int64_t)p.num_slabs * n, 256);
}

__global__ void k_sample_root(int16_t *kk_root, int64_t n) {
  EINET_KERNEL_PROLOGUE();
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < n) kk_root[b] = 0;  // the scalar root carries component 0
}

int launch_sample(Plan &p, const double *params, const uint8_t *wsb, int conditional,
                  const double *x_e, const uint8_t *evidence, int64_t n, uint64_t seed,
                  uint8_t *scratch, double *out, int32_t *status, cudaStream_t st) {
  if (p.k_root != 1) return fail(EINET_ERR_ENGINE, "sampling requires a scalar root (k_root = 1)");
  if (p.k > 32767) return fail(EINET_ERR_USAGE, "k too large for sampling");
  if (n < 1) return EINET_OK;
  WsView ws = ws_view(p, wsb);
  double *cdf = (double *)scratch;
  int16_t *kk = (int16_t *)(scratch + align_up(8 * p.n_w, 256));
  int rc = check_cuda(cudaMemsetAsync(kk, 0xFF, 2 * (size_t)p.num_slabs * n, st), "sample init");
  if (rc) return rc;
  const int nb = ceil_div(n, 128);
  launch_k(k_sample_root, nb, 128, 0, st, kk + (int64_t)p.root_out_slab * n, n);
  count_launch();
  const int K = p.k;
  for (auto &L : p.layers) {
    if (L.kind != EINET_LAYER_EINSUM) continue;
    const int nthr = L.rows * L.k_out;
    launch_k(k_sample_cdf, ceil_div(nthr, 128), 128, 0, st, params + L.w_off, ws, L.d_left_slab,
                                                       L.d_right_slab, L.d_out_slab, L.rows,
                                                       L.k_out, K, conditional, cdf + L.w_off);
    count_launch();
  }
  for (int li = (int)p.layers.size() - 1; li >= 0; --li) {
    const LayerPlan &L = p.layers[li];
    dim3 grid(nb, L.rows);
    if (L.kind == EINET_LAYER_EINSUM) {
      launch_k(k_sample_einsum, grid, 128, 0, st, cdf + L.w_off, kk, n, K, L.k_out, L.d_left_slab,
                                            L.d_right_slab, L.d_out_slab, seed, status);
    } else {
      launch_k(k_sample_mixing, grid, 128, 0, st, params + p.n_w + L.mix_off, ws, kk, n, L.dmax,
                                            L.d_mix_src_slab, L.d_mix_mask, L.d_out_slab,
                                            conditional, seed, status);
    }
    count_launch();
  }
  const int64_t tot = n * p.d_vars;
  launch_k(k_sample_leaves, (int)((tot + 255) / 256), 256, 0, st, 
      params + p.sizes.phi_offset, kk, n, p.d_vars, K, p.num_replicas, p.family, p.num_states,
      p.n_trials, p.d_leaf_of, p.d_leaf_slab, p.num_slabs, x_e, evidence, seed, out);
  count_launch();
  return check_cuda(cudaGetLastError(), "sampling kernels");
}

}  // namespace einet
