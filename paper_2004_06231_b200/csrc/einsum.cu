// EinsumLayer / EinsumMixingLayer kernels (CUDA-core path) and the
// forward / backward orchestration.
//
// Forward  (engine.py:91-122, 143-195): out[b,l,k] = a + c + log sum_ij
//   W[l,k,i,j] e^(N[b,l,i]-a) e^(N'[b,l,j]-c). Slabs carry (shift fp64, offsets
//   fp32): a, c are the fp32 maxima of the child offsets, the new shift is
//   s_left + s_right + a + c and the new offsets are log r (small magnitude).
// Backward (engine.py:247-316): rho_t = rho / r; W statistics
//   n[l,k,i,j] += W sum_b rho_t ea_i eb_j; child responsibilities
//   left_i = ea_i sum_k rho_t_k sum_j W_kij eb_j, right_j likewise, written to
//   per-row slots and gathered by the consumers in a fixed order.
#include <climits>
#include <cmath>

#include "kern_common.cuh"

namespace einet {

int launch_leaf_forward(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                        uint8_t *wsb, int32_t *status, cudaStream_t st);
int launch_leaf_backward(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                         uint8_t *wsb, double *stats, cudaStream_t st);
int launch_einsum_wstats_tc(Plan &p, const LayerPlan &L, const float *EA, const float *EB,
                            WsView &w, int64_t B, int *bsplit, cudaStream_t st);

constexpr int EF_TB = 128;  // samples per CTA, one per thread
constexpr int EF_KC = 8;    // output entries (k) staged per W chunk

// Forward prep: normalised child exponentials EA = exp(off_left - a),
// EB = exp(off_right - c) with a, c the fp32 maxima (engine.py:99-104), kept
// per layer for the backward; the output shift s_left + s_right + a + c
// (engine.py:108); NaN entering the layer -> status.
// One CTA per 32-sample block and row: the block's [K][32] slab tiles and the
// EA/EB tiles are contiguous, so every pass is a coalesced elementwise sweep.
// grid (ceil(B/32), L), block 128.
__global__ void __launch_bounds__(128) k_einsum_prep_fwd(
    WsView ws, const int *__restrict__ left_slab, const int *__restrict__ right_slab,
    const int *__restrict__ out_slab, int64_t B, int K, float *__restrict__ EA,
    float *__restrict__ EB, float *__restrict__ EBM, float *__restrict__ EAM, int kp,
    int layer_index, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  __shared__ float mx[2][32];
  __shared__ float pmx[2][4][32];
  __shared__ unsigned char dead[32];
  const int l = blockIdx.y, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int nb = (int)min((int64_t)32, B - b0);
  const int ls = left_slab[l], rs = right_slab[l];
  if (EBM != nullptr && (kp / 4) * 32 <= 4 * 128) {
    // tensor-core path, one pass: thread = (sample lane, quads q = wid + 4 i);
    // its child values are loaded once, up front, and give both the per-warp
    // maxima and the exponentials (stores only after every load)
    const int nq4 = (kp / 4) * 32;
    const float *ol = ws.off + tb_idx(ls, b0, 0, ws.bc, ws.ks) + lane;
    const float *orr = ws.off + tb_idx(rs, b0, 0, ws.bc, ws.ks) + lane;
    float xl[4][4], xr[4][4];
    float ml = -CUDART_INF_F, mr = -CUDART_INF_F;
    bool nan = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = (t + 128 * i) >> 5;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * q + u;
        const bool ok = t + 128 * i < nq4 && k < K;
        xl[i][u] = ok ? __ldg(ol + k * 32) : -CUDART_INF_F;
        xr[i][u] = ok ? __ldg(orr + k * 32) : -CUDART_INF_F;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        nan |= (xl[i][u] != xl[i][u]) | (xr[i][u] != xr[i][u]);
        ml = fmaxf(ml, xl[i][u]);
        mr = fmaxf(mr, xr[i][u]);
      }
    pmx[0][wid][lane] = ml;
    pmx[1][wid][lane] = mr;
    if (nan && lane < nb) atomicMin(&status[1], layer_index);
    __syncthreads();
    if (t < 32) {
      const float m0 = fmaxf(fmaxf(pmx[0][0][t], pmx[0][1][t]), fmaxf(pmx[0][2][t], pmx[0][3][t]));
      const float m1 = fmaxf(fmaxf(pmx[1][0][t], pmx[1][1][t]), fmaxf(pmx[1][2][t], pmx[1][3][t]));
      mx[0][t] = m0;
      mx[1][t] = m1;
      bool d = true;
      if (t < nb) {
        const int64_t b = b0 + t;
        const double sl = slab_shift(ws, ls)[b], sr = slab_shift(ws, rs)[b];
        if (sl != sl || sr != sr) atomicMin(&status[1], layer_index);
        d = sl == -CUDART_INF || sr == -CUDART_INF || m0 == -CUDART_INF_F || m1 == -CUDART_INF_F;
        slab_shift(ws, out_slab[l])[b] = d ? -CUDART_INF : (sl + (double)m0) + (sr + (double)m1);
      }
      dead[t] = d;
    }
    __syncthreads();
    const bool d = dead[lane];
    const float m0 = mx[0][lane], m1 = mx[1][lane];
    float *ea = EA + ev_idx(l, b0, 0, ws.bc, K), *eb = EB + ev_idx(l, b0, 0, ws.bc, K);
    const int64_t ntl = ws.bc / 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = t + 128 * i;
      if (e >= nq4) break;
      const int q = e >> 5;
      float va[4] = {0.f, 0.f, 0.f, 0.f}, vb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * q + u;
        if (k >= K) break;
        const int xe = k * EV_ROW + lane;
        va[u] = d ? 0.f : expf(xl[i][u] - m0);
        vb[u] = d ? 0.f : expf(xr[i][u] - m1);
        ea[xe] = va[u];
        eb[xe] = vb[u];
      }
      store_bf16_quad(EBM, l, b0 + lane, q, ntl, kp, make_float4(vb[0], vb[1], vb[2], vb[3]));
      if (EAM)
        store_bf16_quad(EAM, l, b0 + lane, q, ntl, kp, make_float4(va[0], va[1], va[2], va[3]));
    }
    return;
  }
  if (wid < 2) {  // warp 0: left maxima, warp 1: right maxima (lane = sample)
    const int slab = wid ? rs : ls;
    const float *o = ws.off + tb_idx(slab, b0, 0, ws.bc, ws.ks) + lane;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F;
    bool nan = false;
    int k = 0;
#pragma unroll 4
    for (; k + 1 < K; k += 2) {
      const float v0 = o[k * 32], v1 = o[(k + 1) * 32];
      nan |= (v0 != v0) | (v1 != v1);
      m0 = fmaxf(m0, v0);
      m1 = fmaxf(m1, v1);
    }
    if (k < K) {
      const float v = o[k * 32];
      nan |= v != v;
      m0 = fmaxf(m0, v);
    }
    const float m = fmaxf(m0, m1);
    if (lane < nb) {
      const double sh = slab_shift(ws, slab)[b0 + lane];
      nan |= sh != sh;
      if (nan) atomicMin(&status[1], layer_index);
    }
    mx[wid][lane] = m;
  }
  __syncthreads();
  if (t < 32) {
    const int64_t b = b0 + t;
    bool d = true;
    if (t < nb) {
      const double sl = slab_shift(ws, ls)[b], sr = slab_shift(ws, rs)[b];
      d = sl == -CUDART_INF || sr == -CUDART_INF || mx[0][t] == -CUDART_INF_F ||
          mx[1][t] == -CUDART_INF_F;
      slab_shift(ws, out_slab[l])[b] =
          d ? -CUDART_INF : (sl + (double)mx[0][t]) + (sr + (double)mx[1][t]);
    }
    dead[t] = d;
  }
  __syncthreads();
  const float *ol = ws.off + tb_idx(ls, b0, 0, ws.bc, ws.ks);
  const float *orr = ws.off + tb_idx(rs, b0, 0, ws.bc, ws.ks);
  float *ea = EA + ev_idx(l, b0, 0, ws.bc, K), *eb = EB + ev_idx(l, b0, 0, ws.bc, K);
  if (EBM == nullptr) {
    for (int e = t; e < K * 32; e += 128) {
      const int bl = e & 31, x = (e >> 5) * EV_ROW + bl;
      const bool d = dead[bl];
      ea[x] = d ? 0.f : expf(ol[e] - mx[0][bl]);
      eb[x] = d ? 0.f : expf(orr[e] - mx[1][bl]);
    }
    return;
  }
  // tensor-core path: also the EB (and for direct child-rho rows
  // EA) bf16 A-operand tiles, width kp (entries K..kp-1 are zero)
  const int64_t ntl = ws.bc / 128;
  for (int e = t; e < (kp / 4) * 32; e += 128) {
    const int bl = e & 31, q = e >> 5;
    const bool d = dead[bl];
    float va[4] = {0.f, 0.f, 0.f, 0.f}, vb[4] = {0.f, 0.f, 0.f, 0.f};
    if (4 * q < K) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (4 * q + u >= K) break;
        const int x = (4 * q + u) * 32 + bl, xe = (4 * q + u) * EV_ROW + bl;
        va[u] = d ? 0.f : expf(ol[x] - mx[0][bl]);
        vb[u] = d ? 0.f : expf(orr[x] - mx[1][bl]);
        ea[xe] = va[u];
        eb[xe] = vb[u];
      }
    }
    store_bf16_quad(EBM, l, b0 + bl, q, ntl, kp, make_float4(vb[0], vb[1], vb[2], vb[3]));
    if (EAM) store_bf16_quad(EAM, l, b0 + bl, q, ntl, kp, make_float4(va[0], va[1], va[2], va[3]));
  }
}

template <int KT>
__device__ __forceinline__ float dot_row(const float *w, const float (&v)[KT]) {
  const float4 *w4 = (const float4 *)w;
  float t0 = 0.f, t1 = 0.f;
#pragma unroll
  for (int j = 0; j < KT / 4; ++j) {
    const float4 q = w4[j];
    t0 = fmaf(q.x, v[4 * j], t0);
    t1 = fmaf(q.y, v[4 * j + 1], t1);
    t0 = fmaf(q.z, v[4 * j + 2], t0);
    t1 = fmaf(q.w, v[4 * j + 3], t1);
  }
  return t0 + t1;
}

// Stage W[l][k0:k0+nk][i][0:K] into smem as [kk][i][KT] (zero padded).
__device__ __forceinline__ void stage_w(float *wsm, const float *__restrict__ Wl, int k0, int nk,
                                        int K, int KT) {
  const int n = nk * K * KT;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int j = e % KT;
    const int i = (e / KT) % K;
    const int kk = e / (KT * K);
    wsm[e] = j < K ? Wl[((int64_t)(k0 + kk) * K + i) * K + j] : 0.f;
  }
}

// SIMT forward GEMM: one sample per thread, ea/eb in registers, W chunk in smem.
// grid (ceil(B/128), L, ceil(Ko/8)), block 128
template <int KT>
__global__ void __launch_bounds__(EF_TB) k_einsum_fwd(WsView ws, const float *__restrict__ EA,
                                                      const float *__restrict__ EB,
                                                      const int *__restrict__ out_slab,
                                                      const float *__restrict__ W, int64_t B,
                                                      int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float wsm[];
  const int l = blockIdx.y;
  const int k0 = blockIdx.z * EF_KC;
  const int nk = min(EF_KC, Ko - k0);
  stage_w(wsm, W + (int64_t)l * Ko * K * K, k0, nk, K, KT);
  const int64_t b = (int64_t)blockIdx.x * EF_TB + threadIdx.x;
  const bool live = b < B;
  const int64_t bb = live ? b : 0;
  float ea[KT], eb[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    ea[i] = (live && i < K) ? EA[ev_idx(l, bb, i, ws.bc, K)] : 0.f;
    eb[i] = (live && i < K) ? EB[ev_idx(l, bb, i, ws.bc, K)] : 0.f;
  }
  __syncthreads();
  if (!live) return;
  const Col32 o = slab_off(ws, out_slab[l], b);
  for (int kk = 0; kk < nk; ++kk) {
    const float *wk = wsm + kk * K * KT;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < KT; ++i)
      if (i < K) acc = fmaf(ea[i], dot_row<KT>(wk + i * KT, eb), acc);
    o[k0 + kk] = acc > 0.f ? logf(acc) : -CUDART_INF_F;
  }
}

// Generic (any K) forward from EA/EB, W read through L1.
__global__ void k_einsum_fwd_generic(WsView ws, const float *__restrict__ EA,
                                     const float *__restrict__ EB, const int *out_slab,
                                     const float *__restrict__ W, int64_t B, int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  const int l = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const Col32 o = slab_off(ws, out_slab[l], b);
  const float *Wl = W + (int64_t)l * Ko * K * K;
  for (int k = 0; k < Ko; ++k) {
    float acc = 0.f;
    for (int i = 0; i < K; ++i) {
      float t = 0.f;
      for (int j = 0; j < K; ++j)
        t = fmaf(Wl[((int64_t)k * K + i) * K + j], EB[ev_idx(l, b, j, ws.bc, K)], t);
      acc = fmaf(EA[ev_idx(l, b, i, ws.bc, K)], t, acc);
    }
    o[k] = acc > 0.f ? logf(acc) : -CUDART_INF_F;
  }
}

// Forward for 64 < K <= 128 on CUDA cores (the register-tile kernel above
// keeps a sample's EA, EB rows in registers, which stops scaling past 64).
// out[b,k] = log sum_i EA[b,i] sum_j W[k,i,j] EB[b,j] (engine.py:91-109) as a
// tiled GEMM per (row, k): the CTA stages W[k] transposed ([j][i]) and the
// tile's EB, EA rows in shared memory; a thread accumulates s[b][i] =
// sum_j W[k,i,j] EB[b,j] for 4 samples x 8 i (per j: one 16-byte EB load, two
// 16-byte W loads, 32 FMAs), folds in EA[b,i] and the 16 i-groups are summed
// in fixed order. grid (ceil(B/64), rows, K_out), block 256.
constexpr int FB_TB = 64, FB_KP = 128, FB_WS = FB_KP + 4;
size_t fwd_big_smem() {
  return sizeof(float) * ((size_t)FB_KP * FB_WS + 2 * FB_KP * FB_TB + 16 * FB_TB);
}
__global__ void __launch_bounds__(256) k_einsum_fwd_big(WsView ws, const float *__restrict__ EA,
                                                        const float *__restrict__ EB,
                                                        const int *out_slab,
                                                        const float *__restrict__ W, int64_t B,
                                                        int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float fsm[];
  float *wt = fsm;                       // [j][FB_WS]: W[k][i][j] at wt[j][i]
  float *ebs = wt + FB_KP * FB_WS;       // [j][64]
  float *eas = ebs + FB_KP * FB_TB;      // [i][64]
  float *red = eas + FB_KP * FB_TB;      // [16][64]
  const int tid = threadIdx.x, l = blockIdx.y, k = blockIdx.z;
  const int64_t b0 = (int64_t)blockIdx.x * FB_TB;
  const float *Wk = W + ((int64_t)l * Ko + k) * K * K;
  for (int e = tid; e < FB_KP * FB_KP; e += 256) {
    const int i = e / FB_KP, j = e - i * FB_KP;
    wt[j * FB_WS + i] = (i < K && j < K) ? Wk[i * K + j] : 0.f;
  }
  for (int e = tid; e < FB_KP * FB_TB; e += 256) {
    const int r = e >> 6, s = e & 63;
    const int64_t b = b0 + s;
    float vb = 0.f, va = 0.f;
    if (r < K && b < ws.bc) {
      const int64_t x = ev_idx(l, b, r, ws.bc, K);
      vb = EB[x];
      va = EA[x];
    }
    ebs[e] = vb;
    eas[e] = va;
  }
  __syncthreads();
  const int sg = tid & 15, ig = tid >> 4;
  float s[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) s[a][c] = 0.f;
  for (int j = 0; j < K; ++j) {
    const float4 eb = *(const float4 *)(ebs + j * FB_TB + sg * 4);
    const float4 w0 = *(const float4 *)(wt + j * FB_WS + ig * 8);
    const float4 w1 = *(const float4 *)(wt + j * FB_WS + ig * 8 + 4);
    const float ebv[4] = {eb.x, eb.y, eb.z, eb.w};
    const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 8; ++c) s[a][c] = fmaf(wv[c], ebv[a], s[a][c]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    float part = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) part = fmaf(eas[(ig * 8 + c) * FB_TB + sg * 4 + a], s[a][c], part);
    red[ig * FB_TB + sg * 4 + a] = part;
  }
  __syncthreads();
  if (tid < FB_TB) {
    const int64_t b = b0 + tid;
    if (b < B) {
      float acc = 0.f;
      for (int g = 0; g < 16; ++g) acc += red[g * FB_TB + tid];
      slab_off(ws, out_slab[l], b)[k] = acc > 0.f ? logf(acc) : -CUDART_INF_F;
    }
  }
}

// ---------------------------------------------------------------------------
// mixing layers (engine.py:112-122, 268-293)
// ---------------------------------------------------------------------------

// Mixing forward, elementwise over (sample, k) of a 32-sample block:
// out = s + mk + log sum_c w_c exp(s_c - s + off_c - mk) with s = max_c s_c
// (engine.py:112-122; masked children never contribute).
// grid (ceil(B/32), M), block 128: a thread keeps one sample (lane) and walks
// k = warp, warp + 4, ...; the sample's child shifts are loaded once, the
// child offsets of one k are independent loads (MC children in registers).
constexpr int MC = 8;  // children handled in registers; larger rows loop over groups
__global__ void __launch_bounds__(128) k_mixing_fwd(
    WsView ws, const int *__restrict__ src_slab, const uint8_t *__restrict__ mask,
    const int *__restrict__ out_slab, const float *__restrict__ w, int64_t B, int Ko, int dmax,
    int layer_index, int32_t *status) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ int msm[];
  int *src = msm;                        // [dmax], -1 = masked
  float *wc = (float *)(msm + dmax);     // [dmax]
  (void)layer_index;
  (void)status;
  const int m = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < dmax; c += 128) {
    src[c] = mask[m * dmax + c] ? src_slab[m * dmax + c] : -1;
    wc[c] = w[m * dmax + c];
  }
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * 32, b = b0 + lane;
  if (b >= B) return;
  const int os = out_slab[m];
  float *o = ws.off + tb_idx(os, b0, 0, ws.bc, ws.ks);
  if (dmax <= MC) {
    double sc[MC];
    const float *oc[MC];
    double sh = -CUDART_INF;
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      sc[c] = -CUDART_INF;
      oc[c] = nullptr;
      if (c < dmax && src[c] >= 0) {
        sc[c] = slab_shift(ws, src[c])[b];
        oc[c] = ws.off + tb_idx(src[c], b0, 0, ws.bc, ws.ks);
        if (sc[c] > sh || sc[c] != sc[c]) sh = sc[c];
      }
    }
    if (wid == 0 && blockIdx.z == 0) slab_shift(ws, os)[b] = sh;
#pragma unroll 4
    for (int k = wid + 4 * blockIdx.z; k < Ko; k += 4 * gridDim.z) {
      const int e = k * 32 + lane;
      if (sh == -CUDART_INF) {
        o[e] = 0.f;
        continue;
      }
      float dv[MC];
      float mk = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        dv[c] = -CUDART_INF_F;
        if (oc[c] && sc[c] != -CUDART_INF) dv[c] = (float)(sc[c] - sh) + oc[c][e];
        mk = fmaxf(mk, dv[c]);
      }
      float out = -CUDART_INF_F;
      if (mk != -CUDART_INF_F) {
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < MC; ++c)
          if (dv[c] != -CUDART_INF_F) sum = fmaf(wc[c < dmax ? c : 0], expf(dv[c] - mk), sum);
        if (sum > 0.f) out = mk + logf(sum);
      }
      o[e] = out;
    }
    return;
  }
  // generic (many children)
  double sh = -CUDART_INF;
  for (int c = 0; c < dmax; ++c) {
    if (src[c] < 0) continue;
    const double scc = slab_shift(ws, src[c])[b];
    if (scc > sh || scc != scc) sh = scc;
  }
  if (wid == 0 && blockIdx.z == 0) slab_shift(ws, os)[b] = sh;
  for (int k = wid + 4 * blockIdx.z; k < Ko; k += 4 * gridDim.z) {
    const int e = k * 32 + lane;
    if (sh == -CUDART_INF) {
      o[e] = 0.f;
      continue;
    }
    float mk = -CUDART_INF_F;
    for (int c = 0; c < dmax; ++c) {
      if (src[c] < 0) continue;
      const double scc = slab_shift(ws, src[c])[b];
      if (scc == -CUDART_INF) continue;
      mk = fmaxf(mk, (float)(scc - sh) + ws.off[tb_idx(src[c], b0, 0, ws.bc, ws.ks) + e]);
    }
    float out = -CUDART_INF_F;
    if (mk != -CUDART_INF_F) {
      float sum = 0.f;
      for (int c = 0; c < dmax; ++c) {
        if (src[c] < 0) continue;
        const double scc = slab_shift(ws, src[c])[b];
        if (scc == -CUDART_INF) continue;
        const float dvv = (float)(scc - sh) + ws.off[tb_idx(src[c], b0, 0, ws.bc, ws.ks) + e];
        sum = fmaf(wc[c], expf(dvv - mk), sum);
      }
      if (sum > 0.f) out = mk + logf(sum);
    }
    o[e] = out;
  }
}

// Responsibility of slab `slab` for element e (= k*32 + sample) of the
// 32-sample block at b0: ordered sum over the slab's contribution slots.
__device__ __forceinline__ float gather_rho_tile(const WsView &ws, int q0, int q1,
                                                 const int *__restrict__ csr_slot, bool one,
                                                 int64_t b0, int e) {
  if (one) return 1.0f;
  float acc = 0.0f;
  for (int q = q0; q < q1; ++q) acc += ws.slots[tb_idx(csr_slot[q], b0, 0, ws.bc, ws.ks) + e];
  return acc;
}

// gather_rho_tile for up to RE_MAX tile entries of one thread at once: slot by
// slot (the same summation order per entry), all entries' loads of one slot in
// flight together. idx(j) = tile entry of item j, or < 0 for none.
constexpr int RE_MAX = 16;
template <typename F>
__device__ __forceinline__ void gather_rho_many(const WsView &ws, int q0, int q1,
                                                const int *__restrict__ csr_slot, bool one,
                                                int64_t b0, F idx, float (&acc)[RE_MAX]) {
#pragma unroll
  for (int j = 0; j < RE_MAX; ++j) acc[j] = one ? 1.0f : 0.0f;
  if (one) return;
  for (int q = q0; q < q1; ++q) {
    const float *sp = ws.slots + tb_idx(csr_slot[q], b0, 0, ws.bc, ws.ks);
#pragma unroll
    for (int j = 0; j < RE_MAX; ++j) {
      const int x = idx(j);
      if (x >= 0) acc[j] += sp[x];
    }
  }
}

// Deterministic CTA sum of one double per thread (fixed tree, 4 warps).
__device__ __forceinline__ double cta_sum128(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const double s = (red[0] + red[1]) + (red[2] + red[3]);
  __syncthreads();
  return s;
}

// Mixing backward: contribution of child c to the responsibility of its slab
// rho_c = rho * w_c * exp(s_c + off_c - s - off) (engine.py:268-293), written
// to the child's slot; the mixing statistics get the per-CTA partial sums.
// grid (ceil(B/32), M), block 128.
__global__ void __launch_bounds__(128) k_mixing_bwd(
    WsView ws, const int *__restrict__ src_slab, const uint8_t *__restrict__ mask,
    const int *__restrict__ out_slab, const int *__restrict__ mix_slot,
    const float *__restrict__ w, const int *csr_off, const int *__restrict__ csr_slot,
    const uint8_t *ones, int64_t B, int Ko, int dmax, double *mixpart, int64_t mix_off,
    int64_t n_mix) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[4];
  const int m = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int os = out_slab[m];
  const int q0 = csr_off[os], q1 = csr_off[os + 1];
  const bool one = ones[os] != 0;
  const float *oo = ws.off + tb_idx(os, b0, 0, ws.bc, ws.ks);
  const int ne = Ko * 32;
  const bool many = ne <= 128 * RE_MAX;
  float rho[RE_MAX];  // this thread's entries e = tid + 128 j of the slab's rho
  if (many)
    gather_rho_many(ws, q0, q1, csr_slot, one, b0,
                    [&](int j) { const int e = threadIdx.x + 128 * j; return e < ne ? e : -1; },
                    rho);
  // one sample per thread (128 = 4 x 32): its shift and output log-densities
  // are loaded once, each child's before any store (dst may alias them for
  // the compiler: interleaved, every entry would wait a full memory trip)
  const int64_t bt = b0 + (threadIdx.x & 31);
  const bool in = bt < B;
  const double so_t = in ? slab_shift(ws, os)[bt] : -CUDART_INF;
  float ov[RE_MAX];
#pragma unroll
  for (int j = 0; j < RE_MAX; ++j) {
    const int e = threadIdx.x + 128 * j;
    ov[j] = (many && e < ne && in) ? __ldg(oo + e) : 0.f;
  }
  for (int c = 0; c < dmax; ++c) {
    float run = 0.f;
    if (mask[m * dmax + c]) {
      const int sl = src_slab[m * dmax + c];
      const float wc = w[m * dmax + c];
      const float *oc = ws.off + tb_idx(sl, b0, 0, ws.bc, ws.ks);
      float *dst = ws.slots + tb_idx(mix_slot[m * dmax + c], b0, 0, ws.bc, ws.ks);
      if (many && in) {
        const double sc = slab_shift(ws, sl)[bt];
        const bool ok = so_t != -CUDART_INF && sc != -CUDART_INF;
        const float dsh = ok ? (float)(sc - so_t) : 0.f;
        float cv[RE_MAX];
#pragma unroll
        for (int j = 0; j < RE_MAX; ++j) {
          const int e = threadIdx.x + 128 * j;
          cv[j] = e < ne ? __ldg(oc + e) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < RE_MAX; ++j) {
          const int e = threadIdx.x + 128 * j;
          if (e >= ne) break;
          const float dk = dsh + cv[j] - ov[j];
          const float ratio = (ok && isfinite(dk)) ? expf(dk) : 0.f;
          const float contrib = rho[j] * wc * ratio;
          dst[e] = contrib;
          run += contrib;
        }
      }
      for (int e = threadIdx.x; !many && e < ne; e += 128) {
        const int64_t b = b0 + (e & 31);
        if (b >= B) continue;
        const double so = slab_shift(ws, os)[b], sc = slab_shift(ws, sl)[b];
        const bool ok = so != -CUDART_INF && sc != -CUDART_INF;
        const float dk = (ok ? (float)(sc - so) : 0.f) + oc[e] - oo[e];
        const float ratio = (ok && isfinite(dk)) ? expf(dk) : 0.f;
        const float contrib = gather_rho_tile(ws, q0, q1, csr_slot, one, b0, e) * wc * ratio;
        dst[e] = contrib;
        run += contrib;
      }
    }
    const double tot = cta_sum128((double)run, red);
    if (threadIdx.x == 0)
      mixpart[(int64_t)blockIdx.x * n_mix + mix_off + (int64_t)m * dmax + c] = tot;
  }
}

// ---------------------------------------------------------------------------
// einsum backward
// ---------------------------------------------------------------------------

// RT = rho / r per row and sample (engine.py:310-311), r = exp(log r) from the
// forward offsets; elementwise over a 32-sample block (contiguous tiles).
// grid (ceil(B/32), L), block 128
__global__ void __launch_bounds__(128) k_einsum_bwd_rt(
    WsView ws, const int *out_slab, const int *csr_off, const int *__restrict__ csr_slot,
    const uint8_t *ones, int64_t B, int Ko, float *RT, float *RTM, int kob, float *RTB, int nn) {
  EINET_KERNEL_PROLOGUE();
  const int l = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int os = out_slab[l];
  const int q0 = csr_off[os], q1 = csr_off[os + 1];
  const bool one = ones[os] != 0;
  const float *oo = ws.off + tb_idx(os, b0, 0, ws.bc, ws.ks);
  float *rt = RT + tb_idx(l, b0, 0, ws.bc, ws.ks);
  if (RTM == nullptr) {
    const int ne = Ko * 32;
    if (ne <= 128 * RE_MAX) {
      float rhos[RE_MAX];
      gather_rho_many(ws, q0, q1, csr_slot, one, b0,
                      [&](int j) { const int e = threadIdx.x + 128 * j; return e < ne ? e : -1; },
                      rhos);
      // every load of the thread before the first store (rt may alias oo for
      // the compiler: interleaved, each entry would wait a full memory trip)
      float ov[RE_MAX];
      const int64_t bt = b0 + (threadIdx.x & 31);  // (128 = 4 x 32: one sample per thread)
      const bool live = bt < B && slab_shift(ws, os)[bt] != -CUDART_INF;
#pragma unroll
      for (int j = 0; j < RE_MAX; ++j) {
        const int e = threadIdx.x + 128 * j;
        ov[j] = e < ne && live ? __ldg(oo + e) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < RE_MAX; ++j) {
        const int e = threadIdx.x + 128 * j;
        if (e >= ne) break;
        const int64_t b = b0 + (e & 31);
        float v = 0.f;
        if (b < B) {
          const float r = live ? expf(ov[j]) : 0.f;
          v = r > 0.f ? rhos[j] / r : 0.f;
        }
        rt[e] = v;  // samples past the batch hold 0 (the W statistics sum whole blocks)
      }
    } else {
      for (int e = threadIdx.x; e < ne; e += 128) {
        const int64_t b = b0 + (e & 31);
        float v = 0.f;
        if (b < B) {
          const float r = slab_shift(ws, os)[b] == -CUDART_INF ? 0.f : expf(oo[e]);
          const float rho = gather_rho_tile(ws, q0, q1, csr_slot, one, b0, e);
          v = r > 0.f ? rho / r : 0.f;
        }
        rt[e] = v;
      }
    }
    if (RTB) {
      __syncthreads();
      bt_tile16(rt, (uint8_t *)RTB + ((int64_t)l * (ws.bc / 32) + b0 / 32) * (nn * 128), Ko, nn);
    }
    return;
  }
  // tensor-core path: also the RT bf16 A-operand tile (width kob, zero padded)
  const int64_t ntl = ws.bc / 128;
  const int ne = (kob / 4) * 32;
  if (ne <= 128 * (RE_MAX / 4)) {
    // all of this thread's entries gathered together: item j = 4 it + u
    float rhos[RE_MAX];
    gather_rho_many(ws, q0, q1, csr_slot, one, b0,
                    [&](int j) {
                      const int e = threadIdx.x + 128 * (j >> 2), k = 4 * (e >> 5) + (j & 3);
                      return (e < ne && k < Ko) ? k * 32 + (e & 31) : -1;
                    },
                    rhos);
    // the thread's sample is the same for every item (128 = 4 x 32): its
    // liveness and all its output log-densities are loaded before any store
    const int64_t bt = b0 + (threadIdx.x & 31);
    const bool live = bt < B && slab_shift(ws, os)[bt] != -CUDART_INF;
    float ov[RE_MAX];
#pragma unroll
    for (int j = 0; j < RE_MAX; ++j) {
      const int e = threadIdx.x + 128 * (j >> 2), k = 4 * (e >> 5) + (j & 3);
      ov[j] = (e < ne && k < Ko && live) ? __ldg(oo + k * 32 + (e & 31)) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < RE_MAX / 4; ++it) {
      const int e = threadIdx.x + 128 * it;
      if (e >= ne) break;
      const int bl = e & 31, q = e >> 5;
      const int64_t b = b0 + bl;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * q + u;
        if (k >= Ko) continue;
        const int x = k * 32 + bl;
        if (b < B) {
          const float r = live ? expf(ov[4 * it + u]) : 0.f;
          v[u] = r > 0.f ? rhos[4 * it + u] / r : 0.f;
        }
        rt[x] = v[u];
      }
      store_bf16_quad(RTM, l, b, q, ntl, kob, make_float4(v[0], v[1], v[2], v[3]));
    }
  } else {
    for (int e = threadIdx.x; e < ne; e += 128) {
      const int bl = e & 31, q = e >> 5;
      const int64_t b = b0 + bl;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      const bool live = b < B && slab_shift(ws, os)[b] != -CUDART_INF;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * q + u;
        if (k >= Ko) continue;
        const int x = k * 32 + bl;
        if (b < B) {
          const float r = live ? expf(oo[x]) : 0.f;
          const float rho = gather_rho_tile(ws, q0, q1, csr_slot, one, b0, x);
          v[u] = r > 0.f ? rho / r : 0.f;
        }
        rt[x] = v[u];
      }
      store_bf16_quad(RTM, l, b, q, ntl, kob, make_float4(v[0], v[1], v[2], v[3]));
    }
  }
  if (RTB) {
    __syncthreads();
    bt_tile16(rt, (uint8_t *)RTB + ((int64_t)l * (ws.bc / 32) + b0 / 32) * (nn * 128), Ko, nn);
  }
}

constexpr int WS_BT = 32;  // samples per fp32 run of the W statistics

// sum_b RT[b,k] EA[b,i] EB[b,j] for one (l, k) per CTA and a batch split.
// Register tile 4x4 of (i, j) per thread; block K4*K4 threads.
__global__ void k_einsum_wstats(const float *__restrict__ EA, const float *__restrict__ EB,
                                const float *__restrict__ RT, int64_t Bc, int ks, int64_t B,
                                int K, int Ko, int L, int bsplit, double *wpart, int ti_per,
                                int kc) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float sm[];
  const int K4 = (K + 3) / 4;
  const int KP = K4 * 4;
  float *ea_s = sm;                     // [WS_BT][KP]
  float *eb_s = ea_s + WS_BT * KP;      // [WS_BT][KP]
  float *rt_s = eb_s + WS_BT * KP;      // [WS_BT][kc]
  // blockIdx.x = (row l, chunk of kc output components): the chunk's slices
  // share the EA / EB staging (small K: kc K4^2 threads instead of K4^2)
  const int nkc = (Ko + kc - 1) / kc;
  const int l = blockIdx.x / nkc, k0 = (blockIdx.x % nkc) * kc;
  const int tpk = ti_per * K4, kk = threadIdx.x / tpk, rr = threadIdx.x - kk * tpk;
  const int k = k0 + kk;
  const int split = blockIdx.y;
  // K > 64: the slice's i-rows of 4 are split over blockIdx.z (<= 256 threads)
  const int ti = blockIdx.z * ti_per + rr / K4, tj = rr % K4;
  const bool act = ti < K4 && k < Ko;
  const int64_t per = (B + bsplit - 1) / bsplit;
  const int64_t bb = split * per, be = min(B, bb + per);
  float acc[4][4];
  double tot[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      acc[u][v] = 0.f;
      tot[u][v] = 0.0;
    }
  for (int64_t t = bb; t < be; t += WS_BT) {
    const int nb = (int)min((int64_t)WS_BT, be - t);
    __syncthreads();
    for (int e = threadIdx.x; e < WS_BT * KP; e += blockDim.x) {
      const int bl = e / KP, i = e % KP;
      const bool ok = bl < nb && i < K;
      ea_s[e] = ok ? EA[ev_idx(l, t + bl, i, Bc, K)] : 0.f;
      eb_s[e] = ok ? EB[ev_idx(l, t + bl, i, Bc, K)] : 0.f;
    }
    for (int e = threadIdx.x; e < WS_BT * kc; e += blockDim.x) {
      const int bl = e / kc, kq = e - bl * kc;
      rt_s[e] = (bl < nb && k0 + kq < Ko) ? RT[tb_idx(l, t + bl, k0 + kq, Bc, ks)] : 0.f;
    }
    __syncthreads();
    for (int bl = 0; act && bl < nb; ++bl) {
      const float r = rt_s[bl * kc + kk];
      const float4 a4 = *(const float4 *)(ea_s + bl * KP + 4 * ti);
      const float4 e4 = *(const float4 *)(eb_s + bl * KP + 4 * tj);
      const float au[4] = {r * a4.x, r * a4.y, r * a4.z, r * a4.w};
      const float ev[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(au[u], ev[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        tot[u][v] += (double)acc[u][v];
        acc[u][v] = 0.f;
      }
  }
  double *dst = wpart + (((int64_t)split * L + l) * Ko + k) * K * K;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = 4 * ti + u, j = 4 * tj + v;
      if (act && i < K && j < K) dst[i * K + j] = tot[u][v];
    }
}

// W statistics of K_out = 1 rows (the root einsum layer):
//   S[l][i,j] = sum_b RT[b,l] EA[b,l,i] EB[b,l,j]
// a K x K x B product per row, on CUDA cores (the tensor-core kernel pads
// K_out to 16). grid (rows, nsplit), block >= K4*K4: thread (ti, tj) owns rows
// ti + K4*u and columns tj + K4*v (u, v < 4), so a warp reads consecutive
// padded rows (conflict-free 16-byte loads). The 32-sample EA / EB / RT blocks
// (contiguous, ev_idx / tb_idx; zero past the batch) are double-buffered with
// cp.async. Each CTA sums its contiguous run of blocks in fp32 and writes an
// fp64 partial per split; the partials are reduced in split order.
__global__ void __launch_bounds__(256) k_wstats_k1(const float *__restrict__ EA,
                                                   const float *__restrict__ EB,
                                                   const float *__restrict__ RT, int64_t Bc,
                                                   int ks, int64_t B, int K, int L, int nsplit,
                                                   double *wpart) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float smk1[];
  const int K4 = (K + 3) / 4;
  const int evf = K * EV_ROW;                       // floats per EA (or EB) block
  const int stage = 2 * evf + 32;                   // EA | EB | RT
  const int l = blockIdx.x, split = blockIdx.y;
  const int nblk = (int)((B + 31) / 32);
  const int c0 = (int)((int64_t)split * nblk / nsplit), c1 = (int)((int64_t)(split + 1) * nblk / nsplit);
  const int tid = threadIdx.x, ti = tid / K4, tj = tid - ti * K4;
  const bool act = ti < K4;
  auto load = [&](int c, int buf) {
    const int64_t b0 = (int64_t)c * 32;
    const float *ea = EA + ev_idx(l, b0, 0, Bc, K), *eb = EB + ev_idx(l, b0, 0, Bc, K);
    const float *rt = RT + tb_idx(l, b0, 0, Bc, ks);
    float *dst = smk1 + buf * stage;
    for (int e = tid; e < evf / 4; e += blockDim.x) {
      cp_async16(dst + 4 * e, ea + 4 * e);
      cp_async16(dst + evf + 4 * e, eb + 4 * e);
    }
    if (tid < 8) cp_async16(dst + 2 * evf + 4 * tid, rt + 4 * tid);
    cp_async_commit();
  };
  float acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
  if (c0 < c1) load(c0, 0);
  for (int c = c0; c < c1; ++c) {
    const int buf = (c - c0) & 1;
    if (c + 1 < c1) {
      load(c + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float *ea_s = smk1 + buf * stage, *eb_s = ea_s + evf, *rt_s = eb_s + evf;
    if (act) {
#pragma unroll 2
      for (int q = 0; q < 8; ++q) {
        const float4 r = *(const float4 *)(rt_s + 4 * q);
        float4 a[4], e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = ti + K4 * u;
          a[u] = i < K ? *(const float4 *)(ea_s + i * EV_ROW + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
          a[u].x *= r.x;
          a[u].y *= r.y;
          a[u].z *= r.z;
          a[u].w *= r.w;
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = tj + K4 * v;
          e[v] = j < K ? *(const float4 *)(eb_s + j * EV_ROW + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            acc[u][v] = fmaf(a[u].x, e[v].x, acc[u][v]);
            acc[u][v] = fmaf(a[u].y, e[v].y, acc[u][v]);
            acc[u][v] = fmaf(a[u].z, e[v].z, acc[u][v]);
            acc[u][v] = fmaf(a[u].w, e[v].w, acc[u][v]);
          }
      }
    }
    __syncthreads();
  }
  if (!act) return;
  double *dst = wpart + ((int64_t)split * L + l) * K * K;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = ti + K4 * u, j = tj + K4 * v;
      if (i < K && j < K) dst[i * K + j] = (double)acc[u][v];
    }
}

// Child responsibilities, one sample per thread; W staged per k-chunk.
template <int KT>
__global__ void __launch_bounds__(EF_TB) k_einsum_childrho(
    const float *__restrict__ EA, const float *__restrict__ EB, const float *__restrict__ RT,
    const float *__restrict__ W, WsView ws, const int *slot_left, const int *slot_right,
    int64_t B, int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float wsm[];
  const int l = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * EF_TB + threadIdx.x;
  const bool live = b < B;
  const int64_t bb = live ? b : 0;
  float ea[KT], eb[KT], left[KT], right[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    ea[i] = (live && i < K) ? EA[ev_idx(l, bb, i, ws.bc, K)] : 0.f;
    eb[i] = (live && i < K) ? EB[ev_idx(l, bb, i, ws.bc, K)] : 0.f;
    left[i] = 0.f;
    right[i] = 0.f;
  }
  const float *Wl = W + (int64_t)l * Ko * K * K;
  for (int k0 = 0; k0 < Ko; k0 += EF_KC) {
    const int nk = min(EF_KC, Ko - k0);
    __syncthreads();
    stage_w(wsm, Wl, k0, nk, K, KT);
    __syncthreads();
    if (!live) continue;
    for (int kk = 0; kk < nk; ++kk) {
      const float rt = RT[tb_idx(l, bb, k0 + kk, ws.bc, ws.ks)];
      if (rt == 0.f) continue;
      const float *wk = wsm + kk * K * KT;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        if (i >= K) break;
        const float *wr = wk + i * KT;
        left[i] = fmaf(rt, dot_row<KT>(wr, eb), left[i]);
        const float ci = rt * ea[i];
        const float4 *w4 = (const float4 *)wr;
#pragma unroll
        for (int j = 0; j < KT / 4; ++j) {
          const float4 q = w4[j];
          right[4 * j] = fmaf(ci, q.x, right[4 * j]);
          right[4 * j + 1] = fmaf(ci, q.y, right[4 * j + 1]);
          right[4 * j + 2] = fmaf(ci, q.z, right[4 * j + 2]);
          right[4 * j + 3] = fmaf(ci, q.w, right[4 * j + 3]);
        }
      }
    }
  }
  if (!live) return;
  const Col32 dl = slot_ptr(ws, slot_left[l], b), dr = slot_ptr(ws, slot_right[l], b);
#pragma unroll
  for (int i = 0; i < KT; ++i)
    if (i < K) {
      dl[i] = ea[i] * left[i];
      dr[i] = eb[i] * right[i];
    }
}

__global__ void k_einsum_childrho_generic(const float *__restrict__ EA,
                                          const float *__restrict__ EB,
                                          const float *__restrict__ RT,
                                          const float *__restrict__ W, WsView ws,
                                          const int *slot_left, const int *slot_right,
                                          int64_t B, int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  const int l = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  auto ea = [&](int i) { return EA[ev_idx(l, b, i, ws.bc, K)]; };
  auto eb = [&](int i) { return EB[ev_idx(l, b, i, ws.bc, K)]; };
  auto rt = [&](int k) { return RT[tb_idx(l, b, k, ws.bc, ws.ks)]; };
  const float *Wl = W + (int64_t)l * Ko * K * K;
  const Col32 dl = slot_ptr(ws, slot_left[l], b), dr = slot_ptr(ws, slot_right[l], b);
  for (int i = 0; i < K; ++i) {
    float acc = 0.f;
    for (int k = 0; k < Ko; ++k) {
      float t = 0.f;
      for (int j = 0; j < K; ++j) t = fmaf(Wl[((int64_t)k * K + i) * K + j], eb(j), t);
      acc = fmaf(rt(k), t, acc);
    }
    dl[i] = ea(i) * acc;
  }
  for (int j = 0; j < K; ++j) {
    float acc = 0.f;
    for (int k = 0; k < Ko; ++k) {
      float t = 0.f;
      for (int i = 0; i < K; ++i) t = fmaf(Wl[((int64_t)k * K + i) * K + j], ea(i), t);
      acc = fmaf(rt(k), t, acc);
    }
    dr[j] = eb(j) * acc;
  }
}

// Child responsibilities for 48 < K <= 128 on CUDA cores (engine.py:294-316):
//   left[b,i]  = EA[b,i] sum_k RT[b,k] sum_j W[k,i,j] EB[b,j]
//   right[b,j] = EB[b,j] sum_k RT[b,k] sum_i W[k,i,j] EA[b,i]
// per (row, 64-sample tile): W[k] staged in shared memory one output component
// at a time, RT folded into the EB / EA operand, a 4-sample x 8-entry register
// tile per thread for each side. grid (ceil(B/64), rows), block 256.
constexpr int CB_WS = FB_KP + 1;  // odd row stride: the 8-row column reads hit 8 banks
size_t childrho_big_smem() {
  return sizeof(float) * ((size_t)FB_KP * CB_WS + 3 * FB_KP * FB_TB);
}
__global__ void __launch_bounds__(256) k_einsum_childrho_big(
    const float *__restrict__ EA, const float *__restrict__ EB, const float *__restrict__ RT,
    const float *__restrict__ W, WsView ws, const int *slot_left, const int *slot_right,
    int64_t B, int K, int Ko) {
  EINET_KERNEL_PROLOGUE();
  extern __shared__ __align__(16) float csm[];
  float *wk = csm;                      // [i][CB_WS] = W[k][i][j]
  float *ebs = wk + FB_KP * CB_WS;      // [j][64]
  float *eas = ebs + FB_KP * FB_TB;     // [i][64]
  float *rts = eas + FB_KP * FB_TB;     // [k][64]
  const int tid = threadIdx.x, l = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * FB_TB;
  for (int e = tid; e < FB_KP * FB_TB; e += 256) {
    const int r = e >> 6, s = e & 63;
    const int64_t b = b0 + s;
    float vb = 0.f, va = 0.f, vr = 0.f;
    if (b < ws.bc) {
      if (r < K) {
        const int64_t x = ev_idx(l, b, r, ws.bc, K);
        vb = EB[x];
        va = EA[x];
      }
      if (r < Ko) vr = RT[tb_idx(l, b, r, ws.bc, ws.ks)];
    }
    ebs[e] = vb;
    eas[e] = va;
    rts[e] = vr;
  }
  const int sg = tid & 15, ig = tid >> 4;  // samples 4 sg .. +3, entries 8 ig .. +7
  float al[4][8], ar[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) al[a][c] = ar[a][c] = 0.f;
  const float *Wl = W + (int64_t)l * Ko * K * K;
  for (int k = 0; k < Ko; ++k) {
    __syncthreads();
    const float *src = Wl + (int64_t)k * K * K;
    for (int e = tid; e < FB_KP * FB_KP; e += 256) {
      const int i = e / FB_KP, j = e - i * FB_KP;
      wk[i * CB_WS + j] = (i < K && j < K) ? src[i * K + j] : 0.f;
    }
    __syncthreads();
    const float4 r4 = *(const float4 *)(rts + k * FB_TB + sg * 4);
    const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
    for (int j = 0; j < K; ++j) {  // left side: entries i = 8 ig + c
      const float4 e4 = *(const float4 *)(ebs + j * FB_TB + sg * 4);
      const float eb[4] = {rv[0] * e4.x, rv[1] * e4.y, rv[2] * e4.z, rv[3] * e4.w};
      float wv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) wv[c] = wk[(ig * 8 + c) * CB_WS + j];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) al[a][c] = fmaf(wv[c], eb[a], al[a][c]);
    }
    for (int i = 0; i < K; ++i) {  // right side: entries j = 8 ig + c
      const float4 a4 = *(const float4 *)(eas + i * FB_TB + sg * 4);
      const float ea[4] = {rv[0] * a4.x, rv[1] * a4.y, rv[2] * a4.z, rv[3] * a4.w};
      float wv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) wv[c] = wk[i * CB_WS + ig * 8 + c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) ar[a][c] = fmaf(wv[c], ea[a], ar[a][c]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int s = sg * 4 + a;
    const int64_t b = b0 + s;
    if (b >= B) continue;
    const Col32 dl = slot_ptr(ws, slot_left[l], b), dr = slot_ptr(ws, slot_right[l], b);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int x = ig * 8 + c;
      if (x >= K) continue;
      dl[x] = eas[x * FB_TB + s] * al[a][c];
      dr[x] = ebs[x * FB_TB + s] * ar[a][c];
    }
  }
}

// ---------------------------------------------------------------------------
// root outputs and the log-likelihood sum
// ---------------------------------------------------------------------------

__global__ void k_root_out(WsView ws, int slab, int64_t B, int kr, double *out,
                           unsigned *ll_ticket) {
  EINET_KERNEL_PROLOGUE();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e == 0) *ll_ticket = 0u;  // k_ll_sum's completion counter
  if (e >= B * kr) return;
  const int64_t b = e / kr;
  const int k = (int)(e % kr);
  const double s = slab_shift(ws, slab)[b];
  out[e] = s == -CUDART_INF ? -CUDART_INF : s + (double)slab_off(ws, slab, b)[k];
}

// Sum of the batch's root log-likelihoods into stats (ll, count): one CTA per
// 256 samples writes a fixed-order partial (strided warp runs, shuffle tree,
// warp order); the last CTA to finish (ticket counter, zeroed by k_root_out in
// the forward pass and reset here) adds the partials in a fixed order (lane
// runs, shuffle tree), so the sum is deterministic whichever CTA finishes last.
__global__ void __launch_bounds__(256) k_ll_sum(WsView ws, int slab, int64_t B, double *ll,
                                                double count, double *part, unsigned *ticket) {
  EINET_KERNEL_PROLOGUE();
  __shared__ double red[8];
  __shared__ bool last;
  const double *sh = slab_shift(ws, slab);
  const int64_t b = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double v = 0.0;
  if (b < B) {
    const double s = sh[b];
    v = s == -CUDART_INF ? -CUDART_INF : s + (double)slab_off(ws, slab, b)[0];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    // fixed order: lane runs over q = lane + 32 i, then the shuffle tree
    __threadfence();
    double t = 0.0;
    for (unsigned q = threadIdx.x; q < gridDim.x; q += 32) t += __ldcg(part + q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      ll[0] += t;
      ll[1] += count;
      *ticket = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------

template <int KT>
static void fwd_simt(const LayerPlan &L, const float *w32, const float *EA, const float *EB,
                     WsView &w, int64_t B, int K, cudaStream_t st) {
  const size_t smem = sizeof(float) * EF_KC * K * KT;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_einsum_fwd<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  dim3 grid(ceil_div(B, EF_TB), L.rows, ceil_div(L.k_out, EF_KC));
  launch_k(k_einsum_fwd<KT>, grid, EF_TB, smem, st, w, EA, EB, L.d_out_slab, w32 + L.w_off, B, K,
                                              L.k_out);
}

template <int KT>
static void childrho_simt(const LayerPlan &L, const float *w32, const float *EA,
                          const float *EB, WsView &w, int64_t B, int K, cudaStream_t st) {
  const size_t smem = sizeof(float) * EF_KC * K * KT;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_einsum_childrho<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  dim3 grid(ceil_div(B, EF_TB), L.rows);
  launch_k(k_einsum_childrho<KT>, grid, EF_TB, smem, st, EA, EB, w.rt, w32 + L.w_off, w,
                                                   L.d_slot_left, L.d_slot_right, B, K,
                                                   L.k_out);
}

static void einsum_forward_simt(const LayerPlan &L, const float *w32, const float *EA,
                                const float *EB, WsView &w, int64_t B, int K,
                                cudaStream_t st) {
  if (K <= 4) fwd_simt<4>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 8) fwd_simt<8>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 12) fwd_simt<12>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 16) fwd_simt<16>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 24) fwd_simt<24>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 32) fwd_simt<32>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 40) fwd_simt<40>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 48) fwd_simt<48>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 64) fwd_simt<64>(L, w32, EA, EB, w, B, K, st);
  else if (K <= FB_KP) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_einsum_fwd_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fwd_big_smem());
      attr = true;
    }
    dim3 grid(ceil_div(B, FB_TB), L.rows, L.k_out);
    launch_k(k_einsum_fwd_big, grid, 256, fwd_big_smem(), st, w, EA, EB, L.d_out_slab, w32 + L.w_off,
                                                       B, K, L.k_out);
  } else {
    dim3 grid(ceil_div(B, 128), L.rows);
    launch_k(k_einsum_fwd_generic, grid, 128, 0, st, w, EA, EB, L.d_out_slab, w32 + L.w_off, B, K,
                                               L.k_out);
  }
}

static void einsum_childrho_simt(const LayerPlan &L, const float *w32, const float *EA,
                                 const float *EB, WsView &w, int64_t B, int K,
                                 cudaStream_t st) {
  if (K <= 4) childrho_simt<4>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 8) childrho_simt<8>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 12) childrho_simt<12>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 16) childrho_simt<16>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 24) childrho_simt<24>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 32) childrho_simt<32>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 40) childrho_simt<40>(L, w32, EA, EB, w, B, K, st);
  else if (K <= 48) childrho_simt<48>(L, w32, EA, EB, w, B, K, st);
  else if (K <= FB_KP) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_einsum_childrho_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)childrho_big_smem());
      attr = true;
    }
    dim3 grid(ceil_div(B, FB_TB), L.rows);
    launch_k(k_einsum_childrho_big, grid, 256, childrho_big_smem(), st, 
        EA, EB, w.rt, w32 + L.w_off, w, L.d_slot_left, L.d_slot_right, B, K, L.k_out);
  } else {
    dim3 grid(ceil_div(B, 128), L.rows);
    launch_k(k_einsum_childrho_generic, grid, 128, 0, st, EA, EB, w.rt, w32 + L.w_off, w,
                                                    L.d_slot_left, L.d_slot_right, B, K,
                                                    L.k_out);
  }
}

static inline const float *layer_ea(const Plan &p, const WsView &w, const LayerPlan &L) {
  return w.ea + (int64_t)L.erow_base * (w.bc / 32) * p.k * EV_ROW;
}
static inline const float *layer_eb(const Plan &p, const WsView &w, const LayerPlan &L) {
  return w.eb + (int64_t)L.erow_base * (w.bc / 32) * p.k * EV_ROW;
}

int launch_forward(Plan &p, const uint8_t *compute, const float *x, int64_t B, uint8_t *wsb,
                   double *root_out, int32_t *status, cudaStream_t st) {
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  int rc = launch_leaf_forward(p, compute, x, B, wsb, status, st);
  if (rc) return rc;
  for (const LayerPlan &L : p.layers) {
    if (L.kind == EINET_LAYER_EINSUM) {
      float *EA = (float *)layer_ea(p, w, L), *EB = (float *)layer_eb(p, w, L);
      {
        ProfScope prof(prof_layer_name("einsum_prep", L.index), st);
        dim3 grid(ceil_div(B, 32), L.rows);
        const bool tcl = p.use_tc && L.tc;
        float *EBM = tcl ? w.ebm + (int64_t)L.erow_base * w.bc * p.kp : nullptr;
        float *EAM = tcl && L.direct ? w.eam + (int64_t)L.erow_base * w.bc * p.kp : nullptr;
        launch_k(k_einsum_prep_fwd, grid, 128, 0, st, w, L.d_left_slab, L.d_right_slab, L.d_out_slab,
                                                B, p.k, EA, EB, EBM, EAM, p.kp, L.index, status);
      }
      ProfScope prof(prof_layer_name("einsum_fwd", L.index), st);
      if (p.use_tc && L.tc)
        rc = launch_contract_tc(p, L, 0, compute, EA, EB, w, B, st);
      else
        einsum_forward_simt(L, c.w32, EA, EB, w, B, p.k, st);
      if (rc) return rc;
      count_launch(2);
    } else {
      ProfScope prof("mixing_fwd", st);
      // small batches: the k-range is split over blockIdx.z to fill the SMs
      const int64_t ctas = (int64_t)ceil_div(B, 32) * L.rows;
      const int kz = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.k_out, 4),
                                                                 ceil_div(2 * p.num_sms, ctas)));
      dim3 grid(ceil_div(B, 32), L.rows, kz);
      launch_k(k_mixing_fwd, grid, 128, 8 * L.dmax, st, w, L.d_mix_src_slab, L.d_mix_mask, L.d_out_slab,
                                         c.mix32 + L.mix_off, B, L.k_out, L.dmax, L.index,
                                         status);
      count_launch();
    }
  }
  const int64_t n = B * p.k_root;
  launch_k(k_root_out, ceil_div(n, 256), 256, 0, st, w, p.root_out_slab, B, p.k_root, root_out,
           (unsigned *)(wsb + p.w_llpart) + 2 * ceil_div(w.bc, 256));
  count_launch();
  return check_cuda(cudaGetLastError(), "forward kernels");
}

static int wstats_bsplit(const Plan &p, const LayerPlan &L, int64_t B, int64_t blocks = -1) {
  if (blocks < 0) blocks = (int64_t)L.rows * L.k_out;
  int64_t bs = std::max<int64_t>(1, (2 * p.num_sms + blocks - 1) / blocks);
  return (int)std::min<int64_t>(bs, std::min<int64_t>(kMaxBSplit, (B + 63) / 64));
}

int launch_backward(Plan &p, const double *params, const uint8_t *compute, const float *x,
                    int64_t B, uint8_t *wsb, double *stats, int32_t *status,
                    cudaStream_t st) {
  (void)status;
  CompView c = comp_view(p, compute);
  WsView w = ws_view(p, wsb);
  const int K = p.k;
  int eo = 0, rc = 0;
  bool red_pending[3] = {false, false, false};
  // log-likelihood sum of the batch (root entry 0) and the sample count: off
  // the critical path on the reduction stream (it only reads the root slab and
  // writes the stats' LL entries), joined with the other reductions at the end
  const bool ll_side = p.red_stream && !profiling_enabled();
  {
    ProfScope prof("ll_sum", st);
    cudaStream_t ls = ll_side ? p.red_stream : st;
    if (ll_side) {
      if ((rc = check_cuda(cudaEventRecord(p.red_fork[4], st), "ll fork")) ||
          (rc = check_cuda(cudaStreamWaitEvent(ls, p.red_fork[4], 0), "ll fork")))
        return rc;
    }
    double *part = (double *)(wsb + p.w_llpart);
    launch_k(k_ll_sum, ceil_div(B, 256), 256, 0, ls, w, p.root_out_slab, B,
             stats + p.sizes.stats_ll_offset, (double)B, part,
             (unsigned *)part + 2 * ceil_div(w.bc, 256));
    count_launch();
    if (ll_side && (rc = check_cuda(cudaEventRecord(p.red_done[4], ls), "ll done"))) return rc;
  }
  for (int li = (int)p.layers.size() - 1; li >= 0; --li) {
    const LayerPlan &L = p.layers[li];
    if (L.kind == EINET_LAYER_MIXING) {
      ProfScope prof("mixing_bwd", st);
      const int nb = ceil_div(B, 32);
      dim3 grid(nb, L.rows);
      launch_k(k_mixing_bwd, grid, 128, 0, st, w, L.d_mix_src_slab, L.d_mix_mask, L.d_out_slab,
                                        L.d_mix_slot, c.mix32 + L.mix_off, p.d_csr_off,
                                        p.d_csr_slot, p.d_slab_ones, B, L.k_out, L.dmax,
                                        w.mixpart, L.mix_off, p.n_mix);
      // the mixing-weight batch reduction on the reduction stream (its
      // partials are per layer: no reuse to guard), joined at the end
      // (the profiler's per-class pass keeps them in line: clean class times)
    cudaStream_t rs = p.red_stream && !profiling_enabled() ? p.red_stream : st;
      if (rs != st) {
        if ((rc = check_cuda(cudaEventRecord(p.red_fork[2], st), "mixing fork")) ||
            (rc = check_cuda(cudaStreamWaitEvent(rs, p.red_fork[2], 0), "mixing fork")))
          return rc;
      }
      launch_reduce_partials(stats + p.n_w + L.mix_off, w.mixpart + L.mix_off, nb,
                             (int64_t)L.rows * L.dmax, p.n_mix, nullptr, rs);
      if (rs != st) {
        if ((rc = check_cuda(cudaEventRecord(p.red_done[2], rs), "mixing done"))) return rc;
        red_pending[2] = true;
      }
      count_launch();
      continue;
    }
    const float *EA = layer_ea(p, w, L), *EB = layer_eb(p, w, L);
    {
      ProfScope prof(prof_layer_name("einsum_bwd_rt", L.index), st);
      dim3 g1(ceil_div(B, 32), L.rows);
      const bool tcl = p.use_tc && L.tc;
      launch_k(k_einsum_bwd_rt, g1, 128, 0, st, w, L.d_out_slab, p.d_csr_off, p.d_csr_slot,
                                          p.d_slab_ones, B, L.k_out, w.rt,
                                          tcl && !L.direct ? w.rtm : nullptr, L.kob,
                                          tcl ? w.rtb : nullptr, L.nn);
    }
    const int64_t lw = (int64_t)L.rows * L.k_out * K * K;
    // W-statistics partials alternate between the two halves of w_wpart by
    // einsum-layer parity; each layer's batch reduction runs on the
    // reduction stream (rs) beside the next layers' kernels, and the layer two
    // steps later waits for it before reusing the half
    const int par = eo++ & 1;
    double *wpart = w.wpart + par * p.wpart_half;
    // (the profiler's per-class pass keeps them in line: clean class times)
    cudaStream_t rs = p.red_stream && !profiling_enabled() ? p.red_stream : st;
    if (red_pending[par] && (rc = check_cuda(cudaStreamWaitEvent(st, p.red_done[par], 0), "wstats join")))
      return rc;
    auto red_fork = [&](cudaStream_t r) -> int {
      if (r == st) return 0;
      int e = check_cuda(cudaEventRecord(p.red_fork[par], st), "wstats fork");
      if (!e) e = check_cuda(cudaStreamWaitEvent(r, p.red_fork[par], 0), "wstats fork");
      return e;
    };
    {
      ProfScope prof(prof_layer_name("einsum_wstats", L.index), st);
      const int K4 = (K + 3) / 4;
      if (L.k_out == 1 && K4 * K4 <= 256 && !getenv("EINET_WK1_OFF")) {
        const int ns = wstats_bsplit(p, L, B, L.rows);
        const size_t smem = sizeof(float) * 2 * (2 * K * EV_ROW + 32);
        const int threads = std::max(128, (K4 * K4 + 31) / 32 * 32);
        launch_k(k_wstats_k1, dim3(L.rows, ns), threads, smem, st, EA, EB, w.rt, w.bc, w.ks, B, K,
                                                             L.rows, ns, wpart);
        if ((rc = red_fork(rs))) return rc;
        launch_reduce_partials(stats + L.w_off, wpart, ns, lw, lw, params + L.w_off, rs);
      } else if (p.use_tc && L.tc) {
        WsView wv = w;
        wv.wpart = wpart;
        if ((rc = launch_wstats_tc(p, L, EA, EB, wv, B, params + L.w_off, stats + L.w_off, st,
                                   rs != st ? rs : nullptr, p.red_fork[par])))
          return rc;
      } else {
        const int K4 = (K + 3) / 4;
        int ti_per = K4;
        while (ti_per * K4 > 256) ti_per = (ti_per + 1) / 2;
        // small K: several output components per CTA (shared EA / EB staging)
        const int kc = wstats_simt_kc(K, L.k_out);
        const int nkc = ceil_div(L.k_out, kc);
        const int bs = wstats_bsplit(p, L, B, (int64_t)L.rows * nkc);
        const size_t smem = sizeof(float) * (2 * WS_BT * K4 * 4 + WS_BT * kc);
        dim3 g2(L.rows * nkc, bs, ceil_div(K4, ti_per));
        launch_k(k_einsum_wstats, g2, kc * ti_per * K4, smem, st, EA, EB, w.rt, w.bc, w.ks, B, K,
                                                            L.k_out, L.rows, bs, wpart, ti_per,
                                                            kc);
        if ((rc = red_fork(rs))) return rc;
        launch_reduce_partials(stats + L.w_off, wpart, bs, lw, lw, params + L.w_off, rs);
      }
    }
    if (rs != st) {
      if ((rc = check_cuda(cudaEventRecord(p.red_done[par], rs), "wstats done"))) return rc;
      red_pending[par] = true;
    }
    {
      ProfScope prof(prof_layer_name("einsum_childrho", L.index), st);
      if (p.use_tc && L.tc) {
        int rc = launch_contract_tc(p, L, 3, compute, EA, EB, w, B, st);
        if (rc) return rc;
      } else {
        einsum_childrho_simt(L, c.w32, EA, EB, w, B, K, st);
      }
    }
    count_launch(3);
  }
  rc = launch_leaf_backward(p, compute, x, B, wsb, stats, st);
  if (rc) return rc;
  if (ll_side && (rc = check_cuda(cudaStreamWaitEvent(st, p.red_done[4], 0), "ll join")))
    return rc;
  for (int q = 0; q < 3; ++q)  // join the reduction stream
    if (red_pending[q] && (rc = check_cuda(cudaStreamWaitEvent(st, p.red_done[q], 0), "wstats join")))
      return rc;
  return check_cuda(cudaGetLastError(), "backward kernels");
}

}  // namespace einet
