// Internal declarations of the B200 Einsum-Network engine.
//
// Data layout in HBM (per chunk of Bc samples):
//   slab  s : one log-density vector per sample, value[b,k] = shift[s][b] (fp64)
//             + off[s][b][k] (fp32). Slabs 0..R-1 are the reference buffer rows
//             (compiler.py:54-99); root einsum rows and the root mixing output
//             get extra slabs so every layer writes a slab.
//   slot  q : one child-responsibility contribution [b][k] (fp32); the
//             responsibility of slab s is the ordered sum over csr(s) -- a
//             deterministic replacement for np.add.at (engine.py:315-316).
#pragma once

#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/einet_b200.h"

namespace einet {

constexpr int kMaxDSplit = 16;     // leaf forward split of a scope across CTAs
constexpr int kMaxBSplit = 64;     // batch split of statistic reductions
constexpr int kReduceThreads = 256;
// per-einsum-layer tile descriptor for the fused M-step (int64 words)
enum TileDescWord {
  TD_SLICE0, TD_ROWS, TD_KO, TD_TC, TD_DIRECT, TD_KG, TD_NG, TD_FW_ROWS, TD_IG, TD_NI,
  TD_UW_ROWS, TD_KOB, TD_RW_ROWS, TD_FW_OFF, TD_FW_TILE, TD_UW_OFF, TD_UW_TILE, TD_VW_OFF,
  TD_RW_TILE, TD_WOFF, TD_IT0, TD_NFW, TD_NUW, TD_NRW, TD_WORDS
};
constexpr int EV_ROW = 36;         // padded row of the EA / EB 32-sample blocks (kern_common.cuh)

struct LayerPlan {
  int kind = 0;        // EINET_LAYER_*
  int index = 0;       // position in circuit.layers (leaf = 0)
  int rows = 0;        // L or M
  int k_out = 0;
  int is_root = 0;
  int dmax = 0;
  // einsum
  int *d_left_slab = nullptr, *d_right_slab = nullptr, *d_out_slab = nullptr;
  int *d_slot_left = nullptr, *d_slot_right = nullptr;  // slot ids per row
  int64_t w_off = 0;   // element offset of this layer's W (L,Ko,K,K)
  // mixing
  int *d_mix_src_slab = nullptr;   // (M*dmax), -1 if masked
  int *d_mix_slot = nullptr;       // (M*dmax), -1 if masked
  uint8_t *d_mix_mask = nullptr;
  int64_t mix_off = 0; // element offset of (M,Dmax) weights in the mixing block
  int erow_base = 0;   // first global einsum row (per-layer EA/EB storage)
  // tensor-core tiling (einsum layers with tc != 0), DESIGN.md "EinsumLayer"
  int tc = 0;
  int kg = 0, ng = 0, fw_rows = 0;  // forward: k per N tile, #tiles, tile rows (N_max)
  int ig = 0, ni = 0, uw_rows = 0;  // child-rho: i per N tile, #tiles, tile rows
  int kob = 0;                      // K_out padded to 16 (child-rho bf16 MMA K dimension)
  int nn = 0;                       // W-stats MMA N: K_out padded to 16
  int64_t fw_off = 0, fw_tile = 0;  // compute byte offset, bytes per forward tile
  int64_t uw_off = 0, uw_tile = 0;  // compute byte offset, bytes per child-rho tile (left)
  int64_t vw_off = 0;               // right child-rho tiles (rows (jl, i)), uw_tile bytes each
  // K_out == 1 (root): child responsibilities as one direct GEMM per side,
  // left = EA * rt * (EB W0^T) (forward tile), right = EB * rt * (EA W0) (rw tile at vw_off)
  int direct = 0, rw_rows = 0;
  int64_t rw_tile = 0;
  std::vector<int> h_out_slab;
  std::vector<int> h_src;          // mixing local src
  std::vector<uint8_t> h_mask;
};

struct Plan {
  // descriptor copy
  int d_vars = 0, k = 0, k_root = 0, ks = 0, num_replicas = 0, nbr = 0;
  int family = 0, num_states = 0, n_trials = 0, suff = 0;
  double var_min = 0, var_max = 0, p_min = 0;
  int n_leaf = 0;
  int max_scope = 0;
  std::vector<int> h_scope_off, h_scope_vars, h_leaf_rep, h_leaf_slab;
  int *d_scope_off = nullptr, *d_scope_vars = nullptr, *d_leaf_rep = nullptr,
      *d_leaf_slab = nullptr;
  int *d_leaf_of = nullptr;        // (R, D): leaf index covering (d, r) or -1
  // leaf-statistics segments (leaf_tc.cu): 128 scope positions each
  int n_lseg = 0;
  int *d_lseg_leaf = nullptr, *d_lseg_v0 = nullptr, *d_phi_seg = nullptr;
  uint8_t *d_lseg_vec = nullptr;
  std::vector<LayerPlan> layers;   // einsum / mixing layers in circuit order
  int root_mix_row = -1;
  // slabs & slots
  int num_slabs = 0, num_slots = 0;
  int root_out_slab = -1;          // slab holding the root vector
  std::vector<int> h_csr_off, h_csr_slot;   // per slab
  int *d_csr_off = nullptr, *d_csr_slot = nullptr;
  std::vector<uint8_t> h_slab_ones;         // slab whose responsibility is 1 (root)
  uint8_t *d_slab_ones = nullptr;
  // parameter / stats / compute layout
  int64_t n_w = 0, n_mix = 0, n_phi = 0;
  int64_t max_layer_w = 0, max_rows = 0, n_mix_entries = 0;
  einet_sizes sizes{};
  // compute segments (byte offsets)
  int64_t c_w32 = 0, c_mix32 = 0, c_leafp = 0, c_center = 0, c_const = 0, c_active = 0,
          c_logh = 0, c_leafimg = 0, c_cm2 = 0;
  // FP64 tensor-core (DMMA) Gaussian leaf forward: scopes padded to 32 variables
  int leaf_dmma = 0;               // eligible (Gaussian, K % 8 == 0, K <= 64)
  std::vector<int> h_leaf_pvo;     // padded variable offset per leaf (n_leaf + 1)
  int *d_leaf_pvo = nullptr;
  int *d_scope_pos = nullptr;      // (R, D): position of d in its leaf's scope, or -1
  // INT8 tensor-core Gaussian leaf forward (leaf_i8.cu): scopes padded to 32
  // like the DMMA image, K padded to 8 (<= 40), 6 digits per column
  int leaf_i8 = 0, i8_k8 = 0, i8_ng = 0;
  int64_t c_i8img = 0, c_i8c = 0;  // compute: digit tiles, per-(leaf, k) scale and C
  int64_t c_i8mask = 0;            // compute: active-variable mask per padded chunk
  int *d_i8_tab = nullptr;         // per padded chunk: leaf, variables, flags, 0
  int *d_i8_col = nullptr;         // per padded chunk: 32 variable indices
  int *d_i8_grp = nullptr;         // first chunk of each leaf pair (pairs + 1)
  std::vector<int> h_i8_grp;
  int64_t w_i8flag = 0;            // workspace: off-grid flag of the last i8 forward
  cudaStream_t side_stream = nullptr;  // captures the fallback body of a conditional node
  cudaStream_t fork_stream = nullptr;  // M-step: leaf branch beside the einsum weights
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // back-pass: the W-statistics batch reductions run on red_stream beside
  // the next layer's kernels (double-buffered partials, w_wpart halves)
  cudaStream_t red_stream = nullptr;
  // (index 3: the leaf P reductions beside the leaf statistics GEMM; 4: the
  // log-likelihood sum beside the back-pass)
  cudaEvent_t red_fork[5] = {}, red_done[5] = {};
  int64_t wpart_half = 0;          // doubles per partial buffer half
  // fused M-step (mstep.cu): per-einsum-layer tile geometry, temp leaf terms
  int64_t *d_tiledesc = nullptr;   // einsum layers x TD_WORDS (mstep.cu)
  int n_tiledesc = 0;
  int64_t n_tile_items = 0;        // k_build_tiles_all work items (16-byte pieces)
  int64_t c_mtmp = 0;              // compute segment: 2 x R*D*K doubles
  // workspace segments (byte offsets)
  int64_t w_off = 0, w_shift = 0, w_slots = 0, w_leafpart = 0, w_ea = 0, w_eb = 0,
          w_rt = 0, w_wpart = 0, w_rho = 0, w_lspart = 0, w_ppart = 0, w_mixpart = 0,
          w_llpart = 0, w_tmp_s = 0, w_tmp_p = 0, w_ebm = 0, w_eam = 0, w_rtm = 0, w_rtb = 0, w_rhob = 0, w_scratch_end = 0;
  int64_t max_chunk = 0;
  int64_t bc = 0;                  // per-chunk sample stride (max_chunk rounded to 32)
  int num_sms = 148;
  int max_lsplit = 1;              // leaf-statistics batch split allocated
  int n_erows = 0;                 // einsum rows over all layers
  int use_tc = 1;                  // tcgen05 EinsumLayer path enabled
  int kp = 0;                      // K padded to 16 (forward bf16 MMA K dimension)
  // mixing rows flattened over layers for the M-step
  int n_mixrows = 0;
  int *d_mixrow_off = nullptr, *d_mixrow_len = nullptr;
  uint8_t *d_mix_mask_all = nullptr;
};

// ---- launches: programmatic dependent launch (PDL) ---------------------------
// Every kernel is launched with programmatic stream serialization and starts
// with EINET_KERNEL_PROLOGUE(): griddepcontrol.wait (the predecessor grid has
// completed and its writes are visible) before anything else, so the launch
// of the next kernel of the stream (or CUDA graph) overlaps this one's drain.
// The dependents are released at grid completion (an early
// griddepcontrol.launch_dependents let waiting CTAs take SM slots and cost
// 2-4% at 16384 samples). Every CTA executes the wait, so dependencies stay
// transitive. EINET_PDL=0 launches without the attribute (A/B timing:
// -2.6% step time at 500 samples, neutral at 16384).
#define EINET_KERNEL_PROLOGUE()                                   \
  do {                                                            \
    asm volatile("griddepcontrol.wait;" ::: "memory");            \
  } while (0)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args &&...args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- error handling ---------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int check_cuda(cudaError_t err, const char *what);
void count_launch(int n = 1);

// Optional per-kernel-class CUDA-event timing (einet_profile_*). When enabled,
// a ProfScope records an event pair on the launching stream around a group of
// launches; einet_profile_query sums the elapsed times per class.
bool profiling_enabled();
void profile_record(const char *name, cudaEvent_t start, cudaEvent_t stop);
// Per-layer class names ("einsum_fwd@3") when EINET_PROFILE_LAYERS is set
// (the C5 sweep times one EinsumLayer of a larger graph); else `base`.
const char *prof_layer_name(const char *base, int layer);
struct ProfScope {
  const char *name;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(const char *n, cudaStream_t s) : name(n), st(s) {
    if (profiling_enabled()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEventRecord(b, st);
      profile_record(name, a, b);
    }
  }
};

// ---- launchers (implemented in the .cu files) -------------------------------
struct CompView;
struct WsView;
int launch_prepare(Plan &p, const double *params, uint8_t *compute, const uint8_t *mask,
                   const double *leaf_offset, cudaStream_t st);
int launch_prepare_leaves(Plan &p, const double *params, uint8_t *compute, cudaStream_t st);
int launch_forward(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                   uint8_t *ws, double *root_out, int32_t *status, cudaStream_t st);
int launch_backward(Plan &p, const double *params, const uint8_t *compute, const float *x,
                    int64_t B, uint8_t *ws, double *stats, int32_t *status,
                    cudaStream_t st);
int launch_mstep(Plan &p, double *params, uint8_t *compute, const double *stats,
                 double lam, double eps_w, const int32_t *status, cudaStream_t st);
int upload_tiledesc(Plan &p);
int launch_expand_acc_p(Plan &p, const double *stats, double *acc_p, cudaStream_t st);
int launch_export_buffer(Plan &p, const uint8_t *ws, int64_t B, double *out,
                         cudaStream_t st);
int launch_export_leaf_rows(Plan &p, const uint8_t *ws, int64_t B, double *out,
                            cudaStream_t st);
int launch_ef_log_prob(Plan &p, const double *params, const float *x, int64_t B,
                       const uint8_t *mask, double *out, int32_t *status,
                       cudaStream_t st);
int launch_status_reset(int32_t *status, cudaStream_t st);
int launch_log_step(const double *ll2, const int32_t *status, double *log_ll, int32_t *log_st,
                    int64_t *cursor, int64_t cap, cudaStream_t st);
int launch_status_to_stats(const int32_t *status, double *flag, cudaStream_t st);
int launch_status_from_stats(const double *flag, int32_t *status, cudaStream_t st);
void plan_tc_tiling(Plan &p);
int64_t wstats_tc_slots(const Plan &p, const LayerPlan &L, int64_t B);
int launch_wstats_tc(Plan &p, const LayerPlan &L, const float *EA, const float *EB, WsView &w,
                     int64_t B, const double *Wl, double *stats, cudaStream_t st,
                     cudaStream_t rst = nullptr, cudaEvent_t fork = nullptr);
int launch_prepare_tc_tiles(Plan &p, uint8_t *compute, cudaStream_t st);
int launch_build_tiles_all(Plan &p, uint8_t *compute, cudaStream_t st);
int launch_prepare_leaf_dmma(Plan &p, uint8_t *compute, cudaStream_t st);
int launch_prepare_leaf_i8(Plan &p, uint8_t *compute, cudaStream_t st);
int launch_i8_img(Plan &p, uint8_t *compute, cudaStream_t st);
void plan_leaf_i8(Plan &p, std::vector<int> &tab, std::vector<int> &col, std::vector<int> &grp);
bool leaf_i8_supported(const Plan &p);
int launch_leaf_finalize_parts(Plan &p, const uint8_t *compute, const double *part, int nsplit,
                               int64_t B, uint8_t *wsb, cudaStream_t st);
int launch_leaf_fwd_i8(Plan &p, const uint8_t *compute, const float *x, int64_t B, uint8_t *wsb,
                       int *flag, cudaGraphConditionalHandle cond, cudaStream_t st);
struct CompView;
struct WsView;
int launch_leaf_fwd_dmma(Plan &p, const CompView &c, const float *x, int64_t B, const WsView &w,
                         int32_t *status, cudaStream_t st, int *ds_out, const int *gate);
int launch_contract_tc(Plan &p, const LayerPlan &L, int mode, const uint8_t *compute,
                       const float *EA, const float *EB, const WsView &w, int64_t B,
                       cudaStream_t st);
int64_t sample_scratch_bytes(const Plan &p, int64_t n);
int launch_decode_u8(const uint8_t *src, int64_t count, double divisor, float *dst,
                     cudaStream_t st);
int host_pack_f64(const double *x, int64_t n, uint8_t *u8, float *f32, int threads);
int launch_crc32(const uint8_t *data, int64_t len, uint32_t *crc, cudaStream_t st);
int launch_blob_to_params(const uint8_t *blob, int64_t blob_len, const int64_t *table,
                          int n_tensors, int64_t max_count, double *params, int32_t *bad,
                          cudaStream_t st);
int launch_params_to_blob(const double *params, const int64_t *table, int n_tensors,
                          int64_t max_count, uint8_t *blob, cudaStream_t st);
int launch_sample(Plan &p, const double *params, const uint8_t *wsb, int conditional,
                  const double *x_e, const uint8_t *evidence, int64_t n, uint64_t seed,
                  uint8_t *scratch, double *out, int32_t *status, cudaStream_t st);
int launch_selftest_gemm(const float *A, const float *B, float *D, int N, int K,
                         cudaStream_t st);
int leaf_lsplit(const Plan &p, int64_t B);
int launch_log_einsum_exp(const double *left, const double *right, const double *w,
                          int64_t B, int L, int K, int Ko, double *out, cudaStream_t st);

// deterministic reduction: dst[i] += (scale ? scale[i] : 1) * sum_p part[p*stride+i]
void launch_reduce_partials(double *dst, const double *part, int nparts, int64_t n,
                            int64_t stride, const double *scale, cudaStream_t st);
// same, overwriting: dst[i] = sum_p part[p*stride+i]
void launch_reduce_partials_store(double *dst, const double *part, int nparts, int64_t n,
                                  int64_t stride, cudaStream_t st);
bool leaf_tc_supported(const Plan &p);
int64_t leaf_stats_slots(const Plan &p, int64_t B);
int launch_leaf_stats_tc(Plan &p, const uint8_t *compute, const float *x, int64_t B,
                         uint8_t *wsb, double *stats, const double *Pcall, cudaStream_t st,
                         cudaEvent_t p_ready = nullptr);

// Split factor s in [lo, hi] for a grid of ctas_per_split * s CTAs on
// `slots` concurrently resident CTAs: the smallest s whose last wave is at
// least `good` full once there are >= 2 waves (else the best-filled one).
int pick_split(int64_t ctas_per_split, int64_t slots, int lo, int hi, double good = 0.85);
// resident CTAs of `kernel` on the whole device for the given block / smem
int64_t device_slots(const void *kernel, int block, size_t smem, int num_sms);

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
// CUDA-core W statistics: output components per CTA (einsum.cu k_einsum_wstats)
inline int wstats_simt_kc(int K, int Ko) {
  const int K4 = (K + 3) / 4;
  return K4 * K4 <= 256 ? std::max(1, std::min(Ko, 256 / (K4 * K4))) : 1;
}
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace einet
