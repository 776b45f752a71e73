// C-ABI entry points and execution-plan construction (include/einet_b200.h).
//
// einet_plan_create turns a compiled LayeredCircuit (compiler.py:54-99) into
// the device execution plan: slab ids for every layer output, responsibility
// slots for every child contribution, the per-slab CSR that replaces
// np.add.at (engine.py:315-316), parameter/statistics offsets and the
// workspace layout for a chunk of max_chunk samples.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <deque>
#include <cstring>
#include <string>
#include <vector>

#include "einet_internal.h"

namespace einet {

static thread_local std::string g_last_error = "";
static std::atomic<long long> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
int check_cuda(cudaError_t err, const char *what) {
  if (err == cudaSuccess) return EINET_OK;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
  return EINET_ERR_CUDA;
}
void count_launch(int n) { g_launches += n; }
bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("EINET_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int pick_split(int64_t per, int64_t slots, int lo, int hi, double good) {
  lo = std::max(lo, 1);
  hi = std::max(hi, lo);
  int best = lo;
  double best_eff = -1.0;
  for (int s = lo; s <= hi; ++s) {
    const int64_t n = per * s;
    const int64_t waves = (n + slots - 1) / slots;
    const double eff = (double)n / (double)(waves * slots);
    if (waves >= 2 && eff >= good) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int64_t device_slots(const void *kernel, int block, size_t smem, int num_sms) {
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (int64_t)per_sm * num_sms;
}

static bool g_profiling = false;
struct ProfClass {
  std::string name;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
};
static std::vector<ProfClass> g_prof;
bool profiling_enabled() { return g_profiling; }
void profile_record(const char *name, cudaEvent_t start, cudaEvent_t stop) {
  for (auto &c : g_prof)
    if (c.name == name) {
      c.events.emplace_back(start, stop);
      return;
    }
  g_prof.push_back(ProfClass{name, {{start, stop}}});
}
const char *prof_layer_name(const char *base, int layer) {
  static const bool per_layer = getenv("EINET_PROFILE_LAYERS") != nullptr;
  if (!per_layer || !g_profiling) return base;
  static std::deque<std::string> pool;  // interned: pointers stay valid
  const std::string name = std::string(base) + "@" + std::to_string(layer);
  for (const auto &n : pool)
    if (n == name) return n.c_str();
  pool.push_back(name);
  return pool.back().c_str();
}
static void profile_clear() {
  for (auto &c : g_prof)
    for (auto &e : c.events) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  g_prof.clear();
}

template <typename T>
int upload(T **dst, const std::vector<T> &src) {
  *dst = nullptr;
  size_t n = std::max<size_t>(src.size(), 1);
  int rc = check_cuda(cudaMalloc((void **)dst, n * sizeof(T)), "cudaMalloc(plan)");
  if (rc) return rc;
  if (!src.empty())
    rc = check_cuda(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T),
                               cudaMemcpyHostToDevice),
                    "cudaMemcpy(plan)");
  return rc;
}

int upload_tiledesc(Plan &p) {
  std::vector<int64_t> td;
  int64_t items = 0;
  const int64_t KK = (int64_t)p.k * p.k;
  for (auto &L : p.layers) {
    if (L.kind != EINET_LAYER_EINSUM) continue;
    int64_t w[TD_WORDS] = {0};
    w[TD_SLICE0] = L.w_off / KK;
    w[TD_ROWS] = L.rows;
    w[TD_KO] = L.k_out;
    w[TD_TC] = L.tc;
    w[TD_DIRECT] = L.direct;
    w[TD_KG] = L.kg;
    w[TD_NG] = L.ng;
    w[TD_FW_ROWS] = L.fw_rows;
    w[TD_IG] = L.ig;
    w[TD_NI] = L.ni;
    w[TD_UW_ROWS] = L.uw_rows;
    w[TD_KOB] = L.kob;
    w[TD_RW_ROWS] = L.rw_rows;
    w[TD_FW_OFF] = L.fw_off;
    w[TD_FW_TILE] = L.fw_tile;
    w[TD_UW_OFF] = L.uw_off;
    w[TD_UW_TILE] = L.uw_tile;
    w[TD_VW_OFF] = L.vw_off;
    w[TD_RW_TILE] = L.rw_tile;
    // k_build_tiles_all items (one 8-element K chunk of one tile row each)
    w[TD_WOFF] = L.w_off;
    w[TD_IT0] = items;
    if (L.tc) {
      w[TD_NFW] = (int64_t)L.rows * L.ng * L.fw_rows * (p.kp / 8);
      w[TD_NUW] = L.direct ? 0 : (int64_t)L.rows * L.ni * L.uw_rows * (L.kob / 8);
      w[TD_NRW] = L.direct ? (int64_t)L.rows * L.rw_rows * (p.kp / 8) : 0;
    }
    items += w[TD_NFW] + 2 * w[TD_NUW] + w[TD_NRW];
    td.insert(td.end(), w, w + TD_WORDS);
  }
  p.n_tile_items = items;
  p.n_tiledesc = (int)(td.size() / TD_WORDS);
  return upload(&p.d_tiledesc, td);
}

static void free_plan_memory(Plan *p) {
  auto f = [](void *ptr) {
    if (ptr) cudaFree(ptr);
  };
  f(p->d_scope_off);
  f(p->d_scope_vars);
  f(p->d_leaf_rep);
  f(p->d_leaf_slab);
  f(p->d_leaf_of);
  f(p->d_lseg_leaf);
  f(p->d_lseg_v0);
  f(p->d_lseg_vec);
  f(p->d_phi_seg);
  f(p->d_leaf_pvo);
  f(p->d_i8_tab);
  if (p->side_stream) cudaStreamDestroy(p->side_stream);
  p->side_stream = nullptr;
  if (p->fork_stream) cudaStreamDestroy(p->fork_stream);
  p->fork_stream = nullptr;
  if (p->fork_ev) cudaEventDestroy(p->fork_ev);
  if (p->join_ev) cudaEventDestroy(p->join_ev);
  p->fork_ev = p->join_ev = nullptr;
  if (p->red_stream) cudaStreamDestroy(p->red_stream);
  p->red_stream = nullptr;
  for (int i = 0; i < 5; ++i) {
    if (p->red_fork[i]) cudaEventDestroy(p->red_fork[i]);
    if (p->red_done[i]) cudaEventDestroy(p->red_done[i]);
    p->red_fork[i] = p->red_done[i] = nullptr;
  }
  f(p->d_i8_col);
  f(p->d_i8_grp);
  f(p->d_scope_pos);
  f(p->d_tiledesc);
  f(p->d_csr_off);
  f(p->d_csr_slot);
  f(p->d_slab_ones);
  f(p->d_mixrow_off);
  f(p->d_mixrow_len);
  f(p->d_mix_mask_all);
  for (auto &L : p->layers) {
    f(L.d_left_slab);
    f(L.d_right_slab);
    f(L.d_out_slab);
    f(L.d_slot_left);
    f(L.d_slot_right);
    f(L.d_mix_src_slab);
    f(L.d_mix_slot);
    f(L.d_mix_mask);
  }
}

static int build_plan(const einet_plan_desc *d, int64_t max_chunk, Plan *p) {
  if (!d) return fail(EINET_ERR_USAGE, "null plan descriptor");
  if (d->d_vars < 1 || d->k < 1 || d->k_root < 1 || d->num_replicas < 1)
    return fail(EINET_ERR_USAGE, "d_vars, k, k_root and num_replicas must be >= 1");
  if (d->n_leaf < 1 || d->n_layers < 1)
    return fail(EINET_ERR_USAGE, "plan needs a leaf layer and at least one einsum layer");
  if (max_chunk < 1) return fail(EINET_ERR_USAGE, "max_chunk must be >= 1");
  if (d->family < 0 || d->family > 2) return fail(EINET_ERR_USAGE, "unknown family id");
  if (d->family == EINET_FAMILY_CATEGORICAL && d->num_states < 1)
    return fail(EINET_ERR_USAGE, "categorical family needs num_states >= 1");
  if (d->family == EINET_FAMILY_BINOMIAL && d->n_trials < 0)
    return fail(EINET_ERR_USAGE, "binomial family needs n_trials >= 0");

  p->d_vars = d->d_vars;
  p->k = d->k;
  p->k_root = d->k_root;
  p->ks = std::max(d->k, d->k_root);
  p->num_replicas = d->num_replicas;
  p->nbr = d->num_buffer_rows;
  p->family = d->family;
  p->num_states = d->num_states;
  p->n_trials = d->n_trials;
  p->suff = d->family == EINET_FAMILY_GAUSSIAN ? 2
            : d->family == EINET_FAMILY_CATEGORICAL ? d->num_states
                                                    : 1;
  p->var_min = d->var_min;
  p->var_max = d->var_max;
  p->p_min = d->p_min;
  p->n_leaf = d->n_leaf;
  p->max_chunk = max_chunk;
  p->root_mix_row = d->root_mix_row;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
        sms > 0)
      p->num_sms = sms;
    cudaGetLastError();
  }
  const int D = p->d_vars, K = p->k, R = p->num_replicas;

  // ---- leaf layer ----------------------------------------------------------
  p->h_scope_off.assign(d->leaf_scope_offsets, d->leaf_scope_offsets + d->n_leaf + 1);
  const int nvars = p->h_scope_off.back();
  p->h_scope_vars.assign(d->leaf_scope_vars, d->leaf_scope_vars + nvars);
  p->h_leaf_rep.assign(d->leaf_replica, d->leaf_replica + d->n_leaf);
  p->h_leaf_slab.assign(d->leaf_out_rows, d->leaf_out_rows + d->n_leaf);
  std::vector<int> leaf_of((size_t)R * D, -1);
  for (int l = 0; l < d->n_leaf; ++l) {
    int r = p->h_leaf_rep[l];
    if (r < 0 || r >= R) return fail(EINET_ERR_USAGE, "leaf replica out of range");
    int len = p->h_scope_off[l + 1] - p->h_scope_off[l];
    if (len < 1) return fail(EINET_ERR_USAGE, "empty leaf scope");
    p->max_scope = std::max(p->max_scope, len);
    for (int q = p->h_scope_off[l]; q < p->h_scope_off[l + 1]; ++q) {
      int v = p->h_scope_vars[q];
      if (v < 0 || v >= D) return fail(EINET_ERR_USAGE, "leaf scope variable out of range");
      leaf_of[(size_t)r * D + v] = l;
    }
  }

  // ---- leaf-statistics segments (128 scope positions; leaf_tc.cu) ------------
  std::vector<int> lseg_leaf, lseg_v0, phi_seg((size_t)R * D, -1);
  std::vector<uint8_t> lseg_vec;
  for (int l = 0; l < d->n_leaf; ++l) {
    const int sb = p->h_scope_off[l], slen = p->h_scope_off[l + 1] - sb;
    for (int v0 = 0; v0 < slen; v0 += 128) {
      const int nv = std::min(128, slen - v0);
      bool vec = nv % 4 == 0;
      for (int g = 0; vec && g < nv; g += 4) {
        const int d0 = p->h_scope_vars[sb + v0 + g];
        vec = d0 % 4 == 0;
        for (int u = 1; vec && u < 4; ++u) vec = p->h_scope_vars[sb + v0 + g + u] == d0 + u;
      }
      for (int q = 0; q < nv; ++q)
        phi_seg[(size_t)p->h_leaf_rep[l] * D + p->h_scope_vars[sb + v0 + q]] = (int)lseg_leaf.size();
      lseg_leaf.push_back(l);
      lseg_v0.push_back(v0);
      lseg_vec.push_back(vec ? 1 : 0);
    }
  }
  p->n_lseg = (int)lseg_leaf.size();

  // ---- layers, slabs -------------------------------------------------------
  int next_slab = p->nbr;
  int64_t w_acc = 0, mix_acc = 0;
  p->layers.resize(d->n_layers);
  for (int i = 0; i < d->n_layers; ++i) {
    const einet_layer_desc &ld = d->layers[i];
    LayerPlan &L = p->layers[i];
    L.kind = ld.kind;
    L.index = i + 1;
    L.rows = ld.rows;
    L.k_out = ld.k_out;
    L.is_root = ld.is_root;
    L.dmax = ld.dmax;
    if (ld.rows < 1) return fail(EINET_ERR_USAGE, "layer with no rows");
    if (ld.k_out != (ld.is_root ? d->k_root : d->k))
      return fail(EINET_ERR_USAGE, "layer k_out does not match k / k_root");
    L.h_out_slab.resize(ld.rows);
    for (int r = 0; r < ld.rows; ++r) {
      int o = ld.out_rows[r];
      if (o >= p->nbr) return fail(EINET_ERR_USAGE, "out row beyond num_buffer_rows");
      L.h_out_slab[r] = o >= 0 ? o : next_slab++;
    }
    p->max_rows = std::max<int64_t>(p->max_rows, ld.rows);
    if (ld.kind == EINET_LAYER_EINSUM) {
      for (int r = 0; r < ld.rows; ++r)
        if (ld.left[r] < 0 || ld.left[r] >= p->nbr || ld.right[r] < 0 ||
            ld.right[r] >= p->nbr)
          return fail(EINET_ERR_USAGE, "einsum child row out of range");
      L.w_off = w_acc;
      L.erow_base = p->n_erows;
      p->n_erows += ld.rows;
      int64_t lw = (int64_t)ld.rows * ld.k_out * K * K;
      w_acc += lw;
      p->max_layer_w = std::max(p->max_layer_w, lw);
    } else if (ld.kind == EINET_LAYER_MIXING) {
      if (i == 0 || d->layers[i - 1].kind != EINET_LAYER_EINSUM)
        return fail(EINET_ERR_USAGE, "mixing layer must follow an einsum layer");
      if (ld.dmax < 1) return fail(EINET_ERR_USAGE, "mixing layer with dmax < 1");
      L.mix_off = mix_acc;
      mix_acc += (int64_t)ld.rows * ld.dmax;
      L.h_src.assign(ld.src, ld.src + (size_t)ld.rows * ld.dmax);
      L.h_mask.assign(ld.mask, ld.mask + (size_t)ld.rows * ld.dmax);
    } else {
      return fail(EINET_ERR_USAGE, "unknown layer kind");
    }
  }
  p->num_slabs = next_slab;
  p->n_w = w_acc;
  p->n_mix = mix_acc;
  p->n_mix_entries = mix_acc;
  p->n_phi = (int64_t)D * K * R * p->suff;

  const LayerPlan &last = p->layers.back();
  if (!last.is_root) return fail(EINET_ERR_USAGE, "last layer must hold the root");
  if (last.kind == EINET_LAYER_MIXING) {
    if (p->root_mix_row < 0 || p->root_mix_row >= last.rows)
      return fail(EINET_ERR_USAGE, "root_mix_row out of range");
    p->root_out_slab = last.h_out_slab[p->root_mix_row];
  } else {
    p->root_out_slab = last.h_out_slab[0];
  }

  // ---- slots and CSR -----------------------------------------------------
  std::vector<std::vector<int>> contrib(p->num_slabs);
  p->h_slab_ones.assign(p->num_slabs, 0);
  int next_slot = 0;
  std::vector<std::vector<int>> slot_left(d->n_layers), slot_right(d->n_layers),
      mix_slot(d->n_layers), mix_src_slab(d->n_layers);
  for (int i = 0; i < d->n_layers; ++i) {
    const einet_layer_desc &ld = d->layers[i];
    LayerPlan &L = p->layers[i];
    if (ld.kind == EINET_LAYER_EINSUM) {
      slot_left[i].resize(ld.rows);
      slot_right[i].resize(ld.rows);
      for (int r = 0; r < ld.rows; ++r) {
        slot_left[i][r] = next_slot++;
        slot_right[i][r] = next_slot++;
      }
    } else {
      const LayerPlan &prev = p->layers[i - 1];
      mix_slot[i].assign((size_t)ld.rows * ld.dmax, -1);
      mix_src_slab[i].assign((size_t)ld.rows * ld.dmax, -1);
      for (int m = 0; m < ld.rows; ++m)
        for (int c = 0; c < ld.dmax; ++c) {
          size_t q = (size_t)m * ld.dmax + c;
          if (!L.h_mask[q]) continue;
          int s = L.h_src[q];
          if (s < 0 || s >= prev.rows) return fail(EINET_ERR_USAGE, "mixing src out of range");
          mix_slot[i][q] = next_slot++;
          mix_src_slab[i][q] = prev.h_out_slab[s];
        }
    }
  }
  p->num_slots = next_slot;
  // contributions ordered top-down (the reference's backward order)
  for (int i = d->n_layers - 1; i >= 0; --i) {
    const einet_layer_desc &ld = d->layers[i];
    if (ld.kind == EINET_LAYER_EINSUM) {
      for (int r = 0; r < ld.rows; ++r) contrib[ld.left[r]].push_back(slot_left[i][r]);
      for (int r = 0; r < ld.rows; ++r) contrib[ld.right[r]].push_back(slot_right[i][r]);
    } else {
      for (size_t q = 0; q < mix_slot[i].size(); ++q)
        if (mix_slot[i][q] >= 0) contrib[mix_src_slab[i][q]].push_back(mix_slot[i][q]);
    }
  }
  p->h_slab_ones[p->root_out_slab] = 1;
  p->h_csr_off.assign(p->num_slabs + 1, 0);
  for (int s = 0; s < p->num_slabs; ++s)
    p->h_csr_off[s + 1] = p->h_csr_off[s] + (int)contrib[s].size();
  p->h_csr_slot.clear();
  for (int s = 0; s < p->num_slabs; ++s)
    p->h_csr_slot.insert(p->h_csr_slot.end(), contrib[s].begin(), contrib[s].end());

  // ---- sizes ---------------------------------------------------------------
  einet_sizes &z = p->sizes;
  z.params_f64 = p->n_w + p->n_mix + p->n_phi;
  z.mixing_offset = p->n_w;
  z.phi_offset = p->n_w + p->n_mix;
  z.stats_acc_pt_offset = p->n_w + p->n_mix;
  z.stats_p_offset = z.stats_acc_pt_offset + p->n_phi;
  z.stats_ll_offset = z.stats_p_offset + (int64_t)p->n_leaf * K;
  z.stats_f64 = z.stats_ll_offset + 3;  // [ll_sum, n, failed ranks]
  z.max_chunk = max_chunk;
  z.suff_dim = p->suff;

  const int64_t A = 256;
  int64_t off = 0;
  auto seg = [&](int64_t bytes) {
    int64_t at = off;
    off = align_up(off + std::max<int64_t>(bytes, 0), A);
    return at;
  };
  const int64_t RDK = (int64_t)R * D * K;
  p->c_w32 = seg(4 * p->n_w);
  p->c_mix32 = seg(4 * std::max<int64_t>(p->n_mix, 1));
  if (p->family == EINET_FAMILY_CATEGORICAL)
    p->c_leafp = seg(8 * RDK * p->num_states);
  else
    p->c_leafp = seg(16 * RDK);
  p->c_center = seg(4 * RDK);
  p->c_const = seg(8 * (int64_t)p->n_leaf * K);
  p->c_active = seg(D + 1);
  p->c_logh = seg(8 * (int64_t)(std::max(p->n_trials, 0) + 1));
  p->leaf_dmma = p->family == EINET_FAMILY_GAUSSIAN && K % 8 == 0 && K <= 64;
  if (p->family == EINET_FAMILY_GAUSSIAN) {
    p->h_leaf_pvo.assign(p->n_leaf + 1, 0);
    for (int l = 0; l < p->n_leaf; ++l)
      p->h_leaf_pvo[l + 1] =
          p->h_leaf_pvo[l] + (int)align_up(p->h_scope_off[l + 1] - p->h_scope_off[l], 32);
  }
  if (p->leaf_dmma) {
    p->c_leafimg = seg(16 * (int64_t)K * p->h_leaf_pvo.back());
    p->c_cm2 = seg(8 * (int64_t)p->n_leaf * K);
  }
  {
    const char *env = getenv("EINET_DISABLE_TC");
    p->use_tc = !(env && env[0] == '1');
  }
  std::vector<int> i8_tab, i8_col, i8_grp;
  if (p->family == EINET_FAMILY_GAUSSIAN) plan_leaf_i8(*p, i8_tab, i8_col, i8_grp);
  if (p->leaf_i8) {
    p->c_i8img = seg((int64_t)p->i8_ng * 96 * (p->h_leaf_pvo.back() / 32));
    p->c_i8c = seg(16 * (int64_t)p->n_leaf * p->i8_k8);
    p->c_i8mask = seg(4 * (int64_t)(p->h_leaf_pvo.back() / 32));
  }
  plan_tc_tiling(*p);
  for (auto &L : p->layers) {
    if (!L.tc) continue;
    L.fw_off = seg(L.fw_tile * L.rows * L.ng);
    L.uw_off = seg(L.uw_tile * L.rows * L.ni);
    L.vw_off = seg(std::max(L.uw_tile * L.ni, L.rw_tile) * L.rows);
  }
  p->c_mtmp = seg(16 * (int64_t)R * D * K);
  z.compute_bytes = off;

  p->bc = align_up(max_chunk, 128);  // 32-sample blocks, 128-sample tensor-core tiles
  const int64_t Bc = p->bc, KS = p->ks;
  off = 0;
  p->w_off = seg(4 * (int64_t)p->num_slabs * Bc * KS);
  p->w_shift = seg(8 * (int64_t)p->num_slabs * Bc);
  p->w_slots = seg(4 * (int64_t)std::max(p->num_slots, 1) * Bc * KS);
  p->w_leafpart = seg(8 * (int64_t)kMaxDSplit * p->n_leaf * Bc * K);
  p->w_ea = seg(4 * (int64_t)p->n_erows * (Bc / 32) * K * EV_ROW);
  p->w_eb = seg(4 * (int64_t)p->n_erows * (Bc / 32) * K * EV_ROW);
  p->w_rt = seg(4 * p->max_rows * Bc * KS);
  // W-stat partials: bsplit chosen per layer by the launcher, bounded here
  int64_t wpart = 0;
  for (auto &L : p->layers) {
    if (L.kind != EINET_LAYER_EINSUM) continue;
    int64_t lw = (int64_t)L.rows * L.k_out * K * K;
    int64_t blocks = (int64_t)L.rows * ((L.k_out + wstats_simt_kc(K, L.k_out) - 1) /
                                        wstats_simt_kc(K, L.k_out));
    int64_t bs = std::min<int64_t>(std::max<int64_t>(1, (2 * p->num_sms + blocks - 1) / blocks),
                                   std::min<int64_t>(kMaxBSplit, (Bc + 63) / 64));
    // tensor-core W statistics: fp32 partials per (segment, slot) (wstats_tc.cu)
    int64_t tc_slots = L.tc ? wstats_tc_slots(*p, L, Bc) : 0;
    wpart = std::max(wpart, std::max(bs * lw, (tc_slots * lw + 1) / 2));
  }
  p->wpart_half = align_up(std::max<int64_t>(wpart, 1), 32);
  p->w_wpart = seg(8 * 2 * p->wpart_half);  // two halves: layer parity
  p->w_rho = seg(4 * (int64_t)p->n_leaf * Bc * K);
  p->max_lsplit = leaf_lsplit(*p, Bc);
  p->w_lspart = seg(std::max(8 * (int64_t)p->max_lsplit * p->n_phi,
                             4 * leaf_stats_slots(*p, Bc) * p->n_phi));
  p->w_ppart = seg(8 * (int64_t)ceil_div(Bc, 32) * p->n_leaf * K);
  p->w_mixpart = seg(8 * (int64_t)ceil_div(Bc, 32) * std::max<int64_t>(p->n_mix, 1));
  p->w_llpart = seg(8 * ((int64_t)ceil_div(Bc, 256) + 1));  // partials + ticket
  p->w_tmp_s = seg(8 * p->n_phi);
  p->w_tmp_p = seg(8 * (int64_t)p->n_leaf * K);
  {
    int kobmax = 0;
    bool any_tc = false;
    for (auto &L : p->layers)
      if (L.tc) {
        any_tc = true;
        kobmax = std::max(kobmax, L.kob);
      }
    // bf16 hi | lo A-operand tiles (contract_tc.cu)
    p->w_ebm = seg(any_tc ? 4 * (int64_t)p->n_erows * Bc * p->kp : 0);
    p->w_eam = seg(any_tc ? 4 * (int64_t)p->n_erows * Bc * p->kp : 0);
    p->w_rtm = seg(any_tc ? 4 * p->max_rows * Bc * kobmax : 0);
    int nnmax = 0;
    for (auto &L : p->layers)
      if (L.tc) nnmax = std::max(nnmax, L.nn);
    p->w_rtb = seg(any_tc ? 8 * p->max_rows * Bc * nnmax : 0);
    p->w_rhob = seg(8 * (int64_t)p->n_leaf * Bc * ((K + 15) / 16 * 16));
  }
  p->w_i8flag = seg(16);
  p->w_scratch_end = off;
  z.workspace_bytes = off;

  // ---- device copies ---------------------------------------------------------
  int rc;
  if ((rc = upload(&p->d_scope_off, p->h_scope_off))) return rc;
  if ((rc = upload(&p->d_scope_vars, p->h_scope_vars))) return rc;
  if ((rc = upload(&p->d_leaf_rep, p->h_leaf_rep))) return rc;
  if ((rc = upload(&p->d_leaf_slab, p->h_leaf_slab))) return rc;
  if ((rc = upload(&p->d_leaf_of, leaf_of))) return rc;
  if ((rc = upload(&p->d_lseg_leaf, lseg_leaf))) return rc;
  if ((rc = upload(&p->d_lseg_v0, lseg_v0))) return rc;
  if ((rc = upload(&p->d_lseg_vec, lseg_vec))) return rc;
  if ((rc = upload(&p->d_phi_seg, phi_seg))) return rc;
  if (!p->h_leaf_pvo.empty() && (rc = upload(&p->d_leaf_pvo, p->h_leaf_pvo))) return rc;
  if (p->leaf_i8 && (rc = upload(&p->d_i8_tab, i8_tab))) return rc;
  if (p->leaf_i8 && (rc = upload(&p->d_i8_col, i8_col))) return rc;
  if (p->leaf_i8 && (rc = upload(&p->d_i8_grp, i8_grp))) return rc;
  p->h_i8_grp = i8_grp;
  if (p->leaf_i8 &&
      (rc = check_cuda(cudaStreamCreateWithFlags(&p->side_stream, cudaStreamNonBlocking),
                       "side stream")))
    return rc;
  if ((rc = check_cuda(cudaStreamCreateWithFlags(&p->fork_stream, cudaStreamNonBlocking),
                       "fork stream")) ||
      (rc = check_cuda(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming), "event")) ||
      (rc = check_cuda(cudaEventCreateWithFlags(&p->join_ev, cudaEventDisableTiming), "event")) ||
      (rc = check_cuda(cudaStreamCreateWithFlags(&p->red_stream, cudaStreamNonBlocking),
                       "reduction stream")))
    return rc;
  for (int i = 0; i < 5; ++i)
    if ((rc = check_cuda(cudaEventCreateWithFlags(&p->red_fork[i], cudaEventDisableTiming), "event")) ||
        (rc = check_cuda(cudaEventCreateWithFlags(&p->red_done[i], cudaEventDisableTiming), "event")))
      return rc;
  {
    std::vector<int> pos((size_t)R * D, -1);
    for (int l = 0; l < d->n_leaf; ++l)
      for (int q = p->h_scope_off[l]; q < p->h_scope_off[l + 1]; ++q)
        pos[(size_t)p->h_leaf_rep[l] * D + p->h_scope_vars[q]] = q - p->h_scope_off[l];
    if ((rc = upload(&p->d_scope_pos, pos))) return rc;
  }
  if ((rc = upload_tiledesc(*p))) return rc;
  if ((rc = upload(&p->d_csr_off, p->h_csr_off))) return rc;
  if ((rc = upload(&p->d_csr_slot, p->h_csr_slot))) return rc;
  if ((rc = upload(&p->d_slab_ones, p->h_slab_ones))) return rc;
  {
    std::vector<int> roff, rlen;
    std::vector<uint8_t> mall;
    for (auto &L : p->layers) {
      if (L.kind != EINET_LAYER_MIXING) continue;
      for (int m = 0; m < L.rows; ++m) {
        roff.push_back((int)(L.mix_off + (int64_t)m * L.dmax));
        rlen.push_back(L.dmax);
      }
      mall.insert(mall.end(), L.h_mask.begin(), L.h_mask.end());
    }
    p->n_mixrows = (int)roff.size();
    if ((rc = upload(&p->d_mixrow_off, roff))) return rc;
    if ((rc = upload(&p->d_mixrow_len, rlen))) return rc;
    if ((rc = upload(&p->d_mix_mask_all, mall))) return rc;
  }
  for (int i = 0; i < d->n_layers; ++i) {
    const einet_layer_desc &ld = d->layers[i];
    LayerPlan &L = p->layers[i];
    if ((rc = upload(&L.d_out_slab, L.h_out_slab))) return rc;
    if (ld.kind == EINET_LAYER_EINSUM) {
      std::vector<int> ls(ld.left, ld.left + ld.rows), rs(ld.right, ld.right + ld.rows);
      if ((rc = upload(&L.d_left_slab, ls))) return rc;
      if ((rc = upload(&L.d_right_slab, rs))) return rc;
      if ((rc = upload(&L.d_slot_left, slot_left[i]))) return rc;
      if ((rc = upload(&L.d_slot_right, slot_right[i]))) return rc;
    } else {
      if ((rc = upload(&L.d_mix_src_slab, mix_src_slab[i]))) return rc;
      if ((rc = upload(&L.d_mix_slot, mix_slot[i]))) return rc;
      if ((rc = upload(&L.d_mix_mask, L.h_mask))) return rc;
    }
  }
  return EINET_OK;
}

}  // namespace einet

using namespace einet;

struct einet_plan {
  Plan impl;
};

extern "C" {

int einet_plan_create(const einet_plan_desc *desc, int64_t max_chunk, einet_plan **out) {
  if (!out) return fail(EINET_ERR_USAGE, "null output pointer");
  *out = nullptr;
  einet_plan *h = new einet_plan();
  int rc = build_plan(desc, max_chunk, &h->impl);
  if (rc) {
    free_plan_memory(&h->impl);
    delete h;
    return rc;
  }
  *out = h;
  return EINET_OK;
}

void einet_plan_destroy(einet_plan *plan) {
  if (!plan) return;
  free_plan_memory(&plan->impl);
  delete plan;
}

int einet_plan_sizes(const einet_plan *plan, einet_sizes *out) {
  if (!plan || !out) return fail(EINET_ERR_USAGE, "null argument");
  *out = plan->impl.sizes;
  return EINET_OK;
}

int einet_prepare(einet_plan *plan, const double *params, void *compute,
                  const uint8_t *marg_mask, const double *leaf_log_offset, void *stream) {
  if (!plan || !params || !compute) return fail(EINET_ERR_USAGE, "null argument");
  return launch_prepare(plan->impl, params, (uint8_t *)compute, marg_mask, leaf_log_offset,
                        (cudaStream_t)stream);
}

int einet_forward(einet_plan *plan, const void *compute, const float *x, int64_t batch,
                  void *workspace, double *root_out, int32_t *status, void *stream) {
  if (!plan || !compute || !x || !workspace || !root_out || !status)
    return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1 || batch > plan->impl.max_chunk)
    return fail(EINET_ERR_USAGE, "batch must be in [1, max_chunk]");
  return launch_forward(plan->impl, (const uint8_t *)compute, x, batch,
                        (uint8_t *)workspace, root_out, status, (cudaStream_t)stream);
}

int einet_backward(einet_plan *plan, const double *params, const void *compute,
                   const float *x, int64_t batch, void *workspace, double *stats,
                   int32_t *status, void *stream) {
  if (!plan || !params || !compute || !x || !workspace || !stats || !status)
    return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1 || batch > plan->impl.max_chunk)
    return fail(EINET_ERR_USAGE, "batch must be in [1, max_chunk]");
  return launch_backward(plan->impl, params, (const uint8_t *)compute, x, batch,
                         (uint8_t *)workspace, stats, status, (cudaStream_t)stream);
}

int einet_status_reset(int32_t *status, void *stream) {
  if (!status) return fail(EINET_ERR_USAGE, "null argument");
  return launch_status_reset(status, (cudaStream_t)stream);
}

int einet_log_step(const double *ll2, const int32_t *status, double *log_ll, int32_t *log_st,
                   int64_t *cursor, int64_t cap, void *stream) {
  if (!ll2 || !status || !log_ll || !log_st || !cursor) return fail(EINET_ERR_USAGE, "null argument");
  if (cap < 0) return fail(EINET_ERR_USAGE, "cap must be >= 0");
  return launch_log_step(ll2, status, log_ll, log_st, cursor, cap, (cudaStream_t)stream);
}

int einet_status_to_stats(einet_plan *plan, const int32_t *status, double *stats,
                          void *stream) {
  if (!plan || !status || !stats) return fail(EINET_ERR_USAGE, "null argument");
  return launch_status_to_stats(status, stats + plan->impl.sizes.stats_ll_offset + 2,
                                (cudaStream_t)stream);
}

int einet_status_from_stats(einet_plan *plan, const double *stats, int32_t *status,
                            void *stream) {
  if (!plan || !status || !stats) return fail(EINET_ERR_USAGE, "null argument");
  return launch_status_from_stats(stats + plan->impl.sizes.stats_ll_offset + 2, status,
                                  (cudaStream_t)stream);
}

int einet_plan_set_tensor_cores(einet_plan *plan, int enable) {
  if (!plan) return fail(EINET_ERR_USAGE, "null argument");
  plan->impl.use_tc = enable != 0;
  return EINET_OK;
}

int einet_stats_zero(einet_plan *plan, double *stats, void *stream) {
  if (!plan || !stats) return fail(EINET_ERR_USAGE, "null argument");
  return check_cuda(cudaMemsetAsync(stats, 0, sizeof(double) * plan->impl.sizes.stats_f64,
                                    (cudaStream_t)stream),
                    "cudaMemsetAsync(stats)");
}

int einet_mstep(einet_plan *plan, double *params, void *compute, const double *stats,
                double lam, double eps_w, const int32_t *status, void *stream) {
  if (!plan || !params || !compute || !stats) return fail(EINET_ERR_USAGE, "null argument");
  if (!(lam > 0.0 && lam <= 1.0)) return fail(EINET_ERR_USAGE, "lam must lie in (0, 1]");
  return launch_mstep(plan->impl, params, (uint8_t *)compute, stats, lam, eps_w, status,
                      (cudaStream_t)stream);
}

int einet_stats_expand_acc_p(einet_plan *plan, const double *stats, double *acc_p,
                             void *stream) {
  if (!plan || !stats || !acc_p) return fail(EINET_ERR_USAGE, "null argument");
  return launch_expand_acc_p(plan->impl, stats, acc_p, (cudaStream_t)stream);
}

int einet_export_buffer(einet_plan *plan, const void *workspace, int64_t batch, double *out,
                        void *stream) {
  if (!plan || !workspace || !out) return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1 || batch > plan->impl.max_chunk)
    return fail(EINET_ERR_USAGE, "batch must be in [1, max_chunk]");
  return launch_export_buffer(plan->impl, (const uint8_t *)workspace, batch, out,
                              (cudaStream_t)stream);
}

int einet_export_leaf_rows(einet_plan *plan, const void *workspace, int64_t batch,
                           double *out, void *stream) {
  if (!plan || !workspace || !out) return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1 || batch > plan->impl.max_chunk)
    return fail(EINET_ERR_USAGE, "batch must be in [1, max_chunk]");
  return launch_export_leaf_rows(plan->impl, (const uint8_t *)workspace, batch, out,
                                 (cudaStream_t)stream);
}

int einet_ef_log_prob(einet_plan *plan, const double *params, const float *x, int64_t batch,
                      const uint8_t *marg_mask, double *out, int32_t *status, void *stream) {
  if (!plan || !params || !x || !out || !status) return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1) return fail(EINET_ERR_USAGE, "batch must be >= 1");
  return launch_ef_log_prob(plan->impl, params, x, batch, marg_mask, out, status,
                            (cudaStream_t)stream);
}

int einet_log_einsum_exp(const double *left, const double *right, const double *w,
                         int64_t batch, int32_t rows, int32_t k, int32_t k_out, double *out,
                         void *stream) {
  if (!left || !right || !w || !out) return fail(EINET_ERR_USAGE, "null argument");
  if (batch < 1 || rows < 1 || k < 1 || k_out < 1)
    return fail(EINET_ERR_USAGE, "sizes must be >= 1");
  return launch_log_einsum_exp(left, right, w, batch, rows, k, k_out, out,
                               (cudaStream_t)stream);
}

int64_t einet_sample_scratch_bytes(const einet_plan *plan, int64_t n) {
  if (!plan || n < 0) return -1;
  return sample_scratch_bytes(plan->impl, n);
}

int einet_sample(einet_plan *plan, const double *params, const void *workspace,
                 int32_t conditional, const double *x_e, const uint8_t *evidence, int64_t n,
                 uint64_t seed, void *scratch, double *out, int32_t *status, void *stream) {
  if (!plan || !params || !scratch || !out || !status)
    return fail(EINET_ERR_USAGE, "null argument");
  if (conditional && (!workspace || !x_e || !evidence))
    return fail(EINET_ERR_USAGE, "conditional sampling needs the forward workspace, x_e and the evidence mask");
  if (n < 0) return fail(EINET_ERR_USAGE, "n must be >= 0");
  return launch_sample(plan->impl, params, (const uint8_t *)workspace, conditional, x_e,
                       evidence, n, seed, (uint8_t *)scratch, out, status,
                       (cudaStream_t)stream);
}

int einet_decode_u8(const uint8_t *src, int64_t count, double divisor, float *dst,
                    void *stream) {
  if (count < 0) return fail(EINET_ERR_USAGE, "count must be >= 0");
  if (count > 0 && (!src || !dst)) return fail(EINET_ERR_USAGE, "null argument");
  if (!(divisor > 0.0) || !std::isfinite(divisor))
    return fail(EINET_ERR_USAGE, "divisor must be finite and > 0");
  return launch_decode_u8(src, count, divisor, dst, (cudaStream_t)stream);
}

int einet_pack_f64(const double *x, int64_t count, uint8_t *u8_out, float *f32_out,
                   int32_t threads, int32_t *kind) {
  if (count < 0) return fail(EINET_ERR_USAGE, "count must be >= 0");
  if (!kind || (count > 0 && (!x || !u8_out)))
    return fail(EINET_ERR_USAGE, "null argument");
  *kind = host_pack_f64(x, count, u8_out, f32_out, threads);
  return EINET_OK;
}

int einet_crc32(const uint8_t *data, int64_t len, uint32_t *crc, void *stream) {
  if (len < 0) return fail(EINET_ERR_USAGE, "len must be >= 0");
  if (!crc || (len > 0 && !data)) return fail(EINET_ERR_USAGE, "null argument");
  return launch_crc32(data, len, crc, (cudaStream_t)stream);
}

int einet_params_from_blob(const uint8_t *blob, int64_t blob_len, const int64_t *table,
                           int32_t n_tensors, int64_t max_count, double *params, int32_t *bad,
                           void *stream) {
  if (n_tensors < 0 || blob_len < 0 || max_count < 0)
    return fail(EINET_ERR_USAGE, "sizes must be >= 0");
  if (n_tensors > 0 && (!blob || !table || !params || !bad))
    return fail(EINET_ERR_USAGE, "null argument");
  return launch_blob_to_params(blob, blob_len, table, n_tensors, max_count, params, bad,
                               (cudaStream_t)stream);
}

int einet_params_to_blob(const double *params, const int64_t *table, int32_t n_tensors,
                         int64_t max_count, uint8_t *blob, void *stream) {
  if (n_tensors < 0 || max_count < 0) return fail(EINET_ERR_USAGE, "sizes must be >= 0");
  if (n_tensors > 0 && (!blob || !table || !params))
    return fail(EINET_ERR_USAGE, "null argument");
  return launch_params_to_blob(params, table, n_tensors, max_count, blob,
                               (cudaStream_t)stream);
}

int einet_selftest_tf32_gemm(const float *A, const float *B, float *D, int32_t N, int32_t K,
                             void *stream) {
  if (!A || !B || !D) return fail(EINET_ERR_USAGE, "null argument");
  return launch_selftest_gemm(A, B, D, N, K, (cudaStream_t)stream);
}

int64_t einet_launch_count(void) { return (int64_t)g_launches.load(); }

int einet_profile_enable(int on) {
  cudaDeviceSynchronize();
  profile_clear();
  g_profiling = on != 0;
  return EINET_OK;
}

int einet_profile_query(int32_t index, char *name, int32_t name_len, double *total_ms,
                        int64_t *count) {
  if (index < 0 || index >= (int)g_prof.size()) return EINET_ERR_USAGE;
  ProfClass &c = g_prof[index];
  double tot = 0.0;
  for (auto &e : c.events) {
    cudaEventSynchronize(e.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.first, e.second);
    tot += ms;
  }
  if (name && name_len > 0) {
    std::strncpy(name, c.name.c_str(), name_len - 1);
    name[name_len - 1] = 0;
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = (int64_t)c.events.size();
  return EINET_OK;
}

const char *einet_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
