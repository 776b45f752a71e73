/*
 * einet_b200.h -- C ABI of the B200-native Einsum-Network EM engine.
 *
 * The reference (arXiv 2004.06231 reimplementation, /root/reference/pkg/src/einet)
 * is pure Python/NumPy and has no FFI; these entry points are the boundary its
 * hot path would bind. Each function names the reference
 * interface it replaces. Plain pointers and sizes only; every device buffer is
 * caller-owned (the Python host mirror passes torch CUDA tensors' data_ptr()).
 *
 * All compute calls are stream-ordered and asynchronous. Data-dependent errors
 * (values outside the leaf family's support, NaN entering an einsum layer) are
 * raised on the device into the caller's int32 status word and mapped to the
 * reference exception types by the host after its next synchronisation point.
 */
#ifndef EINET_B200_H
#define EINET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map 1:1 to reference exception types) ---------------- */
#define EINET_OK 0
#define EINET_ERR_USAGE 1       /* ValueError (bad arguments / shapes)           */
#define EINET_ERR_ENGINE 2      /* EngineError, engine.py:23-24                  */
#define EINET_ERR_UNSUPPORTED 3 /* UnsupportedValueError, expfam.py:19-20        */
#define EINET_ERR_CUDA 4        /* CUDA runtime failure                          */

/* ---- families (expfam.py:82-275) ---------------------------------------- */
#define EINET_FAMILY_GAUSSIAN 0
#define EINET_FAMILY_CATEGORICAL 1
#define EINET_FAMILY_BINOMIAL 2

/* ---- layer kinds (compiler.py:28-45) ------------------------------------ */
#define EINET_LAYER_EINSUM 1
#define EINET_LAYER_MIXING 2

/* Device status words written by forward/backward (int32[4]).
 * [0] lowest variable index with an unsupported value (INT32_MAX = none)
 * [1] lowest layer index with NaN entering an einsum layer (INT32_MAX = none)
 * [2] family-specific detail code (internal)
 * [3] 0 = another rank of the process group failed this EM step
 *     (einet_status_from_stats); sampling: a slab with all-zero weights. */
#define EINET_STATUS_WORDS 4

/* One einsum or mixing layer of a compiled LayeredCircuit (compiler.py:28-45). */
typedef struct {
  int32_t kind;             /* EINET_LAYER_EINSUM | EINET_LAYER_MIXING            */
  int32_t rows;             /* L (einsum rows) or M (mixing rows)                */
  int32_t k_out;            /* K or K_root                                       */
  int32_t is_root;          /* layer holds the root region                       */
  int32_t dmax;             /* mixing: padded child count per row                */
  const int32_t *left;      /* einsum: (rows) global buffer rows, left child     */
  const int32_t *right;     /* einsum: (rows) global buffer rows, right child    */
  const int32_t *out_rows;  /* (rows) global buffer row, -1 = root (unbuffered)  */
  const int32_t *src;       /* mixing: (rows*dmax) local rows of previous layer  */
  const uint8_t *mask;      /* mixing: (rows*dmax) 1 where a child exists        */
} einet_layer_desc;

/* A compiled LayeredCircuit plus the leaf family (compiler.py:54-99). */
typedef struct {
  int32_t d_vars;
  int32_t k;
  int32_t k_root;
  int32_t num_replicas;
  int32_t num_buffer_rows;
  int32_t family;           /* EINET_FAMILY_*                                    */
  int32_t num_states;       /* categorical                                       */
  int32_t n_trials;         /* binomial                                          */
  double var_min, var_max;  /* gaussian projection bounds (expfam.py:112-115)    */
  double p_min;             /* categorical / binomial floor                     */
  int32_t n_leaf;           /* leaf regions (LeafLayer, compiler.py:20-25)       */
  const int32_t *leaf_scope_offsets; /* (n_leaf+1) CSR into leaf_scope_vars      */
  const int32_t *leaf_scope_vars;    /* sorted variable indices per leaf         */
  const int32_t *leaf_replica;       /* (n_leaf)                                 */
  const int32_t *leaf_out_rows;      /* (n_leaf)                                 */
  int32_t n_layers;                  /* einsum/mixing layers after the leaf     */
  const einet_layer_desc *layers;
  int32_t root_mix_row;     /* index of the root region in a root mixing layer   */
} einet_plan_desc;

/* Element counts / byte sizes of the caller-owned buffers of one plan. */
typedef struct {
  int64_t params_f64;       /* master params: [W layers | mixing | phi(D,K,R,T)]   */
  int64_t phi_offset;       /* element offset of phi inside params               */
  int64_t mixing_offset;    /* element offset of the first mixing layer          */
  int64_t stats_f64;        /* EM statistics: [n_W | n_mix | acc_pt | P | ll,n,f] */
  int64_t stats_acc_pt_offset;
  int64_t stats_p_offset;   /* compressed acc_p: (n_leaf, K)                     */
  int64_t stats_ll_offset;  /* [ll_sum, n_samples, failed ranks]                 */
  int64_t compute_bytes;    /* derived device tensors (prepare / mstep output)   */
  int64_t workspace_bytes;  /* per-chunk activations, responsibilities, scratch  */
  int64_t max_chunk;        /* largest batch one forward/backward call accepts  */
  int64_t suff_dim;         /* T of the leaf family                              */
} einet_sizes;

typedef struct einet_plan einet_plan;

/* Build the execution plan (slabs, responsibility slots, CSR, device index
 * arrays). Replaces compiler.compile_graph's consumer side (compiler.py:158-251). */
int einet_plan_create(const einet_plan_desc *desc, int64_t max_chunk, einet_plan **out);
void einet_plan_destroy(einet_plan *plan);
int einet_plan_sizes(const einet_plan *plan, einet_sizes *out);

/* Derive the device compute tensors from fp64 master parameters. marg_mask
 * (uint8 per variable, nullable) and leaf_log_offset (fp64 (D,K,R), nullable)
 * replace forward's marg_mask / leaf_log_offset (engine.py:143-144,
 * expfam.py:297-309). */
int einet_prepare(einet_plan *plan, const double *params, void *compute,
                  const uint8_t *marg_mask, const double *leaf_log_offset,
                  void *stream);

/* Forward pass over B <= max_chunk samples (x: fp32 (B, D) row-major, device).
 * Writes root log-densities (B, k_root) fp64 and keeps the trace in workspace.
 * Replaces engine.forward (engine.py:143-195). */
int einet_forward(einet_plan *plan, const void *compute, const float *x, int64_t batch,
                  void *workspace, double *root_out, int32_t *status, void *stream);

/* Responsibility back-pass over the trace in workspace; ADDS the expected
 * statistics of the batch into stats (reference layout, fp64), including the
 * batch log-likelihood sum. Replaces engine.backward + BackwardStats.merge
 * (engine.py:218-328). */
int einet_backward(einet_plan *plan, const double *params, const void *compute,
                   const float *x, int64_t batch, void *workspace, double *stats,
                   int32_t *status, void *stream);

/* Enable (default) or disable the tcgen05 EinsumLayer kernels of this plan
 * (the CUDA-core kernels are used for layers the tensor-core path does not
 * cover; EINET_DISABLE_TC=1 in the environment disables them at creation). */
int einet_plan_set_tensor_cores(einet_plan *plan, int enable);

/* Set the int32[EINET_STATUS_WORDS] status words to "no error" (INT32_MAX).
 * Call once per step; forward/backward only lower them (atomicMin). */
int einet_status_reset(int32_t *status, void *stream);

/* Per-step device log of a pipelined EM sequence (trainer.em_stochastic_steps,
 * the reference's loop of em_stochastic_step calls, trainer.py:99-117, each
 * returning its mean LL): copies ll2[0..1] (the stats buffer's LL sum and
 * sample count) to log_ll[2 * r] and the status words to
 * log_st[EINET_STATUS_WORDS * r] for r = *cursor (when r < cap), then
 * increments *cursor (device int64). Captured as the last node of the step's
 * CUDA graph. */
int einet_log_step(const double *ll2, const int32_t *status, double *log_ll, int32_t *log_st,
                   int64_t *cursor, int64_t cap, void *stream);

/* One collective per data-parallel EM update (the reference's
 * merge, engine.py:228-236, is the all-reduce(sum) of the stats buffer).
 * einet_status_to_stats: stats[ll+2] = 1 if this rank's status words report
 *   an error, else 0 -- enqueue after the last einet_backward of the step, so
 *   the sum over ranks counts the failing ranks.
 * einet_status_from_stats: after the all-reduce, set status word 3 to 0 when
 *   that count is non-zero; einet_mstep then skips the update on every rank.
 *   Only then does the host need the exact words (a MIN all-reduce). */
int einet_status_to_stats(einet_plan *plan, const int32_t *status, double *stats,
                          void *stream);
int einet_status_from_stats(einet_plan *plan, const double *stats, int32_t *status,
                            void *stream);

/* Zero a stats buffer (engine._zero_stats, engine.py:239-244). */
int einet_stats_zero(einet_plan *plan, double *stats, void *stream);

/* Fused M-step: targets (trainer.py:69-86), gliding average with step lam
 * (trainer.py:110-115), projections (trainer.py:89-96, engine.py:46-54,
 * family.project) and re-derivation of the compute tensors. Skips the
 * update when a status word reports an error (words 0, 1, 3). lam == 0 must not be passed
 * (the host returns early, trainer.py:107-108). */
int einet_mstep(einet_plan *plan, double *params, void *compute, const double *stats,
                double lam, double eps_w, const int32_t *status, void *stream);

/* Expand compressed statistics to the reference acc_p (D, K, R) layout. */
int einet_stats_expand_acc_p(einet_plan *plan, const double *stats, double *acc_p,
                             void *stream);

/* Materialise the forward buffer as log values: (B, num_buffer_rows, K) fp64
 * (ForwardTrace.buffer, engine.py:129) -- debugging / parity only. */
int einet_export_buffer(einet_plan *plan, const void *workspace, int64_t batch,
                        double *out, void *stream);

/* Leaf-region log densities (B, n_leaf, K) fp64 (expfam.leaf_forward) from a
 * completed forward pass in workspace. */
int einet_export_leaf_rows(einet_plan *plan, const void *workspace, int64_t batch,
                           double *out, void *stream);

/* Per-variable log-density tensor E (B, D, K, R) fp64 (expfam.ef_log_prob,
 * expfam.py:278-294); masked variables are exactly 0. */
int einet_ef_log_prob(einet_plan *plan, const double *params, const float *x,
                      int64_t batch, const uint8_t *marg_mask, double *out,
                      int32_t *status, void *stream);

/* Batched ancestral sampling (engine.py:331-423, sample / conditional_sample).
 * Writes n complete assignments to out (n, d_vars) fp64, deterministic in
 * seed: every decision of sample b uses a Philox4x32-10 uniform keyed by
 * (seed, b, decision site). conditional != 0: branch choices follow the
 * posterior of the forward pass of x_e held in `workspace` (einet_forward
 * with batch 1 and the evidence-marginalised compute), observed variables
 * (evidence[d] != 0) are copied from x_e. scratch: einet_sample_scratch_bytes
 * bytes. A sum node whose weights are all zero sets status word 3 (the slab)
 * -> EngineError. Replaces the per-sample Python descent _descend. */
int64_t einet_sample_scratch_bytes(const einet_plan *plan, int64_t n);
int einet_sample(einet_plan *plan, const double *params, const void *workspace,
                 int32_t conditional, const double *x_e, const uint8_t *evidence, int64_t n,
                 uint64_t seed, void *scratch, double *out, int32_t *status, void *stream);

/* Dataset payload decode (modelio.py:145-166, load_dataset): dst[i] =
 * (float)((double)src[i] / divisor) for count u8 values on the device
 * (divisor 255 = the reference's default normalisation of EIND1 u8 payloads,
 * 1 = raw counts). Lets callers ship image batches as bytes: the values are
 * bit-identical to the fp32 staging of the reference's float64 array. */
int einet_decode_u8(const uint8_t *src, int64_t count, double divisor, float *dst,
                    void *stream);

/* Host packing of a float64 batch for the device copy (host memory only, no
 * device call). The reference up-casts every batch to float64
 * (trainer.py:104) and its image datasets are v / 255 (modelio.py:145-166);
 * this writes the smallest exact form of the count values of x: *kind = 255
 * when every value is v / 255 for a byte v (bytes in u8_out; decode with
 * divisor 255), 1 when every value is a byte count v (bytes; divisor 1),
 * else 0 (fp32 values, round to nearest, in f32_out). Either way the fp32
 * values the engine sees equal the host cast of x. NaN, inf, negative zero
 * and off-grid values give kind 0; with f32_out NULL they give kind -1 and
 * nothing is converted (the caller allocates fp32 staging only for batches
 * that need it). threads <= 0: all host threads. */
int einet_pack_f64(const double *x, int64_t count, uint8_t *u8_out, float *f32_out,
                   int32_t threads, int32_t *kind);

/* EINM1 model files (modelio.py:55-134, save_model / load_model) on the
 * device. The host parses the magic, the JSON header and the tensor manifest;
 * the blob section (per tensor: u32 ndim, u32 dims, f64 payload) lives in
 * device memory.
 * einet_crc32: *crc (device) = zlib CRC32 of data[0, len) (the checksum that
 *   closes the file, modelio.py:83 / :100-102).
 * einet_params_from_blob: table (device, int64 [n_tensors][8] = blob offset
 *   of the tensor's u32 ndim, ndim, d0..d3, parameter offset (< 0: check
 *   only), element count)
 *   -> checks each embedded ndim/dims against the table and copies the
 *   payloads into params; *bad (device, caller-initialised to INT32_MAX) =
 *   the first tensor whose embedded shape differs or whose payload runs past
 *   blob_len (ShapeError, modelio.py:106-117). max_count = largest count.
 * einet_params_to_blob: the inverse (writes ndim, dims and payloads). */
int einet_crc32(const uint8_t *data, int64_t len, uint32_t *crc, void *stream);
int einet_params_from_blob(const uint8_t *blob, int64_t blob_len, const int64_t *table,
                           int32_t n_tensors, int64_t max_count, double *params, int32_t *bad,
                           void *stream);
int einet_params_to_blob(const double *params, const int64_t *table, int32_t n_tensors,
                         int64_t max_count, uint8_t *blob, void *stream);

/* Standalone EinsumLayer contraction (engine.log_einsum_exp, engine.py:91-109):
 * left/right (B, L, K) fp64, w (L, K_out, K, K) fp64 -> out (B, L, K_out). */
int einet_log_einsum_exp(const double *left, const double *right, const double *w,
                         int64_t batch, int32_t rows, int32_t k, int32_t k_out,
                         double *out, void *stream);

/* Diagnostic: D[128 x N] = A[128 x K] B[N x K]^T (fp32, row-major, device) on
 * one CTA with tcgen05 3xTF32 MMAs; validates the tensor-core plumbing.
 * Passing -N stages A in tensor memory (tcgen05.st) instead of shared memory. */
int einet_selftest_tf32_gemm(const float *A, const float *B, float *D, int32_t N, int32_t K,
                             void *stream);

/* Number of kernels this library has launched in this process. */
int64_t einet_launch_count(void);

/* Per-kernel-class CUDA-event timing of this library's launches (bench.py).
 * enable(1) clears and starts recording; query(i) returns class i's name,
 * summed device milliseconds and launch-group count (EINET_ERR_USAGE past the
 * last class). */
int einet_profile_enable(int on);
int einet_profile_query(int32_t index, char *name, int32_t name_len, double *total_ms,
                        int64_t *count);

/* Message of the last failing call on this thread (never NULL). */
const char *einet_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* EINET_B200_H */
