/*
 * vsp_gpu.h — C ABI of the B200-native (sm_100a) VS-prefill path.
 *
 * Drop-in for the reference's hot-path operator API (header-only C++, namespace vsp,
 * /root/reference/proj/include/vsprefill). Every entry point here replaces one reference
 * function, batched over heads and operating on caller-owned DEVICE buffers:
 *
 *   vsp_indexer_scores   <- vsp::indexer_forward          indexer.hpp:116-120 (+ :77-113)
 *   vsp_select           <- vsp::select_pattern           sparsity.hpp:105-114
 *                           (cumulative_budget :51-79, topk_indices :83-97,
 *                            inject_offset_zero :99-101)
 *   vsp_vs_attn_fwd      <- vsp::sparse_attention         attention.hpp:150-194
 *                           (merge_row_columns merge.hpp:18-56, fused on the fly)
 *   vsp_dense_attn_fwd   <- vsp::blockwise_attention      attention.hpp:96-145
 *   vsp_vs_aggregate     <- vsp::aggregate_streaming      vsaggregate.hpp:62-127
 *                           + vsp::combine_scores         vsaggregate.hpp:133-157
 *   vsp_recall_from_lse  <- vsp::attention_recall         attention.hpp:198-215
 *   vsp_apply_rope       <- vsp::apply_rope               rope.hpp:63-79 (Q and K, one pass)
 *   vsp_indexer_loss_grad <- vsp::indexer_backward_loss   indexer.hpp:158-272 (KL + backward)
 *   vsp_adamw_step       <- vsp::optimizer_step           indexer.hpp:347-363
 *   vsp_allgather_heads  (the only collective: head-sharded O assembly)
 *   vsp_{write,read}_tensor, vsp_{save,load}_checkpoint, vsp_{write,read}_indices
 *                        <- tensor_io.hpp:49-88, indexer.hpp:450-499, sparsity.hpp:187-245
 *
 * Layouts (all row-major, innermost last):
 *   Q [n, hq, d] bf16, K/V [n, hkv, d] bf16, O [n, hq, d] bf16, LSE [hq, n] fp32,
 *   scores A_v/A_s [hkv, n] fp32, index lists I_v/I_s [hkv, cap] int32 ascending with
 *   counts k_v/k_s [hkv] int32. Q head h uses KV head h / (hq / hkv) (GQA), and a KV
 *   head's pattern is shared by its Q heads (the reference models one KV group as one
 *   head). d must be 128 for the attention kernels.
 *
 * Semantics are the reference's: logit scale 1/sqrt(d) (attention.hpp:31); slash offset
 * o = i - j; offset 0 always injected into I_s; top-k ties to the lower index; output
 * index lists ascending; cumulative threshold with tau - 1e-12 slack.
 *
 * Errors: every call returns a vsp_status. VSP_EINVAL carries the reference's exception
 * text (e.g. "uncovered query row 0") in vsp_last_error() (thread-local). Calls are
 * stream-ordered and asynchronous unless a flag asks for validation. There is no CPU
 * fallback: without a sm_100 device every compute call returns VSP_ECUDA.
 *
 * Concurrency: calls on different streams may run concurrently as long as each in-flight
 * call has its own workspace (the attention kernels keep their work-queue counters there;
 * the dense kernel, which takes no workspace, rotates through 256 internal counters).
 */
#ifndef VSP_GPU_H
#define VSP_GPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VSP_API __attribute__((visibility("default")))
#else
#define VSP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    VSP_OK = 0,
    VSP_EINVAL = 1,   /* std::invalid_argument in the reference */
    VSP_ERUNTIME = 2, /* std::runtime_error */
    VSP_ECUDA = 3,
    VSP_ENCCL = 4
} vsp_status;

/* Slash mapping (reference indexer.hpp:22): 0 = Reverse (default), 1 = Identity. */
enum { VSP_SLASH_REVERSE = 0, VSP_SLASH_IDENTITY = 1 };
/* Group reduce (vsaggregate.hpp:131): 0 = Mean, 1 = Sum. */
enum { VSP_REDUCE_MEAN = 0, VSP_REDUCE_SUM = 1 };
/* vsp_vs_attn_fwd flags */
enum {
    VSP_VALIDATE = 1,     /* sync + check sortedness/range/coverage like the reference */
    VSP_O_HEAD_MAJOR = 2, /* write O head-major [hq, n, 128] (the reference's per-head n x d
                             matrices) instead of token-major [n, hq, 128]; a rank's heads are
                             then one contiguous slab, the in-place all-gather send buffer */
    VSP_DENSE_SWITCH = 4  /* opt-in (vsp_vs_attn_fwd, vsp_vs_prefill, vsp_vs_prefill_units): a
                             query block whose vertical-slash tiles would visit every causal
                             tile anyway runs unmasked causal attention (blockwise_attention's
                             rows) instead of the masked pattern — same tiles, no mask work, recall
                             1 on those rows. Off = the reference's sparse_attention exactly. */
};

/* Reference BudgetConfig (sparsity.hpp:22-36). max_budget < 0 means "no maximum". */
typedef struct {
    double tau_v;
    double tau_s;
    int64_t min_budget;
    int64_t max_budget;
} vsp_budget;

typedef struct vsp_ctx vsp_ctx;

VSP_API const char* vsp_last_error(void);
VSP_API const char* vsp_version(void);
/* Kernels this library has launched in this process so far (every launch site counts), so a
 * caller can attribute the device work of a region to libvsp_gpu.so. */
VSP_API long long vsp_kernel_launches(void);
/* Live timing of the attention (K3) launches made by the layer entry points
 * (vsp_vs_prefill, vsp_vs_prefill_host, vsp_vs_prefill_units): when enabled, every K3 launch
 * is bracketed by a CUDA event pair on the stream it runs on (at most 512 per read).
 * vsp_attn_timing(ctx, 1) enables and resets; vsp_attn_timing_read waits for the recorded
 * launches and returns their summed duration (ms) and count, then resets. */
VSP_API int vsp_attn_timing(vsp_ctx* ctx, int enable);
VSP_API int vsp_attn_timing_read(vsp_ctx* ctx, double* total_ms, int* launches);

VSP_API int vsp_create(vsp_ctx** ctx, int device);
VSP_API int vsp_destroy(vsp_ctx* ctx);

/* ---- the step before the path: RoPE feed ------------------------------------------
 * apply_rope (rope.hpp:63-79) on Q [n, hq, d] and K [n, hkv, d] bf16 in ONE HBM pass:
 * plane p of the vector at position t rotates by t * base^(-2p/d); positions null means
 * t = row index. Out-of-place or in place (q_out == q_in). hq or hkv may be 0 to rotate one
 * tensor. VSP_ROPE_INTERLEAVED pairs (2p, 2p+1) (the reference); VSP_ROPE_HALF_SPLIT pairs
 * (p, p + d/2) (HF LLaMA/Qwen checkpoints). Angles in fp64, rotation in fp32, bf16 out. */
enum { VSP_ROPE_INTERLEAVED = 0, VSP_ROPE_HALF_SPLIT = 1 };
VSP_API int vsp_apply_rope(vsp_ctx* ctx, const void* q_in, const void* k_in, void* q_out, void* k_out, int n,
                           int hq, int hkv, int d, const int64_t* positions, double base, int style, void* stream);

/* ---- K1: VSIndexer scoring -------------------------------------------------------
 * X_t = [K_t | V_t] (per KV head), Z = SiLU(X W_U + b_U), logit_v = Z w_v + b_v,
 * raw_s = Z w_s + b_s, logit_s[o] = raw_s[n-1-o] (Reverse) or raw_s[o] (Identity),
 * A_v = softmax(logit_v), A_s = softmax(logit_s) over all n.
 * w_u: bf16 [hkv, 2d, d_h] (rows 0..d-1 multiply K, d..2d-1 multiply V; indexer.hpp:119),
 * b_u/w_v/w_s: fp32 [hkv, d_h], b_v/b_s: fp32 [hkv]. logits_v/logits_s may be NULL. */
VSP_API size_t vsp_indexer_workspace_size(int n, int hkv, int d_h);
VSP_API int vsp_indexer_scores(vsp_ctx* ctx, const void* k, const void* v, int n, int hkv, int d, int d_h,
                       const void* w_u, const float* b_u, const float* w_v, const float* b_v,
                       const float* w_s, const float* b_s, int slash_mapping, float* a_v,
                       float* a_s, float* logits_v, float* logits_s, void* workspace,
                       void* stream);

/* ---- K2: adaptive cumulative-threshold top-k selection ---------------------------
 * budgets: HOST array [hkv]. Outputs I_v/I_s [hkv, cap] (cap >= n + 1), k_v/k_s [hkv].
 * Index sets are bit-exact with select_pattern on the same scores widened to f64.
 * flags & VSP_VALIDATE: sync and report the reference's score checks (sparsity.hpp:60-61). */
VSP_API size_t vsp_select_workspace_size(int n, int hkv);
VSP_API int vsp_select(vsp_ctx* ctx, const float* a_v, const float* a_s, int n, int hkv,
               const vsp_budget* budgets, int* i_v, int* k_v, int* i_s, int* k_s, int cap,
               void* workspace, int flags, void* stream);

/* ---- K3: fused vertical-slash sparse attention forward --------------------------- */
VSP_API size_t vsp_vs_attn_workspace_size(int n, int hkv, int cap);
VSP_API int vsp_vs_attn_fwd(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                    int hkv, int d, const int* i_v, const int* k_v, const int* i_s,
                    const int* k_s, int cap, float scale, void* o, float* lse, void* workspace,
                    int flags, void* stream);

/* Statistics of the last vsp_vs_attn_fwd on `workspace` (stream-ordered, synchronises):
 * tiles_out[0] = 128x128 KV tiles visited, summed over query blocks and KV heads,
 * tiles_out[1] = tiles the dense causal kernel visits for the same heads,
 * tiles_out[2 + g] = tiles of KV head g (tiles_out holds 2 + hkv entries). */
VSP_API int vsp_vs_attn_tile_stats(vsp_ctx* ctx, int n, int hkv, int cap, const void* workspace,
                                   int64_t* tiles_out, void* stream);

/* ---- distillation: the training half (indexer.hpp:138-434) ---------------------------
 * vsp_indexer_loss_grad = indexer_forward + kl_loss_grad (Forward KL, eps smoothing) +
 * indexer_backward_from_upstream for every KV head: per-head loss KL_v + KL_s into loss[hkv]
 * (device, may be null) and the gradient, flattened in the parameter layout
 *   W_U [hkv, 2d, d_h] | b_U [hkv, d_h] | w_v [hkv, d_h] | w_s [hkv, d_h] | b_v [hkv] | b_s [hkv]
 * The forward reads the bf16 copy of W_U; targets are K5's normalised aggregates.
 * vsp_adamw_step = optimizer_step (:347-363) over a flat fp32 parameter vector with the
 * learning rate of learning_rate (:322-329) supplied by the caller; it also refreshes a
 * bf16 shadow of the first shadow_count parameters (W_U) for the next forward. */
typedef struct {
    double lr;
    double beta1;
    double beta2;
    double adam_eps;
    double weight_decay;
} vsp_adamw;
VSP_API size_t vsp_indexer_grad_workspace_size(int n, int hkv, int d_h);
VSP_API int vsp_indexer_loss_grad(vsp_ctx* ctx, const void* k, const void* v, int n, int hkv, int d, int d_h,
                                  const void* w_u_bf16, const float* b_u, const float* w_v, const float* b_v,
                                  const float* w_s, const float* b_s, int slash_mapping, const float* target_v,
                                  const float* target_s, double kl_eps, float* loss, float* grads, void* workspace,
                                  void* stream);
VSP_API int vsp_adamw_step(vsp_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t count,
                           int64_t step_index, const vsp_adamw* cfg, void* shadow_bf16, int64_t shadow_count,
                           void* stream);

/* ---- the whole VS-prefill layer: K1 -> K2 -> K3 in one call ------------------------
 * Same results as vsp_indexer_scores + vsp_select + vsp_vs_attn_fwd on all heads. With
 * heads_per_chunk = 0 (automatic: one chunk) everything runs in order on `stream`; with
 * KV-head chunks of `heads_per_chunk` heads the scoring, selection and tile planning of
 * chunk c+1 run on a high-priority side stream while chunk c's attention runs on `stream`.
 * a_v/a_s, i_v/k_v/i_s/k_s are outputs (caller-owned, as in the
 * individual calls). Mirrors `vsprefill select` + `vsprefill attend` (tools/vsprefill.cpp
 * :154-185) on the device. */
VSP_API size_t vsp_vs_prefill_workspace_size(int n, int hkv, int d_h, int cap);
VSP_API int vsp_vs_prefill(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq, int hkv,
                           int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                           const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                           const vsp_budget* budgets, float* a_v, float* a_s, int* i_v, int* k_v, int* i_s,
                           int* k_s, int cap, void* o, float* lse, void* workspace, int heads_per_chunk,
                           int flags, void* stream);

/* ---- heads split without an all-gather: mirrored outputs ----------------------------
 * vsp_vs_prefill, and K3's epilogue also stores every O tile (TMA) and LSE row, at the same
 * offsets, into n_mirrors (<= 7) other buffers laid out like o / lse — in the KV-head split,
 * the other ranks' full-layer outputs mapped into this process with vsp_ipc_open (peer HBM
 * over NVLink/NVSwitch). Each rank then holds the assembled layer once every rank's call has
 * completed (a stream-ordered barrier, e.g. a 1-element NCCL all-reduce): the all-gather of
 * vsp_allgather_heads happens inside the attention kernel, overlapped with the math, instead
 * of after it. With n_mirrors = 0 it is vsp_vs_prefill. lse_mirrors must be given iff lse is.
 * Replaces: nothing in the reference (single-process, vsprefill.cpp:176-185); it is the
 * multi-GPU assembly of SURVEY.md §8e. */
VSP_API int vsp_vs_prefill_mirrored(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                                    int hkv, int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                                    const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                                    const vsp_budget* budgets, float* a_v, float* a_s, int* i_v, int* k_v, int* i_s,
                                    int* k_s, int cap, void* o, float* lse, void* workspace, int heads_per_chunk,
                                    int flags, int n_mirrors, void* const* o_mirrors, float* const* lse_mirrors,
                                    void* stream);
/* CUDA IPC for the mirrors: vsp_ipc_alloc allocates device memory on ctx's GPU and returns its
 * 64-byte handle; another process opens it with vsp_ipc_open (peer access enabled lazily);
 * vsp_ipc_close unmaps an opened handle, vsp_ipc_free releases an allocation. */
VSP_API int vsp_ipc_alloc(vsp_ctx* ctx, size_t bytes, void** ptr, unsigned char* handle);
VSP_API int vsp_ipc_open(vsp_ctx* ctx, const unsigned char* handle, void** ptr);
VSP_API int vsp_ipc_close(void* ptr);
VSP_API int vsp_ipc_free(void* ptr);

/* ---- balanced multi-GPU split (SURVEY.md §8e refinement) -----------------------------
 * Adaptive per-head budgets make KV heads unequal (one head can carry 40% of a layer's
 * tiles), so plain head sharding leaves ranks idle. A unit is one KV head g (with its Q
 * heads) on query blocks [qb_lo, qb_hi) of 128 rows; ranks take contiguous runs of units of
 * equal predicted cost (per-(head, block) tile counts from vsp_vs_attn_tile_counts on a
 * calibration prompt) and call vsp_vs_prefill_units with the full (replicated) Q/K/V: it
 * scores, selects and plans each distinct head of its units, then attends each unit. No
 * collective; units write disjoint (head, row) regions of O and LSE (head-major O with
 * VSP_O_HEAD_MAJOR). Same results as vsp_vs_prefill on the rows a unit covers. */
typedef struct {
    int32_t g;
    int32_t qb_lo;
    int32_t qb_hi;
} vsp_unit;
VSP_API int vsp_vs_attn_tile_counts(vsp_ctx* ctx, int n, int hkv, int cap, const void* workspace, int32_t* counts,
                                    void* stream);
VSP_API int vsp_vs_prefill_units(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq, int hkv,
                                 int d, int d_h, const void* w_u, const float* b_u, const float* w_v, const float* b_v,
                                 const float* w_s, const float* b_s, int slash_mapping, const vsp_budget* budgets,
                                 float* a_v, float* a_s, int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* o,
                                 float* lse, void* workspace, const vsp_unit* units, int nunits, int flags,
                                 void* stream);

/* ---- the layer from HOST buffers (the reference's own calling convention) ----------
 * The reference operators take and return host memory (std::vector; attention.hpp:150,
 * tools/vsprefill.cpp:154-185). This entry point does the same: Q/K/V are read from host
 * memory (pinned for asynchronous copies) and O [n, hq, 128] bf16, LSE [hq, n] (nullable)
 * and the per-head budgets k_v/k_s [hkv] (nullable) are written back to host memory. The
 * copies are pipelined with the compute on two copy engines. heads_per_chunk = 0
 * (automatic): K and V first (two contiguous copies; scoring needs all n rows), then Q in 16
 * query-row ranges; range r is attended as soon as its rows land and its O rows / LSE
 * columns return while later ranges are still in flight. heads_per_chunk > 0: per KV-head
 * chunk, chunk c's K/V/Q columns travel while chunk c-1 is scored and attended. workspace:
 * device memory of vsp_vs_prefill_host_workspace_size bytes
 * (it holds the device copies of the inputs and outputs). Stream-ordered on `stream`. */
VSP_API size_t vsp_vs_prefill_host_workspace_size(int n, int hq, int hkv, int d_h);
VSP_API int vsp_vs_prefill_host(vsp_ctx* ctx, const void* q_h, const void* k_h, const void* v_h, int n, int hq,
                                int hkv, int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                                const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                                const vsp_budget* budgets, void* o_h, float* lse_h, int* k_v_h, int* k_s_h,
                                void* workspace, int heads_per_chunk, void* stream);

/* ---- K4: dense causal attention forward (the speed-up denominator) ---------------- */
VSP_API int vsp_dense_attn_fwd(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                       int hkv, int d, float scale, void* o, float* lse, void* stream);

/* ---- K5: ground-truth vertical/slash aggregation ----------------------------------
 * A_v[g][j] = reduce_{h in group g} sum_i A_h[i,j] (/ n if normalized),
 * A_s[g][o] = reduce_{h in group g} sum_i A_h[i,i-o]. lse: [hq, n] from K4 (pass 1),
 * or NULL to compute it. */
VSP_API size_t vsp_aggregate_workspace_size(int n, int hq);
VSP_API int vsp_vs_aggregate(vsp_ctx* ctx, const void* q, const void* k, int n, int hq, int hkv, int d,
                     float scale, const float* lse, int reduce, int normalized, float* a_v,
                     float* a_s, void* workspace, void* stream);

/* ---- standalone selection/merge operators (not on the layer path) -----------------
 * merge.hpp:69-95 (host; the device row merge below uses the same search per thread):
 * balanced p-way cut points of the merge of ascending a[na] and b[nb], a-first ties;
 * cuts int64 [(p + 1), 2] = (a_idx, b_idx). p >= 1 ("merge_path_partition: p must be >= 1"). */
VSP_API int vsp_merge_path_partition(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                                     int64_t* cuts);
/* merge.hpp:18-56 on the device: the ascending duplicate-free column set of each query row
 * rows[0..count) (device int32) under one KV head's lists i_v[k_v], i_s[k_s] (device int32,
 * strictly ascending) -> out int32 [count, out_cap], out_len int32 [count]. One CTA per row,
 * split across its threads by merge path. flags & VSP_VALIDATE: sync and report the
 * reference's messages for unsorted lists (checked on every row, as the reference does) and
 * overflow of out_cap; without it such rows get out_len -1 (i_v) / -2 (i_s) / -3 (cap). */
VSP_API int vsp_merge_row_columns(vsp_ctx* ctx, const int* i_v, int k_v, const int* i_s, int k_s, const int* rows,
                                  int count, int* out, int* out_len, int out_cap, int flags, void* stream);
/* sparsity.hpp:83-97: indices of the k[r] largest entries of each row r of scores [rows, n]
 * (any fp32 values, -0.0 == 0.0; ties to the lower index; ascending) -> out int32 [rows, cap].
 * k is a HOST array, checked like the reference (1 <= k[r] <= n) and k[r] <= cap. */
VSP_API size_t vsp_topk_workspace_size(int rows);
VSP_API int vsp_topk_indices(vsp_ctx* ctx, const float* scores, int n, int rows, const int* k, int* out, int cap,
                             void* workspace, void* stream);
/* vsaggregate.hpp:133-157: group combine of per-head scores v_in/s_in [heads, n] fp32 into
 * v_out/s_out [n] fp32: mean (VSP_REDUCE_MEAN) or sum (VSP_REDUCE_SUM), f64 in head order. */
VSP_API int vsp_combine_scores(vsp_ctx* ctx, const float* v_in, const float* s_in, int heads, int n, int reduce,
                               float* v_out, float* s_out, void* stream);

/* ---- recall from LSE pairs: mean_i exp(lse_sparse - lse_dense) per Q head ---------- */
VSP_API int vsp_recall_from_lse(vsp_ctx* ctx, const float* lse_sparse, const float* lse_dense, int n,
                        int hq, float* recall_per_head, void* stream);

/* ---- multi-GPU output assembly --------------------------------------
 * KV heads shard across ranks with no collective on the data path. The only exchange is
 * assembling O: each rank writes its Q heads with VSP_O_HEAD_MAJOR into their slab of the
 * full head-major O [hq, n, d] (pass o = o_full + first_head * n * d), then
 * vsp_allgather_heads runs ONE in-place ncclAllGather over NVLink (plus one for LSE
 * [hq, n] when lse_full is non-null). Rank r owns heads [r*hq/world, (r+1)*hq/world).
 * NCCL is dlopen'ed on first use. The unique id (vsp_comm_id_bytes() bytes) is made on
 * one rank and shipped to the others by the caller (the reference has no transport). */
typedef struct vsp_comm vsp_comm;
VSP_API size_t vsp_comm_id_bytes(void);
VSP_API int vsp_comm_unique_id(uint8_t* id);
VSP_API int vsp_comm_init(vsp_comm** comm, int world, int rank, const uint8_t* id, int device);
VSP_API int vsp_comm_destroy(vsp_comm* comm);
VSP_API int vsp_allgather_heads(vsp_comm* comm, void* o_full, float* lse_full, int n, int hq, int d, void* stream);
/* Assembly of a (KV head, query-block) unit split (balanced / spread): units int32 [count, 4]
 * = (owner rank, KV head, first query block, end query block), 128-row blocks, the union of
 * all ranks' units; every rank passes the same list. In place on the head-major o_full
 * [hq, n, d] bf16 and lse_full [hq, n] fp32 (optional): one ncclBroadcast per (unit, Q head)
 * from its owner, in one NCCL group. */
VSP_API int vsp_assemble_units(vsp_comm* comm, void* o_full, float* lse_full, int n, int hq, int hkv, int d,
                               const int32_t* units, int count, void* stream);

/* ---- interchange formats (host files; no device work) ------------------------------
 * The reference's on-disk formats, so GPU outputs can be diffed against the reference CLI
 * pipeline and one checkpoint drives both paths. Errors carry the reference's message text;
 * std::runtime_error maps to VSP_ERUNTIME, std::invalid_argument to VSP_EINVAL.
 *
 * VSTN tensor (tensor_io.hpp:14-88): "VSTN", u32 version=1, u32 ndim, u64 dims[ndim],
 * little-endian f64 row-major payload. rank = 1 / 2 reproduce read_vector / read_tensor
 * (rank mismatch is an error with the reference text); rank <= 0 accepts any rank.
 * `count` must equal the product of the file's dims (query it with vsp_tensor_header). */
VSP_API int vsp_tensor_header(const char* path, int* ndim, uint64_t* dims, int max_dims);
VSP_API int vsp_read_tensor(const char* path, int rank, double* data, uint64_t count);
VSP_API int vsp_write_tensor(const char* path, int ndim, const uint64_t* dims, const double* data);

/* VSCK indexer checkpoint, one per KV head (indexer.hpp:450-499, save_checkpoint /
 * load_checkpoint): "VSCK", u32 version=1, u32 d, u32 d_h, then W_U [2d x d_h], b_U [d_h],
 * w_v [d_h], b_v, w_s [d_h], b_s as little-endian f64. */
VSP_API int vsp_checkpoint_header(const char* path, int* d, int* d_h);
VSP_API int vsp_load_checkpoint(const char* path, int d, int d_h, double* w_u, double* b_u, double* w_v,
                                double* b_v, double* w_s, double* b_s);
VSP_API int vsp_save_checkpoint(const char* path, int d, int d_h, const double* w_u, const double* b_u,
                                const double* w_v, double b_v, const double* w_s, double b_s);

/* "V: ..." / "S: ..." index text (sparsity.hpp:187-245, write_indices / read_indices): one line
 * per direction, ascending. vsp_read_indices fills up to `cap` entries per direction and
 * rejects unsorted, negative or malformed lines with the reference's messages. */
VSP_API int vsp_write_indices(const char* path, const int64_t* i_v, int64_t k_v, const int64_t* i_s,
                              int64_t k_s);
VSP_API int vsp_read_indices(const char* path, int64_t* i_v, int64_t* k_v, int64_t* i_s, int64_t* k_s,
                             int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* VSP_GPU_H */
