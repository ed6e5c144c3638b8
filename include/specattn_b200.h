/* specattn_b200.h — C ABI of the B200-native SpecAttn hot path (libspecattn_b200.so).
 *
 * Drop-in boundary for the reference's operator API (/root/reference/proj, namespace specattn):
 *
 *   reference (C++, Eigen, CPU)                                   this ABI (sm_100a, device-resident)
 *   ------------------------------------------------------------  ---------------------------------------
 *   KvStore::KvStore(ModelConfig)        kv_store.hpp:21          sa_cache_create
 *   KvStore::append(keys, values)        kv_store.hpp:33-36       sa_kv_append (n tokens at once)
 *   KvStore::truncate(to_len)            kv_store.hpp:38-40       sa_kv_truncate
 *   KvStore::set_committed(len)          kv_store.hpp:42          sa_kv_set_committed
 *   KvStore::gather(layer, head, idx)    kv_store.hpp:44-46       sa_kv_gather
 *   KvStore::keys()/values() views       kv_store.hpp:48-54       sa_kv_read
 *   KvStore::size()/committed()          kv_store.hpp:23-24       sa_kv_size / sa_kv_committed
 *   KvStore::bytes_per_token()           kv_store.hpp:30          sa_kv_bytes_per_token
 *   attend_collect(q, Kp, Vp, Kw, Vw, s) attention.hpp:63-67      sa_verify_attention (all q-heads x
 *     + LogitMatrix byproduct            attention.hpp:22-41        gamma+1 rows of one layer, fused
 *                                                                   append, fused score byproduct)
 *   score_columns + selection_k          selection.hpp:48-55      sa_select_topk (per layer or per
 *     + topk_indices + select_collect2   selection.hpp:61-69        KV head; Collect-2 / AllDraft rows)
 *     / select_all_draft
 *   KvStore::gather + attend(q, K, V, s) kv_store.hpp:44, attention.hpp:49-53
 *                                                                 sa_draft_attention (index gather fused
 *                                                                   with attention, fused append)
 *   SPEC decode_iteration (absent in code) SPEC.md:350-457        sa_iteration_run (verify -> select ->
 *                                                                   gamma drafts for all layers; CUDA graph)
 *
 * Conventions
 *  - Plain pointers and sizes; device pointers unless a parameter says "host".  Every
 *    device-side call takes a cudaStream_t (passed as void*; NULL = legacy default stream).
 *  - No exceptions cross the ABI.  sa_status mirrors the reference's exception taxonomy
 *    (SURVEY.md §8b): std::invalid_argument -> SA_INVALID_ARGUMENT, std::domain_error ->
 *    SA_DOMAIN_ERROR, std::out_of_range -> SA_OUT_OF_RANGE, std::length_error -> SA_LENGTH_ERROR.
 *    sa_last_error() returns the message of the last failure on the calling thread.
 *  - Device KV storage is bf16 (the reference stores fp32, config.hpp:40-42; bf16 is required to
 *    fit config 3 in one B200's HBM).  fp32 inputs are rounded to nearest-even bf16.
 *  - Threading (kv_store.hpp:16-18): one writer stream per cache; read-only calls may
 *    run on other streams after an event.
 *  - head_dim must be 128 (all BASELINE configs); page_size a power of two >= 128.
 */
#ifndef SPECATTN_B200_H_
#define SPECATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA_API __attribute__((visibility("default")))

typedef enum sa_status {
  SA_OK = 0,
  SA_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  SA_DOMAIN_ERROR = 2,     /* std::domain_error     */
  SA_OUT_OF_RANGE = 3,     /* std::out_of_range     */
  SA_LENGTH_ERROR = 4,     /* std::length_error     */
  SA_CUDA_ERROR = 5,
  SA_NOT_SUPPORTED = 6,
  SA_NCCL_ERROR = 7
} sa_status;

typedef enum sa_dtype { SA_F32 = 0, SA_BF16 = 1 } sa_dtype;

/* selection.hpp:15-22 — the logit-guided strategies on the hot path. */
typedef enum sa_strategy {
  SA_WINDOW = 0,          /* sink + sliding window, query-agnostic (baseline) selection.cpp:209-222 */
  SA_QUEST_LIKE = 1,      /* page min/max bounds vs the live query, re-selected before every draft
                             step (baseline)                                  selection.cpp:224-274 */
  SA_LAST_ACCEPTED = 2,   /* one row: a+1 (needs all rows' raw logits)        selection.cpp:198-207 */
  SA_ALL_DRAFT = 3,       /* all gamma+1 rows                                 selection.cpp:183-185 */
  SA_COLLECT2 = 4,        /* rows {1, gamma+1} (the paper's method)           selection.cpp:187-196 */
  SA_COLLECT2_WEIGHTS = 5 /* rows {1, gamma+1}, softmax-weights metric        selection.cpp:110-135 */
} sa_strategy;

/* Selection granularity.  SA_PER_LAYER is the reference contract (one set per layer shared by
 * all heads, scores averaged over ALL q-heads: selection.cpp:96); SA_PER_KV_HEAD
 * averages over the G q-heads of each KV head and selects per KV head (north star). */
typedef enum sa_select_mode { SA_PER_LAYER = 0, SA_PER_KV_HEAD = 1 } sa_select_mode;

typedef struct sa_cache sa_cache;   /* paged bf16 KV cache for up to max_seqs sequences */
typedef struct sa_runner sa_runner; /* workspaces + batch binding for the fused kernels  */

SA_API const char* sa_status_string(sa_status s);
SA_API const char* sa_last_error(void);
SA_API const char* sa_version(void);

/* ------------------------------------------------------------------------------------ cache */

typedef struct sa_cache_config {
  int64_t n_layers;    /* ModelConfig::n_layers   (kv_store.cpp:8-15 reads these four) */
  int64_t n_kv_heads;  /* ModelConfig::n_kv_heads */
  int64_t head_dim;    /* ModelConfig::head_dim (must be 128) */
  int64_t max_context; /* ModelConfig::max_context, per sequence */
  int64_t max_seqs;    /* sequences addressable by seq id 0..max_seqs-1 (reference: 1) */
  int64_t page_size;   /* tokens per page (power of two >= 128, sa_cache_create checks); 0 -> 256 */
  int64_t num_pages;   /* page pool size; 0 -> max_seqs * ceil(max_context / page_size) */
} sa_cache_config;

SA_API sa_status sa_cache_create(const sa_cache_config* cfg, sa_cache** out);
SA_API sa_status sa_cache_destroy(sa_cache* cache);
SA_API sa_status sa_kv_size(const sa_cache* cache, int32_t seq, int64_t* len);
SA_API sa_status sa_kv_committed(const sa_cache* cache, int32_t seq, int64_t* committed);
/* Reference accounting (fp32: 2*L*Hkv*d*4, kv_store.hpp:30) and the device (bf16) figure. */
SA_API sa_status sa_kv_bytes_per_token(const sa_cache* cache, int64_t* ref_fp32_bytes, int64_t* device_bytes);

/* Append n_tokens tokens (kv_store.cpp:29-49, batched).  keys/values: [n_tokens][n_layers*n_kv_heads]
 * [head_dim] in layer-major row order, dtype SA_F32 or SA_BF16, device or host memory
 * (keys_on_host != 0).  All-or-nothing: SA_LENGTH_ERROR if len + n_tokens > max_context. */
SA_API sa_status sa_kv_append(sa_cache* cache, int32_t seq, int64_t n_tokens, const void* keys,
                              const void* values, sa_dtype dtype, int keys_on_host, void* stream);
/* kv_store.cpp:51-58: SA_OUT_OF_RANGE if to_len > len; committed = min(committed, to_len). */
SA_API sa_status sa_kv_truncate(sa_cache* cache, int32_t seq, int64_t to_len);
/* kv_store.cpp:60-65 */
SA_API sa_status sa_kv_set_committed(sa_cache* cache, int32_t seq, int64_t len);
/* Pre-allocate pages so rows [0, len) are addressable by fused appends (no length change). */
SA_API sa_status sa_kv_reserve(sa_cache* cache, int32_t seq, int64_t len);
/* Set the length after device-side fused appends (verify/draft wrote rows [len, new_len)). */
SA_API sa_status sa_kv_set_size(sa_cache* cache, int32_t seq, int64_t new_len);
/* kv_store.cpp:67-88: host indices, strictly increasing and < len (SA_OUT_OF_RANGE otherwise);
 * K_out/V_out: device fp32 [n][head_dim]. */
SA_API sa_status sa_kv_gather(const sa_cache* cache, int32_t seq, int64_t layer, int64_t kv_head,
                              const int64_t* indices_host, int64_t n, float* K_out, float* V_out,
                              void* stream);
/* keys()/values() rows [begin, begin+n) as device fp32 [n][head_dim] (kv_store.hpp:48-54). */
SA_API sa_status sa_kv_read(const sa_cache* cache, int32_t seq, int64_t layer, int64_t kv_head,
                            int64_t begin, int64_t n, float* K_out, float* V_out, void* stream);

/* ----------------------------------------------------------------------------------- runner */

typedef struct sa_runner_config {
  int32_t max_batch;     /* sequences per call */
  int32_t n_q_heads;     /* Hq (multiple of n_kv_heads); G = Hq/Hkv */
  int32_t max_rows;      /* gamma+1 upper bound; G*max_rows + 2 <= 64 */
  int64_t max_prefix;    /* largest prefix length p0 a call will see */
  double sparse_ratio;   /* SelectorConfig::sparse_ratio (selection.hpp:31) */
  int64_t k_min;         /* SelectorConfig::k_min        (selection.hpp:32) */
  int32_t n_layers_buf;  /* score/index buffers kept per layer (iteration keeps all L) ; 0 -> L */
} sa_runner_config;

SA_API sa_status sa_runner_create(sa_cache* cache, const sa_runner_config* cfg, sa_runner** out);
SA_API sa_status sa_runner_destroy(sa_runner* r);
/* Bind a batch: seq_ids_host[n], prefix_len_host[n] (p0 = columns of the logit matrix; the
 * gamma+1 verify rows sit at p0..p0+gamma).  Reserves pages for p0 + max_rows. */
SA_API sa_status sa_runner_set_batch(sa_runner* r, int32_t n, const int32_t* seq_ids_host,
                                     const int64_t* prefix_len_host);
/* Per-layer device buffers owned by the runner (valid until destroy). */
SA_API float* sa_runner_scores(sa_runner* r, int32_t layer_slot, int64_t* ld);      /* [B][Hkv][ld] */
/* Per-layer score byproduct: int64 column sums in units of 2^-32 ([B][ld]); consumed (zeroed) by
 * sa_select_topk in SA_PER_LAYER mode. */
SA_API int64_t* sa_runner_layer_scores(sa_runner* r, int32_t layer_slot, int64_t* ld);
SA_API int32_t* sa_runner_indices(sa_runner* r, int32_t layer_slot, int32_t* k_cap); /* [B][sets][k_cap] */
SA_API int32_t* sa_runner_counts(sa_runner* r, int32_t layer_slot);                  /* [B][sets] */

/* Verify attention for one layer (attend_collect for every q-head x row):
 * row t = 1..n_rows of q-head h sees prefix [0,p0) and window [p0, p0+t).  Emits the Collect-k
 * score byproduct (raw q.k summed over the G heads of each KV head and the rows in
 * score_row_mask) into the runner's score buffer for layer_slot, fused with the attention pass. */
typedef struct sa_verify_args {
  int32_t layer;            /* cache layer */
  int32_t layer_slot;       /* runner score-buffer slot */
  int32_t n_rows;           /* gamma+1 */
  const void* q;            /* bf16 [B][Hq][n_rows][128] */
  const void* k_new;        /* bf16 [B][n_rows][Hkv][128] appended at p0.. (fused); NULL = in cache */
  const void* v_new;
  float scale;              /* 1/sqrt(d) (attention.hpp:51) */
  uint32_t score_row_mask;  /* bit r -> row r+1 contributes to the score (Collect-2: rows 1,gamma+1) */
  float* out;               /* f32 [B][Hq][n_rows][128] */
  float* logits;            /* optional raw prefix logits f32 [B][Hq][n_collect][ld_logits]; NULL = off */
  int64_t ld_logits;
  uint32_t collect_row_mask;/* rows whose raw logits go to `logits` (n_collect = popcount) */
  int32_t score_layout;     /* sa_select_mode the byproduct is laid out for: SA_PER_LAYER = one
                               fixed-point column sum per (sequence, column) over all KV heads
                               (sa_runner_layer_scores), SA_PER_KV_HEAD = fp32 per-head column
                               sums (sa_runner_scores).  sa_select_topk must use the same mode. */
} sa_verify_args;
SA_API sa_status sa_verify_attention(sa_runner* r, const sa_verify_args* a, void* stream);

/* Top-k selection from the score byproduct (score_columns + selection_k + topk_indices,
 * selection.cpp:89-108,63-66,137-158): k = clamp(llround(ratio*p0), k_min, p0) per sequence,
 * descending score, ties to the lower index, output ascending int32. */
typedef struct sa_select_args {
  int32_t layer_slot;
  sa_select_mode mode;
  int32_t rows_in_score;    /* popcount(score_row_mask) used by verify: divisor = heads*rows */
} sa_select_args;
SA_API sa_status sa_select_topk(sa_runner* r, const sa_select_args* a, void* stream);

/* Collect2Weights metric (score_columns_weights, selection.cpp:110-135): from the raw prefix logits
 * a verify wrote (sa_verify_args.logits, [B][Hq][n_rows][ld_logits] f32, rows = the collected score
 * rows), the softmax-weight column scores for layer_slot, laid out for `mode` (per-layer fixed-point
 * sums or per-KV-head fp32), ready for sa_select_topk with the same mode. */
SA_API sa_status sa_score_weights(sa_runner* r, int32_t layer_slot, const float* logits, int64_t ld_logits,
                                  int32_t n_rows, sa_select_mode mode, void* stream);

/* Baseline selectors of the paper (selection.cpp:209-274), writing the same per-layer index slot the
 * draft kernel reads.  QuestLike needs the cache's page summaries (kv_store.cpp:90-139, enabled once
 * with sa_kv_enable_page_summaries; refreshed lazily); q: bf16 [B][Hq][128], the query rows the
 * bounds are taken over (select_quest's q_heads).  Window: sink + sliding window. */
SA_API sa_status sa_kv_enable_page_summaries(sa_cache* cache, int64_t page_size);
SA_API sa_status sa_select_quest(sa_runner* r, int32_t layer, int32_t layer_slot, const void* q, void* stream);
SA_API sa_status sa_select_window(sa_runner* r, int32_t layer_slot, int64_t sink, int64_t window, void* stream);

/* Sparse draft attention for one layer (gather(T) ++ tail, then attend; kv_store.cpp:67-88,
 * attention.cpp:70-76): query of q-head h at position p0+step-1 attends to the
 * selected prefix T (layer_slot's index list; per-layer or per-KV-head) and the tail rows
 * [p0, p0+step).  If k_new/v_new are given they are row p0+step-1, appended (fused). */
typedef struct sa_draft_args {
  int32_t layer;
  int32_t layer_slot;
  sa_select_mode mode;
  int32_t step;             /* 1..gamma: tail length */
  const void* q;            /* bf16 [B][Hq][128] */
  const void* k_new;        /* bf16 [B][Hkv][128] or NULL */
  const void* v_new;
  float scale;
  float* out;               /* f32 [B][Hq][128] */
} sa_draft_args;
SA_API sa_status sa_draft_attention(sa_runner* r, const sa_draft_args* a, void* stream);

/* One speculation iteration of attention for all layers of the bound batch (SURVEY.md §8d unit):
 * per layer verify (+fused append of gamma+1 rows) -> select (side stream, overlapped with the
 * next layer's verify) ; then gamma draft steps, each over all layers in order (+fused append).
 * Inputs are per-layer contiguous blocks:
 *   qv  [L][B][Hq][gamma+1][128] bf16   kv_new/vv_new [L][B][gamma+1][Hkv][128] bf16
 *   qd  [gamma][L][B][Hq][128] bf16     kd_new/vd_new [gamma][L][B][Hkv][128] bf16
 *   out_v [L][B][Hq][gamma+1][128] f32   out_d [gamma][L][B][Hq][128] f32
 * use_graph != 0 captures the launch sequence into a CUDA graph on first use and replays it. */
typedef struct sa_iteration_args {
  int32_t gamma;
  sa_strategy strategy;     /* any sa_strategy: the logit-guided ones select from the verify byproduct;
                               SA_WINDOW selects once per iteration with the fixed baseline budget
                               sink 4 + window (k_cap - 4), k_cap = selection_k(ratio, max_prefix,
                               k_min); SA_QUEST_LIKE before every draft launch from that step's
                               query (the baselines; not with a KV-head group communicator) */
  sa_select_mode mode;
  float scale;
  const void *qv, *kv_new, *vv_new, *qd, *kd_new, *vd_new;
  float *out_v, *out_d;
  int32_t use_graph;
  uint32_t phases;          /* 0 = all; else a mask of SA_PHASE_* (timing breakdowns: the phases left
                               out are skipped, their buffers are left as the last run wrote them) */
  int32_t accepted;         /* a, 0 <= a <= gamma: the drafts the caller accepts from THIS iteration's
                               verify (sa_accept's result).  SA_LAST_ACCEPTED selects from row a+1
                               (selection.cpp:198-207).  The draft phase is the NEXT draft chain
                               (SPEC.md:382-385): its new rows go to p0+a+1, p0+a+2, ... after the
                               rows [y, x1..xa] the verify wrote, and every draft step's tail is
                               [p0, p0+a+1+step).  Commit with sa_kv_commit_accepted(seq, p0, a):
                               it keeps the verify's rows p0..p0+a (the draft rows beyond are
                               provisional, and the next verify rewrites them). */
} sa_iteration_args;
#define SA_PHASE_VERIFY 1u
#define SA_PHASE_SELECT 2u
#define SA_PHASE_DRAFT 4u
SA_API sa_status sa_iteration_run(sa_runner* r, const sa_iteration_args* a, void* stream);
/* Number of kernels one sa_iteration_run launches (for gpu_launches accounting). */
SA_API int64_t sa_iteration_kernel_count(const sa_runner* r, const sa_iteration_args* a);

/* Development hooks (not part of the reference surface; the product never reads the environment).
 * sa_dev_set_knob sets one dev-only tuning / tracing knob of a runner (internal.h DevConfig: e.g.
 * "verify_impl" 1 = the mma.sync baseline kernel, "iter_skip" phase bits, "trace" 1 = per-CTA
 * globaltimer traces); the defaults are the product settings.  Unknown names: SA_INVALID_ARGUMENT.
 * sa_dev_trace_dump writes the runner's verify + draft trace buffers to `path` after a device sync;
 * returns 0 on success, < 0 otherwise (e.g. tracing not enabled). */
SA_API sa_status sa_dev_set_knob(sa_runner* r, const char* name, int64_t value);
SA_API int sa_dev_trace_dump(sa_runner* r, const char* path);

/* ---------------------------------------------------------------- multi-GPU
 * The path's only collective: when a layer's KV heads are sharded over several GPUs (one process
 * per GPU) and selection is per layer, the per-layer fixed-point column sums are all-reduced over
 * the head group between verify and select (int64 sum: exact, order-independent).  NCCL is
 * loaded at run time (libnccl.so.2).  A group of one rank needs no NCCL. */
typedef struct sa_comm sa_comm;
/* 128-byte NCCL unique id, created on one rank and shared with the group out of band. */
SA_API sa_status sa_comm_unique_id(void* id_out_128);
SA_API sa_status sa_comm_create(const void* id_128, int32_t nranks, int32_t rank, sa_comm** out);
SA_API sa_status sa_comm_destroy(sa_comm* comm);
/* The communicator's size and this rank as NCCL reports them (ncclCommCount / ncclCommUserRank). */
SA_API sa_status sa_comm_info(const sa_comm* comm, int32_t* nranks, int32_t* rank);
/* NCCL asynchronous-error check (ncclCommGetAsyncError): on an error the communicator is aborted
 * (ncclCommAbort, so no kernel of this rank waits on a dead peer) and SA_NCCL_ERROR is returned;
 * every later exchange on it fails.  sa_iteration_run checks it after each launch. */
SA_API sa_status sa_comm_check(sa_comm* comm);
/* Wait for `stream` while watching the communicator: returns when the stream is idle, or aborts the
 * communicator and returns SA_NCCL_ERROR on an asynchronous error or after timeout_ms (< 0: none). */
SA_API sa_status sa_comm_sync(sa_comm* comm, void* stream, int64_t timeout_ms);
/* Attach the head-group communicator: sa_iteration_run then exchanges every layer's sums before
 * its select (per-layer mode).  NULL detaches. */
SA_API sa_status sa_runner_set_comm(sa_runner* r, sa_comm* comm);
/* Exchange one slot's per-layer sums on `stream` (direct-API use between verify and select). */
SA_API sa_status sa_exchange_layer_scores(sa_runner* r, int32_t layer_slot, void* stream);

/* ------------------------------------------------------- speculation glue (§8f)
 * Verification acceptance for B sequences (SPEC-only in the reference; oracle: oracle/speculation.py):
 * p: f32 [B][gamma+1][V] target distributions of the verify rows, q: f32 [B][gamma][V] draft
 * distributions (NULL when greedy), draft: int32 [B][gamma] draft tokens, u: f32 [B][gamma+1]
 * uniforms in [0,1) (u[t] for the accept test of draft t, u[gamma] for the residual / bonus sample;
 * NULL when greedy).  Sample: accept x_t iff u_t < min(1, p_t(x_t)/q_t(x_t)); on the first rejection
 * emit a sample of normalize(max(0, p_t - q_t)); if all accepted emit a bonus ~ p_{gamma+1}.  Greedy:
 * accept iff x_t = argmax p_t (ties to the lower id), trailing token argmax p_{a+1}.
 * Out (device): accepted [B], emitted [B][gamma+1] (accepted drafts, the trailing token, then -1). */
SA_API sa_status sa_accept(const float* p, const float* q, const int32_t* draft, const float* u, int32_t B,
                           int32_t gamma, int32_t V, int32_t greedy, int32_t* accepted, int32_t* emitted, void* stream);
/* Commit after acceptance (kv_store.cpp:51-65): the verify rows [p0, p0+accepted] (y and
 * the accepted drafts, written by sa_verify_attention's fused append) stay; the store's length and
 * committed mark become p0 + accepted + 1.  OUT_OF_RANGE if p0 is past the current length or the
 * kept rows were never reserved. */
SA_API sa_status sa_kv_commit_accepted(sa_cache* cache, int32_t seq, int64_t p0, int32_t accepted);

/* ------------------------------------------------------- model-side producer (§8f rank 4)
 * RMSNorm -> fused Q/K/V projection -> RoPE for the tokens of one layer, emitting exactly the bf16
 * q / k_new / v_new buffers sa_verify_attention (rows = gamma+1) and sa_draft_attention (rows = 1)
 * take.  Weights (device or host memory; repacked into a handle-owned copy at create, so the caller
 * may free them afterwards): w_qkv bf16
 * [n_layers][(Hq + 2 Hkv) * 128][d_model] = per layer the rows of wq^T, wk^T, wv^T (weights.hpp:21-23;
 * Eigen's column-major wq is already this layout), attn_norm_gain f32 [n_layers][d_model]
 * (weights.hpp:25).  norm_eps / rope_theta: config.hpp:32,34.  rope_style 0 = half-split pairs
 * (i, i+64), 1 = interleaved pairs (2j, 2j+1); both rotate pair j by pos * theta^(-2j/128). */
typedef struct sa_qkv sa_qkv;
SA_API sa_status sa_qkv_create(const void* w_qkv, const float* attn_norm_gain, int32_t n_layers, int32_t d_model,
                               int32_t n_q_heads, int32_t n_kv_heads, double norm_eps, double rope_theta,
                               int32_t rope_style, sa_qkv** out);
SA_API sa_status sa_qkv_destroy(sa_qkv* h);
/* Dev-only knobs of a projection ("trace" 1: per-CTA stamps, dumped to /tmp/sa_qkv_trace.bin by
 * sa_qkv_destroy; "dev": variant bits; "impl_tc" 1: the tcgen05 path for every token count). */
SA_API sa_status sa_qkv_dev_set_knob(sa_qkv* h, const char* name, int64_t value);
/* x: f32 [B][rows][d_model] hidden states (device); positions: int32 [B] (device) absolute position of
 * each sequence's row 0 (row r is at positions[b] + r); 1 <= B * rows <= 128.  Out (device, bf16):
 * q [B][Hq][rows][128], k_new / v_new [B][rows][Hkv][128].  Stream-ordered, graph-capturable. */
SA_API sa_status sa_qkv_project(sa_qkv* h, int32_t layer, const float* x, const int32_t* positions, int32_t B,
                                int32_t rows, void* q, void* k_new, void* v_new, void* stream);

/* Reference helper: selection_k (selection.cpp:63-66). */
SA_API int64_t sa_selection_k(double sparse_ratio, int64_t prefix_len, int64_t k_min);

#ifdef __cplusplus
}
#endif
#endif /* SPECATTN_B200_H_ */
