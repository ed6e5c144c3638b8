// internal.h — host-side structures shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/specattn_b200.h"
#include "common.cuh"

namespace sa {

// Thread-local error message set by every failing entry point.
sa_status fail(sa_status st, const std::string& msg);
sa_status cuda_fail(cudaError_t e, const char* where);
#define SA_CUDA_CHECK(expr)                                         \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) return ::sa::cuda_fail(_e, #expr);       \
  } while (0)

// Kernel function attributes (max dynamic smem, non-portable clusters) are per device: `mask` holds one
// bit per device ordinal on which they were set.  Setting them twice is harmless, so races are benign.
inline bool func_attrs_needed(std::atomic<uint64_t>& mask, int* dev_out) {
  int dev = 0;
  cudaGetDevice(&dev);
  *dev_out = dev;
  return dev >= 64 || !(mask.load(std::memory_order_relaxed) & (uint64_t{1} << dev));
}
inline void func_attrs_done(std::atomic<uint64_t>& mask, int dev) {
  if (dev < 64) mask.fetch_or(uint64_t{1} << dev, std::memory_order_relaxed);
}

bool encode_tensor_map(CUtensorMap* map, void* base, uint64_t rows, uint32_t box_rows, std::string* err);
// bf16 [rows][cols] row-major, box {64, box_rows}, SWIZZLE_128B
bool encode_tensor_map_2d(CUtensorMap* map, void* base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                          std::string* err);

}  // namespace sa

struct sa_cache {
  int64_t n_layers = 0, n_kv_heads = 0, head_dim = 0, max_context = 0, max_seqs = 0;
  int64_t page_size = 0, page_shift = 0, num_pages = 0, max_pages_per_seq = 0;
  __nv_bfloat16* k_pool = nullptr;
  __nv_bfloat16* v_pool = nullptr;
  int32_t* d_block_table = nullptr;          // [max_seqs][max_pages_per_seq]
  std::vector<int32_t> h_block_table;
  std::vector<int64_t> len, committed, pages_of_seq;
  std::vector<int32_t> free_pages;           // LIFO free list
  std::vector<int64_t> verified_end;         // p0 + n_rows of the last verify with a fused append (commit bound)
  CUtensorMap tmap_k{}, tmap_v{};            // 2-D [rows][128] bf16, box {64, 64}, SWIZZLE_128B
  CUtensorMap tmap_k128{}, tmap_v128{};      // same tensors, box {64, 128} (tcgen05 verify tiles)
  CUtensorMap tmap_kg{}, tmap_vg{};          // same tensors, box {64, 1}: draft row gathers (tile::gather4)
  // Quest page summaries (kv_store.cpp:90-139): per (layer, page, KV head, quest page) elementwise key
  // min / max, bf16 (exact: min/max of bf16 keys); summ_valid[seq]: tokens whose quest pages are current
  int64_t qpage = 0;
  __nv_bfloat16* qmin = nullptr;
  __nv_bfloat16* qmax = nullptr;
  std::vector<int64_t> summ_valid;
  void summaries_stale_from(int32_t seq, int64_t pos) {  // rows >= pos changed
    if (qpage > 0) summ_valid[seq] = std::min(summ_valid[seq], pos / qpage * qpage);
  }
  int device = 0;

  sa::CacheView view() const {
    sa::CacheView v;
    v.k = k_pool;
    v.v = v_pool;
    v.block_table = d_block_table;
    v.max_pages_per_seq = static_cast<int32_t>(max_pages_per_seq);
    v.num_pages = static_cast<int32_t>(num_pages);
    v.page_shift = static_cast<int32_t>(page_shift);
    v.n_kv_heads = static_cast<int32_t>(n_kv_heads);
    v.n_layers = static_cast<int32_t>(n_layers);
    v.max_context = static_cast<int32_t>(max_context);
    return v;
  }
  sa_status reserve(int32_t seq, int64_t rows);  // allocate pages for [0, rows)
};

namespace sa {

// Dev-only tuning / tracing knobs of one runner (sa_dev_set_knob).  The defaults ARE the product
// settings; nothing here is read from the environment.
struct DevConfig {
  int verify_impl = 0;          // 0: tcgen05 verify (product); 1: the mma.sync baseline kernel (verify.cu)
  int verify_chunk_tiles = 2;   // 128-token tiles per dynamically claimed chunk
  int verify_no_prefill = 0;    // do not fill the ring before griddepcontrol.wait
  int verify_static_first = 1;  // first chunk = split index (else every chunk claimed from the counter)
  int verify_mergers = 6;       // designated merger CTAs (splits 0..n-1) that split the merge's rows
  int verify_full_rows = 0;     // softmax over all N MMA columns instead of MR = roundup4(M)
  int verify_max_splits = 0;    // cap on CTAs per (sequence, KV head) unit (0: automatic)
  int verify_tail_tiles = 72;   // single-tile chunks at the end of the prefix (guided claiming)
  int verify_flush_tiles = 8;   // TMEM accumulation block (warpgroup tiles) folded into Oacc; 0: never
  int verify_flush_min_tiles = 24;  // fold only when a CTA streams more than this many prefix tiles
  int verify_row_split = 1;     // N >= 48: softmax warpgroups split every tile's rows instead of alternating tiles
  int draft_min_cs = 0;         // minimum CTAs per (sequence, KV head) unit (0: automatic)
  int draft_cs = 0;             // forced CTAs per unit (0: automatic)
  int draft_sub = 0;            // forced clusters per unit, two-level merge (0: automatic)
  int draft_stream = -1;        // forced streaming (1) / two-CTA-per-SM (0) mode (-1: automatic)
  int draft_cluster_policy = 1; // cudaClusterSchedulingPolicy: 1 spread (no two CTAs of a cluster share an SM)
  int draft_multi_rounds = 3;   // rounds allowed in the two-CTA-per-SM multi-round mode
  int draft_debug = 0;          // print the draft launch geometry to stderr
  int draft_no_pdl = 0;         // launch iteration drafts without programmatic dependent launch
  int iter_skip = -1;           // phase bits to skip in sa_iteration_run (-1: sa_iteration_args.phases)
  int select_batched = 0;       // one grid-z select launch for all layers after the verify chain
  int select_legacy = 0;        // select kernel: 0 automatic, 1 single-CTA, 2 cluster (dev)
  int stream_priority = 1;      // side stream lowest priority, capture stream highest
  int trace = 0;                // per-CTA globaltimer traces (sa_dev_trace_dump)
};

// ---- kernel launch parameter blocks (also used by the launchers in verify.cu / draft.cu / select.cu)

struct VerifyParams {
  CacheView cache;
  int layer, B, Hkv, G, R, M, MT, hi_row;
  const int32_t* seq_ids;
  const int32_t* p0;
  const __nv_bfloat16* q;
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  float scale_log2;
  uint32_t score_mask;
  float* out;
  float* scores;           // per-KV-head fp32 column sums [B][Hkv][ld] (SA_PER_KV_HEAD layout) or null
  long long* score_fx;     // per-layer fixed-point column sums [B][ld] (SA_PER_LAYER layout) or null
  int64_t ld_scores;
  float* logits;
  int64_t ld_logits;
  uint32_t collect_mask;
  int n_collect;
  int n_splits, chunk;
  float* part_o;   // [B*Hkv][n_splits][MT*16][128]
  float* part_ml;  // [B*Hkv][n_splits][MT*16][2]
  int n_mergers;   // CTAs (the last arrivals of a unit) that split the merge's rows
  int no_prefill;  // dev knob
  int static_first;  // first chunk = split index (else every chunk claimed from the counter)
  int* counters;   // [B*Hkv][4]: [0] arrivals, [1] go (all partials stored), [2] mergers done
  int* chunk_ctr;  // [B*Hkv] dynamic chunk claims (tcgen05 verify), re-armed by the merging CTA
  int* flags;      // [B*Hkv][8 mergers][128 splits]: partial published (tcgen05 verify), reset by the merger
  unsigned long long* trace;  // dev-only pipeline timestamps of CTA (0,0,0); null in production
  int use_pdl;  // programmatic dependent launch after the previous layer's verify (iteration graph)
  int chunk_tiles;  // 128-token tiles per dynamically claimed chunk
  int tail_tiles;   // the last tail_tiles tiles of the prefix are claimed as single-tile chunks
  int flush_tiles;  // TMEM accumulation block length in a warpgroup's tiles (0: never flush)
  int row_split;    // both softmax warpgroups on every tile, each on half of the rows
  int full_rows;    // dev: softmax over all N columns
};

struct DraftParams {
  CUtensorMap tmk, tmv;  // K / V cache rows for tile::gather4 (box {64, 1}, SWIZZLE_128B)
  CacheView cache;
  int layer, B, Hkv, G, step;
  const int32_t* seq_ids;
  const int32_t* p0;
  const __nv_bfloat16* q;
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  const int32_t* idx;
  const int32_t* k_act;
  int n_sets, k_cap;
  float scale_log2;
  float* out;
  int n_splits, chunk;  // n_splits: CTAs per cluster
  int n_sub;            // clusters per (sequence, KV head); > 1: two-level merge through part_o / part_ml
  float* part_o;        // [B*Hkv][n_sub][G*128]
  float* part_ml;       // [B*Hkv][n_sub][n_splits][8][2]
  int* counters;        // [B*Hkv][16] arrivals per output slice, re-armed by the combining CTA
  unsigned long long* trace;  // dev-only per-CTA phase timestamps; null in production
  int use_pdl;  // launch with programmatic stream serialization (iteration graph only)
  int stream;   // double-buffered multi-round chunks (one CTA per SM)
  int cluster_policy;  // cudaClusterSchedulingPolicy of the launch (1: spread a cluster's CTAs over SMs)
  int draft_off;  // this chain's new rows start at p0 + draft_off; the tail is [p0, p0 + draft_off + step)
};

struct SelectParams {
  int B, Hkv, n_sets;
  const int32_t* p0;
  const float* scores;     // per-KV-head fp32 sums (when score_fx is null)
  long long* score_fx;     // per-layer fixed-point sums, zeroed as consumed
  int64_t ld_scores;
  double count;  // (#q-heads in the set) * rows_in_score
  double ratio;
  int64_t k_min;
  int k_cap;
  uint32_t* keys;  // workspace [B][n_sets][ld_scores]
  int32_t* idx;    // [B][n_sets][k_cap]
  int32_t* k_out;  // [B][n_sets]
  int64_t zs_scores = 0, zs_fx = 0, zs_idx = 0, zs_cnt = 0;  // per-slot strides (batched launches)
  int64_t max_n = 0;  // largest p0 of the bound batch (kernel choice)
  int legacy = 0;     // kernel choice: 0 automatic, 1 single-CTA radix select, 2 cluster select (dev)
};

sa_status comm_allreduce_i64(sa_comm* c, long long* buf, size_t count, cudaStream_t s);
cudaError_t launch_quest_summarize(const CacheView& c, const __nv_bfloat16* qmin, const __nv_bfloat16* qmax, int qpage,
                                   int seq, int64_t tok_lo, int64_t len, cudaStream_t s);
cudaError_t launch_quest_select(const CacheView& c, const __nv_bfloat16* qmin, const __nv_bfloat16* qmax, int qpage,
                                int layer, const int32_t* seq_ids, const int32_t* p0, int B, int Hq, int G,
                                const __nv_bfloat16* q, double ratio, int64_t k_min, int k_cap, double* bounds,
                                int64_t max_qpages, int32_t* idx, int32_t* k_out, cudaStream_t s);
cudaError_t launch_window(const int32_t* p0, int B, int64_t sink, int64_t window, int k_cap, int32_t* idx,
                          int32_t* k_out, cudaStream_t s);
cudaError_t launch_accept(const float* p, const float* q, const int32_t* draft, const float* u, int B, int gamma, int V,
                          int greedy, int32_t* accepted, int32_t* emitted, cudaStream_t s);
constexpr int kWeightParts = 8;  // Collect2Weights row statistics: CTAs per logit row
cudaError_t launch_weights(const float* logits, int64_t ld, const int32_t* p0, int B, int Hq, int G, int n_rows,
                           double scale, float2* stats, int n_sets, long long* fx, float* scores, int64_t ld_scores,
                           int64_t max_p, cudaStream_t s);

cudaError_t launch_verify(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s);
cudaError_t launch_verify_tc(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s);
cudaError_t launch_draft(const DraftParams& p, cudaStream_t s);
int draft_max_splits();
int draft_round_rows();
int draft_max_active_clusters(int stream, int cs);
cudaError_t launch_select(const SelectParams& p, cudaStream_t s, int n_slots = 1);
int select_max_smem_keys();
size_t verify_smem_bytes(int MT);
int verify_tc_merge_capacity(int M);  // bytes of smem a merge may fill (tcgen05 verify, rows M)
int verify_max_ctas_per_sm(int MT);

}  // namespace sa
