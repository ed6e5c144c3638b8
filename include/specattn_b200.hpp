// specattn_b200.hpp — C++ host mirror of the reference operator API over the C ABI.
//
// Reference-shaped call sites (namespace specattn, /root/reference/proj/include/specattn/*.hpp)
// switch to these classes: same names, same argument meaning, same exception types:
//   std::invalid_argument (SA_INVALID_ARGUMENT), std::domain_error (SA_DOMAIN_ERROR),
//   std::out_of_range (SA_OUT_OF_RANGE), std::length_error (SA_LENGTH_ERROR),
//   std::runtime_error (CUDA / NCCL / not supported).
// Differences by design: storage is a paged bf16 pool on the device; attention and
// selection run batched over all heads of a layer (sa_verify_attention / sa_select_topk /
// sa_draft_attention) instead of one query per call; device pointers are raw `const void*`.
// Header-only; link with -lspecattn_b200 (paper_2602_07223_b200/lib) and the CUDA runtime.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "specattn_b200.h"

namespace specattn_b200 {

// Rethrow an sa_status as the reference's exception type (SURVEY.md §8b error taxonomy).
inline void check(sa_status st) {
  if (st == SA_OK) return;
  const std::string msg = std::string(sa_status_string(st)) + ": " + sa_last_error();
  switch (st) {
    case SA_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SA_DOMAIN_ERROR: throw std::domain_error(msg);
    case SA_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SA_LENGTH_ERROR: throw std::length_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// selection.hpp:48-49 / selection.cpp:63-66
// speculation::verify acceptance over device buffers; see sa_accept.
inline void accept(const float* p, const float* q, const int32_t* draft, const float* u, int32_t B, int32_t gamma,
                   int32_t V, bool greedy, int32_t* accepted, int32_t* emitted, void* stream = nullptr) {
  check(sa_accept(p, q, draft, u, B, gamma, V, greedy ? 1 : 0, accepted, emitted, stream));
}

inline int64_t selection_k(double sparse_ratio, int64_t prefix_len, int64_t k_min) {
  return sa_selection_k(sparse_ratio, prefix_len, k_min);
}

// The ModelConfig fields KvStore reads (kv_store.cpp:8-15) plus the device-pool shape.
struct ModelConfig {
  int64_t n_layers = 4, n_kv_heads = 2, head_dim = 128, max_context = 4096;
  int64_t max_seqs = 1, page_size = 256, num_pages = 0;
};

// specattn::KvStore (kv_store.hpp:19-89) over the paged device pool; `seq` selects the sequence
// (the reference store holds one).
class KvStore {
 public:
  explicit KvStore(const ModelConfig& cfg) : cfg_(cfg) {
    sa_cache_config c{cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.max_context,
                      cfg.max_seqs, cfg.page_size, cfg.num_pages};
    check(sa_cache_create(&c, &h_));
  }
  ~KvStore() { sa_cache_destroy(h_); }
  KvStore(const KvStore&) = delete;
  KvStore& operator=(const KvStore&) = delete;

  int64_t size(int32_t seq = 0) const {  // kv_store.hpp:23
    int64_t n = 0;
    check(sa_kv_size(h_, seq, &n));
    return n;
  }
  int64_t committed(int32_t seq = 0) const {  // kv_store.hpp:24
    int64_t n = 0;
    check(sa_kv_committed(h_, seq, &n));
    return n;
  }
  int64_t bytes_per_token() const {  // kv_store.hpp:30 (reference fp32 accounting)
    int64_t ref = 0, dev = 0;
    check(sa_kv_bytes_per_token(h_, &ref, &dev));
    return ref;
  }
  // kv_store.cpp:29-49: one token, keys/values row-major [(n_layers * n_kv_heads)][head_dim] fp32
  // in host memory; returns the new length.
  int64_t append(const float* keys, const float* values, int32_t seq = 0, cudaStream_t s = nullptr) {
    return append_n(1, keys, values, SA_F32, /*on_host=*/true, seq, s);
  }
  // n tokens at once, host or device memory, fp32 or bf16.
  int64_t append_n(int64_t n, const void* keys, const void* values, sa_dtype dt, bool on_host, int32_t seq = 0,
                   cudaStream_t s = nullptr) {
    check(sa_kv_append(h_, seq, n, keys, values, dt, on_host ? 1 : 0, s));
    return size(seq);
  }
  void truncate(int64_t to_len, int32_t seq = 0) { check(sa_kv_truncate(h_, seq, to_len)); }  // :51-58
  void set_committed(int64_t len, int32_t seq = 0) { check(sa_kv_set_committed(h_, seq, len)); }  // :60-65
  // keep verify rows [p0, p0+accepted], truncate to p0+accepted+1, commit.
  void commit_accepted(int64_t p0, int32_t accepted, int32_t seq = 0) {
    check(sa_kv_commit_accepted(h_, seq, p0, accepted));
  }
  // kv_store.cpp:67-88: strictly increasing indices -> (K, V) row-major fp32 copies (host).
  std::pair<std::vector<float>, std::vector<float>> gather(int64_t layer, int64_t kv_head,
                                                           const std::vector<int64_t>& indices,
                                                           int32_t seq = 0) const {
    const int64_t n = static_cast<int64_t>(indices.size());
    return read_device(n, [&](float* K, float* V) {
      check(sa_kv_gather(h_, seq, layer, kv_head, indices.data(), n, K, V, nullptr));
    });
  }
  // kv_store.hpp:48-54 keys()/values(): rows [0, size) as host fp32 copies.
  std::pair<std::vector<float>, std::vector<float>> keys_values(int64_t layer, int64_t kv_head,
                                                                int32_t seq = 0) const {
    const int64_t n = size(seq);
    return read_device(n, [&](float* K, float* V) { check(sa_kv_read(h_, seq, layer, kv_head, 0, n, K, V, nullptr)); });
  }
  sa_cache* handle() const { return h_; }
  const ModelConfig& config() const { return cfg_; }

 private:
  template <typename F>
  std::pair<std::vector<float>, std::vector<float>> read_device(int64_t n, F&& fill) const {
    std::vector<float> K(static_cast<size_t>(n * cfg_.head_dim)), V(K.size());
    if (n == 0) return {K, V};
    float* d = nullptr;
    if (cudaMalloc(&d, 2 * K.size() * sizeof(float)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
    try {
      fill(d, d + K.size());
      if (cudaMemcpy(K.data(), d, K.size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(V.data(), d + K.size(), V.size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy");
    } catch (...) {
      cudaFree(d);
      throw;
    }
    cudaFree(d);
    return {K, V};
  }
  ModelConfig cfg_;
  sa_cache* h_ = nullptr;
};

// SelectorConfig fields on this path (selection.hpp:30-38).
struct SelectorConfig {
  double sparse_ratio = 0.25;
  int64_t k_min = 16;
  sa_select_mode mode = SA_PER_LAYER;
};

// Batched verify / select / draft for one bound batch (attend_collect + select_collect2 /
// select_all_draft + gather/attend, all q-heads of a layer per call).
class Runner {
 public:
  Runner(KvStore& kv, int32_t n_q_heads, int32_t max_rows, int64_t max_prefix, int32_t max_batch = 1,
         SelectorConfig sel = {}, int32_t n_layers_buf = 0)
      : sel_(sel) {
    sa_runner_config c{max_batch, n_q_heads, max_rows, max_prefix, sel.sparse_ratio, sel.k_min, n_layers_buf};
    check(sa_runner_create(kv.handle(), &c, &h_));
  }
  ~Runner() { sa_runner_destroy(h_); }
  Runner(const Runner&) = delete;
  Runner& operator=(const Runner&) = delete;

  void set_batch(const std::vector<int32_t>& seq_ids, const std::vector<int64_t>& prefix_lens) {
    if (seq_ids.size() != prefix_lens.size()) throw std::invalid_argument("set_batch: size mismatch");
    check(sa_runner_set_batch(h_, static_cast<int32_t>(seq_ids.size()), seq_ids.data(), prefix_lens.data()));
  }
  // attend_collect for every q-head x verify row of `layer` (attention.cpp:78-87),
  // Collect-2 rows {1, gamma+1} by default (selection.cpp:187-196).
  void verify(int32_t layer, int32_t n_rows, const void* q, float* out, const void* k_new, const void* v_new,
              float scale, cudaStream_t s = nullptr, uint32_t score_row_mask = 0) {
    sa_verify_args a{};
    a.layer = layer;
    a.layer_slot = layer;
    a.n_rows = n_rows;
    a.q = q;
    a.k_new = k_new;
    a.v_new = v_new;
    a.scale = scale;
    a.score_row_mask = score_row_mask ? score_row_mask : (1u | (1u << (n_rows - 1)));
    a.out = out;
    a.score_layout = sel_.mode;
    check(sa_verify_attention(h_, &a, s));
  }
  // score_columns + selection_k + topk_indices (selection.cpp:89-108,63-66,137-158)
  void select(int32_t layer, int32_t rows_in_score = 2, cudaStream_t s = nullptr) {
    sa_select_args a{layer, sel_.mode, rows_in_score};
    check(sa_select_topk(h_, &a, s));
  }
  // gather(T) ++ tail, then attend (kv_store.cpp:67-88, attention.cpp:70-76)
  void draft(int32_t layer, int32_t step, const void* q, float* out, const void* k_new, const void* v_new,
             float scale, cudaStream_t s = nullptr) {
    sa_draft_args a{layer, layer, sel_.mode, step, q, k_new, v_new, scale, out};
    check(sa_draft_attention(h_, &a, s));
  }
  void iteration(const sa_iteration_args& a, cudaStream_t s = nullptr) { check(sa_iteration_run(h_, &a, s)); }
  sa_runner* handle() const { return h_; }

 private:
  SelectorConfig sel_;
  sa_runner* h_ = nullptr;
};

}  // namespace specattn_b200
