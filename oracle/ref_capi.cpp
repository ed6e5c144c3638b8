// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shims over the reference's OWN functions, compiled together with
// the unmodified /root/reference/proj/src/{attention,selection,kv_store}.cpp
// (against oracle/shim/Eigen) into oracle/_ref/libspecattn_ref.so by
// oracle/Makefile.  Used by tests/ to pin the C restatement and the golden
// vectors, and by bench.py --impl reference as the reference CPU arm.
//
// The *_layer functions are the SPEC callers' compositions (SURVEY.md §8a
// a17: SPEC.md:59-62,385,394,447) — harness code, not reference code — and may
// fan out over std::thread because the reference functions are pure and
// reentrant (SPEC.md:220,340; KvStore readers between mutations, :157).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "specattn/attention.hpp"
#include "specattn/kv_store.hpp"
#include "specattn/selection.hpp"

using specattn::RowMatrixXf;

namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::domain_error&) {
    return 2;
  } catch (const std::out_of_range&) {
    return 3;
  } catch (const std::length_error&) {
    return 4;
  } catch (...) {
    return 9;
  }
}

RowMatrixXf rows_of(const float* p, int64_t m, int64_t d) {
  RowMatrixXf M(m, d);
  if (m * d > 0) std::memcpy(M.data(), p, sizeof(float) * static_cast<size_t>(m * d));
  return M;
}

Eigen::VectorXf vec_of(const float* p, int64_t n) {
  Eigen::VectorXf v(n);
  if (n > 0) std::memcpy(v.data(), p, sizeof(float) * static_cast<size_t>(n));
  return v;
}

specattn::LogitMatrix logit_matrix(const float* L, int64_t H, int64_t R, int64_t C, const int* labels,
                                   int64_t head_dim, int64_t layer) {
  specattn::LogitMatrix M;
  M.layer = layer;
  M.head_dim = head_dim;
  for (int64_t h = 0; h < H; ++h) M.head_logits.push_back(rows_of(L + h * R * C, R, C));
  M.row_labels.assign(labels, labels + R);
  return M;
}

specattn::Strategy strategy_of(int s) {
  switch (s) {
    case 2: return specattn::Strategy::kLastAccepted;
    case 3: return specattn::Strategy::kAllDraft;
    case 4: return specattn::Strategy::kCollect2;
    case 5: return specattn::Strategy::kCollect2Weights;
    default: throw std::invalid_argument("strategy");
  }
}

template <typename F>
void parallel_for(int64_t n, int threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(static_cast<size_t>(threads));
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int64_t i = t; i < n; i += threads) f(i);
      } catch (...) {
        errs[static_cast<size_t>(t)] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

int ref_softmax_stable(const float* logits, int64_t n, double scale, double* out) {
  return guard([&] {
    Eigen::VectorXd p = specattn::softmax_stable(vec_of(logits, n), scale);
    for (int64_t i = 0; i < n; ++i) out[i] = p[i];
  });
}

int ref_attend(const float* q, const float* K, const float* V, int64_t m, int64_t d, float scale, float* out) {
  return guard([&] {
    Eigen::VectorXf o = specattn::attend(vec_of(q, d), rows_of(K, m, d), rows_of(V, m, d), scale);
    for (int64_t j = 0; j < d; ++j) out[j] = o[j];
  });
}

int ref_attend_collect(const float* q, const float* Kp, const float* Vp, int64_t m0, const float* Kw,
                       const float* Vw, int64_t m1, int64_t d, float scale, float* out, float* logits) {
  return guard([&] {
    auto r = specattn::attend_collect(vec_of(q, d), rows_of(Kp, m0, d), rows_of(Vp, m0, d), rows_of(Kw, m1, d),
                                      rows_of(Vw, m1, d), scale);
    for (int64_t j = 0; j < d; ++j) out[j] = r.output[j];
    for (int64_t i = 0; i < m0; ++i) logits[i] = r.prefix_logits[i];
  });
}

int64_t ref_selection_k(double ratio, int64_t p, int64_t k_min) { return specattn::selection_k(ratio, p, k_min); }

int ref_score_columns(const float* L, int64_t H, int64_t R, int64_t C, const int* labels, const int* sel,
                      int64_t n_sel, int weights, int64_t head_dim, double* out) {
  return guard([&] {
    auto M = logit_matrix(L, H, R, C, labels, head_dim, 0);
    std::span<const int> rows(sel, static_cast<size_t>(n_sel));
    Eigen::VectorXd s = weights ? specattn::score_columns_weights(M, rows) : specattn::score_columns(M, rows);
    for (int64_t i = 0; i < C; ++i) out[i] = s[i];
  });
}

int ref_topk_indices(const double* scores, int64_t n, int64_t k, int64_t* out, int64_t* n_out) {
  return guard([&] {
    Eigen::VectorXd s(n);
    for (int64_t i = 0; i < n; ++i) s[i] = scores[i];
    auto idx = specattn::topk_indices(s, k);
    for (size_t i = 0; i < idx.size(); ++i) out[i] = idx[i];
    *n_out = static_cast<int64_t>(idx.size());
  });
}

int ref_select(int strategy, const float* L, int64_t H, int64_t R, int64_t C, const int* labels, int64_t head_dim,
               double ratio, int64_t k_min, int accepted, int64_t* out, int64_t* n_out) {
  return guard([&] {
    auto M = logit_matrix(L, H, R, C, labels, head_dim, 0);
    specattn::SelectorConfig cfg;
    cfg.strategy = strategy_of(strategy);
    cfg.sparse_ratio = ratio;
    cfg.k_min = k_min;
    cfg.validate();
    specattn::SelectionSet set;
    if (cfg.strategy == specattn::Strategy::kCollect2 || cfg.strategy == specattn::Strategy::kCollect2Weights)
      set = specattn::select_collect2(M, cfg);
    else if (cfg.strategy == specattn::Strategy::kAllDraft)
      set = specattn::select_all_draft(M, cfg);
    else
      set = specattn::select_last_accepted(M, accepted, cfg);
    for (size_t i = 0; i < set.indices.size(); ++i) out[i] = set.indices[i];
    *n_out = set.k;
  });
}

// ---------------------------------------------------------------- KvStore

void* ref_kv_create(int64_t n_layers, int64_t n_kv_heads, int64_t head_dim, int64_t max_context) {
  specattn::ModelConfig cfg;
  cfg.n_layers = n_layers;
  cfg.n_kv_heads = n_kv_heads;
  cfg.head_dim = head_dim;
  cfg.max_context = max_context;
  return new specattn::KvStore(cfg);
}
void ref_kv_destroy(void* h) { delete static_cast<specattn::KvStore*>(h); }
int64_t ref_kv_size(void* h) { return static_cast<specattn::KvStore*>(h)->size(); }
int64_t ref_kv_committed(void* h) { return static_cast<specattn::KvStore*>(h)->committed(); }
int64_t ref_kv_bytes_per_token(void* h) { return static_cast<specattn::KvStore*>(h)->bytes_per_token(); }

int ref_kv_append(void* h, const float* keys, const float* values) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  const int64_t rows = kv->n_layers() * kv->n_kv_heads(), d = kv->head_dim();
  return guard([&] { kv->append(rows_of(keys, rows, d), rows_of(values, rows, d)); });
}
int ref_kv_truncate(void* h, int64_t to_len) {
  return guard([&] { static_cast<specattn::KvStore*>(h)->truncate(to_len); });
}
int ref_kv_set_committed(void* h, int64_t len) {
  return guard([&] { static_cast<specattn::KvStore*>(h)->set_committed(len); });
}
int ref_kv_gather(void* h, int64_t layer, int64_t head, const int64_t* idx, int64_t n, float* K, float* V) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  return guard([&] {
    auto kvp = kv->gather(layer, head, std::span<const int64_t>(idx, static_cast<size_t>(n)));
    const int64_t d = kv->head_dim();
    if (n > 0) {
      std::memcpy(K, kvp.first.data(), sizeof(float) * static_cast<size_t>(n * d));
      std::memcpy(V, kvp.second.data(), sizeof(float) * static_cast<size_t>(n * d));
    }
  });
}
int ref_kv_rows(void* h, int64_t layer, int64_t head, int64_t begin, int64_t n, float* K, float* V) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  return guard([&] {
    auto Ks = kv->keys(layer, head);
    auto Vs = kv->values(layer, head);
    if (begin < 0 || begin + n > Ks.rows()) throw std::out_of_range("rows");
    for (int64_t r = 0; r < n; ++r)
      for (int64_t j = 0; j < kv->head_dim(); ++j) {
        K[r * kv->head_dim() + j] = Ks(begin + r, j);
        V[r * kv->head_dim() + j] = Vs(begin + r, j);
      }
  });
}

// Quest page summaries and the baseline selectors (kv_store.cpp:90-139, selection.cpp:209-274).
int ref_kv_enable_page_summaries(void* h, int64_t page_size) {
  return guard([&] { static_cast<specattn::KvStore*>(h)->enable_page_summaries(page_size); });
}
// mins/maxs: [n_pages][d] (n_pages = ceil(size / page_size))
int ref_kv_page_minmax(void* h, int64_t layer, int64_t head, float* mins, float* maxs, int64_t* n_pages) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  return guard([&] {
    auto mn = kv->page_min(layer, head);
    auto mx = kv->page_max(layer, head);
    *n_pages = mn.rows();
    for (int64_t r = 0; r < mn.rows(); ++r)
      for (int64_t j = 0; j < kv->head_dim(); ++j) {
        mins[r * kv->head_dim() + j] = mn(r, j);
        maxs[r * kv->head_dim() + j] = mx(r, j);
      }
  });
}
// q_heads: [Hq][d]; out: ascending positions (capacity prefix_len)
int ref_select_quest(void* h, const float* q_heads, int64_t Hq, int64_t layer, int64_t prefix_len, double ratio,
                     int64_t k_min, int64_t* out, int64_t* n_out) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  return guard([&] {
    specattn::SelectorConfig cfg;
    cfg.strategy = specattn::Strategy::kQuestLike;
    cfg.sparse_ratio = ratio;
    cfg.k_min = k_min;
    cfg.page_size = kv->page_size();
    const auto set = specattn::select_quest(rows_of(q_heads, Hq, kv->head_dim()), *kv, layer, prefix_len, cfg);
    *n_out = static_cast<int64_t>(set.indices.size());
    for (size_t i = 0; i < set.indices.size(); ++i) out[i] = set.indices[i];
  });
}
int ref_select_window(int64_t prefix_len, int64_t sink, int64_t window, int64_t* out, int64_t* n_out) {
  return guard([&] {
    specattn::SelectorConfig cfg;
    cfg.strategy = specattn::Strategy::kWindow;
    cfg.sink = sink;
    cfg.window = window;
    const auto set = specattn::select_window(prefix_len, cfg, 0);
    *n_out = static_cast<int64_t>(set.indices.size());
    for (size_t i = 0; i < set.indices.size(); ++i) out[i] = set.indices[i];
  });
}

// ---------------------------------------------------------------- caller compositions

// Verify, one layer: q-head h, row t in 1..R (query at p0+t-1) sees
// prefix keys(l,g).topRows(p0) and window rows [p0, p0+t).  q/out: [Hq][R][d];
// logits (nullable): [Hq][R][p0].
int ref_verify_layer(void* h, int64_t layer, int64_t n_q_heads, const float* q, int64_t p0, int64_t R, float scale,
                     float* out, float* logits, int threads) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  const int64_t d = kv->head_dim(), G = n_q_heads / kv->n_kv_heads();
  return guard([&] {
    if (p0 < 0 || p0 + R > kv->size()) throw std::out_of_range("verify window beyond store");
    parallel_for(n_q_heads * R, threads, [&](int64_t hr) {
      const int64_t hq = hr / R, r = hr % R, t = r + 1;
      auto Ks = kv->keys(layer, hq / G);
      auto Vs = kv->values(layer, hq / G);
      Eigen::VectorXf qv = vec_of(q + hr * d, d);
      auto res = specattn::attend_collect(qv, Ks.topRows(p0), Vs.topRows(p0), Ks.middleRows(p0, t),
                                          Vs.middleRows(p0, t), scale);
      for (int64_t j = 0; j < d; ++j) out[hr * d + j] = res.output[j];
      if (logits)
        for (int64_t i = 0; i < p0; ++i) logits[hr * p0 + i] = res.prefix_logits[i];
    });
  });
}

// Draft, one layer: kv head g attends to gather(T_g) ++ tail rows
// [tail_begin, tail_begin+tail_len).  idx: [n_sets][k_stride] (n_sets 1 = per-layer set shared
// by all heads, Hkv = per-KV-head).  q/out: [Hq][d].
int ref_draft_layer(void* h, int64_t layer, int64_t n_q_heads, const float* q, const int64_t* idx,
                    const int64_t* k, int64_t n_sets, int64_t k_stride, int64_t tail_begin, int64_t tail_len,
                    float scale, float* out, int threads) {
  auto* kv = static_cast<specattn::KvStore*>(h);
  const int64_t d = kv->head_dim(), Hkv = kv->n_kv_heads(), G = n_q_heads / Hkv;
  return guard([&] {
    parallel_for(Hkv, threads, [&](int64_t g) {
      const int64_t set = n_sets == 1 ? 0 : g;
      auto kvp = kv->gather(layer, g, std::span<const int64_t>(idx + set * k_stride, static_cast<size_t>(k[set])));
      auto tailK = kv->keys(layer, g).middleRows(tail_begin, tail_len);
      auto tailV = kv->values(layer, g).middleRows(tail_begin, tail_len);
      const int64_t m = k[set] + tail_len;
      RowMatrixXf K(m, d), V(m, d);
      for (int64_t r = 0; r < k[set]; ++r) {
        K.row(r) = kvp.first.row(r);
        V.row(r) = kvp.second.row(r);
      }
      for (int64_t r = 0; r < tail_len; ++r) {
        K.row(k[set] + r) = tailK.row(r);
        V.row(k[set] + r) = tailV.row(r);
      }
      for (int64_t hq = g * G; hq < (g + 1) * G; ++hq) {
        Eigen::VectorXf o = specattn::attend(vec_of(q + hq * d, d), K, V, scale);
        for (int64_t j = 0; j < d; ++j) out[hq * d + j] = o[j];
      }
    });
  });
}

}  // extern "C"
