/* specattn_oracle.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 * See specattn_oracle.h for the contract.  Build: oracle/Makefile (-O2 -ffp-contract=off). */
#include "specattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ attention */

/* attention.cpp:8-32: max over non-masked double(l)*scale; exp(double(l)*scale - max);
 * masked (-inf) entries get 0; probs /= sum. */
int so_softmax_stable(const float* logits, int64_t n, double scale, double* probs) {
  if (!(scale > 0.0)) return SO_INVALID_ARGUMENT; /* :9-11 */
  double max_scaled = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    const float l = logits[i];
    if (l == -INFINITY) continue;
    const double v = (double)l * scale;
    if (v > max_scaled) max_scaled = v; /* std::max(max_scaled, v) */
  }
  if (!isfinite(max_scaled)) return SO_DOMAIN_ERROR; /* :19-21 */
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const float l = logits[i];
    const double w = (l == -INFINITY) ? 0.0 : exp((double)l * scale - max_scaled);
    probs[i] = w;
    sum += w;
  }
  for (int64_t i = 0; i < n; ++i) probs[i] /= sum; /* :30 probs /= sum */
  return SO_OK;
}

static float dot_f(const float* a, const float* b, int64_t d) {
  float acc = 0.0f; /* Eigen float dot, index order (parity unpinned at the Eigen boundary) */
  for (int64_t j = 0; j < d; ++j) acc += a[j] * b[j];
  return acc;
}

/* attention.cpp:38-66 */
int so_attend_segments(const float* q, int64_t d, const float* K0, const float* V0, int64_t m0,
                       const float* K1, const float* V1, int64_t m1, float scale, float* out,
                       float* raw_prefix_logits) {
  const int64_t m = m0 + m1;
  if (m < 1) return SO_INVALID_ARGUMENT; /* :45-47 */
  float* logits = (float*)malloc((size_t)m * sizeof(float));
  double* w = (double*)malloc((size_t)m * sizeof(double));
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  if (!logits || !w || !acc) abort();
  for (int64_t i = 0; i < m0; ++i) logits[i] = dot_f(q, K0 + i * d, d);      /* :57 */
  for (int64_t i = 0; i < m1; ++i) logits[m0 + i] = dot_f(q, K1 + i * d, d); /* :58 */
  if (raw_prefix_logits) memcpy(raw_prefix_logits, logits, (size_t)m0 * sizeof(float)); /* :59 */
  int st = so_softmax_stable(logits, m, (double)scale, w); /* :61 */
  if (st == SO_OK) {
    for (int64_t i = 0; i < m0; ++i) /* :62 acc += w[i] * V0.row(i).cast<double>() */
      for (int64_t j = 0; j < d; ++j) acc[j] += w[i] * (double)V0[i * d + j];
    for (int64_t i = 0; i < m1; ++i) /* :63 */
      for (int64_t j = 0; j < d; ++j) acc[j] += w[m0 + i] * (double)V1[i * d + j];
    for (int64_t j = 0; j < d; ++j) out[j] = (float)acc[j]; /* :65 cast<float> */
  }
  free(logits);
  free(w);
  free(acc);
  return st;
}

/* attention.cpp:70-76 — empty first segment. */
int so_attend(const float* q, int64_t d, const float* K, const float* V, int64_t m, float scale,
              float* out) {
  return so_attend_segments(q, d, NULL, NULL, 0, K, V, m, scale, out, NULL);
}

/* attention.cpp:78-87 */
int so_attend_collect(const float* q, int64_t d, const float* Kp, const float* Vp, int64_t m0,
                      const float* Kw, const float* Vw, int64_t m1, float scale, float* out,
                      float* prefix_logits) {
  return so_attend_segments(q, d, Kp, Vp, m0, Kw, Vw, m1, scale, out, prefix_logits);
}

/* ------------------------------------------------------------------ selection */

/* selection.cpp:63-66 */
int64_t so_selection_k(double sparse_ratio, int64_t prefix_len, int64_t k_min) {
  const int64_t wanted = (int64_t)llround(sparse_ratio * (double)prefix_len);
  const int64_t lo = wanted > k_min ? wanted : k_min;
  return prefix_len < lo ? prefix_len : lo;
}

/* selection.cpp:70-85 (label -> row index); returns SO_INVALID_ARGUMENT on empty / absent. */
static int resolve_rows(const so_logit_matrix* L, const int* labels, int64_t n, int* rows) {
  if (n < 1) return SO_INVALID_ARGUMENT;
  for (int64_t i = 0; i < n; ++i) {
    int r = -1;
    for (int64_t j = 0; j < L->rows; ++j)
      if (L->row_labels[j] == labels[i]) { r = (int)j; break; } /* attention.hpp:35-40 */
    if (r < 0) return SO_INVALID_ARGUMENT;
    rows[i] = r;
  }
  return SO_OK;
}

#define LOGIT(L, h, r, c) ((L)->logits[((h) * (L)->rows + (r)) * (L)->cols + (c)])

/* selection.cpp:89-108: for each column, heads outer, rows inner, double sum over finite. */
int so_score_columns(const so_logit_matrix* L, const int* labels, int64_t n_labels, double* scores) {
  int* rows = (int*)malloc(sizeof(int) * (size_t)(n_labels > 0 ? n_labels : 1));
  int st = resolve_rows(L, labels, n_labels, rows);
  if (st == SO_OK) {
    for (int64_t i = 0; i < L->cols; ++i) {
      double sum = 0.0;
      int64_t count = 0;
      for (int64_t h = 0; h < L->n_heads; ++h)
        for (int64_t j = 0; j < n_labels; ++j) {
          const float l = LOGIT(L, h, rows[j], i);
          if (l == -INFINITY) continue;
          sum += (double)l;
          ++count;
        }
      scores[i] = count > 0 ? sum / (double)count : -INFINITY;
    }
  }
  free(rows);
  return st;
}

/* selection.cpp:110-135 */
int so_score_columns_weights(const so_logit_matrix* L, const int* labels, int64_t n_labels,
                             double* scores) {
  int* rows = (int*)malloc(sizeof(int) * (size_t)(n_labels > 0 ? n_labels : 1));
  int st = resolve_rows(L, labels, n_labels, rows);
  if (st == SO_OK && L->head_dim < 1) st = SO_INVALID_ARGUMENT; /* :115-117 */
  if (st != SO_OK) { free(rows); return st; }
  const int64_t C = L->cols;
  const double scale = 1.0 / sqrt((double)L->head_dim);
  double* sum = (double*)calloc((size_t)(C > 0 ? C : 1), sizeof(double));
  double* finite_count = (double*)calloc((size_t)(C > 0 ? C : 1), sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)(C > 0 ? C : 1));
  int64_t terms = 0;
  for (int64_t h = 0; h < L->n_heads && st == SO_OK; ++h)
    for (int64_t j = 0; j < n_labels; ++j) {
      const float* row = &LOGIT(L, h, rows[j], 0);
      st = so_softmax_stable(row, C, scale, w); /* :123 */
      if (st != SO_OK) break;
      for (int64_t i = 0; i < C; ++i) sum[i] += w[i];
      ++terms;
      for (int64_t i = 0; i < C; ++i)
        if (row[i] != -INFINITY) finite_count[i] += 1.0;
    }
  if (st == SO_OK)
    for (int64_t i = 0; i < C; ++i) {
      scores[i] = sum[i] / (double)terms;                     /* :130 */
      if (finite_count[i] == 0.0) scores[i] = -INFINITY;      /* :131-133 */
    }
  free(sum);
  free(finite_count);
  free(w);
  free(rows);
  return st;
}

static const double* g_sort_scores;
/* descending score, ties toward the lower index (selection.cpp:145-148) */
static int cmp_desc(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  const double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
  if (sa != sb) return sa > sb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib);
}
static int cmp_asc(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  return ia < ib ? -1 : (ia > ib);
}

/* selection.cpp:137-158 (the comparator is a strict total order on finite, non-NaN scores,
 * so qsort reproduces std::sort's result exactly). Not reentrant (static comparator state). */
int so_topk_indices(const double* scores, int64_t n, int64_t k, int64_t* out, int64_t* n_out) {
  if (k < 0 || k > n) return SO_INVALID_ARGUMENT; /* :139-141 */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  g_sort_scores = scores;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_desc);
  int64_t m = 0;
  for (int64_t i = 0; i < k; ++i) {
    const int64_t idx = order[i];
    if (scores[idx] == -INFINITY) break; /* :153 never select masked */
    out[m++] = idx;
  }
  qsort(out, (size_t)m, sizeof(int64_t), cmp_asc); /* :156 */
  *n_out = m;
  free(order);
  return SO_OK;
}

/* selection.cpp:162-207 */
int so_select(int strategy, const so_logit_matrix* L, double sparse_ratio, int64_t k_min,
              int accepted_count, int64_t* out, int64_t* n_out) {
  int labels[2];
  const int* use = labels;
  int64_t n_labels = 0;
  if (strategy == SO_ALL_DRAFT) { /* :183-185 all collected rows */
    use = L->row_labels;
    n_labels = L->rows;
  } else if (strategy == SO_COLLECT2 || strategy == SO_COLLECT2_WEIGHTS) { /* :187-196 */
    if (L->rows < 1) return SO_INVALID_ARGUMENT;
    int first = L->row_labels[0], last = L->row_labels[0];
    for (int64_t i = 1; i < L->rows; ++i) {
      if (L->row_labels[i] < first) first = L->row_labels[i];
      if (L->row_labels[i] > last) last = L->row_labels[i];
    }
    labels[n_labels++] = first;
    if (last != first) labels[n_labels++] = last;
  } else if (strategy == SO_LAST_ACCEPTED) { /* :198-207 */
    labels[n_labels++] = accepted_count + 1;
    int found = 0;
    for (int64_t i = 0; i < L->rows; ++i) found |= (L->row_labels[i] == labels[0]);
    if (!found) return SO_INVALID_ARGUMENT;
  } else {
    return SO_INVALID_ARGUMENT;
  }
  double* scores = (double*)malloc(sizeof(double) * (size_t)(L->cols > 0 ? L->cols : 1));
  /* score_by_metric :173-179: only the Collect2Weights strategy uses the weights metric */
  int st = (strategy == SO_COLLECT2_WEIGHTS) ? so_score_columns_weights(L, use, n_labels, scores)
                                             : so_score_columns(L, use, n_labels, scores);
  if (st == SO_OK) {
    const int64_t k = so_selection_k(sparse_ratio, L->cols, k_min); /* :166 */
    st = so_topk_indices(scores, L->cols, k, out, n_out);
  }
  free(scores);
  return st;
}

/* ------------------------------------------------------------------ kv store */

struct so_kv {
  int64_t n_layers, n_kv_heads, head_dim, max_context;
  int64_t len, committed, capacity;
  float** keys;   /* [n_layers*n_kv_heads] slabs, capacity x head_dim row-major */
  float** values;
};

so_kv* so_kv_create(int64_t n_layers, int64_t n_kv_heads, int64_t head_dim, int64_t max_context) {
  so_kv* kv = (so_kv*)calloc(1, sizeof(so_kv));
  kv->n_layers = n_layers;
  kv->n_kv_heads = n_kv_heads;
  kv->head_dim = head_dim;
  kv->max_context = max_context;
  const int64_t slabs = n_layers * n_kv_heads;
  kv->keys = (float**)calloc((size_t)(slabs > 0 ? slabs : 1), sizeof(float*));
  kv->values = (float**)calloc((size_t)(slabs > 0 ? slabs : 1), sizeof(float*));
  return kv;
}

void so_kv_destroy(so_kv* kv) {
  if (!kv) return;
  for (int64_t s = 0; s < kv->n_layers * kv->n_kv_heads; ++s) {
    free(kv->keys[s]);
    free(kv->values[s]);
  }
  free(kv->keys);
  free(kv->values);
  free(kv);
}

int64_t so_kv_size(const so_kv* kv) { return kv->len; }
int64_t so_kv_committed(const so_kv* kv) { return kv->committed; }

/* kv_store.cpp:17-27: doubling growth from 128, capped at max_context. */
static void ensure_capacity(so_kv* kv, int64_t rows) {
  if (rows <= kv->capacity) return;
  int64_t next = kv->capacity * 2 > 128 ? kv->capacity * 2 : 128;
  if (next < rows) next = rows;
  if (next > kv->max_context) next = kv->max_context;
  for (int64_t s = 0; s < kv->n_layers * kv->n_kv_heads; ++s) {
    kv->keys[s] = (float*)realloc(kv->keys[s], sizeof(float) * (size_t)(next * kv->head_dim));
    kv->values[s] = (float*)realloc(kv->values[s], sizeof(float) * (size_t)(next * kv->head_dim));
  }
  kv->capacity = next;
}

/* kv_store.cpp:29-49 */
int so_kv_append(so_kv* kv, const float* keys, const float* values) {
  if (kv->len >= kv->max_context) return SO_LENGTH_ERROR; /* :30-32 */
  ensure_capacity(kv, kv->len + 1);
  const int64_t d = kv->head_dim;
  for (int64_t s = 0; s < kv->n_layers * kv->n_kv_heads; ++s) { /* :39-45 row r = layer*Hkv+head */
    memcpy(kv->keys[s] + kv->len * d, keys + s * d, sizeof(float) * (size_t)d);
    memcpy(kv->values[s] + kv->len * d, values + s * d, sizeof(float) * (size_t)d);
  }
  ++kv->len;
  return SO_OK;
}

/* kv_store.cpp:51-58 */
int so_kv_truncate(so_kv* kv, int64_t to_len) {
  if (to_len < 0 || to_len > kv->len) return SO_OUT_OF_RANGE;
  kv->len = to_len;
  if (kv->committed > kv->len) kv->committed = kv->len;
  return SO_OK;
}

/* kv_store.cpp:60-65 */
int so_kv_set_committed(so_kv* kv, int64_t len) {
  if (len < 0 || len > kv->len) return SO_OUT_OF_RANGE;
  kv->committed = len;
  return SO_OK;
}

/* kv_store.cpp:67-88 */
int so_kv_gather(const so_kv* kv, int64_t layer, int64_t kv_head, const int64_t* idx, int64_t n,
                 float* K_out, float* V_out) {
  if (layer < 0 || layer >= kv->n_layers || kv_head < 0 || kv_head >= kv->n_kv_heads)
    return SO_OUT_OF_RANGE; /* :69-71 */
  int64_t prev = -1;
  for (int64_t i = 0; i < n; ++i) { /* :72-78 strictly increasing, in range */
    if (idx[i] <= prev || idx[i] >= kv->len) return SO_OUT_OF_RANGE;
    prev = idx[i];
  }
  const int64_t d = kv->head_dim, s = layer * kv->n_kv_heads + kv_head;
  for (int64_t r = 0; r < n; ++r) { /* :83-86 */
    memcpy(K_out + r * d, kv->keys[s] + idx[r] * d, sizeof(float) * (size_t)d);
    memcpy(V_out + r * d, kv->values[s] + idx[r] * d, sizeof(float) * (size_t)d);
  }
  return SO_OK;
}

const float* so_kv_keys(const so_kv* kv, int64_t layer, int64_t kv_head) {
  return kv->keys[layer * kv->n_kv_heads + kv_head];
}
const float* so_kv_values(const so_kv* kv, int64_t layer, int64_t kv_head) {
  return kv->values[layer * kv->n_kv_heads + kv_head];
}

/* ------------------------------------------------------------------ caller compositions */

int so_verify_layer(const so_kv* kv, int64_t layer, int64_t n_q_heads, const float* q, int64_t p0,
                    int64_t R, float scale, float* out, float* logits) {
  const int64_t d = kv->head_dim, G = n_q_heads / kv->n_kv_heads;
  if (p0 < 0 || p0 + R > kv->len) return SO_OUT_OF_RANGE;
  for (int64_t h = 0; h < n_q_heads; ++h) {
    const float* Ks = so_kv_keys(kv, layer, h / G);
    const float* Vs = so_kv_values(kv, layer, h / G);
    for (int64_t t = 1; t <= R; ++t) { /* row t: query at p0+t-1 sees prefix + window [p0,p0+t) */
      const int64_t r = t - 1;
      int st = so_attend_collect(q + (h * R + r) * d, d, Ks, Vs, p0, Ks + p0 * d, Vs + p0 * d, t,
                                 scale, out + (h * R + r) * d,
                                 logits ? logits + (h * R + r) * p0 : NULL);
      if (st != SO_OK) return st;
    }
  }
  return SO_OK;
}

int so_draft_layer(const so_kv* kv, int64_t layer, int64_t n_q_heads, const float* q,
                   const int64_t* idx, const int64_t* k, int64_t n_sets, int64_t k_stride,
                   int64_t tail_begin, int64_t tail_len, float scale, float* out) {
  const int64_t d = kv->head_dim, Hkv = kv->n_kv_heads, G = n_q_heads / Hkv;
  if (tail_begin < 0 || tail_begin + tail_len > kv->len) return SO_OUT_OF_RANGE;
  for (int64_t g = 0; g < Hkv; ++g) {
    const int64_t set = n_sets == 1 ? 0 : g;
    const int64_t kk = k[set], m = kk + tail_len;
    float* K = (float*)malloc(sizeof(float) * (size_t)((m > 0 ? m : 1) * d));
    float* V = (float*)malloc(sizeof(float) * (size_t)((m > 0 ? m : 1) * d));
    int st = so_kv_gather(kv, layer, g, idx + set * k_stride, kk, K, V);
    if (st == SO_OK) {
      memcpy(K + kk * d, so_kv_keys(kv, layer, g) + tail_begin * d, sizeof(float) * (size_t)(tail_len * d));
      memcpy(V + kk * d, so_kv_values(kv, layer, g) + tail_begin * d, sizeof(float) * (size_t)(tail_len * d));
      for (int64_t h = g * G; h < (g + 1) * G && st == SO_OK; ++h)
        st = so_attend(q + h * d, d, K, V, m, scale, out + h * d);
    }
    free(K);
    free(V);
    if (st != SO_OK) return st;
  }
  return SO_OK;
}

/* ------------------------------------------------------------------ rng (rng.hpp:17-62) */

#define SO_GOLDEN 0x9E3779B97F4A7C15ull
uint64_t so_rng_mix64(uint64_t z) { /* rng.hpp:53-58 */
  z += SO_GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t so_rng_seeded_key(uint64_t seed) { return so_rng_mix64(seed ^ 0x537065634174746Eull); }
uint64_t so_rng_derive_key(uint64_t key, uint64_t label) {
  return so_rng_mix64(key ^ so_rng_mix64(label + 0xA5A5A5A5DEADBEEFull));
}
uint64_t so_rng_at(uint64_t key, uint64_t i) { return so_rng_mix64(key + (i + 1) * SO_GOLDEN); }
void so_rng_normals(uint64_t key, int64_t n, double* out) { /* rng.hpp:37-45 Box-Muller */
  uint64_t c = 0;
  for (int64_t i = 0; i < n; ++i) {
    double u1 = (double)(so_rng_at(key, c++) >> 11) * 0x1.0p-53;
    double u2 = (double)(so_rng_at(key, c++) >> 11) * 0x1.0p-53;
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    out[i] = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
  }
}
