/* specattn_oracle.h — CPU restatement of the SpecAttn reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline — never as the product path.
 *
 * Plain C11 restatement of /root/reference/proj/src/{attention,selection,
 * kv_store}.cpp.  Every function cites the reference lines it follows.  The
 * arithmetic order mirrors the reference exactly (float dot in index order,
 * double softmax / value accumulation), and the build uses -ffp-contract=off
 * so it is bit-identical to the reference TUs compiled against
 * oracle/shim/Eigen (checked in tests/test_oracle.py).
 *
 * Status codes mirror the reference's exception taxonomy
 * (SURVEY.md §8b): 0 ok, 1 std::invalid_argument, 2 std::domain_error,
 * 3 std::out_of_range, 4 std::length_error.
 */
#ifndef SPECATTN_ORACLE_H_
#define SPECATTN_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SO_OK = 0, SO_INVALID_ARGUMENT = 1, SO_DOMAIN_ERROR = 2, SO_OUT_OF_RANGE = 3, SO_LENGTH_ERROR = 4 };

/* Strategy tags, selection.hpp:15-22 (logit-guided subset used on the path). */
enum { SO_LAST_ACCEPTED = 2, SO_ALL_DRAFT = 3, SO_COLLECT2 = 4, SO_COLLECT2_WEIGHTS = 5 };

/* attention.cpp:8-32 */
int so_softmax_stable(const float* logits, int64_t n, double scale, double* probs);

/* attention.cpp:38-66 — K0/V0 (m0 x d) then K1/V1 (m1 x d), row-major, contiguous rows. */
int so_attend_segments(const float* q, int64_t d, const float* K0, const float* V0, int64_t m0,
                       const float* K1, const float* V1, int64_t m1, float scale, float* out,
                       float* raw_prefix_logits /* nullable, m0 */);

/* attention.cpp:70-76 */
int so_attend(const float* q, int64_t d, const float* K, const float* V, int64_t m, float scale,
              float* out);

/* attention.cpp:78-87 */
int so_attend_collect(const float* q, int64_t d, const float* Kp, const float* Vp, int64_t m0,
                      const float* Kw, const float* Vw, int64_t m1, float scale, float* out,
                      float* prefix_logits);

/* selection.cpp:63-66 */
int64_t so_selection_k(double sparse_ratio, int64_t prefix_len, int64_t k_min);

/* LogitMatrix (attention.hpp:22-41) flattened: logits[h][r][c], n_heads x rows x cols,
 * row_labels[rows] (1-based t).  selection.cpp:70-85 resolves labels to rows. */
typedef struct so_logit_matrix {
  const float* logits;
  int64_t n_heads, rows, cols;
  const int* row_labels;
  int64_t head_dim;
  int64_t layer;
} so_logit_matrix;

/* selection.cpp:89-108 */
int so_score_columns(const so_logit_matrix* L, const int* labels, int64_t n_labels, double* scores);
/* selection.cpp:110-135 */
int so_score_columns_weights(const so_logit_matrix* L, const int* labels, int64_t n_labels,
                             double* scores);
/* selection.cpp:137-158 — out must hold k entries; *n_out = selected count. */
int so_topk_indices(const double* scores, int64_t n, int64_t k, int64_t* out, int64_t* n_out);

/* selection.cpp:162-207 — strategy in {SO_ALL_DRAFT, SO_COLLECT2, SO_COLLECT2_WEIGHTS,
 * SO_LAST_ACCEPTED}; out holds selection_k(...) entries. */
int so_select(int strategy, const so_logit_matrix* L, double sparse_ratio, int64_t k_min,
              int accepted_count, int64_t* out, int64_t* n_out);

/* KvStore (kv_store.hpp:19-89, kv_store.cpp:1-88): fp32 slabs per (layer, kv_head). */
typedef struct so_kv so_kv;
so_kv* so_kv_create(int64_t n_layers, int64_t n_kv_heads, int64_t head_dim, int64_t max_context);
void so_kv_destroy(so_kv* kv);
int64_t so_kv_size(const so_kv* kv);
int64_t so_kv_committed(const so_kv* kv);
/* kv_store.cpp:29-49: keys/values are (n_layers*n_kv_heads) x head_dim, layer-major rows. */
int so_kv_append(so_kv* kv, const float* keys, const float* values);
int so_kv_truncate(so_kv* kv, int64_t to_len);      /* kv_store.cpp:51-58 */
int so_kv_set_committed(so_kv* kv, int64_t len);    /* kv_store.cpp:60-65 */
/* kv_store.cpp:67-88 */
int so_kv_gather(const so_kv* kv, int64_t layer, int64_t kv_head, const int64_t* idx, int64_t n,
                 float* K_out, float* V_out);
/* Zero-copy views keys()/values() (kv_store.hpp:48-54): pointer to row 0 of the slab. */
const float* so_kv_keys(const so_kv* kv, int64_t layer, int64_t kv_head);
const float* so_kv_values(const so_kv* kv, int64_t layer, int64_t kv_head);

/* ---- Caller compositions (SPEC-only callers) ---- */

/* Verify for one layer: query head h (kv head h / G) row t (1..R, position p0+t-1) attends to
 * prefix rows [0,p0) and window rows [p0, p0+t) of the store.
 * q: [Hq][R][d]; out: [Hq][R][d]; logits (nullable): [Hq][R][p0] raw prefix logits. */
int so_verify_layer(const so_kv* kv, int64_t layer, int64_t n_q_heads, const float* q, int64_t p0,
                    int64_t R, float scale, float* out, float* logits);

/* Draft for one layer: kv head g attends to gather(T_g) ++ rows [tail_begin, tail_begin+tail_len)
 * (SPEC.md:385,447).  idx: [n_sets][k_stride] with counts k[n_sets]; n_sets == 1 shares one set
 * across heads (per-layer selection), n_sets == Hkv is per-KV-head. q/out: [Hq][d]. */
int so_draft_layer(const so_kv* kv, int64_t layer, int64_t n_q_heads, const float* q,
                   const int64_t* idx, const int64_t* k, int64_t n_sets, int64_t k_stride,
                   int64_t tail_begin, int64_t tail_len, float scale, float* out);

/* CounterRng (rng.hpp:17-62), used to generate the synthetic inputs. */
uint64_t so_rng_mix64(uint64_t z);
uint64_t so_rng_seeded_key(uint64_t seed);
uint64_t so_rng_derive_key(uint64_t key, uint64_t label);
uint64_t so_rng_at(uint64_t key, uint64_t i);
/* n standard normals from stream `key` starting at draw counter 0 (two uniforms each). */
void so_rng_normals(uint64_t key, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SPECATTN_ORACLE_H_ */
