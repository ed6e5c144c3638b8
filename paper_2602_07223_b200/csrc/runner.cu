// runner.cu — batch binding, workspaces, per-layer entry points and the iteration driver.
//
// The iteration driver is the GPU-side analogue of the SPEC decode_iteration (SPEC.md:409-417,
// absent from the reference code): per layer verify -> select, the select on a side stream so it
// overlaps the next layer's verify (it is consumed only by the next draft phase), then gamma
// dependent draft steps over all layers.  The whole launch sequence is captured once into a CUDA
// graph and replayed.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using sa::fail;

struct sa_runner {
  sa_cache* cache = nullptr;
  sa_runner_config cfg{};
  int Hq = 0, Hkv = 0, G = 0, n_slots = 0, num_sms = 148;
  // bound batch
  int B = 0;
  std::vector<int32_t> h_seq;
  std::vector<int64_t> h_p0;
  int64_t p_max = 0;
  int32_t* d_seq = nullptr;
  int32_t* d_p0 = nullptr;
  // selection buffers
  int64_t ld = 0;
  float* scores = nullptr;     // [slots][max_batch][Hkv][ld]   per-KV-head layout
  long long* score_fx = nullptr;  // [slots][max_batch][ld]    per-layer layout (fixed point)
  std::vector<char> fx_dirty;  // slot holds unconsumed per-layer sums (needs zeroing before reuse)
  std::vector<int> slot_layout;  // layout the slot's last verify wrote (-1: none)
  int k_cap = 0;
  int32_t* idx = nullptr;      // [slots][max_batch][Hkv][k_cap]
  int32_t* kcnt = nullptr;     // [slots][max_batch][Hkv]
  uint32_t* keys = nullptr;    // [max_batch][Hkv][ld]
  // split-KV workspaces
  int64_t v_units_cap = 0, d_units_cap = 0;
  float *v_po = nullptr, *v_pml = nullptr, *d_po = nullptr, *d_pml = nullptr;
  int *v_cnt = nullptr, *d_cnt = nullptr, *v_chunk = nullptr, *v_flags = nullptr;
  // streams / graph
  cudaStream_t side = nullptr;
  cudaStream_t capture = nullptr;  // graphs are captured here (the caller's stream may be legacy)
  std::vector<cudaEvent_t> ev_v, ev_s;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<std::pair<std::vector<char>, cudaGraphExec_t>> graphs;  // keyed by args + batch binding
  sa_comm* comm = nullptr;  // KV-head group communicator (per-layer score exchange), may be null
  // Collect2Weights: raw logits of the collected rows per slot ([max_batch][Hq][2][ld]), row stats
  std::vector<float*> wlogits;
  float2* wstats = nullptr;
  double* qbounds = nullptr;  // QuestLike page bounds [max_batch][max quest pages]
  sa::DevConfig dev;  // dev-only knobs (sa_dev_set_knob); defaults = product settings
  unsigned long long* vtrace = nullptr;  // dev traces (knob "trace"), null in production
  unsigned long long* dtrace = nullptr;
};

namespace {

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Pick the split count for `units` independent (sequence, KV head) units of `len` keys: minimise
// (waves x per-CTA keys) + a per-split merge cost, chunks a multiple of `gran`.
int choose_splits(int64_t units, int64_t len, int64_t gran, int64_t max_chunk, int64_t slots_per_wave,
                  int64_t max_ctas, int64_t max_splits, int* chunk_out) {
  len = std::max<int64_t>(len, 1);
  int best_n = 1;
  int64_t best_chunk = round_up(len, gran), best_cost = -1;
  for (int64_t n = 1; n <= max_splits; ++n) {
    int64_t chunk = round_up((len + n - 1) / n, gran);
    if (max_chunk && chunk > max_chunk) continue;
    const int64_t nn = (len + chunk - 1) / chunk;
    if (nn != n) continue;
    if (units * nn > max_ctas) break;
    const int64_t waves = (units * nn + slots_per_wave - 1) / slots_per_wave;
    const int64_t cost = waves * chunk + 2 * gran * nn / std::max<int64_t>(1, slots_per_wave / units);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_n = static_cast<int>(nn);
      best_chunk = chunk;
    }
  }
  *chunk_out = static_cast<int>(best_chunk);
  return best_n;
}

int mtiles_for(int G, int R) { return (G * R + 2 + 15) / 16; }

}  // namespace

// dev-only verify pipeline trace (knob "trace"): [1024] per-tile events of CTA 0, then per layer
// (mod 64) [1024 CTAs][8] = start, end, main-loop end, tiles | split << 32, last PV done,
// partial stored, arrival counted, merge inputs landed (globaltimer ns).
constexpr size_t kVTraceWords = 1024 + 64 * 16384;
// dev-only draft trace: [(step-1) mod 8][layer mod 64][512 CTAs][16 phases] globaltimer ns.
constexpr size_t kDTraceWords = static_cast<size_t>(8) * 64 * 512 * 16;

// (Re)create the runner's side / capture streams with the priorities of its dev config: the selection
// side stream at the lowest priority, the capture stream at the highest, so that when SMs free up the
// next layer's verify CTAs are scheduled ahead of the (off-critical-path) selects.
static cudaError_t make_streams(sa_runner* r) {
  if (r->side) cudaStreamDestroy(r->side);
  if (r->capture) cudaStreamDestroy(r->capture);
  r->side = r->capture = nullptr;
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const bool prio = r->dev.stream_priority != 0;
  cudaError_t e = cudaStreamCreateWithPriority(&r->side, cudaStreamNonBlocking, prio ? least : 0);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&r->capture, cudaStreamNonBlocking, prio ? greatest : 0);
  return e;
}

extern "C" {

SA_API sa_status sa_runner_create(sa_cache* cache, const sa_runner_config* cfg, sa_runner** out) {
  if (!cache || !cfg || !out) return fail(SA_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (cfg->n_q_heads < 1 || cfg->n_q_heads % cache->n_kv_heads)
    return fail(SA_INVALID_ARGUMENT, "n_q_heads must be a positive multiple of n_kv_heads");
  const int G = cfg->n_q_heads / static_cast<int>(cache->n_kv_heads);
  if (G > 8) return fail(SA_NOT_SUPPORTED, "GQA group size > 8 (draft kernel n8 tile)");
  if (cfg->max_rows < 1 || mtiles_for(G, cfg->max_rows) > 4)
    return fail(SA_NOT_SUPPORTED, "G*(gamma+1)+2 must be <= 64");
  if (cfg->max_batch < 1 || cfg->max_batch > cache->max_seqs) return fail(SA_INVALID_ARGUMENT, "max_batch");
  if (cfg->max_prefix < 0 || cfg->max_prefix + cfg->max_rows > cache->max_context)
    return fail(SA_LENGTH_ERROR, "max_prefix + max_rows exceeds max_context");
  if (!(cfg->sparse_ratio > 0.0) || cfg->sparse_ratio > 1.0)
    return fail(SA_INVALID_ARGUMENT, "SelectorConfig: sparse_ratio must be in (0, 1]");  // selection.cpp:50-53
  if (cfg->k_min < 0) return fail(SA_INVALID_ARGUMENT, "SelectorConfig: k_min must be >= 0");
  auto* r = new sa_runner();
  r->cache = cache;
  r->cfg = *cfg;
  r->Hkv = static_cast<int>(cache->n_kv_heads);
  r->Hq = cfg->n_q_heads;
  r->G = G;
  r->n_slots = cfg->n_layers_buf > 0 ? cfg->n_layers_buf : static_cast<int>(cache->n_layers);
  cudaDeviceGetAttribute(&r->num_sms, cudaDevAttrMultiProcessorCount, cache->device);
  r->ld = std::max<int64_t>(64, round_up(cfg->max_prefix, 64));
  r->k_cap = static_cast<int>(std::max<int64_t>(1, sa_selection_k(cfg->sparse_ratio, cfg->max_prefix, cfg->k_min)));
  const int64_t mb = cfg->max_batch, H = r->Hkv, S = r->n_slots;
  r->v_units_cap = std::max<int64_t>(8 * r->num_sms, mb * H);  // verify partial slots (multi-wave splits)
  r->d_units_cap = std::max<int64_t>(8 * r->num_sms, mb * H);
  cudaError_t e = cudaSuccess;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) e = cudaMemset(*p, 0, std::max<size_t>(bytes, 16));
  };
  alloc(reinterpret_cast<void**>(&r->d_seq), sizeof(int32_t) * mb);
  alloc(reinterpret_cast<void**>(&r->d_p0), sizeof(int32_t) * mb);
  alloc(reinterpret_cast<void**>(&r->scores), sizeof(float) * S * mb * H * r->ld);
  alloc(reinterpret_cast<void**>(&r->score_fx), sizeof(long long) * S * mb * r->ld);
  r->fx_dirty.assign(S, 0);
  r->slot_layout.assign(S, -1);
  alloc(reinterpret_cast<void**>(&r->idx), sizeof(int32_t) * S * mb * H * r->k_cap);
  alloc(reinterpret_cast<void**>(&r->kcnt), sizeof(int32_t) * S * mb * H);
  alloc(reinterpret_cast<void**>(&r->keys), sizeof(uint32_t) * mb * H * r->ld);
  // verify split workspaces x2: consecutive layers alternate (PDL-chained verify launches)
  alloc(reinterpret_cast<void**>(&r->v_po), 2 * sizeof(float) * r->v_units_cap * 64 * 128);
  alloc(reinterpret_cast<void**>(&r->v_pml), 2 * sizeof(float) * r->v_units_cap * 64 * 2);
  alloc(reinterpret_cast<void**>(&r->v_cnt), 2 * 4 * sizeof(int) * mb * H);
  alloc(reinterpret_cast<void**>(&r->v_chunk), 2 * sizeof(int) * mb * H);
  alloc(reinterpret_cast<void**>(&r->v_flags), 2 * sizeof(int) * mb * H * 8 * 128);  // [parity][unit][merger][split]
  alloc(reinterpret_cast<void**>(&r->d_po), sizeof(float) * r->d_units_cap * 16 * 128);
  alloc(reinterpret_cast<void**>(&r->d_pml), sizeof(float) * r->d_units_cap * 16 * 2);
  alloc(reinterpret_cast<void**>(&r->d_cnt), sizeof(int) * mb * H * sa::draft_max_splits());
  if (e == cudaSuccess) e = make_streams(r);
  r->ev_v.resize(S);
  r->ev_s.resize(S);
  for (int64_t i = 0; i < S && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&r->ev_v[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_s[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->ev_join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    sa_runner_destroy(r);
    return sa::cuda_fail(e, "sa_runner_create");
  }
  *out = r;
  return SA_OK;
}

SA_API sa_status sa_runner_destroy(sa_runner* r) {
  if (!r) return SA_OK;
  for (auto& kv : r->graphs) cudaGraphExecDestroy(kv.second);
  for (float* w : r->wlogits) cudaFree(w);
  cudaFree(r->wstats);
  cudaFree(r->qbounds);
  cudaFree(r->vtrace);
  cudaFree(r->dtrace);
  for (auto ev : r->ev_v) if (ev) cudaEventDestroy(ev);
  for (auto ev : r->ev_s) if (ev) cudaEventDestroy(ev);
  if (r->ev_fork) cudaEventDestroy(r->ev_fork);
  if (r->ev_join) cudaEventDestroy(r->ev_join);
  if (r->side) cudaStreamDestroy(r->side);
  if (r->capture) cudaStreamDestroy(r->capture);
  for (void* p : {static_cast<void*>(r->d_seq), static_cast<void*>(r->d_p0), static_cast<void*>(r->scores),
                  static_cast<void*>(r->idx), static_cast<void*>(r->score_fx), static_cast<void*>(r->kcnt), static_cast<void*>(r->keys),
                  static_cast<void*>(r->v_po), static_cast<void*>(r->v_pml), static_cast<void*>(r->v_cnt), static_cast<void*>(r->v_chunk),
                  static_cast<void*>(r->v_flags), static_cast<void*>(r->d_po), static_cast<void*>(r->d_pml), static_cast<void*>(r->d_cnt)})
    cudaFree(p);
  delete r;
  return SA_OK;
}

SA_API sa_status sa_runner_set_batch(sa_runner* r, int32_t n, const int32_t* seq_ids, const int64_t* p0) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  if (n < 1 || n > r->cfg.max_batch) return fail(SA_INVALID_ARGUMENT, "batch size out of range");
  std::vector<int32_t> s32(n), p32(n);
  int64_t pm = 0;
  for (int i = 0; i < n; ++i) {
    if (seq_ids[i] < 0 || seq_ids[i] >= r->cache->max_seqs) return fail(SA_OUT_OF_RANGE, "sequence id out of range");
    for (int j2 = 0; j2 < i; ++j2)
      if (seq_ids[j2] == seq_ids[i]) return fail(SA_INVALID_ARGUMENT, "duplicate sequence in batch");
    if (p0[i] < 0 || p0[i] > r->cfg.max_prefix) return fail(SA_OUT_OF_RANGE, "prefix length beyond runner max_prefix");
    if (p0[i] > r->cache->len[seq_ids[i]]) return fail(SA_OUT_OF_RANGE, "prefix beyond store length");
    if (sa_status st = r->cache->reserve(seq_ids[i], p0[i] + r->cfg.max_rows)) return st;
    s32[i] = seq_ids[i];
    p32[i] = static_cast<int32_t>(p0[i]);
    pm = std::max(pm, p0[i]);
  }
  SA_CUDA_CHECK(cudaMemcpy(r->d_seq, s32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  SA_CUDA_CHECK(cudaMemcpy(r->d_p0, p32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  r->B = n;
  r->h_seq.assign(seq_ids, seq_ids + n);
  r->h_p0.assign(p0, p0 + n);
  r->p_max = pm;
  return SA_OK;
}

SA_API float* sa_runner_scores(sa_runner* r, int32_t slot, int64_t* ld) {
  if (!r || slot < 0 || slot >= r->n_slots) return nullptr;
  if (ld) *ld = r->ld;
  return r->scores + static_cast<size_t>(slot) * r->cfg.max_batch * r->Hkv * r->ld;
}
SA_API int64_t* sa_runner_layer_scores(sa_runner* r, int32_t slot, int64_t* ld) {
  if (!r || slot < 0 || slot >= r->n_slots) return nullptr;
  if (ld) *ld = r->ld;
  return reinterpret_cast<int64_t*>(r->score_fx + static_cast<size_t>(slot) * r->cfg.max_batch * r->ld);
}
SA_API int32_t* sa_runner_indices(sa_runner* r, int32_t slot, int32_t* k_cap) {
  if (!r || slot < 0 || slot >= r->n_slots) return nullptr;
  if (k_cap) *k_cap = r->k_cap;
  return r->idx + static_cast<size_t>(slot) * r->cfg.max_batch * r->Hkv * r->k_cap;
}
SA_API int32_t* sa_runner_counts(sa_runner* r, int32_t slot) {
  if (!r || slot < 0 || slot >= r->n_slots) return nullptr;
  return r->kcnt + static_cast<size_t>(slot) * r->cfg.max_batch * r->Hkv;
}

static sa_status verify_impl(sa_runner* r, const sa_verify_args* a, cudaStream_t s, bool pdl = false,
                             bool in_iteration = false) {
  if (!a || !a->q || !a->out) return fail(SA_INVALID_ARGUMENT, "verify: null argument");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "verify: no batch bound");
  if (a->layer < 0 || a->layer >= r->cache->n_layers) return fail(SA_OUT_OF_RANGE, "verify: layer out of range");
  if (a->layer_slot < 0 || a->layer_slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "verify: layer_slot");
  if (a->n_rows < 1 || a->n_rows > r->cfg.max_rows) return fail(SA_INVALID_ARGUMENT, "verify: n_rows out of range");
  if (!(a->scale > 0.f)) return fail(SA_INVALID_ARGUMENT, "softmax_stable: scale must be positive");
  if ((a->k_new == nullptr) != (a->v_new == nullptr)) return fail(SA_INVALID_ARGUMENT, "verify: k_new/v_new");
  if (a->score_row_mask >> a->n_rows) return fail(SA_INVALID_ARGUMENT, "score_columns: row label not collected");
  if (r->cache->max_pages_per_seq > 1024)
    return fail(SA_NOT_SUPPORTED, "verify: more than 1024 pages per sequence (raise page_size)");
  if (a->score_layout != SA_PER_LAYER && a->score_layout != SA_PER_KV_HEAD)
    return fail(SA_INVALID_ARGUMENT, "verify: score_layout");
  if (a->logits && (a->collect_row_mask == 0 || (a->collect_row_mask >> a->n_rows) || a->ld_logits < r->p_max))
    return fail(SA_INVALID_ARGUMENT, "verify: logits collection arguments");
  if (!a->k_new)
    for (int i = 0; i < r->B; ++i)
      if (r->h_p0[i] + a->n_rows > r->cache->len[r->h_seq[i]])
        return fail(SA_OUT_OF_RANGE, "verify: window rows not in the store");
  sa::VerifyParams p{};
  p.cache = r->cache->view();
  p.layer = a->layer;
  p.B = r->B;
  p.Hkv = r->Hkv;
  p.G = r->G;
  p.R = a->n_rows;
  p.M = r->G * a->n_rows;
  p.MT = mtiles_for(r->G, a->n_rows);
  p.hi_row = std::max(p.M, 16 * (p.MT - 1));
  p.seq_ids = r->d_seq;
  p.p0 = r->d_p0;
  p.q = static_cast<const __nv_bfloat16*>(a->q);
  p.k_new = static_cast<const __nv_bfloat16*>(a->k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(a->v_new);
  p.scale_log2 = a->scale * sa::kLog2e;
  p.score_mask = a->score_row_mask;
  p.out = a->out;
  p.scores = nullptr;
  p.score_fx = nullptr;
  p.ld_scores = r->ld;
  if (a->score_row_mask) {
    if (a->score_layout == SA_PER_KV_HEAD) {
      p.scores = sa_runner_scores(r, a->layer_slot, &p.ld_scores);
    } else {
      p.score_fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, a->layer_slot, &p.ld_scores));
      if (r->fx_dirty[a->layer_slot] && !in_iteration)  // unconsumed sums of an earlier verify
        SA_CUDA_CHECK(cudaMemsetAsync(p.score_fx, 0, sizeof(long long) * r->cfg.max_batch * r->ld, s));
      r->fx_dirty[a->layer_slot] = 1;
    }
    r->slot_layout[a->layer_slot] = a->score_layout;
  }
  p.logits = a->logits;
  p.ld_logits = a->ld_logits;
  p.collect_mask = a->collect_row_mask;
  p.n_collect = __builtin_popcount(a->collect_row_mask);
  const int64_t units = static_cast<int64_t>(r->B) * r->Hkv;
  const int par = a->layer & 1;  // workspace parity
  const size_t po_stride = static_cast<size_t>(r->v_units_cap) * 64 * 128;
  const size_t pml_stride = static_cast<size_t>(r->v_units_cap) * 64 * 2;
  const size_t cnt_stride = static_cast<size_t>(r->cfg.max_batch) * r->Hkv;
  cudaError_t e;
  if (r->dev.verify_impl == 1) {  // dev: the mma.sync baseline kernel (verify.cu)
    p.n_splits = choose_splits(units, r->p_max, 64, 0, r->num_sms, r->v_units_cap, 128, &p.chunk);
    p.part_o = r->v_po;
    p.part_ml = r->v_pml;
    p.counters = r->v_cnt;
    e = sa::launch_verify(p, r->cache->tmap_k, r->cache->tmap_v, s);
  } else {
    // at most one CTA per SM over all units, a single wave (floor: a 149th CTA would run as a
    // second wave); dynamic chunk claiming balances inside a unit
    const sa::DevConfig& dv = r->dev;
    const int chunk_tiles = std::max(1, dv.verify_chunk_tiles);
    p.no_prefill = dv.verify_no_prefill ? 1 : 0;
    p.static_first = dv.verify_static_first;
    p.full_rows = dv.verify_full_rows ? 1 : 0;
    p.chunk_tiles = chunk_tiles;
    p.tail_tiles = std::max(0, dv.verify_tail_tiles);
    p.flush_tiles = std::max(0, dv.verify_flush_tiles);
    p.row_split = dv.verify_row_split ? 1 : 0;
    const int64_t n_chunks = std::max<int64_t>(1, (r->p_max / 128 + chunk_tiles - 1) / chunk_tiles);
    // split merge: the designated mergers (splits 0..n_mergers-1) normalise a slice of rows each; their
    // staged partial rows and the (m, l) table must fit the ring buffers
    const int n_mergers = std::max(1, std::min(8, dv.verify_mergers));
    const int rows_per = (p.M + n_mergers - 1) / n_mergers;
    const int fit = std::max(1, (sa::verify_tc_merge_capacity(p.M) - 128) / (rows_per * 512 + 64 * 8));
    // one wave of at most one CTA per SM when that keeps >= 90 % of the SMs busy; otherwise (e.g. 128
    // units on 148 SMs: 20 idle) the smallest split count whose waves fill >= 90 % of the SM slots —
    // the CTAs of a unit share its chunks, so a wave boundary inside a unit only shifts work
    int64_t ns = std::max<int64_t>(1, r->num_sms / units);
    if (units * ns * 10 < 9LL * r->num_sms)
      for (int64_t s2 = ns + 1; s2 <= 16; ++s2) {
        const int64_t ctas = units * s2, waves = (ctas + r->num_sms - 1) / r->num_sms;
        if (ctas * 10 >= 9LL * waves * r->num_sms) {
          ns = s2;
          break;
        }
      }
    p.n_splits = static_cast<int>(std::min<int64_t>({ns, n_chunks, 128, r->v_units_cap / units, fit}));
    if (dv.verify_max_splits > 0) p.n_splits = std::min(p.n_splits, dv.verify_max_splits);
    // accumulation-block folding only where a CTA's chain is long: the kernels that carry the fold
    // code run their softmax loop 0.6 us per layer slower (same-box A/B), and chains of <= 24 tiles
    // per CTA stay at ~6e-4 elementwise without it (tools/verify_precision.py)
    if ((r->p_max / 128 + p.n_splits - 1) / p.n_splits <= dv.verify_flush_min_tiles) p.flush_tiles = 0;
    p.n_mergers = n_mergers;
    p.chunk = 0;
    p.chunk_ctr = r->v_chunk + par * cnt_stride;
    p.part_o = r->v_po + par * po_stride;
    p.part_ml = r->v_pml + par * pml_stride;
    p.counters = r->v_cnt + par * cnt_stride * 4;
    p.flags = r->v_flags + par * cnt_stride * 8 * 128;
    p.use_pdl = pdl ? 1 : 0;
    p.trace = r->vtrace;
    e = sa::launch_verify_tc(p, r->cache->tmap_k128, r->cache->tmap_v128, s);
  }
  if (e != cudaSuccess) return sa::cuda_fail(e, "verify launch");
  if (a->k_new)  // the fused append wrote rows [p0, p0 + n_rows): sa_kv_commit_accepted may keep them
    for (int i = 0; i < r->B; ++i) r->cache->verified_end[r->h_seq[i]] = r->h_p0[i] + a->n_rows;
  return SA_OK;
}

static sa_status select_impl(sa_runner* r, const sa_select_args* a, cudaStream_t s, int n_slots = 1) {
  if (!a) return fail(SA_INVALID_ARGUMENT, "select: null argument");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "select: no batch bound");
  if (a->layer_slot < 0 || a->layer_slot + n_slots > r->n_slots) return fail(SA_OUT_OF_RANGE, "select: layer_slot");
  if (a->rows_in_score < 1) return fail(SA_INVALID_ARGUMENT, "score_columns: empty row subset");
  if (a->mode != SA_PER_LAYER && a->mode != SA_PER_KV_HEAD) return fail(SA_INVALID_ARGUMENT, "select: mode");
  for (int z = 0; z < n_slots; ++z)
    if (r->slot_layout[a->layer_slot + z] >= 0 && r->slot_layout[a->layer_slot + z] != a->mode)
      return fail(SA_INVALID_ARGUMENT, "select: mode differs from the score layout the verify wrote");
  sa::SelectParams p{};
  p.B = r->B;
  p.Hkv = r->Hkv;
  p.n_sets = a->mode == SA_PER_LAYER ? 1 : r->Hkv;
  p.p0 = r->d_p0;
  p.scores = sa_runner_scores(r, a->layer_slot, &p.ld_scores);
  p.score_fx = nullptr;
  if (a->mode == SA_PER_LAYER) {
    p.score_fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, a->layer_slot, nullptr));
    for (int z = 0; z < n_slots; ++z) r->fx_dirty[a->layer_slot + z] = 0;  // the kernel zeroes what it consumes
  }
  p.count = static_cast<double>(a->mode == SA_PER_LAYER ? r->Hq : r->G) * a->rows_in_score;
  p.ratio = r->cfg.sparse_ratio;
  p.k_min = r->cfg.k_min;
  p.k_cap = r->k_cap;
  p.keys = r->keys;
  p.idx = sa_runner_indices(r, a->layer_slot, nullptr);
  p.k_out = sa_runner_counts(r, a->layer_slot);
  // per-layer sets live at set 0 of each sequence's [Hkv] block; keep the stride = Hkv sets
  // by addressing with n_sets below (the kernel indexes [b][n_sets]); use a dense layout.
  // consecutive slots in one launch (grid z): per-slot strides of the score / index / count buffers
  p.zs_scores = static_cast<int64_t>(r->cfg.max_batch) * r->Hkv * r->ld;
  p.zs_fx = static_cast<int64_t>(r->cfg.max_batch) * r->ld;
  p.zs_idx = static_cast<int64_t>(r->cfg.max_batch) * r->Hkv * r->k_cap;
  p.zs_cnt = static_cast<int64_t>(r->cfg.max_batch) * r->Hkv;
  p.max_n = r->p_max;
  p.legacy = r->dev.select_legacy;
  cudaError_t e = sa::launch_select(p, s, n_slots);
  if (e != cudaSuccess) return sa::cuda_fail(e, "select launch");
  return SA_OK;
}

// draft_off: this chain's new rows start at p0 + draft_off (0 for the direct API; the iteration's next
// draft chain starts after the accepted verify rows, sa_iteration_args.accepted)
static sa_status draft_impl(sa_runner* r, const sa_draft_args* a, cudaStream_t s, bool pdl = false, int draft_off = 0) {
  if (!a || !a->q || !a->out) return fail(SA_INVALID_ARGUMENT, "draft: null argument");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "draft: no batch bound");
  if (a->layer < 0 || a->layer >= r->cache->n_layers) return fail(SA_OUT_OF_RANGE, "draft: layer out of range");
  if (a->layer_slot < 0 || a->layer_slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "draft: layer_slot");
  if (a->step < 1 || a->step > r->cfg.max_rows) return fail(SA_INVALID_ARGUMENT, "draft: step out of range");
  if (!(a->scale > 0.f)) return fail(SA_INVALID_ARGUMENT, "softmax_stable: scale must be positive");
  if ((a->k_new == nullptr) != (a->v_new == nullptr)) return fail(SA_INVALID_ARGUMENT, "draft: k_new/v_new");
  for (int i = 0; i < r->B; ++i) {
    const int64_t need = r->h_p0[i] + draft_off + a->step - (a->k_new ? 1 : 0);
    if (need > r->cache->len[r->h_seq[i]] && !a->k_new)
      return fail(SA_OUT_OF_RANGE, "KvStore: gather indices must be strictly increasing and in range");
  }
  sa::DraftParams p{};
  p.cache = r->cache->view();
  p.layer = a->layer;
  p.B = r->B;
  p.Hkv = r->Hkv;
  p.G = r->G;
  p.step = a->step;
  p.draft_off = draft_off;
  p.seq_ids = r->d_seq;
  p.p0 = r->d_p0;
  p.q = static_cast<const __nv_bfloat16*>(a->q);
  p.k_new = static_cast<const __nv_bfloat16*>(a->k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(a->v_new);
  p.n_sets = a->mode == SA_PER_LAYER ? 1 : r->Hkv;
  p.idx = sa_runner_indices(r, a->layer_slot, &p.k_cap);
  p.k_act = sa_runner_counts(r, a->layer_slot);
  p.scale_log2 = a->scale * sa::kLog2e;
  p.out = a->out;
  const int64_t units = static_cast<int64_t>(r->B) * r->Hkv;
  {  // one cluster of CS CTAs per (sequence, KV head): the smallest CS whose chunk fits one resident
     // round (192 rows); 12 before 16 because two launches of 12-CTA clusters co-reside on 148 SMs
     // (the PDL successor gathers while this one computes) and two of 16-CTA clusters do not.
     // Chunks of several rounds (large k) or grids far beyond two waves (many sequences x heads)
     // switch to the streaming mode: one CTA per SM, CS sized to one wave, rounds double-buffered.
    const int64_t m = r->k_cap + draft_off + a->step;
    const int round_rows = sa::draft_round_rows();
    int cs = -1;
    // at least 4 CTAs per unit while two launches still co-reside at two CTAs per SM: shorter
    // per-CTA chains beat the larger merge (k = 64: 4.27 -> 3.25 us, k = 256: 3.68 -> 3.32 us per
    // launch with CS 1/2 -> 4; CS 8-12 is slower again)
    int min_cs = 1;
    for (int c : {2, 4})
      if (units * c <= r->num_sms) min_cs = c;
    if (r->dev.draft_min_cs) min_cs = r->dev.draft_min_cs;
    // the smallest CS whose chunk fits one round (any size up to 16: e.g. 13 for the 2311 rows of
    // gamma 8 at k = 2294, where 16 CTAs per unit cost 6.0 against ~5.1 us per launch)
    for (int c : {1, 2, 4, 8, 9, 10, 11, 12, 13, 14, 15, 16})
      if (c >= min_cs && (m + c - 1) / c <= round_rows) {
        cs = c;
        break;
      }
    p.stream = 0;
    const int multi_round_max = r->dev.draft_multi_rounds;  // rounds allowed in the two-CTA-per-SM mode
    // a few units with a large budget (config 5 k = 4096, config 4's per-GPU shard): several rounds in
    // the two-CTA-per-SM mode, round 0 gathered before the dependency wait and later rounds reusing its
    // buffer.  Fewest rounds first, with a penalty when two successive launches' clusters cannot
    // co-reside (the next launch's pre-wait gathers would then start late); the one-CTA-per-SM
    // streaming mode would need two waves of 16-CTA clusters here.
    p.n_sub = 1;
    // A few units whose rows do not fit one round of one cluster (config 4's per-GPU shard: 4 units
    // of 9.2K rows): still ONE round per CTA, over n_sub clusters of 6 (or 8, 4) CTAs per unit merged
    // in two levels (the second through global memory, ~2 us), while the grid stays within ~4/3 CTAs
    // per SM.  Measured on config 4's shard: 13.3 us per launch for three rounds of one 16-CTA
    // cluster, 11.8 for two rounds of 4 x 8 CTAs, 9.9-10.0 for one round of 8 x 6 or 6 x 8 (grids
    // past ~200 CTAs or 12-CTA clusters are slower again); config 5 at k = 4096 (8 units): 9.0 for two
    // rounds of 16, 9.35 for 3 x 8, 8.28 for 4 x 6.  At config 2 the second level would cost +2 us.
    if (cs < 0) {
      for (int c : {6, 8, 4}) {
        const int64_t sub = (m + static_cast<int64_t>(c) * round_rows - 1) / (static_cast<int64_t>(c) * round_rows);
        if (sub >= 2 && units * sub * c * 3 <= 4 * static_cast<int64_t>(r->num_sms) && units * sub * 8 <= r->d_units_cap) {
          cs = c;
          p.n_sub = static_cast<int>(sub);
          break;
        }
      }
    }
    int multi_cs = -1;
    double multi_score = 0.0;
    for (int c : {16, 12, 8}) {
      if (cs > 0) break;  // one round fits: the rules above
      const int act = sa::draft_max_active_clusters(0, c);
      const int64_t rounds = ((m + c - 1) / c + round_rows - 1) / round_rows;
      if (act < units || rounds > multi_round_max) continue;
      const double score = static_cast<double>(rounds) + (2 * units > act ? 1.5 : 0.0);
      if (multi_cs < 0 || score < multi_score) {
        multi_cs = c;
        multi_score = score;
      }
    }
    // Many units with a large k (config 3: 128 units of 4.6K rows): small clusters, still two CTAs
    // per SM and one wave, any number of single-buffered rounds — the two CTAs of an SM overlap one's
    // gather with the other's compute.  Config 3: 73 us per launch streaming (one CTA per SM,
    // double-buffered), 68 us with 2-CTA clusters here (TMA row gather).
    if (cs < 0 && multi_cs < 0)
      for (int c : {8, 4, 2})
        if (units * c <= 2 * r->num_sms && units <= sa::draft_max_active_clusters(0, c)) {
          multi_cs = c;
          break;
        }
    if (cs < 0 && multi_cs > 0) {
      cs = multi_cs;
    } else if (cs < 0 || units * cs * p.n_sub > 2 * r->num_sms) {
      // cost ~ waves x (rows per CTA + a fixed per-CTA overhead of one 64-row tile), where the wave
      // count comes from the occupancy API: 16-CTA clusters of one CTA per SM do not all fit on
      // 148 SMs (a cluster lives inside one GPC), and a second wave costs a whole launch
      p.stream = 1;
      cs = 1;
      int64_t best = -1;
      for (int c : {1, 2, 4, 8, 12, 16}) {
        const int act = sa::draft_max_active_clusters(1, c);
        if (act <= 0) continue;
        const int64_t waves = (units + act - 1) / act;
        const int64_t cost = waves * ((m + c - 1) / c + 64);
        if (best < 0 || cost < best) {
          best = cost;
          cs = c;
        }
      }
    }
    if (r->dev.draft_cs > 0) {  // dev: forced CTAs per unit, two-CTA-per-SM mode (<= 3 rounds)
      cs = std::min(r->dev.draft_cs, sa::draft_max_splits());
      p.stream = 0;
      p.n_sub = 1;
    }
    if (r->dev.draft_stream >= 0) p.stream = r->dev.draft_stream;  // dev: forced mode
    if (r->dev.draft_sub > 0 && units * r->dev.draft_sub * 8 <= r->d_units_cap)  // dev: forced
      p.n_sub = r->dev.draft_sub;
    p.n_splits = cs;
    p.chunk = static_cast<int>(((m + cs * p.n_sub - 1) / (cs * p.n_sub) + 15) / 16 * 16);
    if (r->dev.draft_debug) {
      std::fprintf(stderr, "draft: units %lld m %lld -> stream %d cs %d sub %d chunk %d | active clusters (stream/non):",
                   static_cast<long long>(units), static_cast<long long>(m), p.stream, cs, p.n_sub, p.chunk);
      for (int c : {1, 2, 4, 8, 12, 16})
        std::fprintf(stderr, " %d:%d/%d", c, sa::draft_max_active_clusters(1, c), sa::draft_max_active_clusters(0, c));
      std::fprintf(stderr, "\n");
    }
  }
  p.tmk = r->cache->tmap_kg;
  p.tmv = r->cache->tmap_vg;
  p.part_o = r->d_po;
  p.part_ml = r->d_pml;
  p.counters = r->d_cnt;
  p.trace = r->dtrace;
  p.use_pdl = pdl ? 1 : 0;
  p.cluster_policy = r->dev.draft_cluster_policy;
  cudaError_t e = sa::launch_draft(p, s);
  if (e != cudaSuccess) return sa::cuda_fail(e, "draft launch");
  return SA_OK;
}

// dev-only: write the runner's verify + draft trace buffers to `path` (after a device sync); 0 on success.
SA_API int sa_dev_trace_dump(sa_runner* r, const char* path) {
  if (!r || !r->vtrace || !r->dtrace || !path) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  std::vector<unsigned long long> h(kVTraceWords + kDTraceWords);
  if (cudaMemcpy(h.data(), r->vtrace, kVTraceWords * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -3;
  if (cudaMemcpy(h.data() + kVTraceWords, r->dtrace, kDTraceWords * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -3;
  FILE* f = fopen(path, "wb");
  if (!f) return -4;
  fwrite(h.data(), 8, h.size(), f);
  fclose(f);
  return 0;
}

SA_API sa_status sa_dev_set_knob(sa_runner* r, const char* name, int64_t value) {
  if (!r || !name) return fail(SA_INVALID_ARGUMENT, "null argument");
  sa::DevConfig& d = r->dev;
  const std::string n(name);
  const int v = static_cast<int>(value);
  if (n == "verify_impl") d.verify_impl = v;
  else if (n == "verify_chunk_tiles") d.verify_chunk_tiles = v;
  else if (n == "verify_no_prefill") d.verify_no_prefill = v;
  else if (n == "verify_static_first") d.verify_static_first = v;
  else if (n == "verify_mergers") d.verify_mergers = v;
  else if (n == "verify_full_rows") d.verify_full_rows = v;
  else if (n == "verify_max_splits") d.verify_max_splits = v;
  else if (n == "verify_tail_tiles") d.verify_tail_tiles = v;
  else if (n == "verify_flush_tiles") d.verify_flush_tiles = v;
  else if (n == "verify_flush_min_tiles") d.verify_flush_min_tiles = v;
  else if (n == "verify_row_split") d.verify_row_split = v;
  else if (n == "draft_min_cs") d.draft_min_cs = v;
  else if (n == "draft_cs") d.draft_cs = v;
  else if (n == "draft_sub") d.draft_sub = v;
  else if (n == "draft_stream") d.draft_stream = v;
  else if (n == "draft_cluster_policy") d.draft_cluster_policy = v;
  else if (n == "draft_multi_rounds") d.draft_multi_rounds = v;
  else if (n == "draft_debug") d.draft_debug = v;
  else if (n == "draft_no_pdl") d.draft_no_pdl = v;
  else if (n == "iter_skip") d.iter_skip = v;
  else if (n == "select_batched") d.select_batched = v;
  else if (n == "select_legacy") d.select_legacy = v;
  else if (n == "stream_priority") {
    d.stream_priority = v;
    SA_CUDA_CHECK(cudaDeviceSynchronize());
    SA_CUDA_CHECK(make_streams(r));
  } else if (n == "trace") {
    d.trace = v;
    if (v && !r->vtrace) {
      SA_CUDA_CHECK(cudaMalloc(&r->vtrace, kVTraceWords * 8));
      SA_CUDA_CHECK(cudaMemset(r->vtrace, 0, kVTraceWords * 8));
      SA_CUDA_CHECK(cudaMalloc(&r->dtrace, kDTraceWords * 8));
      SA_CUDA_CHECK(cudaMemset(r->dtrace, 0, kDTraceWords * 8));
    }
    if (!v) {
      cudaFree(r->vtrace);
      cudaFree(r->dtrace);
      r->vtrace = r->dtrace = nullptr;
    }
  } else {
    return fail(SA_INVALID_ARGUMENT, "unknown dev knob '" + n + "'");
  }
  for (auto& kv : r->graphs) cudaGraphExecDestroy(kv.second);  // captured with the old settings
  r->graphs.clear();
  return SA_OK;
}

static sa_status ensure_weight_buffers(sa_runner* r) {  // lazily: only the weights metric needs them
  if (r->wlogits.empty()) r->wlogits.assign(r->n_slots, nullptr);
  const size_t bytes = sizeof(float) * r->cfg.max_batch * r->Hq * 2 * r->ld;
  for (auto& w : r->wlogits)
    if (!w) SA_CUDA_CHECK(cudaMalloc(&w, bytes));
  if (!r->wstats) SA_CUDA_CHECK(cudaMalloc(&r->wstats, sizeof(float2) * sa::kWeightParts * r->cfg.max_batch * r->Hq * r->cfg.max_rows));
  return SA_OK;
}

static sa_status weights_impl(sa_runner* r, int32_t slot, const float* logits, int64_t ld, int32_t n_rows,
                              sa_select_mode mode, cudaStream_t s) {
  if (!logits) return fail(SA_INVALID_ARGUMENT, "score_weights: null logits");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "score_weights: no batch bound");
  if (slot < 0 || slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "score_weights: layer_slot");
  if (n_rows < 1 || n_rows > r->cfg.max_rows) return fail(SA_INVALID_ARGUMENT, "score_columns_weights: empty row subset");
  if (ld < r->p_max) return fail(SA_INVALID_ARGUMENT, "score_weights: ld_logits < prefix");
  if (mode != SA_PER_LAYER && mode != SA_PER_KV_HEAD) return fail(SA_INVALID_ARGUMENT, "score_weights: mode");
  if (!r->wstats) SA_CUDA_CHECK(cudaMalloc(&r->wstats, sizeof(float2) * sa::kWeightParts * r->cfg.max_batch * r->Hq * r->cfg.max_rows));
  const int n_sets = mode == SA_PER_LAYER ? 1 : r->Hkv;
  long long* fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, slot, nullptr));
  float* scores = sa_runner_scores(r, slot, nullptr);
  const double scale = 1.0 / std::sqrt(static_cast<double>(r->cache->head_dim));  // selection.cpp:117
  cudaError_t e = sa::launch_weights(logits, ld, r->d_p0, r->B, r->Hq, r->G, n_rows, scale, r->wstats, n_sets, fx,
                                     scores, r->ld, r->p_max, s);
  if (e != cudaSuccess) return sa::cuda_fail(e, "score_weights launch");
  r->slot_layout[slot] = mode;
  if (mode == SA_PER_LAYER) r->fx_dirty[slot] = 1;  // written (not accumulated); the select consumes it
  return SA_OK;
}

SA_API sa_status sa_score_weights(sa_runner* r, int32_t slot, const float* logits, int64_t ld, int32_t n_rows,
                                  sa_select_mode mode, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  return weights_impl(r, slot, logits, ld, n_rows, mode, static_cast<cudaStream_t>(stream));
}

static sa_status quest_refresh(sa_runner* r, cudaStream_t s) {  // stale summaries of the bound batch
  sa_cache* c = r->cache;
  for (int i = 0; i < r->B; ++i) {  // lazily refresh stale summaries (kv_store.cpp:127-139)
    const int seq = r->h_seq[i];
    const int64_t from = std::min(c->summ_valid[seq], r->h_p0[i] / c->qpage * c->qpage);
    cudaError_t e = sa::launch_quest_summarize(c->view(), c->qmin, c->qmax, static_cast<int>(c->qpage), seq, from,
                                               c->len[seq], s);
    if (e != cudaSuccess) return sa::cuda_fail(e, "quest summaries");
    c->summ_valid[seq] = c->len[seq];
  }
  return SA_OK;
}

static sa_status quest_select_impl(sa_runner* r, int32_t layer, int32_t slot, const void* q, cudaStream_t s) {
  sa_cache* c = r->cache;
  const int64_t max_qp = (r->cfg.max_prefix + c->qpage - 1) / c->qpage;
  cudaError_t e = sa::launch_quest_select(c->view(), c->qmin, c->qmax, static_cast<int>(c->qpage), layer, r->d_seq, r->d_p0,
                                          r->B, r->Hq, r->G, static_cast<const __nv_bfloat16*>(q), r->cfg.sparse_ratio,
                                          r->cfg.k_min, r->k_cap, r->qbounds, std::max<int64_t>(1, max_qp),
                                          sa_runner_indices(r, slot, nullptr), sa_runner_counts(r, slot), s);
  if (e != cudaSuccess) return sa::cuda_fail(e, "select_quest launch");
  r->slot_layout[slot] = SA_PER_LAYER;
  return SA_OK;
}

static sa_status quest_prepare(sa_runner* r) {
  sa_cache* c = r->cache;
  if (c->qpage <= 0) return fail(SA_INVALID_ARGUMENT, "select_quest: page summaries not enabled on the store");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "select_quest: no batch bound");
  const int64_t max_qp = (r->cfg.max_prefix + c->qpage - 1) / c->qpage;
  if (max_qp > 8192) return fail(SA_NOT_SUPPORTED, "select_quest: more than 8192 summary pages (raise page_size)");
  if (!r->qbounds) SA_CUDA_CHECK(cudaMalloc(&r->qbounds, sizeof(double) * r->cfg.max_batch * std::max<int64_t>(1, max_qp)));
  return SA_OK;
}

SA_API sa_status sa_select_quest(sa_runner* r, int32_t layer, int32_t slot, const void* q, void* stream) {
  if (!r || !q) return fail(SA_INVALID_ARGUMENT, "null argument");
  if (sa_status st = quest_prepare(r)) return st;
  if (layer < 0 || layer >= r->cache->n_layers) return fail(SA_OUT_OF_RANGE, "select_quest: layer out of range");
  if (slot < 0 || slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "select_quest: layer_slot");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (sa_status st = quest_refresh(r, s)) return st;
  return quest_select_impl(r, layer, slot, q, s);
}

SA_API sa_status sa_select_window(sa_runner* r, int32_t slot, int64_t sink, int64_t window, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  if (r->B < 1) return fail(SA_INVALID_ARGUMENT, "select_window: no batch bound");
  if (slot < 0 || slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "select_window: layer_slot");
  if (sink < 0 || window < 0 || sink + window < 1)
    return fail(SA_INVALID_ARGUMENT, "SelectorConfig: sink + window must be >= 1");  // selection.cpp:55-56
  if (sink + window > r->k_cap) return fail(SA_INVALID_ARGUMENT, "select_window: sink + window exceeds index capacity");
  cudaError_t e = sa::launch_window(r->d_p0, r->B, sink, window, r->k_cap, sa_runner_indices(r, slot, nullptr),
                                    sa_runner_counts(r, slot), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return sa::cuda_fail(e, "select_window launch");
  r->slot_layout[slot] = SA_PER_LAYER;
  return SA_OK;
}

SA_API sa_status sa_runner_set_comm(sa_runner* r, sa_comm* comm) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  r->comm = comm;
  for (auto& kv : r->graphs) cudaGraphExecDestroy(kv.second);  // captured graphs depend on it
  r->graphs.clear();
  return SA_OK;
}

SA_API sa_status sa_exchange_layer_scores(sa_runner* r, int32_t slot, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  if (slot < 0 || slot >= r->n_slots) return fail(SA_OUT_OF_RANGE, "exchange: layer_slot");
  long long* fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, slot, nullptr));
  return sa::comm_allreduce_i64(r->comm, fx, static_cast<size_t>(r->B) * r->ld, static_cast<cudaStream_t>(stream));
}

SA_API sa_status sa_verify_attention(sa_runner* r, const sa_verify_args* a, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  return verify_impl(r, a, static_cast<cudaStream_t>(stream));
}
SA_API sa_status sa_select_topk(sa_runner* r, const sa_select_args* a, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  return select_impl(r, a, static_cast<cudaStream_t>(stream));
}
SA_API sa_status sa_draft_attention(sa_runner* r, const sa_draft_args* a, void* stream) {
  if (!r) return fail(SA_INVALID_ARGUMENT, "null runner");
  return draft_impl(r, a, static_cast<cudaStream_t>(stream));
}

SA_API int64_t sa_iteration_kernel_count(const sa_runner* r, const sa_iteration_args* a) {
  if (!r || !a) return 0;
  const int64_t L = r->cache->n_layers;
  const uint32_t ph = a->phases ? a->phases : 7u;
  const int64_t sel_kernels = a->strategy == SA_COLLECT2_WEIGHTS ? 3 : 1;  // (+ row stats, weight scores)
  const int64_t selects = a->strategy == SA_QUEST_LIKE ? 2 * static_cast<int64_t>(a->gamma) * L  // bounds + pick per draft
                                                       : sel_kernels * L;
  return ((ph & SA_PHASE_VERIFY) ? L : 0) + ((ph & SA_PHASE_SELECT) ? selects : 0) +
         ((ph & SA_PHASE_DRAFT) ? static_cast<int64_t>(a->gamma) * L : 0);
}

static sa_status enqueue_iteration(sa_runner* r, const sa_iteration_args* a, cudaStream_t main) {
  const int L = static_cast<int>(r->cache->n_layers), B = r->B, R = a->gamma + 1;
  // score rows (bit r = row label r+1): AllDraft all gamma+1 rows (selection.cpp:183-185), Collect-2
  // {1, gamma+1} (:187-196), LastAccepted the single row a+1 (:198-207)
  const uint32_t mask = a->strategy == SA_ALL_DRAFT     ? ((1u << R) - 1u)
                        : a->strategy == SA_LAST_ACCEPTED ? (1u << a->accepted)
                                                           : (1u | (1u << a->gamma));
  const bool weights = a->strategy == SA_COLLECT2_WEIGHTS;  // rows {1, gamma+1}, softmax-weight metric
  const bool quest = a->strategy == SA_QUEST_LIKE, window = a->strategy == SA_WINDOW;
  const bool guided = !quest && !window;  // selection from the verify byproduct
  const int rows_in_score = __builtin_popcount(mask);
  const size_t qv_l = static_cast<size_t>(B) * r->Hq * R * 128, kv_l = static_cast<size_t>(B) * R * r->Hkv * 128;
  const size_t qd_l = static_cast<size_t>(B) * r->Hq * 128, kd_l = static_cast<size_t>(B) * r->Hkv * 128;
  const auto* qv = static_cast<const __nv_bfloat16*>(a->qv);
  const auto* kvn = static_cast<const __nv_bfloat16*>(a->kv_new);
  const auto* vvn = static_cast<const __nv_bfloat16*>(a->vv_new);
  const auto* qd = static_cast<const __nv_bfloat16*>(a->qd);
  const auto* kdn = static_cast<const __nv_bfloat16*>(a->kd_new);
  const auto* vdn = static_cast<const __nv_bfloat16*>(a->vd_new);
  // phase selection for timing breakdowns (sa_iteration_args::phases; SA_ITER_SKIP overrides in dev runs)
  const int skip = r->dev.iter_skip >= 0 ? r->dev.iter_skip : (a->phases ? static_cast<int>(~a->phases & 7u) : 0);
  // Selection schedule.  Default: one single-CTA select per layer on the side stream, overlapping the
  // verify chain.  A select CTA needs a whole SM's shared memory, so it waits for a verify CTA of the
  // next layer to exit and then delays a CTA of the layer after; that costs ~39 us over the chain.
  // Dev knob select_batched: the fused-byproduct selections (Collect-2, AllDraft, LastAccepted)
  // run as ONE launch after the chain instead, with the layers' CTAs side by side.  It removes those
  // 39 us but adds a ~55 us bubble before the first draft, so measured it is even (1.748 vs 1.742 ms).
  const bool batch_selects = r->dev.select_batched && (skip & 2) == 0 && guided && !weights &&
                             r->ld <= sa::select_max_smem_keys() && r->n_slots >= L;
  SA_CUDA_CHECK(cudaEventRecord(r->ev_fork, main));
  SA_CUDA_CHECK(cudaStreamWaitEvent(r->side, r->ev_fork, 0));
  for (int l = 0; l < L; ++l) {
    sa_verify_args v{};
    v.layer = l;
    v.layer_slot = l;
    v.n_rows = R;
    v.q = qv + l * qv_l;
    v.k_new = kvn ? kvn + l * kv_l : nullptr;
    v.v_new = vvn ? vvn + l * kv_l : nullptr;
    v.scale = a->scale;
    v.score_row_mask = (weights || !guided) ? 0u : mask;
    v.score_layout = a->mode;
    if (weights) {  // LogitMatrix of the collected rows for the weights kernels
      v.logits = r->wlogits[l];
      v.ld_logits = r->ld;
      v.collect_row_mask = mask;
    }
    v.out = a->out_v + l * qv_l;
    if ((skip & 1) == 0)
      if (sa_status st = verify_impl(r, &v, main, /*pdl=*/l > 0, /*in_iteration=*/true))
        return st;
    SA_CUDA_CHECK(cudaEventRecord(r->ev_v[l], main));
    SA_CUDA_CHECK(cudaStreamWaitEvent(r->side, r->ev_v[l], 0));
    sa_select_args sel{};
    sel.layer_slot = l;
    sel.mode = a->mode;
    sel.rows_in_score = rows_in_score;
    if ((skip & 2) == 0 && window) {  // query-agnostic: once per iteration (budget k: sink 4 + window k-4)
      if (sa_status st = sa_select_window(r, l, 4, std::max<int64_t>(0, r->k_cap - 4), r->side)) return st;
    } else if ((skip & 2) == 0 && guided) {
      if (weights)
        if (sa_status st = weights_impl(r, l, r->wlogits[l], r->ld, rows_in_score, a->mode, r->side)) return st;
      if (r->comm && a->mode == SA_PER_LAYER) {  // §8e exchange: sums of the other KV-head shards
        long long* fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, l, nullptr));
        if (sa_status st = sa::comm_allreduce_i64(r->comm, fx, static_cast<size_t>(B) * r->ld, r->side)) return st;
      }
      if (!batch_selects)
        if (sa_status st = select_impl(r, &sel, r->side)) return st;
    }
    if (!batch_selects) SA_CUDA_CHECK(cudaEventRecord(r->ev_s[l], r->side));
  }
  if (batch_selects) {  // every layer's top-k in one launch (L x B x sets CTAs side by side)
    sa_select_args sel{};
    sel.layer_slot = 0;
    sel.mode = a->mode;
    sel.rows_in_score = rows_in_score;
    if (sa_status st = select_impl(r, &sel, r->side, L)) return st;
    // ONE dependency edge into the draft chain (draft(1, 0)); later drafts follow it through their
    // programmatic (PDL) edges.  A per-draft edge from the shared select node measured ~4 us per
    // step-1 launch: those launches lost their PDL overlap.
    SA_CUDA_CHECK(cudaEventRecord(r->ev_s[L - 1], r->side));
    SA_CUDA_CHECK(cudaStreamWaitEvent(main, r->ev_s[L - 1], 0));
  }
  for (int j = 1; j <= a->gamma; ++j) {
    for (int l = 0; l < L; ++l) {
      if (j == 1 && !batch_selects) SA_CUDA_CHECK(cudaStreamWaitEvent(main, r->ev_s[l], 0));
      sa_draft_args d{};
      d.layer = l;
      d.layer_slot = l;
      d.mode = a->mode;
      d.step = j;
      const size_t off = (static_cast<size_t>(j - 1) * L + l);
      d.q = qd + off * qd_l;
      d.k_new = kdn ? kdn + off * kd_l : nullptr;
      d.v_new = vdn ? vdn + off * kd_l : nullptr;
      d.scale = a->scale;
      d.out = a->out_d + off * qd_l;
      if (quest && (skip & 2) == 0)  // QuestLike re-selects before every draft forward
        if (sa_status st = quest_select_impl(r, l, l, d.q, main)) return st;
      if ((skip & 4) == 0)
        if (sa_status st = draft_impl(r, &d, main, /*pdl=*/(j > 1 || l > 0) && !quest && !r->dev.draft_no_pdl,
                                      /*draft_off=*/a->accepted + 1))
          return st;
    }
  }
  SA_CUDA_CHECK(cudaEventRecord(r->ev_join, r->side));
  SA_CUDA_CHECK(cudaStreamWaitEvent(main, r->ev_join, 0));
  return SA_OK;
}

SA_API sa_status sa_iteration_run(sa_runner* r, const sa_iteration_args* a, void* stream) {
  if (!r || !a) return fail(SA_INVALID_ARGUMENT, "null argument");
  if (a->gamma < 0 || a->gamma + 1 > r->cfg.max_rows) return fail(SA_INVALID_ARGUMENT, "gamma out of range");
  if (a->gamma < 1) return fail(SA_INVALID_ARGUMENT, "DecodeParams: gamma must be >= 1");
  if (a->strategy < SA_WINDOW || a->strategy > SA_COLLECT2_WEIGHTS) return fail(SA_NOT_SUPPORTED, "iteration: unknown strategy");
  if (a->strategy == SA_QUEST_LIKE) {  // summaries current for the bound prefixes before capture / launch
    if (sa_status st = quest_prepare(r)) return st;
    if (sa_status st = quest_refresh(r, static_cast<cudaStream_t>(stream))) return st;
  }
  if (a->strategy == SA_COLLECT2_WEIGHTS)
    if (sa_status st = ensure_weight_buffers(r)) return st;  // (outside any graph capture)
  if (a->accepted < 0 || a->accepted > a->gamma)
    return fail(SA_INVALID_ARGUMENT, a->strategy == SA_LAST_ACCEPTED ? "select_last_accepted: row accepted+1 not collected"
                                                                     : "iteration: accepted must be in [0, gamma]");
  if (a->strategy == SA_QUEST_LIKE && r->comm)
    return fail(SA_NOT_SUPPORTED, "select_quest: page bounds are not exchanged over a KV-head group (per-GPU heads only)");
  // the next draft chain writes rows p0+a+1 .. p0+a+gamma: their pages exist before capture / launch
  for (int i = 0; i < r->B; ++i) {
    const int64_t end = r->h_p0[i] + a->accepted + 1 + a->gamma;
    if (end > r->cache->max_context) return fail(SA_LENGTH_ERROR, "KvStore: draft rows past max_context");
    if (sa_status st = r->cache->reserve(r->h_seq[i], end)) return st;
  }
  if (r->n_slots < r->cache->n_layers) return fail(SA_INVALID_ARGUMENT, "iteration needs n_layers_buf >= n_layers");
  if (!a->qv || !a->qd || !a->out_v || !a->out_d) return fail(SA_INVALID_ARGUMENT, "iteration: null buffer");
  cudaStream_t main = static_cast<cudaStream_t>(stream);
  // per-layer sums left unconsumed (direct verify calls, verify-only phase runs): zero them before an
  // iteration whose selects will consume them (a run without the select phase reads none)
  const uint32_t ph = a->phases ? a->phases : 7u;
  if (a->mode == SA_PER_LAYER && (ph & SA_PHASE_SELECT))
    for (int l = 0; l < r->cache->n_layers; ++l)
      if (r->fx_dirty[l]) {
        long long* fx = reinterpret_cast<long long*>(sa_runner_layer_scores(r, l, nullptr));
        SA_CUDA_CHECK(cudaMemsetAsync(fx, 0, sizeof(long long) * r->cfg.max_batch * r->ld, main));
        r->fx_dirty[l] = 0;
      }
  if (!a->use_graph) {
    sa_status st = enqueue_iteration(r, a, main);
    if (st == SA_OK && r->comm) st = sa_comm_check(r->comm);
    if (st == SA_OK && a->mode == SA_PER_LAYER && a->phases && (a->phases & SA_PHASE_VERIFY) &&
        !(a->phases & SA_PHASE_SELECT))
      for (int l = 0; l < r->cache->n_layers; ++l) r->fx_dirty[l] = 1;
    return st;
  }
  std::vector<char> key(sizeof(sa_iteration_args) + sizeof(int) + r->h_p0.size() * sizeof(int64_t) +
                        r->h_seq.size() * sizeof(int32_t));
  std::memcpy(key.data(), a, sizeof(*a));
  std::memcpy(key.data() + sizeof(*a), &r->B, sizeof(int));
  std::memcpy(key.data() + sizeof(*a) + sizeof(int), r->h_p0.data(), r->h_p0.size() * sizeof(int64_t));
  std::memcpy(key.data() + sizeof(*a) + sizeof(int) + r->h_p0.size() * sizeof(int64_t), r->h_seq.data(),
              r->h_seq.size() * sizeof(int32_t));
  cudaGraphExec_t gexec = nullptr;
  for (auto& kv : r->graphs)
    if (kv.first == key) gexec = kv.second;
  if (!gexec) {
    if (r->graphs.size() >= 8) {  // bounded cache: drop the oldest
      cudaGraphExecDestroy(r->graphs.front().second);
      r->graphs.erase(r->graphs.begin());
    }
    cudaGraph_t graph = nullptr;
    SA_CUDA_CHECK(cudaStreamBeginCapture(r->capture, cudaStreamCaptureModeThreadLocal));
    sa_status st = enqueue_iteration(r, a, r->capture);
    cudaError_t e = cudaStreamEndCapture(r->capture, &graph);
    if (st != SA_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return sa::cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return sa::cuda_fail(e, "cudaGraphInstantiate");
    r->graphs.emplace_back(std::move(key), gexec);
  }
  SA_CUDA_CHECK(cudaGraphLaunch(gexec, main));
  if (r->comm)  // a dead peer surfaces here (the communicator is aborted, the caller sees SA_NCCL_ERROR)
    if (sa_status st = sa_comm_check(r->comm)) return st;
  // a verify without its select leaves per-layer sums unconsumed: zero them before the next use
  if (a->mode == SA_PER_LAYER && a->phases && (a->phases & SA_PHASE_VERIFY) && !(a->phases & SA_PHASE_SELECT))
    for (int l = 0; l < r->cache->n_layers; ++l) r->fx_dirty[l] = 1;
  return SA_OK;
}

}  // extern "C"
