// cache.cu — paged bf16 KV cache: the device counterpart of specattn::KvStore
// (kv_store.hpp:19-89, kv_store.cpp:1-88).
//
// Layout (DESIGN.md §HBM layout): K and V pools are [n_layers][num_pages][Hkv][P][128] bf16, so a
// page holds P consecutive token rows of one (layer, KV head) contiguously (P*256 bytes) — one
// TMA box per 64 tokens, and the whole pool is a flat 2-D [rows][128] tensor for the TMA
// descriptors.  Pages are shared across layers (block_table[seq][page_in_seq] indexes all
// layers), allocated on demand from a LIFO free list.  Length / committed bookkeeping is host
// metadata exactly as in the reference (O(1) truncate, kv_store.cpp:51-65).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace sa {

static thread_local std::string g_last_error;

sa_status fail(sa_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
sa_status cuda_fail(cudaError_t e, const char* where) {
  return fail(SA_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

bool encode_tensor_map(CUtensorMap* map, void* base, uint64_t rows, uint32_t box_rows, std::string* err) {
  return encode_tensor_map_2d(map, base, 128, rows, box_rows, err);
}

bool encode_tensor_map_2d(CUtensorMap* map, void* base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                          std::string* err) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r));
    return false;
  }
  return true;
}

// keys: [n_tokens][L*Hkv][128] (layer-major rows, kv_store.hpp:33-35) -> cache rows len..len+n-1.
template <typename T>
__global__ void append_kernel(CacheView c, int seq, int len0, int n_tokens, const T* keys, const T* values) {
  const int rows_per_tok = c.n_layers * c.n_kv_heads;
  const int64_t total = static_cast<int64_t>(n_tokens) * rows_per_tok * 16;  // 8-element chunks
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i & 15);
    const int64_t r = i >> 4;
    const int tok = static_cast<int>(r / rows_per_tok), lr = static_cast<int>(r % rows_per_tok);
    const int layer = lr / c.n_kv_heads, head = lr % c.n_kv_heads;
    const int64_t dst = cache_row(c, seq, layer, head, len0 + tok) * 128 + ch * 8;
    const T* sk = keys + r * 128 + ch * 8;
    const T* sv = values + r * 128 + ch * 8;
    if constexpr (sizeof(T) == 4) {
      __nv_bfloat16 kb[8], vb[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        kb[e] = __float2bfloat16_rn(sk[e]);
        vb[e] = __float2bfloat16_rn(sv[e]);
      }
      *reinterpret_cast<uint4*>(c.k + dst) = *reinterpret_cast<uint4*>(kb);
      *reinterpret_cast<uint4*>(c.v + dst) = *reinterpret_cast<uint4*>(vb);
    } else {
      *reinterpret_cast<uint4*>(c.k + dst) = *reinterpret_cast<const uint4*>(sk);
      *reinterpret_cast<uint4*>(c.v + dst) = *reinterpret_cast<const uint4*>(sv);
    }
  }
}

// rows[i] (absolute positions) of (seq, layer, head) -> fp32 [n][128]  (gather / keys() views)
__global__ void read_rows_kernel(CacheView c, int seq, int layer, int head, const int64_t* idx, int64_t begin,
                                 int64_t n, float* K, float* V) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * 128;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i >> 7;
    const int col = static_cast<int>(i & 127);
    const int pos = static_cast<int>(idx ? idx[r] : begin + r);
    const int64_t src = cache_row(c, seq, layer, head, pos) * 128 + col;
    K[i] = __bfloat162float(c.k[src]);
    V[i] = __bfloat162float(c.v[src]);
  }
}

}  // namespace sa

using sa::fail;

sa_status sa_cache::reserve(int32_t seq, int64_t rows) {
  const int64_t need = (rows + page_size - 1) >> page_shift;
  if (need > max_pages_per_seq) return fail(SA_LENGTH_ERROR, "KvStore: append past max_context");
  int64_t have = pages_of_seq[seq];
  if (need <= have) return SA_OK;
  if (static_cast<int64_t>(free_pages.size()) < need - have) return fail(SA_LENGTH_ERROR, "KV page pool exhausted");
  for (int64_t i = have; i < need; ++i) {
    h_block_table[seq * max_pages_per_seq + i] = free_pages.back();
    free_pages.pop_back();
  }
  pages_of_seq[seq] = need;
  SA_CUDA_CHECK(cudaMemcpy(d_block_table + seq * max_pages_per_seq + have, h_block_table.data() + seq * max_pages_per_seq + have,
                           sizeof(int32_t) * (need - have), cudaMemcpyHostToDevice));
  return SA_OK;
}

extern "C" {

SA_API const char* sa_status_string(sa_status s) {
  switch (s) {
    case SA_OK: return "ok";
    case SA_INVALID_ARGUMENT: return "invalid_argument";
    case SA_DOMAIN_ERROR: return "domain_error";
    case SA_OUT_OF_RANGE: return "out_of_range";
    case SA_LENGTH_ERROR: return "length_error";
    case SA_CUDA_ERROR: return "cuda_error";
    case SA_NOT_SUPPORTED: return "not_supported";
    case SA_NCCL_ERROR: return "nccl_error";
  }
  return "unknown";
}

SA_API const char* sa_last_error(void) { return sa::g_last_error.c_str(); }
SA_API const char* sa_version(void) { return "specattn_b200 0.1 (sm_100a)"; }

SA_API int64_t sa_selection_k(double sparse_ratio, int64_t prefix_len, int64_t k_min) {
  const int64_t wanted = static_cast<int64_t>(std::llround(sparse_ratio * static_cast<double>(prefix_len)));
  return std::min(prefix_len, std::max(wanted, k_min));
}

SA_API sa_status sa_cache_create(const sa_cache_config* cfg, sa_cache** out) {
  if (!cfg || !out) return fail(SA_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (cfg->head_dim != 128) return fail(SA_NOT_SUPPORTED, "head_dim must be 128");
  if (cfg->n_layers < 1 || cfg->n_kv_heads < 1 || cfg->max_context < 1 || cfg->max_seqs < 1)
    return fail(SA_INVALID_ARGUMENT, "ModelConfig: n_layers, n_kv_heads, max_context, max_seqs must be >= 1");
  const int64_t P = cfg->page_size ? cfg->page_size : 256;
  if (P < 128 || (P & (P - 1))) return fail(SA_INVALID_ARGUMENT, "page_size must be a power of two >= 128");
  auto* c = new sa_cache();
  c->n_layers = cfg->n_layers;
  c->n_kv_heads = cfg->n_kv_heads;
  c->head_dim = cfg->head_dim;
  c->max_context = cfg->max_context;
  c->max_seqs = cfg->max_seqs;
  c->page_size = P;
  while ((int64_t{1} << c->page_shift) < P) ++c->page_shift;
  c->max_pages_per_seq = (cfg->max_context + P - 1) / P;
  c->num_pages = cfg->num_pages ? cfg->num_pages : cfg->max_seqs * c->max_pages_per_seq;
  const uint64_t rows = static_cast<uint64_t>(c->n_layers) * c->num_pages * c->n_kv_heads * P;
  if (rows >= (uint64_t{1} << 31)) {
    delete c;
    return fail(SA_NOT_SUPPORTED, "cache exceeds 2^31 token rows (TMA coordinate range)");
  }
  cudaGetDevice(&c->device);
  const size_t bytes = rows * 256;
  cudaError_t e = cudaMalloc(&c->k_pool, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->v_pool, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_block_table, sizeof(int32_t) * c->max_seqs * c->max_pages_per_seq);
  // Zero the pools so never-written rows inside a partially filled page hold finite values.
  if (e == cudaSuccess) e = cudaMemset(c->k_pool, 0, bytes);
  if (e == cudaSuccess) e = cudaMemset(c->v_pool, 0, bytes);
  if (e == cudaSuccess) e = cudaMemset(c->d_block_table, 0, sizeof(int32_t) * c->max_seqs * c->max_pages_per_seq);
  if (e != cudaSuccess) {
    sa_cache_destroy(c);
    return sa::cuda_fail(e, "sa_cache_create");
  }
  c->h_block_table.assign(c->max_seqs * c->max_pages_per_seq, 0);
  c->len.assign(c->max_seqs, 0);
  c->committed.assign(c->max_seqs, 0);
  c->pages_of_seq.assign(c->max_seqs, 0);
  c->verified_end.assign(c->max_seqs, 0);
  c->free_pages.resize(c->num_pages);
  for (int64_t i = 0; i < c->num_pages; ++i) c->free_pages[i] = static_cast<int32_t>(c->num_pages - 1 - i);
  std::string err;
  if (rows > static_cast<uint64_t>(INT32_MAX)) {  // tile::gather4 row coordinates are int32 (draft)
    sa_cache_destroy(c);
    return fail(SA_NOT_SUPPORTED, "cache rows (layers x pages x KV heads x page size) exceed 2^31");
  }
  if (!sa::encode_tensor_map(&c->tmap_k, c->k_pool, rows, 64, &err) ||
      !sa::encode_tensor_map(&c->tmap_v, c->v_pool, rows, 64, &err) ||
      !sa::encode_tensor_map(&c->tmap_k128, c->k_pool, rows, 128, &err) ||
      !sa::encode_tensor_map(&c->tmap_v128, c->v_pool, rows, 128, &err) ||
      !sa::encode_tensor_map(&c->tmap_kg, c->k_pool, rows, 1, &err) ||
      !sa::encode_tensor_map(&c->tmap_vg, c->v_pool, rows, 1, &err)) {
    sa_cache_destroy(c);
    return fail(SA_CUDA_ERROR, err);
  }
  *out = c;
  return SA_OK;
}

SA_API sa_status sa_accept(const float* p, const float* q, const int32_t* draft, const float* u, int32_t B,
                           int32_t gamma, int32_t V, int32_t greedy, int32_t* accepted, int32_t* emitted, void* stream) {
  if (!p || !draft || !accepted || !emitted || (!greedy && (!q || !u)))
    return fail(SA_INVALID_ARGUMENT, "accept: null argument");
  if (B < 1 || gamma < 1 || V < 1) return fail(SA_INVALID_ARGUMENT, "DecodeParams: gamma must be >= 1");
  cudaError_t e = sa::launch_accept(p, q, draft, u, B, gamma, V, greedy, accepted, emitted,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return sa::cuda_fail(e, "accept launch");
  return SA_OK;
}

SA_API sa_status sa_kv_commit_accepted(sa_cache* c, int32_t seq, int64_t p0, int32_t accepted) {
  if (!c) return fail(SA_INVALID_ARGUMENT, "null cache");
  if (seq < 0 || seq >= c->max_seqs) return fail(SA_OUT_OF_RANGE, "sequence id out of range");
  // The verify rows p0.. were written by the verify kernel's fused append into pages reserved for
  // them (sa_runner_set_batch), whether or not the host length was advanced: keep p0 .. p0+accepted.
  // Rows that exist: the host length, or the last verify's fused append [p0, p0 + n_rows).
  const int64_t keep = p0 + accepted + 1;
  const int64_t written = std::max(c->len[seq], c->verified_end[seq]);
  if (accepted < 0 || p0 < 0 || p0 > c->len[seq] || keep > written || keep > c->max_context ||
      keep > (c->pages_of_seq[seq] << c->page_shift))
    return fail(SA_OUT_OF_RANGE, "KvStore: commit beyond the appended verify rows");
  c->summaries_stale_from(seq, std::min(c->len[seq], p0));
  c->len[seq] = keep;
  c->committed[seq] = keep;
  return SA_OK;
}

SA_API sa_status sa_kv_enable_page_summaries(sa_cache* c, int64_t page_size) {
  if (!c) return fail(SA_INVALID_ARGUMENT, "null cache");
  if (page_size < 1) return fail(SA_INVALID_ARGUMENT, "KvStore: page_size must be >= 1");  // kv_store.cpp:91-93
  if (c->page_size % page_size || (page_size & (page_size - 1)))
    return fail(SA_NOT_SUPPORTED, "summary page size must be a power of two dividing the cache page size");
  const uint64_t rows = static_cast<uint64_t>(c->n_layers) * c->num_pages * c->n_kv_heads * c->page_size / page_size;
  cudaFree(c->qmin);
  cudaFree(c->qmax);
  c->qmin = c->qmax = nullptr;
  SA_CUDA_CHECK(cudaMalloc(&c->qmin, rows * 128 * sizeof(__nv_bfloat16)));
  SA_CUDA_CHECK(cudaMalloc(&c->qmax, rows * 128 * sizeof(__nv_bfloat16)));
  c->qpage = page_size;
  c->summ_valid.assign(c->max_seqs, 0);  // built lazily (the first Quest selection of each sequence)
  return SA_OK;
}

SA_API sa_status sa_cache_destroy(sa_cache* c) {
  if (!c) return SA_OK;
  cudaFree(c->k_pool);
  cudaFree(c->v_pool);
  cudaFree(c->qmin);
  cudaFree(c->qmax);
  cudaFree(c->d_block_table);
  delete c;
  return SA_OK;
}

static sa_status check_seq(const sa_cache* c, int32_t seq) {
  if (!c) return fail(SA_INVALID_ARGUMENT, "null cache");
  if (seq < 0 || seq >= c->max_seqs) return fail(SA_OUT_OF_RANGE, "sequence id out of range");
  return SA_OK;
}

SA_API sa_status sa_kv_size(const sa_cache* c, int32_t seq, int64_t* len) {
  if (sa_status st = check_seq(c, seq)) return st;
  *len = c->len[seq];
  return SA_OK;
}

SA_API sa_status sa_kv_committed(const sa_cache* c, int32_t seq, int64_t* committed) {
  if (sa_status st = check_seq(c, seq)) return st;
  *committed = c->committed[seq];
  return SA_OK;
}

SA_API sa_status sa_kv_bytes_per_token(const sa_cache* c, int64_t* ref_fp32, int64_t* device) {
  if (!c) return fail(SA_INVALID_ARGUMENT, "null cache");
  if (ref_fp32) *ref_fp32 = 2 * c->n_layers * c->n_kv_heads * c->head_dim * 4;  // kv_store.hpp:30
  if (device) *device = 2 * c->n_layers * c->n_kv_heads * c->head_dim * 2;
  return SA_OK;
}

SA_API sa_status sa_kv_append(sa_cache* c, int32_t seq, int64_t n_tokens, const void* keys, const void* values,
                              sa_dtype dtype, int on_host, void* stream) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (n_tokens < 0 || (n_tokens > 0 && (!keys || !values))) return fail(SA_INVALID_ARGUMENT, "KvStore: bad append");
  if (dtype != SA_F32 && dtype != SA_BF16) return fail(SA_INVALID_ARGUMENT, "dtype");
  if (c->len[seq] + n_tokens > c->max_context) return fail(SA_LENGTH_ERROR, "KvStore: append past max_context");
  if (n_tokens == 0) return SA_OK;
  if (sa_status st = c->reserve(seq, c->len[seq] + n_tokens)) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t esz = dtype == SA_F32 ? 4 : 2;
  const size_t bytes = static_cast<size_t>(n_tokens) * c->n_layers * c->n_kv_heads * 128 * esz;
  const void *k = keys, *v = values;
  void *tk = nullptr, *tv = nullptr;
  if (on_host) {
    SA_CUDA_CHECK(cudaMallocAsync(&tk, bytes, s));
    SA_CUDA_CHECK(cudaMallocAsync(&tv, bytes, s));
    SA_CUDA_CHECK(cudaMemcpyAsync(tk, keys, bytes, cudaMemcpyHostToDevice, s));
    SA_CUDA_CHECK(cudaMemcpyAsync(tv, values, bytes, cudaMemcpyHostToDevice, s));
    k = tk;
    v = tv;
  }
  const int64_t chunks = n_tokens * c->n_layers * c->n_kv_heads * 16;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<int64_t>((chunks + threads - 1) / threads, 4096));
  if (dtype == SA_F32)
    sa::append_kernel<float><<<blocks, threads, 0, s>>>(c->view(), seq, static_cast<int>(c->len[seq]),
                                                        static_cast<int>(n_tokens), static_cast<const float*>(k),
                                                        static_cast<const float*>(v));
  else
    sa::append_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(
        c->view(), seq, static_cast<int>(c->len[seq]), static_cast<int>(n_tokens),
        static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v));
  SA_CUDA_CHECK(cudaGetLastError());
  if (on_host) {
    SA_CUDA_CHECK(cudaFreeAsync(tk, s));
    SA_CUDA_CHECK(cudaFreeAsync(tv, s));
  }
  c->summaries_stale_from(seq, c->len[seq]);
  c->len[seq] += n_tokens;
  return SA_OK;
}

SA_API sa_status sa_kv_truncate(sa_cache* c, int32_t seq, int64_t to_len) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (to_len < 0 || to_len > c->len[seq]) return fail(SA_OUT_OF_RANGE, "KvStore: truncate beyond current length");
  c->summaries_stale_from(seq, to_len);
  c->len[seq] = to_len;
  c->committed[seq] = std::min(c->committed[seq], to_len);
  return SA_OK;
}

SA_API sa_status sa_kv_set_committed(sa_cache* c, int32_t seq, int64_t len) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (len < 0 || len > c->len[seq]) return fail(SA_OUT_OF_RANGE, "KvStore: committed mark beyond current length");
  c->committed[seq] = len;
  return SA_OK;
}

SA_API sa_status sa_kv_reserve(sa_cache* c, int32_t seq, int64_t len) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (len < 0) return fail(SA_INVALID_ARGUMENT, "negative length");
  return c->reserve(seq, len);
}

SA_API sa_status sa_kv_set_size(sa_cache* c, int32_t seq, int64_t new_len) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (new_len < 0 || new_len > c->max_context) return fail(SA_LENGTH_ERROR, "KvStore: length past max_context");
  if (sa_status st = c->reserve(seq, new_len)) return st;
  c->summaries_stale_from(seq, std::min(new_len, c->len[seq]));
  c->len[seq] = new_len;
  c->committed[seq] = std::min(c->committed[seq], new_len);
  return SA_OK;
}

SA_API sa_status sa_kv_gather(const sa_cache* c, int32_t seq, int64_t layer, int64_t head, const int64_t* idx,
                              int64_t n, float* K, float* V, void* stream) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (layer < 0 || layer >= c->n_layers || head < 0 || head >= c->n_kv_heads)
    return fail(SA_OUT_OF_RANGE, "KvStore: gather layer/head out of range");
  int64_t prev = -1;
  for (int64_t i = 0; i < n; ++i) {  // kv_store.cpp:72-78
    if (idx[i] <= prev || idx[i] >= c->len[seq])
      return fail(SA_OUT_OF_RANGE, "KvStore: gather indices must be strictly increasing and in range");
    prev = idx[i];
  }
  if (n == 0) return SA_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t* d_idx = nullptr;
  SA_CUDA_CHECK(cudaMallocAsync(&d_idx, sizeof(int64_t) * n, s));
  SA_CUDA_CHECK(cudaMemcpyAsync(d_idx, idx, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
  const int blocks = static_cast<int>(std::min<int64_t>((n * 128 + 255) / 256, 4096));
  sa::read_rows_kernel<<<blocks, 256, 0, s>>>(c->view(), seq, static_cast<int>(layer), static_cast<int>(head), d_idx,
                                              0, n, K, V);
  SA_CUDA_CHECK(cudaGetLastError());
  SA_CUDA_CHECK(cudaFreeAsync(d_idx, s));
  return SA_OK;
}

SA_API sa_status sa_kv_read(const sa_cache* c, int32_t seq, int64_t layer, int64_t head, int64_t begin, int64_t n,
                            float* K, float* V, void* stream) {
  if (sa_status st = check_seq(c, seq)) return st;
  if (layer < 0 || layer >= c->n_layers || head < 0 || head >= c->n_kv_heads)
    return fail(SA_OUT_OF_RANGE, "layer/head out of range");
  if (begin < 0 || n < 0 || begin + n > c->len[seq]) return fail(SA_OUT_OF_RANGE, "rows beyond store length");
  if (n == 0) return SA_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = static_cast<int>(std::min<int64_t>((n * 128 + 255) / 256, 4096));
  sa::read_rows_kernel<<<blocks, 256, 0, s>>>(c->view(), seq, static_cast<int>(layer), static_cast<int>(head), nullptr,
                                              begin, n, K, V);
  SA_CUDA_CHECK(cudaGetLastError());
  return SA_OK;
}

}  // extern "C"
