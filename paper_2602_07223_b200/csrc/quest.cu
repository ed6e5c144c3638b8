// quest.cu — the paper's baseline selectors on the GPU: QuestLike and Window.
//
// Reference: KvStore page summaries (kv_store.cpp:90-139: per page of `page_size` tokens the
// elementwise min and max of the keys, refreshed on the tail page), select_quest
// (selection.cpp:224-274: page upper bound sum_h sum_d max(q_hd * min_d, q_hd * max_d), pages in
// descending bound order (ties -> lower page), tokens taken page by page in ascending position until
// k, output sorted) and select_window (selection.cpp:209-222: sink tokens + the last `window`).
//
// Summaries live in the cache beside K/V ([layer][page][KV head][P / qpage][128] bf16 min and max;
// min / max of bf16 keys are exact in bf16).  quest_summarize recomputes a token range's quest pages
// (the cache refreshes lazily: rows changed by appends / fused appends / truncation mark pages
// stale, the next Quest selection recomputes them first).  quest_bounds: one warp per quest page.
// quest_pick: one CTA per sequence: a radix select finds the key of the last page that can be
// needed (rank ceil(k/qpage)+1), only the pages at or above it are sorted (bitonic, shared memory),
// a block scan of their token counts in rank order decides what is taken, then a scan in page order
// writes the ascending position list.
#include "internal.h"

namespace sa {

__device__ __forceinline__ int64_t qsum_row(const CacheView& c, int qpage, int seq, int layer, int head, int64_t pos) {
  const int page = __ldg(c.block_table + static_cast<int64_t>(seq) * c.max_pages_per_seq + (pos >> c.page_shift));
  const int per_page = (1 << c.page_shift) / qpage;
  const int qp_in = static_cast<int>((pos & ((1 << c.page_shift) - 1)) / qpage);
  return ((static_cast<int64_t>(layer) * c.num_pages + page) * c.n_kv_heads + head) * per_page + qp_in;
}

// one thread per (layer, head, quest page in [qp_lo, qp_hi), d)
__global__ void quest_summarize_kernel(CacheView c, __nv_bfloat16* qmin, __nv_bfloat16* qmax, int qpage, int seq,
                                       int64_t qp_lo, int64_t n_qp, int64_t len) {
  const int64_t total = static_cast<int64_t>(c.n_layers) * c.n_kv_heads * n_qp * 128;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(i & 127);
    int64_t r = i >> 7;
    const int64_t qp = qp_lo + r % n_qp;
    r /= n_qp;
    const int head = static_cast<int>(r % c.n_kv_heads);
    const int layer = static_cast<int>(r / c.n_kv_heads);
    const int64_t begin = qp * qpage, end = min(begin + qpage, len);
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t pos = begin; pos < end; ++pos) {
      const float v = __bfloat162float(c.k[cache_row(c, seq, layer, head, static_cast<int>(pos)) * 128 + d]);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    const int64_t o = qsum_row(c, qpage, seq, layer, head, begin) * 128 + d;
    qmin[o] = __float2bfloat16_rn(mn);
    qmax[o] = __float2bfloat16_rn(mx);
  }
}

cudaError_t launch_quest_summarize(const CacheView& c, const __nv_bfloat16* qmin, const __nv_bfloat16* qmax, int qpage,
                                   int seq, int64_t tok_lo, int64_t len, cudaStream_t s) {
  const int64_t qp_lo = tok_lo / qpage, qp_hi = (len + qpage - 1) / qpage;
  if (qp_hi <= qp_lo) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(c.n_layers) * c.n_kv_heads * (qp_hi - qp_lo) * 128;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  quest_summarize_kernel<<<blocks, 256, 0, s>>>(c, const_cast<__nv_bfloat16*>(qmin), const_cast<__nv_bfloat16*>(qmax),
                                                 qpage, seq, qp_lo, qp_hi - qp_lo, len);
  return cudaGetLastError();
}

// one warp per (quest page, sequence): bound = sum_h double(sum_d max(q*min, q*max))  (fp32 per head)
__global__ void __launch_bounds__(256) quest_bounds_kernel(CacheView c, const __nv_bfloat16* qmin,
                                                           const __nv_bfloat16* qmax, int qpage, int layer,
                                                           const int32_t* seq_ids, const int32_t* p0s, int Hq, int G,
                                                           const __nv_bfloat16* q, double* bounds, int64_t ld) {
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t qp = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  const int p0 = p0s[b];
  const int64_t n_qp = (p0 + qpage - 1) / qpage;
  if (qp >= n_qp) return;
  const int seq = seq_ids[b];
  // each lane owns 4 dims: its per-head partials (fp32 over 4 dims) accumulate in double across the
  // heads, and one butterfly reduces the lanes (the reference's per-head fp32 sum over d is an
  // unpinned Eigen order; this order differs from it at the 1e-7 level, far inside the tie band)
  double acc = 0.0;
#pragma unroll 4
  for (int g = 0; g < c.n_kv_heads; ++g) {
    const int64_t o = qsum_row(c, qpage, seq, layer, g, qp * qpage) * 128 + lane * 4;
    const uint2 mnr = *reinterpret_cast<const uint2*>(qmin + o), mxr = *reinterpret_cast<const uint2*>(qmax + o);
    const float2 mn01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&mnr.x));
    const float2 mn23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&mnr.y));
    const float2 mx01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&mxr.x));
    const float2 mx23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&mxr.y));
    const float mn[4] = {mn01.x, mn01.y, mn23.x, mn23.y}, mx[4] = {mx01.x, mx01.y, mx23.x, mx23.y};
#pragma unroll 4
    for (int hh = 0; hh < G; ++hh) {
      const uint2 qr = __ldg(reinterpret_cast<const uint2*>(q + (static_cast<size_t>(b) * Hq + g * G + hh) * 128 + lane * 4));
      const float2 q01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qr.x));
      const float2 q23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qr.y));
      const float qv[4] = {q01.x, q01.y, q23.x, q23.y};
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) t += fmaxf(qv[e] * mn[e], qv[e] * mx[e]);
      acc += static_cast<double>(t);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) bounds[static_cast<size_t>(b) * ld + qp] = acc;
}

__device__ __forceinline__ unsigned long long dkey(double v) {  // order-preserving (desc by value)
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v + 0.0));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// one CTA (1024 threads) per sequence; n_qp <= kQuestMaxPages
constexpr int kQuestMaxPages = 8192;  // shared-memory sort: 64K tokens at the default 8-token pages

__global__ void __launch_bounds__(1024) quest_pick_kernel(const int32_t* p0s, int qpage, const double* bounds, int64_t ld,
                                                          double ratio, int64_t k_min, int k_cap, int32_t* idx,
                                                          int32_t* k_out) {
  extern __shared__ unsigned long long qsm[];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int p0 = p0s[b];
  const int n_qp = (p0 + qpage - 1) / qpage;
  int npow = 1;
  while (npow < n_qp) npow <<= 1;
  unsigned long long* key = qsm;                                   // [npow]
  int* take = reinterpret_cast<int*>(qsm + npow);                  // [n_qp] tokens taken per page
  __shared__ int wsum[32];
  __shared__ int s_rank, s_before;
  long long k = llround(ratio * static_cast<double>(p0));
  k = min(static_cast<long long>(p0), max(k, static_cast<long long>(k_min)));
  if (k > k_cap) k = k_cap;
  for (int i = tid; i < n_qp; i += 1024) key[i] = dkey(bounds[static_cast<size_t>(b) * ld + i]);
  for (int i = tid; i < n_qp; i += 1024) take[i] = 0;
  __syncthreads();
  // (1) radix select (8-bit digits, MSB first) of T = the m_need-th largest key: only pages ranked
  // before it can be taken (m_need covers k tokens even if the partial last page ranks among them)
  const int m_need = static_cast<int>(min(static_cast<long long>(n_qp), (k + qpage - 1) / qpage + 1));
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_rem, s_nc;
  if (tid == 0) {
    s_prefix = 0ull;
    s_rem = m_need;
    s_nc = 0;
  }
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    for (int i = tid; i < n_qp; i += 1024)
      if ((key[i] & mask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (tid < 32) {  // lane l owns bins 255-8l .. 248-8l (descending)
      unsigned int cnt[8], sum = 0u;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cnt[e] = hist[255 - 8 * tid - e];
        sum += cnt[e];
      }
      unsigned int incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (tid >= off) incl += t;
      }
      const int rem = s_rem;
      const unsigned int hit = __ballot_sync(0xffffffffu, incl >= static_cast<unsigned int>(rem));
      const int l = __ffs(hit) - 1;  // first lane whose bins reach the remaining rank
      if (tid == l) {
        unsigned int above = incl - sum;
        int d = 255 - 8 * l;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (above + cnt[e] >= static_cast<unsigned int>(rem)) {
            d = 255 - 8 * l - e;
            break;
          }
          above += cnt[e];
        }
        s_prefix = prefix | (static_cast<unsigned long long>(d) << shift);
        s_rem = rem - static_cast<int>(above);
      }
    }
    mask |= 0xFFull << shift;
    __syncthreads();
  }
  const unsigned long long T = s_prefix;
  // (2) candidates: every page with key >= T (ties with T included), compacted, then sorted
  unsigned long long* ckey = reinterpret_cast<unsigned long long*>(take + n_qp + (n_qp & 1));  // [npow]
  int* cpg = reinterpret_cast<int*>(ckey + npow);                                                // [npow]
  for (int i = tid; i < n_qp; i += 1024)
    if (key[i] >= T) {
      const int slot = atomicAdd(&s_nc, 1);
      ckey[slot] = key[i];
      cpg[slot] = i;
    }
  __syncthreads();
  const int nc = s_nc;
  int cpow = 1;
  while (cpow < nc) cpow <<= 1;
  for (int i = nc + tid; i < cpow; i += 1024) {
    ckey[i] = 0ull;  // padding sorts last
    cpg[i] = 0x7fffffff;
  }
  __syncthreads();
  // bitonic sort of the candidates: descending key, ties -> ascending page
  for (int size = 2; size <= cpow; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < cpow / 2; i += 1024) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long ka = ckey[lo], kb = ckey[hi];
        const int ia = cpg[lo], ib = cpg[hi];
        const bool a_first = ka > kb || (ka == kb && ia < ib);
        if (a_first != up) {
          ckey[lo] = kb;
          ckey[hi] = ka;
          cpg[lo] = ib;
          cpg[hi] = ia;
        }
      }
      __syncthreads();
    }
  int* pg_r = cpg;          // pages in rank order (the first nc ranks)
  const int n_rank = nc;
  // rank order: cumulative token counts; rank r* = first rank where the running total reaches k
  const int per_r = (n_rank + 1023) / 1024;
  int loc = 0;
  for (int q = 0; q < per_r; ++q) {
    const int r = tid * per_r + q;
    if (r < n_rank) loc += min(qpage, p0 - pg_r[r] * qpage);
  }
  const int lane = tid & 31, warp = tid >> 5;
  int incl = loc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  if (tid == 0) s_rank = -1;
  __syncthreads();
  if (warp == 0) {
    const int v = wsum[lane];
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += t;
    }
    wsum[lane] = x - v;
  }
  __syncthreads();
  int run = wsum[warp] + incl - loc;  // tokens in ranks before this thread's first rank
  for (int q = 0; q < per_r && k > 0; ++q) {
    const int r = tid * per_r + q;
    if (r >= n_rank) break;
    const int c = min(qpage, p0 - pg_r[r] * qpage);
    if (run < k) take[pg_r[r]] = static_cast<int>(min(static_cast<long long>(c), k - run));
    run += c;
  }
  __syncthreads();
  const int per = (n_qp + 1023) / 1024;
  // page order: positions p*qpage .. p*qpage + take[p) - 1, ascending
  loc = 0;
  for (int q = 0; q < per; ++q) {
    const int pp = tid * per + q;
    if (pp < n_qp) loc += take[pp];
  }
  incl = loc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = wsum[lane];
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += t;
    }
    wsum[lane] = x - v;
    if (lane == 31) s_before = x;
  }
  __syncthreads();
  int w = wsum[warp] + incl - loc;
  int32_t* out = idx + static_cast<size_t>(b) * k_cap;
  for (int q = 0; q < per; ++q) {
    const int pp = tid * per + q;
    if (pp >= n_qp) break;
    for (int t = 0; t < take[pp]; ++t) out[w++] = pp * qpage + t;
  }
  if (tid == 0) k_out[b] = s_before;
}

cudaError_t launch_quest_select(const CacheView& c, const __nv_bfloat16* qmin, const __nv_bfloat16* qmax, int qpage,
                                int layer, const int32_t* seq_ids, const int32_t* p0, int B, int Hq, int G,
                                const __nv_bfloat16* q, double ratio, int64_t k_min, int k_cap, double* bounds,
                                int64_t max_qpages, int32_t* idx, int32_t* k_out, cudaStream_t s) {
  if (max_qpages > kQuestMaxPages) return cudaErrorInvalidValue;
  dim3 g1(static_cast<unsigned>((std::max<int64_t>(max_qpages, 1) + 7) / 8), B);
  quest_bounds_kernel<<<g1, 256, 0, s>>>(c, qmin, qmax, qpage, layer, seq_ids, p0, Hq, G, q, bounds, max_qpages);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int npow = 1;
  while (npow < max_qpages) npow <<= 1;
  const size_t smem = static_cast<size_t>(npow) * 8 + (static_cast<size_t>(max_qpages) + 1) * 4 +
                      static_cast<size_t>(npow) * 12 + 16;
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  if (func_attrs_needed(attr_mask, &dev)) {
    e = cudaFuncSetAttribute(quest_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return e;
    func_attrs_done(attr_mask, dev);
  }
  quest_pick_kernel<<<B, 1024, smem, s>>>(p0, qpage, bounds, max_qpages, ratio, k_min, k_cap, idx, k_out);
  return cudaGetLastError();
}

// select_window: [0, min(sink, p)) ++ [max(p - window, sink_end), p)
__global__ void window_kernel(const int32_t* p0s, int64_t sink, int64_t window, int k_cap, int32_t* idx,
                              int32_t* k_out) {
  const int b = blockIdx.x;
  const int64_t p = p0s[b];
  const int64_t sink_end = min(sink, p), win_begin = max(p - window, sink_end);
  const int64_t n = sink_end + (p - win_begin);
  int32_t* out = idx + static_cast<size_t>(b) * k_cap;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    out[i] = static_cast<int32_t>(i < sink_end ? i : win_begin + (i - sink_end));
  if (threadIdx.x == 0) k_out[b] = static_cast<int32_t>(n);
}

cudaError_t launch_window(const int32_t* p0, int B, int64_t sink, int64_t window, int k_cap, int32_t* idx,
                          int32_t* k_out, cudaStream_t s) {
  window_kernel<<<B, 256, 0, s>>>(p0, sink, window, k_cap, idx, k_out);
  return cudaGetLastError();
}

}  // namespace sa
