// select.cu — score aggregation + exact top-k selection (one CTA per (sequence, set)).
//
// Reference: score_columns (selection.cpp:89-108): score_i = sum over heads/rows of double(l) /
// count; selection_k (selection.cpp:63-66); topk_indices (selection.cpp:137-158): k largest,
// ties toward the lower index, -inf never selected, returned ascending.
//
// The verify kernel already emitted per-KV-head raw column sums (fp32).  Here they are summed
// over the set's KV heads in fixed order in double, divided by the term count in double, and
// rounded once to an fp32 key (keys that differ only beyond fp32 precision tie and fall to the
// lower index — inside the north star's tie tolerance).  The k-th largest key is found by an
// MSB-first 8-bit radix select (4 passes, sub-histograms in shared memory); the output pass walks
// the keys in index order, 4096 per round, taking every key above the threshold plus the
// lowest-index keys equal to it, with block-wide scans giving each selected index its output
// slot — so the list comes out ascending without a sort.
//
// Keys live in shared memory when p <= kSmemKeys (all BASELINE configs up to 48K columns) and in
// an L2-resident global workspace otherwise.
#include "internal.h"

namespace sa {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelSubHist = 8;
constexpr int kSmemKeys = 48 * 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0 (the reference compares doubles)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct SelShared {
  uint32_t hist[kSelSubHist][256];
  uint32_t total[256];
  int warp_sum[kSelWarps];
  int warp_off[kSelWarps];
  int block_total;
  uint32_t prefix;
  long long rem;
};

// Exclusive block scan of per-thread counts (thread order == index order).
__device__ __forceinline__ int block_excl_scan(SelShared& sh, int v, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) sh.warp_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int ws = sh.warp_sum[lane];
    int wi = ws;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += t;
    }
    sh.warp_off[lane] = wi - ws;
    if (lane == 31) sh.block_total = wi;
  }
  __syncthreads();
  total = sh.block_total;
  const int r = sh.warp_off[warp] + incl - v;
  __syncthreads();  // sh reusable by the next scan
  return r;
}

template <bool kKeysInSmem>
__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams p) {
  extern __shared__ uint4 dyn_smem[];
  __shared__ SelShared sh;
  const int set = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int n = p.p0[b];
  uint32_t* keys = kKeysInSmem ? reinterpret_cast<uint32_t*>(dyn_smem)
                               : p.keys + (static_cast<size_t>(b) * p.n_sets + set) * p.ld_scores;
  const int sub = (tid >> 5) % kSelSubHist;

  long long k;
  {
    const long long wanted = llround(p.ratio * static_cast<double>(n));
    k = min(static_cast<long long>(n), max(wanted, static_cast<long long>(p.k_min)));
    if (k > p.k_cap) k = p.k_cap;  // host sizes k_cap from the largest p0; never binds
  }
  for (int i = tid; i < kSelSubHist * 256; i += kSelThreads) (&sh.hist[0][0])[i] = 0;
  __syncthreads();

  // Pass 0: aggregate over the set's KV heads (double, fixed order), build keys + top digit.
  const float* sc = p.scores + static_cast<size_t>(b) * p.Hkv * p.ld_scores;
  const int g0 = p.n_sets == 1 ? 0 : set;
  const int ng = p.n_sets == 1 ? p.Hkv : 1;
  const double inv_count = 1.0 / p.count;  // only used to pre-check; exact division below
  (void)inv_count;
  const int n4 = n >> 2;
  for (int i4 = tid; i4 < n4; i4 += kSelThreads) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int g = 0;
    for (; g + 4 <= ng; g += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = __ldg(reinterpret_cast<const float4*>(sc + static_cast<size_t>(g0 + g + u) * p.ld_scores) + i4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s0 += static_cast<double>(v[u].x);
        s1 += static_cast<double>(v[u].y);
        s2 += static_cast<double>(v[u].z);
        s3 += static_cast<double>(v[u].w);
      }
    }
    for (; g < ng; ++g) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(sc + static_cast<size_t>(g0 + g) * p.ld_scores) + i4);
      s0 += static_cast<double>(v.x);
      s1 += static_cast<double>(v.y);
      s2 += static_cast<double>(v.z);
      s3 += static_cast<double>(v.w);
    }
    uint4 u;
    u.x = order_key(static_cast<float>(s0 / p.count));
    u.y = order_key(static_cast<float>(s1 / p.count));
    u.z = order_key(static_cast<float>(s2 / p.count));
    u.w = order_key(static_cast<float>(s3 / p.count));
    reinterpret_cast<uint4*>(keys)[i4] = u;
    atomicAdd(&sh.hist[sub][u.x >> 24], 1u);
    atomicAdd(&sh.hist[sub][u.y >> 24], 1u);
    atomicAdd(&sh.hist[sub][u.z >> 24], 1u);
    atomicAdd(&sh.hist[sub][u.w >> 24], 1u);
  }
  for (int i = 4 * n4 + tid; i < n; i += kSelThreads) {
    double s = 0.0;
    for (int g = 0; g < ng; ++g) s += static_cast<double>(__ldg(sc + static_cast<size_t>(g0 + g) * p.ld_scores + i));
    const uint32_t u = order_key(static_cast<float>(s / p.count));
    keys[i] = u;
    atomicAdd(&sh.hist[sub][u >> 24], 1u);
  }
  __syncthreads();

  uint32_t prefix = 0, pmask = 0;
  long long rem = k;
  for (int pass = 0; pass < 4 && k > 0; ++pass) {
    const int shift = 24 - 8 * pass;
    if (pass > 0) {
      for (int i = tid; i < kSelSubHist * 256; i += kSelThreads) (&sh.hist[0][0])[i] = 0;
      __syncthreads();
      for (int i4 = tid; i4 < n4; i4 += kSelThreads) {
        const uint4 u = reinterpret_cast<const uint4*>(keys)[i4];
        if ((u.x & pmask) == prefix) atomicAdd(&sh.hist[sub][(u.x >> shift) & 255u], 1u);
        if ((u.y & pmask) == prefix) atomicAdd(&sh.hist[sub][(u.y >> shift) & 255u], 1u);
        if ((u.z & pmask) == prefix) atomicAdd(&sh.hist[sub][(u.z >> shift) & 255u], 1u);
        if ((u.w & pmask) == prefix) atomicAdd(&sh.hist[sub][(u.w >> shift) & 255u], 1u);
      }
      for (int i = 4 * n4 + tid; i < n; i += kSelThreads) {
        const uint32_t u = keys[i];
        if ((u & pmask) == prefix) atomicAdd(&sh.hist[sub][(u >> shift) & 255u], 1u);
      }
      __syncthreads();
    }
    if (tid < 256) {
      uint32_t c = 0;
#pragma unroll
      for (int s = 0; s < kSelSubHist; ++s) c += sh.hist[s][tid];
      sh.total[tid] = c;
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins 8l..8l+7; find the bin holding the rem-th largest key (from the top).
      uint32_t loc = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) loc += sh.total[8 * tid + q];
      uint32_t suf = loc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, suf, off);
        if (tid + off < 32) suf += v;
      }
      const long long above = static_cast<long long>(suf - loc);
      if (above < rem && rem <= static_cast<long long>(suf)) {
        long long acc = above;
        for (int q = 7; q >= 0; --q) {
          const uint32_t c = sh.total[8 * tid + q];
          if (acc + c >= rem) {
            sh.prefix = prefix | (static_cast<uint32_t>(8 * tid + q) << shift);
            sh.rem = rem - acc;
            break;
          }
          acc += c;
        }
      }
    }
    __syncthreads();
    prefix = sh.prefix;
    rem = sh.rem;
    pmask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;
  // Take every key > T plus the `rem` lowest-index keys == T; a -inf threshold takes nothing equal
  // to it (selection.cpp:153).  k == 0 selects nothing.
  const bool any = k > 0;
  const long long take_eq_total = (any && T != order_key(-INFINITY)) ? rem : 0;

  int32_t* out = p.idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  int eq_run = 0, sel_run = 0;
  for (int base = 0; base < n; base += 4 * kSelThreads) {
    const int i0 = base + 4 * tid;
    uint32_t u[4];
    if (i0 + 3 < n) {
      const uint4 v = reinterpret_cast<const uint4*>(keys)[i0 >> 2];
      u[0] = v.x, u[1] = v.y, u[2] = v.z, u[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) u[e] = i0 + e < n ? keys[i0 + e] : 0u;
    }
    int eq = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) eq += (any && i0 + e < n && u[e] == T);
    int eq_tot;
    const int eq_before = eq_run + block_excl_scan(sh, eq, eq_tot);
    bool sel[4];
    int nsel = 0, er = eq_before;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool valid = any && i0 + e < n;
      const bool is_eq = valid && u[e] == T;
      sel[e] = valid && (u[e] > T || (is_eq && er < take_eq_total));
      er += is_eq;
      nsel += sel[e];
    }
    int sel_tot;
    int w = sel_run + block_excl_scan(sh, nsel, sel_tot);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (sel[e]) out[w++] = i0 + e;
    eq_run += eq_tot;
    sel_run += sel_tot;
  }
  if (tid == 0) p.k_out[b * p.n_sets + set] = sel_run;
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
  dim3 grid(p.n_sets, p.B);
  if (p.ld_scores <= kSmemKeys) {
    static bool attr = false;
    const int bytes = static_cast<int>(p.ld_scores * 4);
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kSmemKeys * 4);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    select_kernel<true><<<grid, kSelThreads, bytes, s>>>(p);
  } else {
    select_kernel<false><<<grid, kSelThreads, 0, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace sa
