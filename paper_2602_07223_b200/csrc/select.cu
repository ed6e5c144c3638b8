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
// MSB-first 8-bit radix select (4 passes, warp-aggregated shared-memory histograms); the output
// pass takes every key above the threshold plus the lowest-index keys equal to it, writing
// indices through a block-wide exclusive scan so the list comes out ascending without a sort.
#include <cub/block/block_scan.cuh>

#include "internal.h"

namespace sa {

constexpr int kSelThreads = 1024;
constexpr int kSelSubHist = 8;  // sub-histograms (4 warps each) to cut atomic contention

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0 (the reference compares doubles)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams p) {
  __shared__ uint32_t hist[kSelSubHist][256];
  __shared__ uint32_t total[256];
  __shared__ long long s_k;
  __shared__ uint32_t s_prefix;
  __shared__ long long s_rem;
  using Scan = cub::BlockScan<int, kSelThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;

  const int set = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int n = p.p0[b];
  uint32_t* keys = p.keys + (static_cast<size_t>(b) * p.n_sets + set) * p.ld_scores;
  const int sub = (tid >> 5) % kSelSubHist;

  long long k;
  {
    const long long wanted = llround(p.ratio * static_cast<double>(n));
    k = min(static_cast<long long>(n), max(wanted, static_cast<long long>(p.k_min)));
    if (k > p.k_cap) k = p.k_cap;  // host sizes k_cap from the largest p0; never binds
  }

  for (int i = tid; i < kSelSubHist * 256; i += kSelThreads) (&hist[0][0])[i] = 0;
  __syncthreads();
  // Pass 0: aggregate, build keys, top-digit histogram.
  const float* sc = p.scores + static_cast<size_t>(b) * p.Hkv * p.ld_scores;
  for (int i = tid; i < n; i += kSelThreads) {
    double sum = 0.0;
    if (p.n_sets == 1) {
      for (int g = 0; g < p.Hkv; ++g) sum += static_cast<double>(__ldg(sc + static_cast<size_t>(g) * p.ld_scores + i));
    } else {
      sum = static_cast<double>(__ldg(sc + static_cast<size_t>(set) * p.ld_scores + i));
    }
    const uint32_t u = order_key(static_cast<float>(sum / p.count));
    keys[i] = u;
    atomicAdd(&hist[sub][u >> 24], 1u);
  }
  __syncthreads();

  uint32_t prefix = 0, pmask = 0;
  long long rem = k;
  for (int pass = 0; pass < 4 && k > 0; ++pass) {
    const int shift = 24 - 8 * pass;
    if (pass > 0) {
      for (int i = tid; i < kSelSubHist * 256; i += kSelThreads) (&hist[0][0])[i] = 0;
      __syncthreads();
      for (int i = tid; i < n; i += kSelThreads) {
        const uint32_t u = keys[i];
        if ((u & pmask) == prefix) atomicAdd(&hist[sub][(u >> shift) & 255u], 1u);
      }
      __syncthreads();
    }
    if (tid < 256) {
      uint32_t c = 0;
#pragma unroll
      for (int s = 0; s < kSelSubHist; ++s) c += hist[s][tid];
      total[tid] = c;
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins 8l..8l+7; find the bin holding the rem-th largest (scan from the top).
      uint32_t loc = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) loc += total[8 * tid + q];
      uint32_t suf = loc;  // inclusive suffix sum over lanes >= tid
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, suf, off);
        if (tid + off < 32) suf += v;
      }
      const long long above = static_cast<long long>(suf - loc);
      const bool mine = above < rem && rem <= static_cast<long long>(suf);
      if (mine) {
        long long acc = above;
        for (int q = 7; q >= 0; --q) {
          const uint32_t c = total[8 * tid + q];
          if (acc + c >= rem) {
            s_prefix = prefix | (static_cast<uint32_t>(8 * tid + q) << shift);
            s_rem = rem - acc;
            break;
          }
          acc += c;
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    rem = s_rem;
    pmask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;
  // The threshold key: every key > T is taken plus the `rem` lowest-index keys == T.  A -inf
  // threshold takes nothing equal to it (selection.cpp:153).
  const long long take_eq_total = (k > 0 && T != order_key(-INFINITY)) ? rem : 0;
  const uint32_t gt_floor = k > 0 ? T : 0xFFFFFFFFu;  // k == 0 selects nothing

  // Output pass over contiguous per-thread segments (index order preserved by the scans).
  const int seg = (n + kSelThreads - 1) / kSelThreads;
  const int beg = min(n, tid * seg), end = min(n, beg + seg);
  int gt = 0, eq = 0;
  for (int i = beg; i < end; ++i) {
    const uint32_t u = keys[i];
    gt += (k > 0) && (u > gt_floor);
    eq += (k > 0) && (u == T);
  }
  int eq_base;
  Scan(scan_tmp).ExclusiveSum(eq, eq_base);
  __syncthreads();
  const int take_eq = static_cast<int>(max(0LL, min(static_cast<long long>(eq), take_eq_total - eq_base)));
  int out_base, n_sel;
  Scan(scan_tmp).ExclusiveSum(gt + take_eq, out_base, n_sel);
  int32_t* out = p.idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  int w = out_base, taken = 0;
  for (int i = beg; i < end; ++i) {
    const uint32_t u = keys[i];
    if (k > 0 && u > gt_floor) {
      out[w++] = i;
    } else if (k > 0 && u == T && taken < take_eq) {
      out[w++] = i;
      ++taken;
    }
  }
  if (tid == 0) p.k_out[b * p.n_sets + set] = n_sel;
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
  dim3 grid(p.n_sets, p.B);
  select_kernel<<<grid, kSelThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace sa
