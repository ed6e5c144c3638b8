// select.cu — score aggregation + exact top-k selection (one CTA per (sequence, set)).
//
// Reference: score_columns (selection.cpp:89-108): score_i = sum over heads/rows of double(l) /
// count; selection_k (selection.cpp:63-66); topk_indices (selection.cpp:137-158): k largest,
// ties toward the lower index, -inf never selected, returned ascending.
//
// Inputs (written by the verify kernel as a fused byproduct, no LogitMatrix):
//  - per-layer mode: one int64 fixed-point column sum per (sequence, column), accumulated by the
//    verify CTAs of all KV heads with integer atomics (order-independent, hence deterministic)
//    from each head's fp32 sum of its G x |rows| raw logits (2^32 units).  This kernel zeroes the
//    sums it consumes, re-arming the slot for the next verify.
//  - per-KV-head mode: the fp32 per-head column sums.
// Dividing by the positive term count is monotone, so the ordering key is the fp32 rounding of
// the sum itself (order_key: IEEE bits mapped to an unsigned order, -0 -> +0): columns whose
// scores differ only below fp32 resolution tie and fall to the lower index, inside the north
// star's tie tolerance.
//
// The k-th largest key is found by an MSB-first radix select over 12 + 10 + 10 bits (histograms in
// shared memory, two sub-histograms against same-bin contention, early exit once the threshold
// bin is taken whole).  The output pass is warp-ballot based: each warp owns a contiguous index
// range, counts keys above / equal to the threshold, one 32-entry scan gives every warp its output
// base, and a second sweep writes the selected indices in ascending order without a sort.
//
// Keys live in shared memory when p <= kSmemKeys and in an L2-resident global workspace otherwise.
#include "internal.h"

namespace sa {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSmemKeys = 40 * 1024;
constexpr int kBins1 = 4096;  // first digit: key bits [20, 32)
constexpr int kBins2 = 1024;  // then [10, 20) and [0, 10)
constexpr uint32_t kKeyNegInf = 0x007FFFFFu;  // order_key(-inf)

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0 (the reference compares doubles)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct SelShared {
  uint32_t hist[2][kBins1];
  uint32_t part[64];
  int wgt[kSelWarps], weq[kSelWarps];
  uint32_t bin;
  uint32_t bin_count;
  long long rem;
};

// Find the bin (of nb) holding the rem-th largest key; bins hold counts in sh.hist[0] (+hist[1]
// when `two`).  Thread t owns nb/1024 consecutive bins.  Writes sh.bin, sh.rem (rank inside the
// bin) and sh.bin_count.
__device__ __forceinline__ void find_bin(SelShared& sh, int nb, long long rem, bool two) {
  const int tid = threadIdx.x, per = nb / kSelThreads;
  uint32_t loc = 0;
  for (int q = 0; q < per; ++q) {
    const int bin = tid * per + q;
    const uint32_t c = sh.hist[0][bin] + (two ? sh.hist[1][bin] : 0u);
    sh.hist[0][bin] = c;
    loc += c;
  }
  // inclusive suffix sums over threads: warp shuffles, then the 32 warp totals
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t suf_w = loc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_down_sync(0xffffffffu, suf_w, off);
    if (lane + off < 32) suf_w += v;
  }
  if (lane == 0) sh.part[warp] = suf_w;  // warp total
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = sh.part[lane];
    uint32_t st = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_down_sync(0xffffffffu, st, off);
      if (lane + off < 32) st += v;
    }
    sh.part[32 + lane] = st - t;  // total of the warps after this one
  }
  __syncthreads();
  const long long suf = static_cast<long long>(suf_w) + sh.part[32 + warp];
  const long long above = suf - loc;
  if (above < rem && rem <= suf) {
    long long acc = above;
    for (int q = per - 1; q >= 0; --q) {
      const uint32_t c = sh.hist[0][tid * per + q];
      if (acc + c >= rem) {
        sh.bin = static_cast<uint32_t>(tid * per + q);
        sh.rem = rem - acc;
        sh.bin_count = c;
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
}

template <bool kFixed, bool kKeysInSmem>
__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams p) {
  extern __shared__ uint4 dyn_smem[];
  __shared__ SelShared sh;
  const int set = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // blockIdx.z: layer slot within a batched launch (per-slot strides; keys in shared memory only)
  const size_t z = blockIdx.z;
  long long* const p_score_fx = p.score_fx ? p.score_fx + z * p.zs_fx : nullptr;
  const float* const p_scores = p.scores ? p.scores + z * p.zs_scores : nullptr;
  int32_t* const p_idx = p.idx + z * p.zs_idx;
  int32_t* const p_k_out = p.k_out + z * p.zs_cnt;
  const int n = p.p0[b];
  uint32_t* keys = kKeysInSmem ? reinterpret_cast<uint32_t*>(dyn_smem)
                               : p.keys + (static_cast<size_t>(b) * p.n_sets + set) * p.ld_scores;
  long long k;
  {
    const long long wanted = llround(p.ratio * static_cast<double>(n));
    k = min(static_cast<long long>(n), max(wanted, static_cast<long long>(p.k_min)));
    if (k > p.k_cap) k = p.k_cap;  // host sizes k_cap from the largest p0; never binds
  }
  for (int i = tid; i < 2 * kBins1; i += kSelThreads) (&sh.hist[0][0])[i] = 0;
  __syncthreads();

  // ---- pass 1: keys + first-digit histogram
  uint32_t* h1 = sh.hist[warp & 1];
  if constexpr (kFixed) {
    long long* fx = p_score_fx + static_cast<size_t>(b) * p.ld_scores;
    const int n2 = n >> 1;
    for (int i2 = tid; i2 < n2; i2 += kSelThreads) {
      longlong2 v = __ldcg(reinterpret_cast<const longlong2*>(fx) + i2);
      __stcg(reinterpret_cast<longlong2*>(fx) + i2, make_longlong2(0, 0));  // re-arm the slot
      const uint32_t u0 = order_key(__ll2float_rn(v.x)), u1 = order_key(__ll2float_rn(v.y));
      reinterpret_cast<uint2*>(keys)[i2] = make_uint2(u0, u1);
      atomicAdd(&h1[u0 >> 20], 1u);
      atomicAdd(&h1[u1 >> 20], 1u);
    }
    for (int i = 2 * n2 + tid; i < n; i += kSelThreads) {
      const long long v = __ldcg(fx + i);
      fx[i] = 0;
      const uint32_t u = order_key(__ll2float_rn(v));
      keys[i] = u;
      atomicAdd(&h1[u >> 20], 1u);
    }
  } else {
    const float* sc = p_scores + (static_cast<size_t>(b) * p.Hkv + set) * p.ld_scores;
    const int n4 = n >> 2;
    for (int i4 = tid; i4 < n4; i4 += kSelThreads) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(sc) + i4);
      const uint4 u = make_uint4(order_key(v.x), order_key(v.y), order_key(v.z), order_key(v.w));
      reinterpret_cast<uint4*>(keys)[i4] = u;
      atomicAdd(&h1[u.x >> 20], 1u);
      atomicAdd(&h1[u.y >> 20], 1u);
      atomicAdd(&h1[u.z >> 20], 1u);
      atomicAdd(&h1[u.w >> 20], 1u);
    }
    for (int i = 4 * n4 + tid; i < n; i += kSelThreads) {
      const uint32_t u = order_key(__ldcg(sc + i));
      keys[i] = u;
      atomicAdd(&h1[u >> 20], 1u);
    }
  }
  __syncthreads();

  if (k <= 0) {  // nothing to select (the fixed-point slot has been re-armed above)
    if (tid == 0) p_k_out[b * p.n_sets + set] = 0;
    return;
  }
  // ---- radix select: threshold prefix T at resolution `shift`
  uint32_t T = 0;
  int shift = 32;
  long long rem = k;
  {
    find_bin(sh, kBins1, rem, true);
    T = sh.bin;
    shift = 20;
    rem = sh.rem;
    for (int lvl = 0; lvl < 2 && static_cast<long long>(sh.bin_count) != rem; ++lvl) {
      const int nshift = shift - 10;
      for (int i = tid; i < kBins2; i += kSelThreads) sh.hist[0][i] = sh.hist[1][i] = 0;
      __syncthreads();
      uint32_t* h = sh.hist[warp & 1];
      const int n4 = n >> 2;
      for (int i4 = tid; i4 < n4; i4 += kSelThreads) {
        const uint4 u = reinterpret_cast<const uint4*>(keys)[i4];
        if ((u.x >> shift) == T) atomicAdd(&h[(u.x >> nshift) & 1023u], 1u);
        if ((u.y >> shift) == T) atomicAdd(&h[(u.y >> nshift) & 1023u], 1u);
        if ((u.z >> shift) == T) atomicAdd(&h[(u.z >> nshift) & 1023u], 1u);
        if ((u.w >> shift) == T) atomicAdd(&h[(u.w >> nshift) & 1023u], 1u);
      }
      for (int i = 4 * n4 + tid; i < n; i += kSelThreads) {
        const uint32_t u = keys[i];
        if ((u >> shift) == T) atomicAdd(&h[(u >> nshift) & 1023u], 1u);
      }
      __syncthreads();
      find_bin(sh, kBins2, rem, true);
      T = (T << 10) | sh.bin;
      shift = nshift;
      rem = sh.rem;
    }
  }
  // Selected: (key >> shift) > T, plus the `rem` lowest-index keys with (key >> shift) == T; never
  // a -inf key (selection.cpp:153).  k == 0 selects nothing.
  const long long take_eq_ll = rem;

  // ---- output, common case: every key of the threshold bin is taken (no tie straddles the
  // boundary), so the selection is the predicate (key >> shift) >= T: ballot stream compaction,
  // warp w owning the contiguous range [w*R1, (w+1)*R1), 32 keys per step.
  if (static_cast<long long>(sh.bin_count) == take_eq_ll) {
    const int R1 = ((n + kSelThreads - 1) / kSelThreads) * 32;
    const int lo = warp * R1, hi = min(n, lo + R1);
    int cnt = 0;
    for (int base = lo; base < hi; base += 32) {
      const int i = base + lane;
      const uint32_t u = i < hi ? keys[i] : kKeyNegInf;
      cnt += __popc(__ballot_sync(0xffffffffu, u != kKeyNegInf && (u >> shift) >= T));
    }
    if (lane == 0) sh.wgt[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
      const int c = sh.wgt[lane];
      int ci = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ci, off);
        if (lane >= off) ci += t;
      }
      sh.wgt[lane] = ci - c;
      if (lane == 31) p_k_out[b * p.n_sets + set] = ci;
    }
    __syncthreads();
    int32_t* out = p_idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
    int run = sh.wgt[warp];
    const unsigned lt = (1u << lane) - 1u;
    for (int base = lo; base < hi; base += 32) {
      const int i = base + lane;
      const uint32_t u = i < hi ? keys[i] : kKeyNegInf;
      const bool sel = u != kKeyNegInf && (u >> shift) >= T;
      const unsigned bs = __ballot_sync(0xffffffffu, sel);
      if (sel) out[run + __popc(bs & lt)] = i;
      run += __popc(bs);
    }
    return;
  }

  // ---- output, general case (ties straddle the boundary: the lowest-index equal keys win):
  // warp w owns [w*R, min(n, (w+1)*R)), R a multiple of 128; lane l takes keys
  // [base + 4l, base + 4l + 4) of each 128-key step, so (lane, element) order is index order.
  const int R = ((n + kSelWarps * 128 - 1) / (kSelWarps * 128)) * 128;
  const int w_lo = warp * R, w_hi = min(n, w_lo + R);
  const int take_eq = static_cast<int>(take_eq_ll);
  auto classify = [&](int i0, int& cg, int& ce, uint32_t (&u)[4]) {
    if (i0 + 3 < w_hi) {
      const uint4 v = reinterpret_cast<const uint4*>(keys)[i0 >> 2];
      u[0] = v.x, u[1] = v.y, u[2] = v.z, u[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) u[e] = i0 + e < w_hi ? keys[i0 + e] : kKeyNegInf;
    }
    cg = ce = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t d = u[e] >> shift;
      const bool ok = u[e] != kKeyNegInf;
      cg += ok && d > T;
      ce += ok && d == T;
    }
  };
  int gt = 0, eq = 0;
  for (int base = w_lo; base < w_hi; base += 128) {
    uint32_t u[4];
    int cg, ce;
    classify(base + 4 * lane, cg, ce, u);
    gt += cg;
    eq += ce;
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  if (lane == 0) {
    sh.wgt[warp] = gt;
    sh.weq[warp] = eq;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scans of the warps' counts
    const int g = sh.wgt[lane], e = sh.weq[lane];
    int gi = g, ei = e;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int tg = __shfl_up_sync(0xffffffffu, gi, off), te = __shfl_up_sync(0xffffffffu, ei, off);
      if (lane >= off) {
        gi += tg;
        ei += te;
      }
    }
    sh.wgt[lane] = gi - g;
    sh.weq[lane] = ei - e;
    if (lane == 31) p_k_out[b * p.n_sets + set] = gi + min(ei, take_eq);
  }
  __syncthreads();
  int32_t* out = p_idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  int gt_run = sh.wgt[warp], eq_run = sh.weq[warp];
  for (int base = w_lo; base < w_hi; base += 128) {
    const int i0 = base + 4 * lane;
    uint32_t u[4];
    int cg, ce;
    classify(i0, cg, ce, u);
    // warp-exclusive scan of the packed (gt | eq << 16) counts
    const int packed = cg | (ce << 16);
    int incl = packed;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += t;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - packed;
    int g_before = gt_run + (excl & 0xFFFF), e_before = eq_run + (excl >> 16);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t d = u[e] >> shift;
      const bool ok = u[e] != kKeyNegInf;
      const bool is_gt = ok && d > T, is_eq = ok && d == T;
      // selected before this key = gt before + min(eq before, take_eq)
      if (is_gt || (is_eq && e_before < take_eq)) out[g_before + min(e_before, take_eq)] = i0 + e;
      g_before += is_gt;
      e_before += is_eq;
    }
    gt_run += tot & 0xFFFF;
    eq_run += tot >> 16;
  }
}

// ------------------------------------------------------------------------------------------------
// select_cluster_kernel: the same selection spread over a cluster of kCsC CTAs (one selection per
// cluster; CTA c holds columns [c*S, (c+1)*S) in registers, S = 512 * KPT): the single-CTA select above
// is instruction bound (~100 instructions per key at ~2 IPC on one SM).  Radix digits are
// data-adaptive: 8-bit digits of (key - min) over the finite keys' range.  Every exchange is a push:
// each CTA writes its statistics / histogram / counts into every CTA's inbox with st.async (remote
// shared stores completing as transaction bytes on the receiver's mbarrier), so there is no cluster
// barrier (and none of its GPU-scope fence) inside the passes; every CTA sums the same kCsC copies
// in the same order and finds the same threshold bin.  Output: each CTA compacts its own columns
// with ballots (ascending), at the offset given by the counts of the CTAs before it; exact ties at the
// threshold go to the lowest indices (selection.cpp:145-156).
constexpr int kCsC = 8;
constexpr int kCsThreads = 512;
constexpr int kCsWarps = kCsThreads / 32;
constexpr int kCsBins = 256;
constexpr int kCsBits = 8;

struct CsShared {
  uint32_t hist_in[2][kCsC][kCsBins];  // per pass parity: every CTA's histogram (pushed)
  uint32_t hist[kCsBins];              // this CTA's histogram of the current pass
  uint4 stat_in[kCsC];                 // every CTA's (min, max, finite count, -) (pushed)
  int4 cnt_in[kCsC];                   // every CTA's (gt, eq, -, -) output counts (pushed)
  uint64_t bar_stat, bar_cnt, bar_hist[2];
  uint32_t wmin[kCsWarps], wmax[kCsWarps];
  int wgt[kCsWarps], weq[kCsWarps];
  uint32_t part[16];
  uint32_t gstat[4];
  int off[2];
  uint32_t bin, bin_count;
  long long rem;
};

template <bool kFixed, int KPT>
__global__ void __launch_bounds__(kCsThreads) select_cluster_kernel(const SelectParams p) {
  constexpr int E = kFixed ? 2 : 4;  // keys per vector load
  constexpr int J = KPT / E;
  constexpr int kWarpSpan = 32 * KPT;
  constexpr int kCtaSpan = kCsWarps * kWarpSpan;
  __shared__ __align__(16) CsShared sh;
  const int c = blockIdx.x % kCsC, set = blockIdx.x / kCsC, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t z = blockIdx.z;
  int32_t* const p_idx = p.idx + z * p.zs_idx;
  int32_t* const p_k_out = p.k_out + z * p.zs_cnt;
  const int n = p.p0[b];
  const int wbase = c * kCtaSpan + warp * kWarpSpan;
  if (tid == 0) {
    mbar_init(&sh.bar_stat, 1);
    mbar_init(&sh.bar_cnt, 1);
    mbar_init(&sh.bar_hist[0], 1);
    mbar_init(&sh.bar_hist[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < kCsBins; i += kCsThreads) sh.hist[i] = 0;
  cluster_arrive_release();  // inbox barriers initialised (waited on before the first push)
  uint32_t u[KPT];
  if constexpr (kFixed) {
    long long* fx = p.score_fx + z * p.zs_fx + static_cast<size_t>(b) * p.ld_scores;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int i0 = wbase + 64 * j + 2 * lane;
      long long v0 = 0, v1 = 0;
      if (i0 + 1 < n) {
        const longlong2 v = __ldcg(reinterpret_cast<const longlong2*>(fx + i0));
        __stcg(reinterpret_cast<longlong2*>(fx + i0), make_longlong2(0, 0));  // re-arm the slot
        v0 = v.x;
        v1 = v.y;
      } else if (i0 < n) {
        v0 = __ldcg(fx + i0);
        fx[i0] = 0;
      }
      u[2 * j] = i0 < n ? order_key(__ll2float_rn(v0)) : kKeyNegInf;
      u[2 * j + 1] = i0 + 1 < n ? order_key(__ll2float_rn(v1)) : kKeyNegInf;
    }
  } else {
    const float* sc = p.scores + z * p.zs_scores + (static_cast<size_t>(b) * p.Hkv + set) * p.ld_scores;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int i0 = wbase + 128 * j + 4 * lane;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + 3 < n) {
        v = __ldcg(reinterpret_cast<const float4*>(sc + i0));
      } else {
        if (i0 < n) v.x = __ldcg(sc + i0);
        if (i0 + 1 < n) v.y = __ldcg(sc + i0 + 1);
        if (i0 + 2 < n) v.z = __ldcg(sc + i0 + 2);
      }
      u[4 * j] = i0 < n ? order_key(v.x) : kKeyNegInf;
      u[4 * j + 1] = i0 + 1 < n ? order_key(v.y) : kKeyNegInf;
      u[4 * j + 2] = i0 + 2 < n ? order_key(v.z) : kKeyNegInf;
      u[4 * j + 3] = i0 + 3 < n ? order_key(v.w) : kKeyNegInf;
    }
  }
  // ---- range and count of the finite keys over the cluster (-inf is never selected, selection.cpp:153)
  {
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    int nf = 0;
#pragma unroll
    for (int i = 0; i < KPT; ++i)
      if (u[i] != kKeyNegInf) {
        kmin = min(kmin, u[i]);
        kmax = max(kmax, u[i]);
        ++nf;
      }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    nf = __reduce_add_sync(0xffffffffu, nf);
    if (lane == 0) {
      sh.wmin[warp] = kmin;
      sh.wmax[warp] = kmax;
      sh.wgt[warp] = nf;
    }
    __syncthreads();
    cluster_wait_acquire();  // every CTA's inbox barriers are initialised
    if (warp == 0) {
      const bool ok = lane < kCsWarps;
      kmin = __reduce_min_sync(0xffffffffu, ok ? sh.wmin[lane] : 0xFFFFFFFFu);
      kmax = __reduce_max_sync(0xffffffffu, ok ? sh.wmax[lane] : 0u);
      nf = __reduce_add_sync(0xffffffffu, ok ? sh.wgt[lane] : 0);
      if (lane == 0) mbar_arrive_expect_tx(&sh.bar_stat, kCsC * 16u);
      if (lane < kCsC) {  // push (min, max, count) to CTA `lane`
        const uint32_t dst = mapa_shared(smem_u32(&sh.stat_in[c]), lane);
        st_async_v4(dst, make_float4(__uint_as_float(kmin), __uint_as_float(kmax), __int_as_float(nf), 0.f),
                    mapa_shared(smem_u32(&sh.bar_stat), lane));
      }
      mbar_wait_cluster(&sh.bar_stat, 0);
      const uint4 st = lane < kCsC ? sh.stat_in[lane] : make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
      const uint32_t gmin = __reduce_min_sync(0xffffffffu, st.x), gmax = __reduce_max_sync(0xffffffffu, st.y);
      const uint32_t gn = __reduce_add_sync(0xffffffffu, st.z);
      if (lane == 0) {
        sh.gstat[0] = gmin;
        sh.gstat[1] = gmax;
        sh.gstat[2] = gn;
      }
    }
    __syncthreads();
  }
  const uint32_t kmin = sh.gstat[0], kmax = sh.gstat[1];
  const long long nfin = sh.gstat[2];
  long long k;
  {
    const long long wanted = llround(p.ratio * static_cast<double>(n));
    k = min(static_cast<long long>(n), max(wanted, static_cast<long long>(p.k_min)));
    if (k > p.k_cap) k = p.k_cap;
    if (k > nfin) k = nfin;  // topk_indices stops at the first -inf (selection.cpp:153)
  }
  int32_t* out = p_idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  if (k <= 0) {  // every CTA took the same branch; nothing else is pushed
    if (c == 0 && tid == 0) p_k_out[b * p.n_sets + set] = 0;
    return;
  }
  // ---- adaptive radix select over d = key - kmin, kCsBits per pass, histograms pushed to every CTA
  const int nbits = 32 - __clz((kmax - kmin) | 1u);
  int shift = max(0, nbits - kCsBits), prev = 32;
  uint32_t T = 0;
  long long rem = k;
  for (int pass = 0;; ++pass) {
    const bool first = pass == 0;
    const int width = (first ? nbits : prev) - shift;
    const uint32_t mask = (1u << width) - 1u;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const uint32_t d = u[i] - kmin;
      if (u[i] != kKeyNegInf && (first || (d >> prev) == T)) atomicAdd(&sh.hist[(d >> shift) & mask], 1u);
    }
    __syncthreads();
    const int par = pass & 1;
    if (tid == 0) mbar_arrive_expect_tx(&sh.bar_hist[par], kCsC * kCsBins * 4u);
    if (tid < (kCsBins / 4) * kCsC) {  // 64 bin-quads x 8 receivers: one 16-byte push each
      const int q = tid & (kCsBins / 4 - 1), r = tid / (kCsBins / 4);
      const uint4 v = reinterpret_cast<const uint4*>(sh.hist)[q];
      st_async_v4(mapa_shared(smem_u32(&sh.hist_in[par][c][4 * q]), r),
                  make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)),
                  mapa_shared(smem_u32(&sh.bar_hist[par]), r));
    }
    __syncthreads();  // pushes read sh.hist; clear it for the next pass below
    if (tid < kCsBins) {
      sh.hist[tid] = 0;
      mbar_wait_cluster(&sh.bar_hist[par], (pass >> 1) & 1);
      uint32_t cnt = 0;
#pragma unroll
      for (int r = 0; r < kCsC; ++r) cnt += sh.hist_in[par][r][tid];
      uint32_t suf = cnt;  // suffix sums over the 256 bins (8 warps): bins >= tid
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, suf, off);
        if (lane + off < 32) suf += v;
      }
      if (lane == 0) sh.part[warp] = suf;
      named_bar_sync(1, kCsBins);
      uint32_t after = 0;
      for (int w2 = warp + 1; w2 < kCsBins / 32; ++w2) after += sh.part[w2];
      const long long s_incl = static_cast<long long>(suf) + after;
      const long long above = s_incl - cnt;
      if (above < rem && rem <= s_incl) {
        sh.bin = tid;
        sh.rem = rem - above;
        sh.bin_count = cnt;
      }
    }
    __syncthreads();
    T = first ? sh.bin : ((T << width) | sh.bin);
    rem = sh.rem;
    if (static_cast<long long>(sh.bin_count) == rem || shift == 0) break;
    prev = shift;
    shift = max(0, shift - kCsBits);
  }
  // ---- output: finite keys with (d >> shift) > T, plus the `rem` lowest-index ones with (d >> shift) == T
  const int take_eq = static_cast<int>(rem);
  const bool all_eq = static_cast<long long>(sh.bin_count) == rem;
  auto cls = [&](uint32_t key, bool& gt, bool& eq) {
    const uint32_t d = (key - kmin) >> shift;
    const bool ok = key != kKeyNegInf;
    gt = ok && (d > T || (all_eq && d == T));
    eq = ok && !all_eq && d == T;
  };
  int gt = 0, eq = 0;
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool g, e;
    cls(u[i], g, e);
    gt += g;
    eq += e;
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  if (lane == 0) {
    sh.wgt[warp] = gt;
    sh.weq[warp] = eq;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scans of the warps' counts; the CTA totals pushed to every CTA
    const int g = lane < kCsWarps ? sh.wgt[lane] : 0, e = lane < kCsWarps ? sh.weq[lane] : 0;
    int gi = g, ei = e;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int tg = __shfl_up_sync(0xffffffffu, gi, off), te = __shfl_up_sync(0xffffffffu, ei, off);
      if (lane >= off) {
        gi += tg;
        ei += te;
      }
    }
    if (lane < kCsWarps) {
      sh.wgt[lane] = gi - g;
      sh.weq[lane] = ei - e;
    }
    const int gt_cta = __shfl_sync(0xffffffffu, gi, 31), eq_cta = __shfl_sync(0xffffffffu, ei, 31);
    if (lane == 0) mbar_arrive_expect_tx(&sh.bar_cnt, kCsC * 16u);
    if (lane < kCsC)
      st_async_v4(mapa_shared(smem_u32(&sh.cnt_in[c]), lane),
                  make_float4(__int_as_float(gt_cta), __int_as_float(eq_cta), 0.f, 0.f),
                  mapa_shared(smem_u32(&sh.bar_cnt), lane));
    mbar_wait_cluster(&sh.bar_cnt, 0);
    const int4 cn = lane < kCsC ? sh.cnt_in[lane] : make_int4(0, 0, 0, 0);
    const int gb = __reduce_add_sync(0xffffffffu, lane < c ? cn.x : 0), eb = __reduce_add_sync(0xffffffffu, lane < c ? cn.y : 0);
    const int gt_all = __reduce_add_sync(0xffffffffu, cn.x), eq_all = __reduce_add_sync(0xffffffffu, cn.y);
    if (lane == 0) {
      sh.off[0] = gb;
      sh.off[1] = eb;
      if (c == 0) p_k_out[b * p.n_sets + set] = gt_all + min(eq_all, take_eq);
    }
  }
  __syncthreads();
  int g_run = sh.off[0] + sh.wgt[warp], e_run = sh.off[1] + sh.weq[warp];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    unsigned bg[E], be[E];
    bool isg[E], ise[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      cls(u[E * j + e], isg[e], ise[e]);
      bg[e] = __ballot_sync(0xffffffffu, isg[e]);
      be[e] = __ballot_sync(0xffffffffu, ise[e]);
    }
    int g_before = g_run, e_before = e_run;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      g_before += __popc(bg[e] & lt);
      e_before += __popc(be[e] & lt);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (isg[e] || (ise[e] && e_before < take_eq)) out[g_before + min(e_before, take_eq)] = wbase + 32 * E * j + E * lane + e;
      g_before += isg[e];
      e_before += ise[e];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      g_run += __popc(bg[e]);
      e_run += __popc(be[e]);
    }
  }
}

template <bool kFixed, int KPT>
static cudaError_t launch_select_cluster(const SelectParams& p, cudaStream_t s, int n_slots) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCsC * p.n_sets, p.B, n_slots);
  cfg.blockDim = dim3(kCsThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCsC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, select_cluster_kernel<kFixed, KPT>, p);
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s, int n_slots) {
  dim3 grid(p.n_sets, p.B, n_slots);
  const bool fixed = p.score_fx != nullptr;
  // the cluster select takes the selection from ~16 to ~6 us but holds 8 SMs (48 SM-us against ~13):
  // inside the verify chain, where every SM it holds delays the next layer, the single-CTA kernel costs
  // less (config 2 iteration 1.759 against 1.773 ms); past its shared-memory key capacity (64K, 128K
  // contexts: the global-memory key path) the cluster kernel is used
  if ((p.legacy == 0 && p.max_n > kSmemKeys && p.max_n <= static_cast<int64_t>(kCsC) * kCsThreads * 32) ||
      p.legacy == 2) {  // cluster select, keys in registers
    const int64_t per = (p.max_n + kCsC * kCsThreads - 1) / (kCsC * kCsThreads);
    if (per <= 8) return fixed ? launch_select_cluster<true, 8>(p, s, n_slots) : launch_select_cluster<false, 8>(p, s, n_slots);
    if (per <= 16) return fixed ? launch_select_cluster<true, 16>(p, s, n_slots) : launch_select_cluster<false, 16>(p, s, n_slots);
    if (per <= 32) return fixed ? launch_select_cluster<true, 32>(p, s, n_slots) : launch_select_cluster<false, 32>(p, s, n_slots);
  }
  if (n_slots > 1 && p.ld_scores > kSmemKeys) return cudaErrorInvalidValue;  // the keys workspace is per launch
  if (p.ld_scores <= kSmemKeys) {
    static std::atomic<uint64_t> attr_mask{0};  // per device (internal.h)
    int dev = 0;
    const int bytes = static_cast<int>(p.ld_scores * 4);
    if (func_attrs_needed(attr_mask, &dev)) {
      cudaError_t e = cudaFuncSetAttribute(select_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kSmemKeys * 4);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(select_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemKeys * 4);
      if (e != cudaSuccess) return e;
      func_attrs_done(attr_mask, dev);
    }
    if (fixed) select_kernel<true, true><<<grid, kSelThreads, bytes, s>>>(p);
    else select_kernel<false, true><<<grid, kSelThreads, bytes, s>>>(p);
  } else {
    if (fixed) select_kernel<true, false><<<grid, kSelThreads, 0, s>>>(p);
    else select_kernel<false, false><<<grid, kSelThreads, 0, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace sa

namespace sa {
int select_max_smem_keys() { return kSmemKeys; }
}  // namespace sa
