// accept.cu — verification acceptance: the step that turns the verify pass into a decode loop.
//
// Reference: SPEC-only (the reference ships no speculation code): speculation::verify
// — for t = 1..gamma accept draft x_t iff u_t < min(1, p_t(x_t) / q_t(x_t)); on
// the first rejection emit a sample of residual_distribution(p_t, q_t) = normalize(max(0, p_t - q_t))
// and stop; if every draft is accepted emit the bonus token ~ p_{gamma+1}.
// Greedy mode: accept iff x_t == argmax p_t (ties -> lower token id); the trailing token is
// argmax p_{a+1}.  The caller then commits: the KV of [y, x_1..x_a] (verify rows p0..p0+a) stays, the
// store is truncated to p0 + a + 1 ("truncates KV to committed prefix + emitted").
//
// One CTA (1024 threads) per sequence; distributions are fp32 rows of V entries.  Samples use inverse
// CDF sampling with one uniform per sequence (u[gamma]): the smallest token i whose inclusive
// prefix sum (double, the fixed order of block_sample) exceeds u * total.
#include "internal.h"

namespace sa {

constexpr int kAccThreads = 1024;

struct AccShared {
  double part[32];
  double base, target;
  float fmax[32];
  int imax[32];
  int pick, res;
};

// Block argmax of row[0..V): ties -> lower index.
__device__ int block_argmax(const float* row, int V, AccShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = tid; i < V; i += kAccThreads) {
    const float v = row[i];
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    sh.fmax[warp] = best;
    sh.imax[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float b = sh.fmax[0];
    int ix = sh.imax[0];
    for (int w = 1; w < 32; ++w)
      if (sh.fmax[w] > b || (sh.fmax[w] == b && sh.imax[w] < ix)) {
        b = sh.fmax[w];
        ix = sh.imax[w];
      }
    sh.pick = ix;
  }
  __syncthreads();
  const int r = sh.pick;
  __syncthreads();
  return r;
}

// Sum of w over [lo, hi) by one warp in a fixed order: coalesced rounds of 32, lane sums over rounds,
// then a __shfl_xor butterfly (every lane ends with the same value).
template <typename W>
__device__ __forceinline__ double warp_range_sum(int lo, int hi, int lane, W& w) {
  double s = 0.0;
#pragma unroll 8
  for (int i = lo + lane; i < hi; i += 32) s += w(i);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// Thread 0: first of 32 sums whose running total (from `run`) exceeds target; the last range with
// mass if rounding left none.  Returns the index; *base = running total before it.
__device__ __forceinline__ int pick_range(const double* part, double run, double target, double* base) {
  const double run0 = run;
  for (int t = 0; t < 32; ++t) {
    if (run + part[t] > target) {
      *base = run;
      return t;
    }
    run += part[t];
  }
  int c = 0;
  for (int t = 0; t < 32; ++t)
    if (part[t] > 0.0) c = t;
  run = run0;
  for (int t = 0; t < c; ++t) run += part[t];
  *base = run;
  return c;
}

// Inverse-CDF sample of weights w(i) >= 0 (unnormalised): the smallest i whose inclusive prefix sum
// exceeds u * total, in double with a fixed summation order (oracle/speculation.py restates it).
// Level 1: warp w sums the contiguous range [w*per1, (w+1)*per1) (per1 = ceil(V/32) rounded up to
// 32); thread 0 totals them in warp order and picks the range the target falls in.  Level 2: the
// 32 warps split that range into sub-ranges of per2 = ceil(per1/32) rounded up to 32, same sums and
// pick.  Level 3: one warp rescans the picked sub-range in rounds of 32 with an inclusive
// (Hillis-Steele) warp scan on top of the running base.
template <typename W>
__device__ int block_sample(int V, double u, W w, AccShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per1 = ((V + 31) / 32 + 31) / 32 * 32;
  {
    const int lo = warp * per1, hi = min(V, lo + per1);
    const double s = warp_range_sum(lo, hi, lane, w);
    if (lane == 0) sh.part[warp] = s;
  }
  __syncthreads();
  if (tid == 0) {
    double total = 0.0;
    for (int t = 0; t < 32; ++t) total += sh.part[t];
    sh.target = u * total;
    sh.pick = pick_range(sh.part, 0.0, sh.target, &sh.base);
  }
  __syncthreads();
  const int lo1 = sh.pick * per1, hi1 = min(V, lo1 + per1);
  const int per2 = ((per1 + 31) / 32 + 31) / 32 * 32;
  const double base1 = sh.base;
  __syncthreads();
  {
    const int lo = min(hi1, lo1 + warp * per2), hi = min(hi1, lo + per2);
    const double s = warp_range_sum(lo, hi, lane, w);
    if (lane == 0) sh.part[warp] = s;
  }
  __syncthreads();
  if (tid == 0) sh.pick = pick_range(sh.part, base1, sh.target, &sh.base);
  __syncthreads();
  if (warp == 0) {
    const int lo = min(hi1, lo1 + sh.pick * per2), hi = min(hi1, lo + per2);
    double base = sh.base;
    const double target = sh.target;
    int r = -1, last_mass = -1;
    for (int i0 = lo; i0 < hi; i0 += 32) {
      const int i = i0 + lane;
      const double e = i < hi ? w(i) : 0.0;
      double v = e;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += o;
      }
      const unsigned cross = __ballot_sync(0xffffffffu, base + v > target);
      const unsigned mass = __ballot_sync(0xffffffffu, e > 0.0);
      if (mass) last_mass = i0 + 31 - __clz(mass);
      if (cross) {
        r = i0 + __ffs(cross) - 1;
        break;
      }
      base += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) sh.res = r >= 0 ? r : last_mass;  // fallback: the last token with mass
  }
  __syncthreads();
  const int r = sh.res;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kAccThreads) accept_kernel(const float* p, const float* q, const int32_t* draft,
                                                             const float* u, int gamma, int V, int greedy,
                                                             int32_t* accepted, int32_t* emitted) {
  __shared__ AccShared sh;
  const int b = blockIdx.x;
  const float* pb = p + static_cast<size_t>(b) * (gamma + 1) * V;
  const float* qb = q ? q + static_cast<size_t>(b) * gamma * V : nullptr;
  const int32_t* xb = draft + static_cast<size_t>(b) * gamma;
  const float* ub = u ? u + static_cast<size_t>(b) * (gamma + 1) : nullptr;
  int32_t* eb = emitted + static_cast<size_t>(b) * (gamma + 1);
  int a = 0;
  int trailing = -1;
  for (int t = 0; t < gamma; ++t) {
    const float* pt = pb + static_cast<size_t>(t) * V;
    const int x = xb[t];
    bool accept;
    if (greedy) {
      const int am = block_argmax(pt, V, sh);
      accept = x == am;
      if (!accept) trailing = am;  // corrected token = argmax p_t
    } else {
      const float* qt = qb + static_cast<size_t>(t) * V;
      const float ratio = pt[x] / qt[x];
      accept = ub[t] < fminf(1.f, ratio);
      if (!accept)  // residual_distribution(p_t, q_t) = normalize(max(0, p_t - q_t))
        trailing = block_sample(V, static_cast<double>(ub[gamma]),
                                [&](int i) { return static_cast<double>(fmaxf(0.f, pt[i] - qt[i])); }, sh);
    }
    if (!accept) break;
    if (threadIdx.x == 0) eb[a] = x;
    ++a;
  }
  if (a == gamma) {  // every draft accepted: bonus token from p_{gamma+1}
    const float* pl = pb + static_cast<size_t>(gamma) * V;
    trailing = greedy ? block_argmax(pl, V, sh)
                      : block_sample(V, static_cast<double>(ub[gamma]),
                                     [&](int i) { return static_cast<double>(pl[i]); }, sh);
  }
  if (threadIdx.x == 0) {
    eb[a] = trailing;
    for (int j = a + 1; j <= gamma; ++j) eb[j] = -1;
    accepted[b] = a;
  }
}

cudaError_t launch_accept(const float* p, const float* q, const int32_t* draft, const float* u, int B, int gamma, int V,
                          int greedy, int32_t* accepted, int32_t* emitted, cudaStream_t s) {
  accept_kernel<<<B, kAccThreads, 0, s>>>(p, q, draft, u, gamma, V, greedy, accepted, emitted);
  return cudaGetLastError();
}

}  // namespace sa
