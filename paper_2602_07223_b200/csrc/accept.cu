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
// prefix sum (double, fixed order: 1024 contiguous chunks, then a scan over chunks) exceeds u * total.
#include "internal.h"

namespace sa {

constexpr int kAccThreads = 1024;

struct AccShared {
  double part[kAccThreads];
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

// Inverse-CDF sample of weights w(i) >= 0 (unnormalised): the smallest i whose inclusive prefix sum
// exceeds u * total.  Prefix sums in double in a fixed order: contiguous chunks of ceil(V/1024)
// tokens per thread, then the chunk totals in thread order (oracle/speculation.py restates it).
template <typename W>
__device__ int block_sample(int V, double u, W w, AccShared& sh) {
  const int tid = threadIdx.x;
  const int per = (V + kAccThreads - 1) / kAccThreads;
  const int lo = tid * per, hi = min(V, lo + per);
  double loc = 0.0;
  for (int i = lo; i < hi; ++i) loc += w(i);
  sh.part[tid] = loc;
  __syncthreads();
  if (tid == 0) {
    double total = 0.0;
    for (int t = 0; t < kAccThreads; ++t) total += sh.part[t];
    const double target = u * total;
    double run = 0.0;
    int c = -1;
    for (int t = 0; t < kAccThreads; ++t) {
      if (run + sh.part[t] > target) {
        c = t;
        break;
      }
      run += sh.part[t];
    }
    if (c < 0) {  // u * total rounded up to the total: the last chunk with mass
      run = 0.0;
      for (int t = 0; t < kAccThreads; ++t)
        if (sh.part[t] > 0.0) c = t;
      for (int t = 0; t < c; ++t) run += sh.part[t];
    }
    sh.base = run;
    sh.target = target;
    sh.pick = c;
  }
  __syncthreads();
  if (tid == sh.pick) {
    double run = sh.base;
    int r = -1;
    for (int i = lo; i < hi; ++i) {
      const double wi = w(i);
      run += wi;
      if (wi > 0.0) r = i;  // fallback: the last token with mass
      if (run > sh.target) {
        r = i;
        break;
      }
    }
    sh.res = r;
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
    accepted[b] = a;
  }
}

cudaError_t launch_accept(const float* p, const float* q, const int32_t* draft, const float* u, int B, int gamma, int V,
                          int greedy, int32_t* accepted, int32_t* emitted, cudaStream_t s) {
  accept_kernel<<<B, kAccThreads, 0, s>>>(p, q, draft, u, gamma, V, greedy, accepted, emitted);
  return cudaGetLastError();
}

}  // namespace sa
