// weights.cu — the Collect2Weights metric (softmax-weight scores) from the verify kernel's raw logits.
//
// Reference: score_columns_weights (selection.cpp:110-135): for every (q-head, collected row) the
// softmax of the raw prefix logits row with scale 1/sqrt(head_dim) (softmax_stable,
// attention.cpp:8-32), summed over heads and rows and divided by the number of terms.  Unlike the
// raw-logit metric this one needs each row's max and normaliser over ALL prefix columns, known only
// after the verify pass, so the verify kernel writes the collected rows' raw logits (its LogitMatrix
// output, [B][Hq][n_rows][ld]) and two small kernels follow on the selection stream:
//   weight_row_stats  kWeightParts CTAs per (sequence, q-head, row): per chunk m = max l_i and
//                     Z = sum 2^((l_i - m) c), merged in part order by weight_scores
//   weight_scores     four threads per (sequence, column): sum over the set's (head, row) terms of
//                     2^((l - m) c) / Z, / terms -> the per-layer int64 fixed-point sums (2^-32 units)
//                     or the per-KV-head fp32 sums the select kernel consumes.
// fp32 exp2 with the row max subtracted: per-weight relative error ~1e-7, inside the tie band.
#include "internal.h"

namespace sa {

// grid (B * Hq * n_rows, kWeightParts): chunk `part` of one row -> (chunk max, chunk sum of
// 2^((l - max) c)); weight_scores merges the parts in part order (deterministic).  Spreading a row
// over several CTAs puts 4x more SMs on the 128 KB rows (32K context).
__global__ void __launch_bounds__(256) weight_row_stats(const float* logits, int64_t ld, const int32_t* p0_arr,
                                                         int Hq, int n_rows, float c, float2* stats) {
  const int row_id = blockIdx.x, part = blockIdx.y;  // row_id = (b * Hq + h) * n_rows + r
  const int b = row_id / (Hq * n_rows);
  const int n = p0_arr[b];
  const int lo = static_cast<int>(static_cast<int64_t>(n) * part / kWeightParts);
  const int hi = static_cast<int>(static_cast<int64_t>(n) * (part + 1) / kWeightParts);
  const float* l = logits + static_cast<size_t>(row_id) * ld;
  __shared__ float red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 8 independent accumulators per thread, clamped addresses: 8 loads in flight, no branches between
  float mx8[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
  if (hi > lo)
    for (int i0 = lo + tid; i0 < hi; i0 += 256 * 8) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(l + min(i0 + u * 256, hi - 1));
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], x[u]);  // duplicates of l[hi-1]: max unchanged
    }
  float mx = mx8[0];
#pragma unroll
  for (int u = 1; u < 8; ++u) mx = fmaxf(mx, mx8[u]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float z8[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) z8[u] = 0.f;
  if (hi > lo)
    for (int i0 = lo + tid; i0 < hi; i0 += 256 * 8) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(l + min(i0 + u * 256, hi - 1));
#pragma unroll
      for (int u = 0; u < 8; ++u) z8[u] += i0 + u * 256 < hi ? exp2f((x[u] - mx) * c) : 0.f;
    }
  float z = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) z += z8[u];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  if (tid == 0) {
    float zs = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) zs += red[w];
    stats[static_cast<size_t>(row_id) * kWeightParts + part] = make_float2(mx, zs);
  }
}

// grid (ceil(ld / 64), B, n_sets), 256 threads = 64 columns x 4 term groups: the (head, row) terms'
// (max, 1 / normaliser) are merged from the row-stat parts into shared memory first; then each thread
// sums its quarter of the terms (16 loads in flight) and the 4 quarters are added in group order
// (deterministic).  4 threads per column quadruple the loads in flight per SM (the kernel is
// latency-bound: 8 MB of logits per layer at 32K context).
__global__ void __launch_bounds__(256) weight_scores(const float* logits, int64_t ld, const int32_t* p0_arr, int Hq,
                                                      int G, int n_rows, float c, const float2* stats, int n_sets,
                                                      long long* fx, float* scores, int64_t ld_scores) {
  extern __shared__ float2 term_stats[];  // [terms] (max, 1 / normaliser), then [4][64] partial sums
  const int b = blockIdx.y, set = blockIdx.z;
  const int col = threadIdx.x & 63, grp = threadIdx.x >> 6;
  const int i = blockIdx.x * 64 + col;
  const int n = p0_arr[b];
  const int h0 = n_sets == 1 ? 0 : set * G, h1 = n_sets == 1 ? Hq : h0 + G;
  const int t0 = (b * Hq + h0) * n_rows, nt = (h1 - h0) * n_rows;  // (head, row) terms, row-major
  float* part = reinterpret_cast<float*>(term_stats + nt);
  for (int t = threadIdx.x; t < nt; t += 256) {
    float2 pp[kWeightParts];
#pragma unroll
    for (int k = 0; k < kWeightParts; ++k) pp[k] = __ldg(stats + static_cast<size_t>(t0 + t) * kWeightParts + k);
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < kWeightParts; ++k) m = fmaxf(m, pp[k].x);
    float z = 0.f;
#pragma unroll
    for (int k = 0; k < kWeightParts; ++k) z += pp[k].x == -INFINITY ? 0.f : pp[k].y * exp2f((pp[k].x - m) * c);
    term_stats[t] = make_float2(m, 1.f / z);
  }
  __syncthreads();
  const int q = (nt + 3) / 4, ta = min(nt, grp * q), tb = min(nt, ta + q);
  const int ic = min(i, max(n - 1, 0));  // clamped column: loads stay valid, the result is discarded
  float acc = 0.f;
  const float* lp = logits + static_cast<size_t>(t0) * ld + ic;
  for (int t = ta; t < tb; t += 16) {
    float x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = __ldg(lp + static_cast<size_t>(min(t + u, tb - 1)) * ld);
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // terms in (head, row) order
      const float2 st = term_stats[min(t + u, tb - 1)];
      acc += t + u < tb ? exp2f((x[u] - st.x) * c) * st.y : 0.f;
    }
  }
  part[grp * 64 + col] = acc;
  __syncthreads();
  if (grp != 0 || i >= n) return;
  const float score = (((part[col] + part[64 + col]) + part[128 + col]) + part[192 + col]) / static_cast<float>(nt);
  if (n_sets == 1)
    fx[static_cast<size_t>(b) * ld_scores + i] = __float2ll_rn(score * kScoreFxScale);
  else
    scores[(static_cast<size_t>(b) * n_sets + set) * ld_scores + i] = score;
}

cudaError_t launch_weights(const float* logits, int64_t ld, const int32_t* p0, int B, int Hq, int G, int n_rows,
                           double scale, float2* stats, int n_sets, long long* fx, float* scores, int64_t ld_scores,
                           int64_t max_p, cudaStream_t s) {
  const float c = static_cast<float>(scale * 1.4426950408889634);  // natural-exp scale in log2 units
  weight_row_stats<<<dim3(B * Hq * n_rows, kWeightParts), 256, 0, s>>>(logits, ld, p0, Hq, n_rows, c, stats);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((max_p + 63) / 64), B, n_sets);
  const int nt = (n_sets == 1 ? Hq : G) * n_rows;
  if (max_p > 0)
    weight_scores<<<grid, 256, nt * sizeof(float2) + 256 * sizeof(float), s>>>(logits, ld, p0, Hq, G, n_rows, c, stats,
                                                                              n_sets, fx, scores, ld_scores);
  return cudaGetLastError();
}

}  // namespace sa
