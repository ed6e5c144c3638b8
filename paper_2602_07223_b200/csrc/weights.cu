// weights.cu — the Collect2Weights metric (softmax-weight scores) from the verify kernel's raw logits.
//
// Reference: score_columns_weights (selection.cpp:110-135): for every (q-head, collected row) the
// softmax of the raw prefix logits row with scale 1/sqrt(head_dim) (softmax_stable,
// attention.cpp:8-32), summed over heads and rows and divided by the number of terms.  Unlike the
// raw-logit metric this one needs each row's max and normaliser over ALL prefix columns, known only
// after the verify pass, so the verify kernel writes the collected rows' raw logits (its LogitMatrix
// output, [B][Hq][n_rows][ld]) and two small kernels follow on the selection stream:
//   weight_row_stats  one CTA per (sequence, q-head, row): m = max_i l_i, Z = sum_i 2^((l_i - m) c)
//   weight_scores     one thread per (sequence, column): sum over the set's (head, row) terms of
//                     2^((l - m) c) / Z, / terms -> the per-layer int64 fixed-point sums (2^-32 units)
//                     or the per-KV-head fp32 sums the select kernel consumes.
// fp32 exp2 with the row max subtracted: per-weight relative error ~1e-7, inside the tie band.
#include "internal.h"

namespace sa {

__global__ void __launch_bounds__(256) weight_row_stats(const float* logits, int64_t ld, const int32_t* p0_arr,
                                                         int Hq, int n_rows, float c, float2* stats) {
  const int row_id = blockIdx.x;  // (b * Hq + h) * n_rows + r
  const int b = row_id / (Hq * n_rows);
  const int n = p0_arr[b];
  const float* l = logits + static_cast<size_t>(row_id) * ld;
  __shared__ float red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float mx = -INFINITY;
  for (int i = tid; i < n; i += 256) mx = fmaxf(mx, l[i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float z = 0.f;
  for (int i = tid; i < n; i += 256) z += exp2f((l[i] - mx) * c);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  if (tid == 0) {
    float zs = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) zs += red[w];
    stats[row_id] = make_float2(mx, zs);
  }
}

// grid (ceil(ld / 256), B, n_sets)
__global__ void __launch_bounds__(256) weight_scores(const float* logits, int64_t ld, const int32_t* p0_arr, int Hq,
                                                      int G, int n_rows, float c, const float2* stats, int n_sets,
                                                      long long* fx, float* scores, int64_t ld_scores) {
  const int b = blockIdx.y, set = blockIdx.z;
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int n = p0_arr[b];
  if (i >= n) return;
  const int h0 = n_sets == 1 ? 0 : set * G, h1 = n_sets == 1 ? Hq : h0 + G;
  float acc = 0.f;
  for (int h = h0; h < h1; ++h)
    for (int r = 0; r < n_rows; ++r) {
      const int row_id = (b * Hq + h) * n_rows + r;
      const float2 st = stats[row_id];
      acc += exp2f((logits[static_cast<size_t>(row_id) * ld + i] - st.x) * c) / st.y;
    }
  const float score = acc / static_cast<float>((h1 - h0) * n_rows);
  if (n_sets == 1)
    fx[static_cast<size_t>(b) * ld_scores + i] = __float2ll_rn(score * kScoreFxScale);
  else
    scores[(static_cast<size_t>(b) * n_sets + set) * ld_scores + i] = score;
}

cudaError_t launch_weights(const float* logits, int64_t ld, const int32_t* p0, int B, int Hq, int G, int n_rows,
                           double scale, float2* stats, int n_sets, long long* fx, float* scores, int64_t ld_scores,
                           int64_t max_p, cudaStream_t s) {
  const float c = static_cast<float>(scale * 1.4426950408889634);  // natural-exp scale in log2 units
  weight_row_stats<<<B * Hq * n_rows, 256, 0, s>>>(logits, ld, p0, Hq, n_rows, c, stats);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((max_p + 255) / 256), B, n_sets);
  if (max_p > 0)
    weight_scores<<<grid, 256, 0, s>>>(logits, ld, p0, Hq, G, n_rows, c, stats, n_sets, fx, scores, ld_scores);
  return cudaGetLastError();
}

}  // namespace sa
