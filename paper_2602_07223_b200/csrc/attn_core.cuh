// attn_core.cuh — warp-level flash-attention step shared by the verify and draft kernels.
//
// One warp owns a 16-row query tile (mt) and walks 16-token sub-blocks of K/V tiles that sit in
// shared memory in the TMA SWIZZLE_128B layout (see sa::swz).  Per sub-block:
//   S(16x16) = Q(16x128) K^T            8 x ldmatrix.x4 + 16 x mma.m16n8k16 (bf16 in, f32 acc)
//   online softmax in the exp2 domain, lazily rescaling O only when a row max grows
//   O(16x128) += P V                    P split into bf16 hi + lo (P ~= hi + lo to 2^-17), so the
//                                       PV product keeps ~fp32 accuracy against the reference's
//                                       double accumulation (attention.cpp:62-65)
// Each thread holds C fragments for rows gid and gid+8 (gid = lane/4) and token/column pairs
// 2*(lane%4)+{0,1} of every n8 tile.
#pragma once

#include "common.cuh"

namespace sa {

struct WarpAttn {
  float o[16][4];   // O accumulator: 16 n8 tiles of d
  float m[2];       // running row max (scaled, log2 domain), rows gid / gid+8
  float l[2];       // per-thread partial row sums
  uint32_t qa[8][4];  // Q A-fragments for the 8 k16 steps of d = 128

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
  }

  // Q tile rows [mt*16, mt*16+16) from a swizzled [rows][256B] smem tile (half = rows*128 bytes).
  __device__ __forceinline__ void load_q(uint32_t q_smem, uint32_t q_half, int mt, int lane) {
    const int mi = lane >> 3;
    const int row = mt * 16 + (mi & 1) * 8 + (lane & 7);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int chunk = 2 * kk + (mi >> 1);
      ldsm_x4(q_smem + swz(row, chunk, q_half), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
    }
  }

  // Raw logits S for tokens [r0, r0+16) of the K tile at k_smem.
  __device__ __forceinline__ void qk(uint32_t k_smem, uint32_t k_half, int r0, int lane, float (&s)[2][4]) const {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
    const int mi = lane >> 3;
    const int tok = r0 + (mi >> 1) * 8 + (lane & 7);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(k_smem + swz(tok, 2 * kk + (mi & 1), k_half), b0, b1, b2, b3);
      mma_bf16(s[0], qa[kk], b0, b1);
      mma_bf16(s[1], qa[kk], b2, b3);
    }
  }

  // Online softmax over masked raw logits s (-inf = masked) and O += P V for tokens [r0, r0+16).
  // c = scale * log2(e).
  __device__ __forceinline__ void softmax_pv(float (&s)[2][4], uint32_t v_smem, uint32_t v_half, int r0, int lane,
                                             float c) {
    float tmax[2];
    tmax[0] = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
    tmax[1] = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      tmax[sl] = fmaxf(tmax[sl], __shfl_xor_sync(0xffffffffu, tmax[sl], 1));
      tmax[sl] = fmaxf(tmax[sl], __shfl_xor_sync(0xffffffffu, tmax[sl], 2));
    }
    float mnew[2];
    bool grow = false;
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      mnew[sl] = fmaxf(m[sl], tmax[sl] * c);
      grow |= mnew[sl] > m[sl];
    }
    if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const float f = (mnew[sl] == -INFINITY || m[sl] == mnew[sl]) ? 1.f : fast_exp2(m[sl] - mnew[sl]);
        l[sl] *= f;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          o[nt][2 * sl] *= f;
          o[nt][2 * sl + 1] *= f;
        }
        m[sl] = mnew[sl];
      }
    }
    const float base0 = m[0] == -INFINITY ? 0.f : m[0];
    const float base1 = m[1] == -INFINITY ? 0.f : m[1];
    float pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      pr[nt][0] = fast_exp2(fmaf(s[nt][0], c, -base0));
      pr[nt][1] = fast_exp2(fmaf(s[nt][1], c, -base0));
      pr[nt][2] = fast_exp2(fmaf(s[nt][2], c, -base1));
      pr[nt][3] = fast_exp2(fmaf(s[nt][3], c, -base1));
      l[0] += pr[nt][0] + pr[nt][1];
      l[1] += pr[nt][2] + pr[nt][3];
    }
    uint32_t ah[4], al[4];
    split_bf16(pr[0][0], pr[0][1], ah[0], al[0]);  // row gid,   tokens 0-7
    split_bf16(pr[0][2], pr[0][3], ah[1], al[1]);  // row gid+8, tokens 0-7
    split_bf16(pr[1][0], pr[1][1], ah[2], al[2]);  // row gid,   tokens 8-15
    split_bf16(pr[1][2], pr[1][3], ah[3], al[3]);  // row gid+8, tokens 8-15
    const int mi = lane >> 3;
    const int tok = r0 + (mi & 1) * 8 + (lane & 7);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(v_smem + swz(tok, 2 * jj + (mi >> 1), v_half), v0, v1, v2, v3);
      mma_bf16(o[2 * jj], ah, v0, v1);
      mma_bf16(o[2 * jj], al, v0, v1);
      mma_bf16(o[2 * jj + 1], ah, v2, v3);
      mma_bf16(o[2 * jj + 1], al, v2, v3);
    }
  }

  __device__ __forceinline__ void finalize_l() {
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      l[sl] += __shfl_xor_sync(0xffffffffu, l[sl], 1);
      l[sl] += __shfl_xor_sync(0xffffffffu, l[sl], 2);
    }
  }
};

// Per-warp partial in shared memory: O [16][kWpStride] floats, then m[16], l[16].
constexpr int kWpStride = 132;
constexpr int kWpFloats = 16 * kWpStride + 32;

__device__ __forceinline__ void store_warp_partial(const WarpAttn& w, float* wp, int lane) {
  const int gid = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int col = 8 * nt + 2 * t4;
    *reinterpret_cast<float2*>(wp + gid * kWpStride + col) = make_float2(w.o[nt][0], w.o[nt][1]);
    *reinterpret_cast<float2*>(wp + (gid + 8) * kWpStride + col) = make_float2(w.o[nt][2], w.o[nt][3]);
  }
  if (t4 == 0) {
    wp[16 * kWpStride + gid] = w.m[0];
    wp[16 * kWpStride + gid + 8] = w.m[1];
    wp[16 * kWpStride + 16 + gid] = w.l[0];
    wp[16 * kWpStride + 16 + gid + 8] = w.l[1];
  }
}

// Combine the TG warp partials of each of the MT row tiles (warp index = tg*MT + mt) into the
// CTA's split partial in global memory: part_o [MT*16][128], part_ml [MT*16][2] (m, l).
// Fixed summation order (tg ascending) keeps results deterministic.
template <int MT, int TG>
__device__ __forceinline__ void cta_partial_to_global(const float* wps, float* part_o, float* part_ml, int tid,
                                                      int nthreads) {
  for (int i = tid; i < MT * 16 * 128; i += nthreads) {
    const int row = i >> 7, col = i & 127, mt = row >> 4, r = row & 15;
    float mstar = -INFINITY;
#pragma unroll
    for (int tg = 0; tg < TG; ++tg) mstar = fmaxf(mstar, wps[(tg * MT + mt) * kWpFloats + 16 * kWpStride + r]);
    float acc = 0.f, lsum = 0.f;
    if (mstar != -INFINITY) {
#pragma unroll
      for (int tg = 0; tg < TG; ++tg) {
        const float* wp = wps + (tg * MT + mt) * kWpFloats;
        const float f = fast_exp2(wp[16 * kWpStride + r] - mstar);
        acc += wp[r * kWpStride + col] * f;
        lsum += wp[16 * kWpStride + 16 + r] * f;
      }
    }
    part_o[i] = acc;
    if (col == 0) {
      part_ml[2 * row] = mstar;
      part_ml[2 * row + 1] = lsum;
    }
  }
}

// Last-arriving CTA of a (b, kv-head) unit merges the n_splits partials (split order fixed) and
// writes normalised rows.  out_row(r) returns the f32 destination of output row r < rows_out.
// Latency-aware: (m, l) of every (split, row) are staged in shared memory in one pass, the per-row
// merge weights w[s][r] = 2^(m_s - m*) / L are computed once, and each thread then streams float4
// column groups with all split loads independent (unrolled) so the L2 round trips overlap.
// `smem_w` must hold n_splits * rows_out * 2 floats.  Called by all `nthreads` threads.
template <typename OutRow>
__device__ __forceinline__ void combine_splits(const float* part_o_unit, const float* part_ml_unit, int n_splits,
                                               int rows_pad, int rows_out, int* counter, int* smem_flag,
                                               float* smem_w, int tid, int nthreads, int bar_id, OutRow out_row,
                                               bool arrived = false) {
  if (!arrived) {  // arrival (skipped when the caller already counted this CTA in)
    __threadfence();
    named_bar_sync(bar_id, nthreads);
    if (tid == 0) *smem_flag = atomicAdd(counter, 1);
    named_bar_sync(bar_id, nthreads);
    if (*smem_flag != n_splits - 1) return;
  }
  __threadfence();
  float2* ml = reinterpret_cast<float2*>(smem_w);  // [n_splits][rows_out] (m, l) -> (w, -)
  for (int i = tid; i < n_splits * rows_out; i += nthreads) {
    const int s = i / rows_out, row = i % rows_out;
    ml[i] = __ldcg(reinterpret_cast<const float2*>(part_ml_unit) + s * rows_pad + row);
  }
  named_bar_sync(bar_id, nthreads);
  for (int row = tid; row < rows_out; row += nthreads) {
    float mstar = -INFINITY;
    for (int s = 0; s < n_splits; ++s) mstar = fmaxf(mstar, ml[s * rows_out + row].x);
    float lsum = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float2 v = ml[s * rows_out + row];
      const float f = v.x == -INFINITY ? 0.f : fast_exp2(v.x - mstar);
      ml[s * rows_out + row].x = f;
      lsum += v.y * f;
    }
    const float inv = 1.f / lsum;
    for (int s = 0; s < n_splits; ++s) ml[s * rows_out + row].x *= inv;
  }
  named_bar_sync(bar_id, nthreads);
  for (int i = tid; i < rows_out * 32; i += nthreads) {
    const int row = i >> 5, c4 = i & 31;
    const float4* src = reinterpret_cast<const float4*>(part_o_unit) + row * 32 + c4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int s = 0;
    for (; s + 4 <= n_splits; s += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(src + (s + u) * rows_pad * 32);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float w = ml[(s + u) * rows_out + row].x;
        acc.x += v[u].x * w;
        acc.y += v[u].y * w;
        acc.z += v[u].z * w;
        acc.w += v[u].w * w;
      }
    }
    for (; s < n_splits; ++s) {
      const float4 v = __ldcg(src + s * rows_pad * 32);
      const float w = ml[s * rows_out + row].x;
      acc.x += v.x * w;
      acc.y += v.y * w;
      acc.z += v.z * w;
      acc.w += v.w * w;
    }
    reinterpret_cast<float4*>(out_row(row))[c4] = acc;
  }
  if (tid == 0) *counter = 0;  // re-arm for the next launch (stream/graph ordered)
}

}  // namespace sa
