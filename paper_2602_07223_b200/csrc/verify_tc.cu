// verify_tc.cu — tcgen05 (5th-gen tensor core) verify attention with the fused Collect-k byproduct.
//
// Reference: attend_collect / attend_segments / softmax_stable (attention.cpp:8-87) for every
// q-head and verify row t = 1..gamma+1 and the score_columns aggregation that
// consumes the LogitMatrix (selection.cpp:89-108).
//
// Swap-AB formulation (the GQA group x (gamma+1) rows are few, the keys many):
//   S^T[tok][row] = K[tok][:] . Q[row][:]        tcgen05.mma M=128 tokens, N=rows (<=64), K=d=128
//   O^T[d][row]  += V^T[d][tok] . P^T[tok][row]   M=d=128, N=rows, K=128 tokens (P = bf16 hi + lo)
// TMEM lane = token for S and lane = d for O, so each softmax thread owns ONE token and all of its
// query rows: the Collect-2 score byproduct (sum over the G heads and the collected rows of raw
// q.k, selection.cpp:93-106) is a thread-local sum, written as one coalesced float per token — no
// LogitMatrix, no second pass over the KV.
//
// Softmax runs in two ping-pong warpgroups (even / odd tiles), each with its own S and O^T
// accumulators in TMEM and its own running row max / sums, merged once in the epilogue.  The row
// max is kept lazily: a tile whose logits all sit within 2^8 of the warpgroup's reference max needs
// no cross-thread work; otherwise the warpgroup reduces the tile's row max, rescales its l partials
// and O^T columns in TMEM, and continues (exact: every p uses the same reference as its O/l terms).
//
// Warp roles (352 threads): w0 K producer, w1 V producer (TMA, 128-token SWIZZLE_128B boxes, separate
// rings so K is recycled right after QK^T), w2 MMA issuer (single elected thread; owns the TMEM
// allocation), w3-6 softmax warpgroup 0, w7-10 softmax warpgroup 1.  The last split appends the
// gamma+1 window rows to the cache (fused KvStore::append) and reads them back through TMA as part of
// its final tile, masked causally inside the window (row t sees window keys j < t).
#include "attn_core.cuh"
#include "internal.h"

namespace sa {

template <int N>
struct TCfg {
  static constexpr int kTile = 128;
  static constexpr int kSK = (N <= 32) ? 3 : 2;       // K ring stages
  static constexpr int kSV = 2;                       // V ring stages
  static constexpr int kHalf = kTile * 128;           // one 64-column half of a K or V tile (16 KB)
  static constexpr int kTileBytes = 2 * kHalf;         // K or V tile (32 KB)
  static constexpr int kQHalf = N * 128;
  static constexpr int kPAtoms = (N + 31) / 32;        // 32-row MN atoms of the SW64 P layout
  static constexpr int kPBytes = kPAtoms * kTile * 64; // hi (or lo) P plane
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kSK * kTileBytes;
  static constexpr int kOffQ = kOffV + kSV * kTileBytes;
  static constexpr int kOffP = kOffQ + 2 * kQHalf;     // [wg][hi, lo]
  static constexpr int kOffBar = kOffP + 4 * kPBytes;
  static constexpr int kNumBars = 2 * kSK + 2 * kSV + 10;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  // misc: tmem slot, flag | mref[2][64] fac[2][64] ltot[2][64] wsc[64] lim[64] | red[2][4][64]
  static constexpr int kMiscBytes = 16 + (2 + 2 + 2 + 1 + 1) * 64 * 4 + 2 * 4 * 64 * 4;
  static constexpr int kSmem = kOffMisc + kMiscBytes + 1024;
  static constexpr int kThreads = 352;
  static constexpr uint32_t kTmemCols = (4 * N <= 128) ? 128 : 256;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

constexpr float kLazyMaxThresh = 8.0f;  // log2 units: p <= 2^8 before a forced max update

template <int N>
__global__ void __launch_bounds__(352, 1)
    verify_tc_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const VerifyParams p) {
  using C = TCfg<N>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // keep the pointer in the shared window (integer offset, not a generic round trip)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + C::kSK;
  uint64_t* v_full = k_empty + C::kSK;
  uint64_t* v_empty = v_full + C::kSV;
  uint64_t* s_full = v_empty + C::kSV;  // [2] per warpgroup
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* pv_done = p_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  int* flag = reinterpret_cast<int*>(smem + C::kOffMisc + 4);
  float* mref_all = reinterpret_cast<float*>(smem + C::kOffMisc + 16);  // [2][64]
  float* fac_all = mref_all + 128;                                       // [2][64]
  float* ltot = fac_all + 128;                                           // [2][64]
  float* wsc = ltot + 128;                                               // [64] score weights 0/1
  int* lim = reinterpret_cast<int*>(wsc + 64);                           // [64]
  float* red_all = reinterpret_cast<float*>(lim + 64);                   // [2][4][64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int seq = p.seq_ids[b];
  const int p0 = p.p0[b];
  const int R = p.R, M = p.M, Hq = p.Hkv * p.G;
  const bool last = split == p.n_splits - 1;
  int lo = split * p.chunk, hi;
  if (!last) {
    hi = min(lo + p.chunk, p0);
  } else {
    lo = min(lo, p0);
    hi = p0 + R;
  }
  const int tile0 = lo & ~(C::kTile - 1);
  const int n_tiles = hi > lo ? (hi - tile0 + C::kTile - 1) / C::kTile : 0;
  const int pre_hi = min(hi, p0);  // end of this CTA's prefix columns (score byproduct range)

  // ------------------------------------------------------------------ prologue (all threads)
  if (tid == 0) {
    for (int s = 0; s < C::kSK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::kSV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&p_empty[i], 1);
      mbar_init(&pv_done[i], 1);
    }
    fence_mbar_init();
  }
  uint8_t* sq = smem + C::kOffQ;
  const __nv_bfloat16* qb = p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
  for (int i = tid; i < N * 16; i += C::kThreads) {
    const int row = i >> 4, ch = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < M) v = __ldg(reinterpret_cast<const uint4*>(qb + row * 128 + ch * 8));
    *reinterpret_cast<uint4*>(sq + swz(row, ch, C::kQHalf)) = v;
  }
  if (tid < 64) {
    mref_all[tid] = -INFINITY;
    mref_all[64 + tid] = -INFINITY;
    lim[tid] = tid < M ? p0 + tid % R : -1;  // last key position row m may see (causal window)
    wsc[tid] = (tid < M && ((p.score_mask >> (tid % R)) & 1u)) ? 1.f : 0.f;
  }
  if (last && p.k_new) {  // fused KvStore::append of the window rows, read back below by TMA
    for (int i = tid; i < 2 * R * 16; i += C::kThreads) {
      const int which = i / (R * 16), row = (i >> 4) % R, ch = i & 15;
      const __nv_bfloat16* src =
          (which ? p.v_new : p.k_new) + ((static_cast<size_t>(b) * R + row) * p.Hkv + g) * 128;
      const int64_t cr = cache_row(p.cache, seq, p.layer, g, p0 + row);
      __nv_bfloat16* dst = (which ? p.cache.v : p.cache.k) + cr * 128;
      reinterpret_cast<uint4*>(dst)[ch] = __ldg(reinterpret_cast<const uint4*>(src) + ch);
    }
    fence_proxy_async();  // generic-proxy global writes -> async-proxy (TMA) reads
  }
  fence_proxy_async_smem();  // Q tile: generic smem writes -> tensor-core reads
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp <= 1) {
    // ---------------------------------------------------------------- TMA producers (K: w0, V: w1)
    if (lane == 0 && n_tiles > 0) {
      const CUtensorMap* map = warp == 0 ? &tmk : &tmv;
      const int S = warp == 0 ? C::kSK : C::kSV;
      uint64_t* full = warp == 0 ? k_full : v_full;
      uint64_t* empty = warp == 0 ? k_empty : v_empty;
      uint8_t* ring = smem + (warp == 0 ? C::kOffK : C::kOffV);
      tma_prefetch_desc(map);
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % S;
        if (t >= S) mbar_wait(&empty[st], ((t / S) & 1) ^ 1);
        const int row = static_cast<int>(cache_row(p.cache, seq, p.layer, g, tile0 + t * C::kTile));
        uint8_t* dst = ring + st * C::kTileBytes;
        mbar_expect_tx(&full[st], C::kTileBytes);
        tma_load_2d(dst, map, &full[st], 0, row, pol);
        tma_load_2d(dst + C::kHalf, map, &full[st], 64, row, pol);
      }
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(N, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(N, 1, 1);
      const uint32_t q_base = smem_u32(sq);
      const uint32_t p_base = smem_u32(smem + C::kOffP);
      auto issue_pv = [&](int u) {
        const int wg = u & 1, sv = u % C::kSV;
        mbar_wait(&v_full[sv], (u / C::kSV) & 1);
        mbar_wait(&p_full[wg], (u >> 1) & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + C::kOffV + sv * C::kTileBytes);
        const uint32_t p_hi = p_base + wg * 2 * C::kPBytes, p_lo = p_hi + C::kPBytes;
        const uint32_t o_tm = tmem + 2 * N + wg * N;
#pragma unroll
        for (int kt = 0; kt < 8; ++kt) {  // 16 tokens per MMA
          const uint64_t a = umma_desc(v_base + kt * 2048, C::kHalf, 1024, kLayoutSW128);
          const uint64_t bh = umma_desc(p_hi + kt * 1024, C::kTile * 64, 512, kLayoutSW64);
          const uint64_t bl = umma_desc(p_lo + kt * 1024, C::kTile * 64, 512, kLayoutSW64);
          umma_bf16(o_tm, a, bh, idesc_pv, ((u >> 1) > 0 || kt > 0) ? 1u : 0u);
          umma_bf16(o_tm, a, bl, idesc_pv, 1u);
        }
        umma_commit(&v_empty[sv]);
        umma_commit(&p_empty[wg]);
        umma_commit(&pv_done[wg]);
      };
      for (int t = 0; t < n_tiles; ++t) {
        const int sk = t % C::kSK;
        mbar_wait(&k_full[sk], (t / C::kSK) & 1);
        if (t >= 2) mbar_wait(&s_empty[t & 1], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(smem + C::kOffK + sk * C::kTileBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // d in steps of 16
          const uint64_t a = umma_desc(k_base + (kk >> 2) * C::kHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
          const uint64_t bq = umma_desc(q_base + (kk >> 2) * C::kQHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
          umma_bf16(tmem + (t & 1) * N, a, bq, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t & 1]);
        umma_commit(&k_empty[sk]);
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    const int wg = (warp - 3) >> 2;     // 0: even tiles, 1: odd tiles
    const int q4 = warp & 3;            // TMEM lane quarter this warp may access
    const int tk = q4 * 32 + lane;      // token within the tile (S) / d (O)
    const int ts = (warp - 3) * 32 + lane - wg * 128;  // 0..127 within the warpgroup
    const int bar_wg = 2 + wg;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float c = p.scale_log2;
    float* mref = mref_all + wg * 64;
    float* fac = fac_all + wg * 64;
    float* red = red_all + wg * 256;
    float* score_out = p.scores ? p.scores + (static_cast<size_t>(b) * p.Hkv + g) * p.ld_scores : nullptr;
    uint8_t* p_hi = smem + C::kOffP + wg * 2 * C::kPBytes;
    const uint32_t s_tm = tmem + lane_off + wg * N;
    const uint32_t o_tm = tmem + lane_off + 2 * N + wg * N;
    float l[N];
#pragma unroll
    for (int m = 0; m < N; ++m) l[m] = 0.f;

    int i = 0;
    for (int t = wg; t < n_tiles; t += 2, ++i) {
      mbar_wait(&s_full[wg], i & 1);
      tc_fence_after();
      float s[N];
      tmem_ld_n<N>(s_tm, s);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[wg]);
      const int tstart = tile0 + t * C::kTile;
      const int pos = tstart + tk;
      const bool full = tstart >= lo && tstart + C::kTile <= pre_hi;  // every row sees every token
      const bool in_range = pos >= lo && pos < hi;
      if (score_out && pos >= lo && pos < pre_hi) {  // fused Collect-k column sum (raw logits)
        float sc = 0.f;
#pragma unroll
        for (int m = 0; m < N; ++m) sc = fmaf(wsc[m], s[m], sc);
        score_out[pos] = sc;
      }
      if (p.logits && pos >= lo && pos < pre_hi) {  // debug / variant path: raw prefix logits
#pragma unroll
        for (int m = 0; m < N; ++m) {
          if (m >= M) continue;
          const int r = m % R;
          if (!((p.collect_mask >> r) & 1u)) continue;
          const int ci = __popc(p.collect_mask & ((1u << r) - 1u));
          p.logits[((static_cast<size_t>(b) * Hq + g * p.G + m / R) * p.n_collect + ci) * p.ld_logits + pos] = s[m];
        }
      }
      // pass 1: does any logit exceed the lazy reference by more than 2^8?
      bool exceed = false;
      if (full) {
#pragma unroll
        for (int m = 0; m < N; ++m) exceed |= fmaf(s[m], c, -mref[m]) > kLazyMaxThresh;
      } else {
#pragma unroll
        for (int m = 0; m < N; ++m)
          exceed |= (in_range && pos <= lim[m]) && fmaf(s[m], c, -mref[m]) > kLazyMaxThresh;
      }
      if (named_bar_or(bar_wg, 128, exceed)) {
        // slow path: exact row max of this tile, rescale l partials and this warpgroup's O^T
#pragma unroll
        for (int m = 0; m < N; ++m) {
          float x = (full || (in_range && pos <= lim[m])) ? s[m] * c : -INFINITY;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, off));
          if (lane == 0) red[q4 * 64 + m] = x;
        }
        named_bar_sync(bar_wg, 128);
        if (ts < N) {
          const float mo = mref[ts];
          const float mx = fmaxf(fmaxf(red[ts], red[64 + ts]), fmaxf(red[128 + ts], red[192 + ts]));
          const float mn = fmaxf(mo, mx);
          fac[ts] = (mo == -INFINITY) ? 0.f : (mn == mo ? 1.f : fast_exp2(mo - mn));
          mref[ts] = mn;
        }
        named_bar_sync(bar_wg, 128);
#pragma unroll
        for (int m = 0; m < N; ++m) l[m] *= fac[m];
        if (i > 0) {  // O^T of this warpgroup is final through its previous tile once that PV is done
          mbar_wait(&pv_done[wg], (i - 1) & 1);
          tc_fence_after();
          float v[N];
          tmem_ld_n<N>(o_tm, v);
          tc_wait_ld();
#pragma unroll
          for (int m = 0; m < N; ++m) v[m] *= fac[m];
          tmem_st_n<N>(o_tm, v);
          tc_wait_st();
        }
      }
      if (i > 0) mbar_wait(&p_empty[wg], (i - 1) & 1);  // previous PV finished reading this P plane
      // pass 2: p = 2^(s*c - mref), l += p, P^T -> smem as bf16 hi + lo (MN-major SWIZZLE_64B)
#pragma unroll
      for (int a = 0; a < C::kPAtoms; ++a)
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float x[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int m = 32 * a + 8 * ch + 2 * e + u;
              if (m < N) {
                const bool valid = full || (in_range && pos <= lim[m]);
                x[u] = valid ? fast_exp2(fmaf(s[m], c, -mref[m])) : 0.f;
                l[m] += x[u];
              } else {
                x[u] = 0.f;
              }
            }
            split_bf16(x[0], x[1], hw[e], lw[e]);
          }
          const uint32_t off = a * (C::kTile * 64) + tk * 64 + ((ch ^ ((tk >> 1) & 3)) << 4);
          *reinterpret_cast<uint4*>(p_hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(p_hi + C::kPBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[wg]);
    }

    // ---------------------------------------------------------------- epilogue
    const int my_tiles = i;  // tiles this warpgroup processed
    if (my_tiles > 0) {
      mbar_wait(&pv_done[wg], (my_tiles - 1) & 1);
      tc_fence_after();
    }
#pragma unroll
    for (int m = 0; m < N; ++m) {
      float x = l[m];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      if (lane == 0) red[q4 * 64 + m] = x;
    }
    named_bar_sync(bar_wg, 128);
    if (ts < N) ltot[wg * 64 + ts] = red[ts] + red[64 + ts] + red[128 + ts] + red[192 + ts];
    named_bar_sync(1, 256);  // both warpgroups' (mref, ltot) final
    const int unit = b * p.Hkv + g;
    float* po = p.part_o + static_cast<size_t>(unit) * p.n_splits * N * 128;
    float* pml = p.part_ml + static_cast<size_t>(unit) * p.n_splits * N * 2;
    float* my_o = po + static_cast<size_t>(split) * N * 128;
    const bool has0 = n_tiles > 0, has1 = n_tiles > 1;
    // merge the two warpgroups' O^T: warpgroup 0 takes even 16-column chunks, warpgroup 1 odd ones
    for (int c16 = wg; c16 < N / 16; c16 += 2) {
      float o0[16], o1[16];
      if (has0) tmem_ld16(tmem + lane_off + 2 * N + 16 * c16, o0);
      if (has1) tmem_ld16(tmem + lane_off + 3 * N + 16 * c16, o1);
      tc_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = 16 * c16 + j;
        const float m0 = mref_all[m], m1 = mref_all[64 + m];
        const float ms = fmaxf(m0, m1);
        float acc = 0.f;
        if (has0 && m0 != -INFINITY) acc += o0[j] * fast_exp2(m0 - ms);
        if (has1 && m1 != -INFINITY) acc += o1[j] * fast_exp2(m1 - ms);
        my_o[m * 128 + tk] = acc;
      }
    }
    if (wg == 0 && ts < N) {
      const float m0 = mref_all[ts], m1 = mref_all[64 + ts];
      const float ms = fmaxf(m0, m1);
      float lsum = 0.f;
      if (m0 != -INFINITY) lsum += ltot[ts] * fast_exp2(m0 - ms);
      if (m1 != -INFINITY) lsum += ltot[64 + ts] * fast_exp2(m1 - ms);
      pml[(split * N + ts) * 2] = ms;
      pml[(split * N + ts) * 2 + 1] = lsum;
    }
    tc_fence_before();
    float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
    combine_splits(po, pml, p.n_splits, N, M, p.counters + unit, flag, reinterpret_cast<float*>(smem),
                   wg * 128 + ts, 256, 1, [&](int row) { return out_unit + static_cast<size_t>(row) * 128; });
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

template <int N>
static cudaError_t launch_n(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  auto kern = verify_tc_kernel<N>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TCfg<N>::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(p.n_splits, p.Hkv, p.B);
  kern<<<grid, TCfg<N>::kThreads, TCfg<N>::kSmem, s>>>(tk, tv, p);
  return cudaGetLastError();
}

cudaError_t launch_verify_tc(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  const int n = (p.M + 15) / 16 * 16;
  switch (n) {
    case 16: return launch_n<16>(p, tk, tv, s);
    case 32: return launch_n<32>(p, tk, tv, s);
    case 48: return launch_n<48>(p, tk, tv, s);
    case 64: return launch_n<64>(p, tk, tv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sa
