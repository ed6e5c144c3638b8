// verify_tc.cu — tcgen05 (5th-gen tensor core) verify attention with the fused Collect-k byproduct.
//
// Reference: attend_collect / attend_segments / softmax_stable (attention.cpp:8-87) for every
// q-head and verify row t = 1..gamma+1 and the score_columns aggregation that
// consumes the LogitMatrix (selection.cpp:89-108).
//
// Swap-AB formulation (the GQA group x (gamma+1) rows are few, the keys many):
//   S^T[tok][row] = K[tok][:] . Q[row][:]     tcgen05.mma M=128 tokens, N=rows (<=64), K=d=128
//   O^T[d][row]  += V^T[d][tok] . P^T[tok][row]  M=d=128, N=rows, K=128 tokens (P split bf16 hi+lo)
// so TMEM lane = token for S and lane = d for O: each softmax thread owns ONE token and all of its
// query rows.  The Collect-2 score byproduct (sum over the G heads and the collected rows of raw
// q.k, selection.cpp:93-106) is therefore a thread-local sum written as one coalesced float per
// token — no LogitMatrix, no second pass.  The running row max is kept lazily: a tile whose logits
// all sit within 2^8 of the current reference max (the common case) needs no cross-thread work;
// otherwise the softmax warps reduce the row max, rescale their l partials and the O^T columns in
// TMEM, and continue (exact: every p is computed against the same reference as its O/l terms).
//
// Roles (192 threads): warp 0 TMA producer (128-token SWIZZLE_128B K/V tiles, 2-3 stage mbarrier
// ring), warp 1 MMA issuer (one elected thread issues tcgen05.mma and tcgen05.commit; owns the TMEM
// allocation), warps 2-5 softmax / epilogue (tcgen05.ld of S^T, P to shared memory in the
// MN-major SWIZZLE_64B layout, O^T readout).  The last split appends the gamma+1 window rows to the
// cache (fused KvStore::append) and then reads them back through TMA as part of its final tile,
// masking causally within the window (row t sees window keys j < t).
#include "attn_core.cuh"
#include "internal.h"

namespace sa {

template <int N>
struct TCfg {
  static constexpr int kTile = 128;
  static constexpr int kStages = (N <= 32) ? 3 : 2;
  static constexpr int kHalf = kTile * 128;            // one 64-column half of a K or V tile (16 KB)
  static constexpr int kTileBytes = 2 * kHalf;          // K or V tile (32 KB)
  static constexpr int kStageBytes = 2 * kTileBytes;    // K + V (64 KB)
  static constexpr int kQHalf = N * 128;
  static constexpr int kPAtoms = (N + 31) / 32;         // 32-row MN atoms of the SW64 P layout
  static constexpr int kPBytes = kPAtoms * kTile * 64;  // hi (or lo) P buffer
  static constexpr int kOffQ = kStages * kStageBytes;
  static constexpr int kOffP = kOffQ + 2 * kQHalf;
  static constexpr int kOffBar = kOffP + 2 * kPBytes;
  static constexpr int kNumBars = 2 * kStages + 7;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kMiscBytes = 16 + 4 * 64 * 4 + 4 * 64 * 4;  // slot/flag, mref/fac/lim/rmod, red[4][64]
  static constexpr int kSmem = kOffMisc + kMiscBytes + 1024;
  static constexpr int kThreads = 192;
  static constexpr uint32_t kTmemCols = (3 * N <= 128) ? 128 : 256;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

constexpr float kLazyMaxThresh = 8.0f;  // log2 units: p <= 2^8 before a forced max update

template <int N>
__global__ void __launch_bounds__(192, 1)
    verify_tc_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const VerifyParams p) {
  using C = TCfg<N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + C::kStages;
  uint64_t* s_full = bars + 2 * C::kStages;       // [2]
  uint64_t* s_empty = s_full + 2;                  // [2]
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 1;
  uint64_t* pv_done = p_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  int* flag = reinterpret_cast<int*>(smem + C::kOffMisc + 4);
  float* mref = reinterpret_cast<float*>(smem + C::kOffMisc + 16);
  float* fac = mref + 64;
  int* lim = reinterpret_cast<int*>(fac + 64);
  int* rmod = lim + 64;
  float* red = reinterpret_cast<float*>(rmod + 64);  // [4][64]

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

  // ------------------------------------------------------------------ prologue (all threads)
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(p_empty, 1);
    mbar_init(pv_done, 1);
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
    mref[tid] = -INFINITY;
    lim[tid] = tid < M ? p0 + tid % R : -1;  // key position limit of row m (causal window)
    rmod[tid] = tid < M ? tid % R : 0;
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
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t o_col = 2 * N;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % C::kStages;
        if (t >= C::kStages) mbar_wait(&kv_empty[st], ((t / C::kStages) & 1) ^ 1);
        const int row = static_cast<int>(cache_row(p.cache, seq, p.layer, g, tile0 + t * C::kTile));
        uint8_t* sk = smem + st * C::kStageBytes;
        uint8_t* sv = sk + C::kTileBytes;
        mbar_expect_tx(&kv_full[st], C::kStageBytes);
        tma_load_2d(sk, &tmk, &kv_full[st], 0, row, pol);
        tma_load_2d(sk + C::kHalf, &tmk, &kv_full[st], 64, row, pol);
        tma_load_2d(sv, &tmv, &kv_full[st], 0, row, pol);
        tma_load_2d(sv + C::kHalf, &tmv, &kv_full[st], 64, row, pol);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(N, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(N, 1, 1);
      const uint32_t q_base = smem_u32(sq);
      const uint32_t p_hi = smem_u32(smem + C::kOffP), p_lo = p_hi + C::kPBytes;
      auto issue_pv = [&](int u) {
        mbar_wait(p_full, u & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + (u % C::kStages) * C::kStageBytes + C::kTileBytes);
#pragma unroll
        for (int kt = 0; kt < 8; ++kt) {  // 16 tokens per MMA
          const uint64_t a = umma_desc(v_base + kt * 2048, C::kHalf, 1024, kLayoutSW128);
          const uint64_t bh = umma_desc(p_hi + kt * 1024, C::kTile * 64, 512, kLayoutSW64);
          const uint64_t bl = umma_desc(p_lo + kt * 1024, C::kTile * 64, 512, kLayoutSW64);
          umma_bf16(tmem + o_col, a, bh, idesc_pv, (u > 0 || kt > 0) ? 1u : 0u);
          umma_bf16(tmem + o_col, a, bl, idesc_pv, 1u);
        }
        umma_commit(&kv_empty[u % C::kStages]);
        umma_commit(p_empty);
        umma_commit(pv_done);
      };
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % C::kStages;
        mbar_wait(&kv_full[st], (t / C::kStages) & 1);
        if (t >= 2) mbar_wait(&s_empty[t & 1], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(smem + st * C::kStageBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // d in steps of 16
          const uint64_t a = umma_desc(k_base + (kk >> 2) * C::kHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
          const uint64_t bq = umma_desc(q_base + (kk >> 2) * C::kQHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
          umma_bf16(tmem + (t & 1) * N, a, bq, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t & 1]);
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue warps
    const int q4 = warp & 3;             // TMEM lane quarter this warp may access
    const int tk = q4 * 32 + lane;       // token within the tile (S) / d (O)
    const int ts = tid - 64;             // 0..127 among the softmax threads
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float c = p.scale_log2;
    uint64_t score_rows = 0, collect_rows = 0;
    for (int m = 0; m < M; ++m) {
      if ((p.score_mask >> (m % R)) & 1u) score_rows |= uint64_t{1} << m;
      if ((p.collect_mask >> (m % R)) & 1u) collect_rows |= uint64_t{1} << m;
    }
    float* score_out = p.scores ? p.scores + (static_cast<size_t>(b) * p.Hkv + g) * p.ld_scores : nullptr;
    uint8_t* pbuf = smem + C::kOffP;
    float l[N];
#pragma unroll
    for (int m = 0; m < N; ++m) l[m] = 0.f;

    for (int t = 0; t < n_tiles; ++t) {
      mbar_wait(&s_full[t & 1], (t >> 1) & 1);
      tc_fence_after();
      float s[N];
      tmem_ld_n<N>(tmem + lane_off + (t & 1) * N, s);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[t & 1]);
      const int pos = tile0 + t * C::kTile + tk;
      const bool in_range = pos >= lo && pos < hi;
      if (score_out && in_range && pos < p0) {  // fused Collect-k column sum (raw logits)
        float sc = 0.f;
#pragma unroll
        for (int m = 0; m < N; ++m)
          if ((score_rows >> m) & 1) sc += s[m];
        score_out[pos] = sc;
      }
      if (p.logits && in_range && pos < p0) {
#pragma unroll
        for (int m = 0; m < N; ++m)
          if ((collect_rows >> m) & 1) {
            const int r = rmod[m];
            const int ci = __popc(p.collect_mask & ((1u << r) - 1u));
            p.logits[((static_cast<size_t>(b) * Hq + g * p.G + m / R) * p.n_collect + ci) * p.ld_logits + pos] = s[m];
          }
      }
      float tv[N];
      bool exceed = false;
#pragma unroll
      for (int m = 0; m < N; ++m) {
        const bool valid = in_range && pos <= lim[m];
        tv[m] = valid ? fmaf(s[m], c, -mref[m]) : -INFINITY;
        exceed |= tv[m] > kLazyMaxThresh;
      }
      if (named_bar_or(2, 128, exceed)) {
        // Slow path: exact row max over this tile, rescale l partials and O^T columns.
#pragma unroll
        for (int m = 0; m < N; ++m) {
          float x = (in_range && pos <= lim[m]) ? s[m] * c : -INFINITY;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, off));
          if (lane == 0) red[q4 * 64 + m] = x;
        }
        named_bar_sync(2, 128);
        if (ts < N) {
          const float mo = mref[ts];
          const float mx = fmaxf(fmaxf(red[ts], red[64 + ts]), fmaxf(red[128 + ts], red[192 + ts]));
          const float mn = fmaxf(mo, mx);
          fac[ts] = (mo == -INFINITY) ? 0.f : (mn == mo ? 1.f : fast_exp2(mo - mn));
          mref[ts] = mn;
        }
        named_bar_sync(2, 128);
#pragma unroll
        for (int m = 0; m < N; ++m) l[m] *= fac[m];
        if (t > 0) {  // O^T accumulated through tile t-1 is final once PV(t-1) completes
          mbar_wait(pv_done, (t - 1) & 1);
          tc_fence_after();
          float v[N];
          tmem_ld_n<N>(tmem + lane_off + o_col, v);
          tc_wait_ld();
#pragma unroll
          for (int m = 0; m < N; ++m) v[m] *= fac[m];
          tmem_st_n<N>(tmem + lane_off + o_col, v);
          tc_wait_st();
        }
#pragma unroll
        for (int m = 0; m < N; ++m) {
          const bool valid = in_range && pos <= lim[m];
          tv[m] = valid ? fmaf(s[m], c, -mref[m]) : -INFINITY;
        }
      }
#pragma unroll
      for (int m = 0; m < N; ++m) {
        tv[m] = fast_exp2(tv[m]);  // p, in place
        l[m] += tv[m];
      }
      if (t >= 1) mbar_wait(p_empty, (t - 1) & 1);  // PV(t-1) finished reading the P buffer
#pragma unroll
      for (int a = 0; a < C::kPAtoms; ++a)
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint4 h, lw;
          uint32_t* hp = reinterpret_cast<uint32_t*>(&h);
          uint32_t* lp = reinterpret_cast<uint32_t*>(&lw);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = 32 * a + 8 * ch + 2 * e;
            const float x0 = m < N ? tv[m] : 0.f, x1 = m + 1 < N ? tv[m + 1] : 0.f;
            split_bf16(x0, x1, hp[e], lp[e]);
          }
          const uint32_t off = a * (C::kTile * 64) + tk * 64 + ((ch ^ ((tk >> 1) & 3)) << 4);
          *reinterpret_cast<uint4*>(pbuf + off) = h;
          *reinterpret_cast<uint4*>(pbuf + C::kPBytes + off) = lw;
        }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }

    // ---------------------------------------------------------------- epilogue
    if (n_tiles > 0) {
      mbar_wait(pv_done, (n_tiles - 1) & 1);
      tc_fence_after();
    }
#pragma unroll
    for (int m = 0; m < N; ++m) {
      float x = l[m];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      if (lane == 0) red[q4 * 64 + m] = x;
    }
    named_bar_sync(2, 128);
    const int unit = b * p.Hkv + g;
    float* po = p.part_o + static_cast<size_t>(unit) * p.n_splits * N * 128;
    float* pml = p.part_ml + static_cast<size_t>(unit) * p.n_splits * N * 2;
    float* my_o = po + static_cast<size_t>(split) * N * 128;
    {
      float v[N];
      if (n_tiles > 0) {
        tmem_ld_n<N>(tmem + lane_off + o_col, v);
        tc_wait_ld();
      } else {
#pragma unroll
        for (int m = 0; m < N; ++m) v[m] = 0.f;
      }
#pragma unroll
      for (int m = 0; m < N; ++m) my_o[m * 128 + tk] = v[m];
    }
    if (ts < N) {
      pml[(split * N + ts) * 2] = n_tiles > 0 ? mref[ts] : -INFINITY;
      pml[(split * N + ts) * 2 + 1] = red[ts] + red[64 + ts] + red[128 + ts] + red[192 + ts];
    }
    tc_fence_before();
    float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
    combine_splits(po, pml, p.n_splits, N, M, p.counters + unit, flag, reinterpret_cast<float*>(smem), ts, 128, 3,
                   [&](int row) { return out_unit + static_cast<size_t>(row) * 128; });
  }
  __syncthreads();
  if (warp == 1) {
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
