// verify.cu — fused verify attention + Collect-k logit byproduct (+ fused KV append).
//
// Reference: attend_collect / attend_segments / softmax_stable (attention.cpp:8-87) called by the
// SPEC verify pass for every q-head and row t = 1..gamma+1, and the
// score_columns aggregation (selection.cpp:89-108) that consumes its LogitMatrix.
//
// Grid (n_splits, Hkv, B): one CTA streams a contiguous chunk of one (sequence, KV head)'s prefix
// through shared memory with TMA (SWIZZLE_128B boxes of 64 tokens x 64 dims, 4-stage mbarrier
// ring, one producer warp), and MT x TG consumer warps run the mma.sync flash step of attn_core.cuh
// for all G*(gamma+1) query rows of the GQA group at once, so every K/V byte is read once per
// KV head rather than once per (q-head, row) as in the reference.
//
// Fused byproduct: two extra query rows hold hi/lo bf16 halves of q_sum = sum of the q rows whose
// logits the selector averages (Collect-2: rows 1 and gamma+1 of the G heads).  Their S entries sum
// to sum_{h,r} q_{h,r}.k_i = the selector's column sum for KV head g, emitted straight from the
// accumulator into scores[b][g][i] — no LogitMatrix round trip (selection.cpp:93-106).
//
// The last split of each unit also attends the gamma+1 window rows (causal within the window),
// read from k_new/v_new; split 0 appends them to the cache (fused KvStore::append).
#include "attn_core.cuh"
#include "internal.h"

namespace sa {

template <int MT, int TG>
struct VCfg {
  static constexpr int kTile = 64;
  static constexpr int kStages = 4;
  static constexpr int kNCW = MT * TG;
  static constexpr int kThreads = (kNCW + 1) * 32;
  static constexpr int kSubPerWarp = 4 / TG;
  static constexpr int kHalf = kTile * 128;
  static constexpr int kTileBytes = 2 * kHalf;
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kWinHalf = 16 * 128;
  static constexpr int kQHalf = MT * 16 * 128;
  static constexpr int kOffWinK = kStages * kStageBytes;
  static constexpr int kOffWinV = kOffWinK + 2 * kWinHalf;
  static constexpr int kOffQ = kOffWinV + 2 * kWinHalf;
  static constexpr int kOffBar = kOffQ + 2 * kQHalf;
  static constexpr int kOffMisc = kOffBar + 2 * kStages * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr int kMaxSplits = 128;
  static_assert(kNCW * kWpFloats * 4 <= kOffWinK && kMaxSplits * 64 * 8 <= kOffWinK, "epilogue scratch must fit");
};

template <int MT, int TG>
__global__ void __launch_bounds__(VCfg<MT, TG>::kThreads, 1)
    verify_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const VerifyParams p) {
  using Cfg = VCfg<MT, TG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
  uint64_t* empty = full + Cfg::kStages;
  int* misc = reinterpret_cast<int*>(smem + Cfg::kOffMisc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int seq = p.seq_ids[b];
  const int p0 = p.p0[b];
  const int R = p.R, M = p.M;
  const int tok_begin = split * p.chunk;
  const int tok_end = min(p0, tok_begin + p.chunk);
  const int n_tiles = tok_end > tok_begin ? ceil_div(tok_end - tok_begin, Cfg::kTile) : 0;
  const bool last_split = split == p.n_splits - 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kNCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------------ producer warp (TMA)
  if (warp == Cfg::kNCW) {
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % Cfg::kStages;
        if (t >= Cfg::kStages) mbar_wait(&empty[st], ((t / Cfg::kStages) & 1) ^ 1);
        const int row = static_cast<int>(cache_row(p.cache, seq, p.layer, g, tok_begin + t * Cfg::kTile));
        uint8_t* sk = smem + st * Cfg::kStageBytes;
        uint8_t* sv = sk + Cfg::kTileBytes;
        mbar_expect_tx(&full[st], Cfg::kStageBytes);
        tma_load_2d(sk, &tmk, &full[st], 0, row, pol);
        tma_load_2d(sk + Cfg::kHalf, &tmk, &full[st], 64, row, pol);
        tma_load_2d(sv, &tmv, &full[st], 0, row, pol);
        tma_load_2d(sv + Cfg::kHalf, &tmv, &full[st], 64, row, pol);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  const int tid = threadIdx.x;
  constexpr int nct = Cfg::kNCW * 32;
  const int mt = warp % MT, tg = warp / MT;
  const int Hq = p.Hkv * p.G;
  uint8_t* sq = smem + Cfg::kOffQ;
  uint8_t* swk = smem + Cfg::kOffWinK;
  uint8_t* swv = smem + Cfg::kOffWinV;

  // Q tile (rows m = gl*R + r of the G heads of KV head g), zero-padded to MT*16 rows.
  const __nv_bfloat16* qb = p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
  for (int i = tid; i < MT * 16 * 16; i += nct) {
    const int row = i >> 4, ch = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < M) v = __ldg(reinterpret_cast<const uint4*>(qb + row * 128 + ch * 8));
    *reinterpret_cast<uint4*>(sq + swz(row, ch, Cfg::kQHalf)) = v;
  }
  // Window rows p0..p0+R-1 (last split), zero-padded to 16.
  if (last_split) {
    for (int i = tid; i < 2 * 16 * 16; i += nct) {
      const int which = i >> 8, row = (i >> 4) & 15, ch = i & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (row < R) {
        const __nv_bfloat16* src;
        if (p.k_new) {
          src = (which ? p.v_new : p.k_new) + ((static_cast<size_t>(b) * R + row) * p.Hkv + g) * 128;
        } else {
          const int64_t cr = cache_row(p.cache, seq, p.layer, g, p0 + row);
          src = (which ? p.cache.v : p.cache.k) + cr * 128;
        }
        v = __ldg(reinterpret_cast<const uint4*>(src + ch * 8));
      }
      *reinterpret_cast<uint4*>((which ? swv : swk) + swz(row, ch, Cfg::kWinHalf)) = v;
    }
  }
  // Fused append of the window rows (KvStore::append, kv_store.cpp:39-45) by split 0.
  if (split == 0 && p.k_new) {
    for (int i = tid; i < 2 * R * 16; i += nct) {
      const int which = i / (R * 16), row = (i / 16) % R, ch = i & 15;
      const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + ((static_cast<size_t>(b) * R + row) * p.Hkv + g) * 128;
      const int64_t cr = cache_row(p.cache, seq, p.layer, g, p0 + row);
      __nv_bfloat16* dst = (which ? p.cache.v : p.cache.k) + cr * 128;
      reinterpret_cast<uint4*>(dst)[ch] = __ldg(reinterpret_cast<const uint4*>(src) + ch);
    }
  }
  named_bar_sync(1, nct);
  // q_sum rows (hi at hi_row, lo at hi_row+1) for the fused score byproduct.
  if ((p.scores || p.score_fx) && tid < 128) {
    float acc = 0.f;
    const uint32_t off = swz(0, tid >> 3, Cfg::kQHalf) + (tid & 7) * 2;  // row 0 position of column tid
    for (int m = 0; m < M; ++m) {
      if (!((p.score_mask >> (m % R)) & 1u)) continue;
      const uint32_t o = swz(m, tid >> 3, Cfg::kQHalf) + (tid & 7) * 2;
      acc += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(sq + o));
    }
    (void)off;
    const __nv_bfloat16 hi = __float2bfloat16_rn(acc);
    const __nv_bfloat16 lo = __float2bfloat16_rn(acc - __bfloat162float(hi));
    *reinterpret_cast<__nv_bfloat16*>(sq + swz(p.hi_row, tid >> 3, Cfg::kQHalf) + (tid & 7) * 2) = hi;
    *reinterpret_cast<__nv_bfloat16*>(sq + swz(p.hi_row + 1, tid >> 3, Cfg::kQHalf) + (tid & 7) * 2) = lo;
  }
  named_bar_sync(1, nct);

  WarpAttn w;
  w.init();
  w.load_q(smem_u32(sq), Cfg::kQHalf, mt, lane);
  const float c = p.scale_log2;
  const int gid = lane >> 2, t4 = lane & 3;
  const bool score_warp = (mt == MT - 1) && (p.scores != nullptr || p.score_fx != nullptr);
  long long* score_fx = p.score_fx ? p.score_fx + static_cast<size_t>(b) * p.ld_scores : nullptr;
  const int hi_local = p.hi_row - 16 * (MT - 1), lo_local = hi_local + 1;
  float* score_out = p.scores ? p.scores + (static_cast<size_t>(b) * p.Hkv + g) * p.ld_scores : nullptr;

  for (int t = 0; t < n_tiles; ++t) {
    const int st = t % Cfg::kStages;
    mbar_wait(&full[st], (t / Cfg::kStages) & 1);
    const uint32_t kt = smem_u32(smem + st * Cfg::kStageBytes);
    const uint32_t vt = kt + Cfg::kTileBytes;
    const int tile_tok0 = tok_begin + t * Cfg::kTile;
#pragma unroll
    for (int sb = 0; sb < Cfg::kSubPerWarp; ++sb) {
      const int r0 = (tg + sb * TG) * 16;
      float s[2][4];
      w.qk(kt, Cfg::kHalf, r0, lane, s);
      if (score_warp) {  // fused Collect-k column sums (raw, unscaled: attention.hpp:18-21)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          float v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float vh = (hi_local >> 3) ? s[nt][2 + e] : s[nt][e];
            const float vl = (lo_local >> 3) ? s[nt][2 + e] : s[nt][e];
            v[e] = vh + __shfl_sync(0xffffffffu, vl, (lo_local & 7) * 4 + t4);
          }
          const int pos = tile_tok0 + r0 + 8 * nt + 2 * t4;
          if (gid == (hi_local & 7)) {
            if (score_fx) {  // per-layer: integer atomics over the KV heads (order-independent)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (pos + e < tok_end)
                  atomicAdd(reinterpret_cast<unsigned long long*>(score_fx + pos + e),
                            static_cast<unsigned long long>(__float2ll_rn(v[e] * kScoreFxScale)));
            } else if (pos + 1 < tok_end) {
              *reinterpret_cast<float2*>(score_out + pos) = make_float2(v[0], v[1]);
            } else if (pos < tok_end) {
              score_out[pos] = v[0];
            }
          }
        }
      }
      if (p.logits) {  // debug / variant path: raw prefix logits of the collected rows
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          const int m = mt * 16 + gid + 8 * sl;
          if (m >= M) continue;
          const int r = m % R;
          if (!((p.collect_mask >> r) & 1u)) continue;
          const int ci = __popc(p.collect_mask & ((1u << r) - 1u));
          float* dst = p.logits + ((static_cast<size_t>(b) * Hq + g * p.G + m / R) * p.n_collect + ci) * p.ld_logits;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int pos = tile_tok0 + r0 + 8 * nt + 2 * t4 + e;
              if (pos < tok_end) dst[pos] = s[nt][2 * sl + e];
            }
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (tile_tok0 + r0 + 8 * nt + 2 * t4 + (e & 1) >= tok_end) s[nt][e] = -INFINITY;
      w.softmax_pv(s, vt, Cfg::kHalf, r0, lane, c);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // Window tile: key j (position p0+j) is visible to row t = r+1 iff j <= r (causal window).
  if (last_split && tg == 0) {
    float s[2][4];
    w.qk(smem_u32(swk), Cfg::kWinHalf, 0, lane, s);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 8 * nt + 2 * t4 + (e & 1);
        const int m = mt * 16 + gid + 8 * (e >> 1);
        if (j >= R || j > m % R) s[nt][e] = -INFINITY;
      }
    w.softmax_pv(s, smem_u32(swv), Cfg::kWinHalf, 0, lane, c);
  }
  w.finalize_l();

  // Epilogue: warp partials -> CTA split partial -> last CTA merges splits.
  named_bar_sync(1, nct);  // every consumer is done with the stage ring
  float* wps = reinterpret_cast<float*>(smem);
  store_warp_partial(w, wps + warp * kWpFloats, lane);
  named_bar_sync(1, nct);
  const int unit = b * p.Hkv + g;
  const int rows_pad = MT * 16;
  float* po = p.part_o + static_cast<size_t>(unit) * p.n_splits * rows_pad * 128;
  float* pml = p.part_ml + static_cast<size_t>(unit) * p.n_splits * rows_pad * 2;
  cta_partial_to_global<MT, TG>(wps, po + static_cast<size_t>(split) * rows_pad * 128,
                                pml + static_cast<size_t>(split) * rows_pad * 2, tid, nct);
  float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
  combine_splits(po, pml, p.n_splits, rows_pad, M, p.counters + unit, misc, wps, tid, nct,
                 1, [&](int row) { return out_unit + static_cast<size_t>(row) * 128; });
}

size_t verify_smem_bytes(int MT) {
  switch (MT) {
    case 1: return VCfg<1, 4>::kSmem;
    case 2: return VCfg<2, 4>::kSmem;
    case 3: return VCfg<3, 4>::kSmem;
    default: return VCfg<4, 2>::kSmem;
  }
}

int verify_max_ctas_per_sm(int) { return 1; }

template <int MT, int TG>
static cudaError_t launch_mt(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  using Cfg = VCfg<MT, TG>;
  auto kern = verify_kernel<MT, TG>;
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  if (func_attrs_needed(attr_mask, &dev)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return e;
    func_attrs_done(attr_mask, dev);
  }
  dim3 grid(p.n_splits, p.Hkv, p.B);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, s>>>(tk, tv, p);
  return cudaGetLastError();
}

cudaError_t launch_verify(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  switch (p.MT) {
    case 1: return launch_mt<1, 4>(p, tk, tv, s);
    case 2: return launch_mt<2, 4>(p, tk, tv, s);
    case 3: return launch_mt<3, 4>(p, tk, tv, s);
    case 4: return launch_mt<4, 2>(p, tk, tv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sa
