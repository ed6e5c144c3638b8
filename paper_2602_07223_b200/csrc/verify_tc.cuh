#pragma once
// verify_tc.cuh — tcgen05 (5th-gen tensor core) verify attention with the fused Collect-k byproduct.
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
// Warp roles (384 threads, setmaxnreg-rebalanced): w0 TMA producer (one thread, 128-token SWIZZLE_128B
// boxes, separate K and V rings so K is recycled right after QK^T), w1 MMA issuer (single thread; owns
// the TMEM allocation), w2-3 spare (warpgroup 0 drops to 72 registers), w4-7 softmax warpgroup 0,
// w8-11 softmax warpgroup 1 (216 registers each).  The last split appends the
// gamma+1 window rows to the cache (fused KvStore::append) and reads them back through TMA as part of
// its final tile, masked causally inside the window (row t sees window keys j < t).
#include "attn_core.cuh"
#include <cstdlib>

#include "internal.h"

namespace sa {

template <int N>
struct TCfg {
  static constexpr int kTile = 128;
  // K ring stages (K is recycled right after QK^T); N = 64 keeps one so the three P planes fit
  static constexpr int kSK = N <= 48 ? 2 : 1;
  static constexpr int kSV = (N <= 32) ? 3 : 2;       // V ring stages (V is held until PV retires)
  static constexpr int kHalf = kTile * 128;           // one 64-column half of a K or V tile (16 KB)
  static constexpr int kTileBytes = 2 * kHalf;         // K or V tile (32 KB)
  static constexpr int kQHalf = N * 128;
  // P^T planes (bf16, MN-major SWIZZLE_32B, 16-row atoms): P = hi + mid + lo to ~2^-27 relative
  // (the tau = 1e-3 elementwise bar of SURVEY §8c needs more than the ~2^-17 of hi + lo: two planes
  // measured 2.3e-3 at G*(gamma+1) = 56)
  static constexpr int kPlanes = 3;
  static constexpr int kPAtoms = N / 16;               // 16-row MN atoms of the SW32 P layout
  static constexpr int kPBytes = kPAtoms * kTile * 32; // one P plane (N rows x 128 tokens)
  static constexpr int kNP = kPlanes * N;              // merged PV width: [P_hi | P_mid | P_lo] columns
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kSK * kTileBytes;
  static constexpr int kOffQ = kOffV + kSV * kTileBytes;
  static constexpr int kOffP = kOffQ + 2 * kQHalf;     // [wg][planes]
  static constexpr int kOffBar = kOffP + 2 * kPlanes * kPBytes;
  static constexpr int kPosRing = 8;                  // published tile positions (consumer-visible)
  static constexpr int kNumBars = 2 * kSK + 2 * kSV + 8 + kPosRing + 2;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  // misc: tmem slot, flag, ntiles[2] | mref[2][64] fac[2][64] ltot[2][64] wsc[64] lim[64] | red[2][4][64]
  //       | tile_pos[kPosRing] | producer ring pring[32]
  static constexpr int kBtMax = 1024;                  // block-table entries staged in smem
  static constexpr int kMiscBytes = 16 + (2 + 2 + 2 + 1 + 1) * 64 * 4 + 2 * 4 * 64 * 4 + kPosRing * 4 + 32 * 4 +
                                    kBtMax * 4 + 64 * 4;
  static constexpr int kSmem = kOffMisc + kMiscBytes + 1024;
  static constexpr int kThreads = 384;
  // TMEM columns: S[2] (N each), O[2] (kNP each: one N-column block per P plane), then Oacc[2] (N each)
  static constexpr int kOCol = 2 * N;
  static constexpr int kACol = 2 * N + 2 * kNP;
  static constexpr int kColsBase = 2 * N + 2 * kNP;  // without Oacc (flushing off)
  static constexpr bool kFlushable = 4 * N + 2 * kNP <= 512;  // Oacc fits TMEM (N <= 48)
  static constexpr int kCols = kFlushable ? 4 * N + 2 * kNP : kColsBase;
  static constexpr uint32_t kTmemCols = kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  static constexpr uint32_t kTmemColsBase = kColsBase <= 128 ? 128 : kColsBase <= 256 ? 256 : 512;
  static_assert(kCols <= 512, "TMEM columns");
  // Accumulation blocks: the tensor core's fp32 accumulate is not IEEE round-to-nearest, so its error
  // grows with the number of MMAs chained into one accumulator (one CTA streaming a whole 64K prefix,
  // config 3: 2.6e-2 elementwise against the reference).  Every kFlush tiles of a warpgroup, the
  // softmax threads fold the O^T planes into Oacc with IEEE fp32 adds and the next PV restarts
  // the accumulator, so no chain is longer than flush * 8 MMAs (p.flush_tiles; 0: one block per CTA).
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

constexpr float kLazyMaxThresh = 8.0f;

// Butterfly all-reduce of N independent values across the warp, level-outer so the N shuffles of
// each level pipeline instead of forming N serial 5-deep chains.
// Float max across the warp with one REDUX per value: IEEE bits mapped to an order-preserving s32
// (negative values get their magnitude bits flipped), redux.sync.max.s32, mapped back.
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : (i ^ 0x7FFFFFFF);
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : (i ^ 0x7FFFFFFF)); }
template <int N>
__device__ __forceinline__ void warp_allreduce_max(float (&x)[N]) {
#pragma unroll
  for (int m = 0; m < N; ++m) x[m] = ord2f(__reduce_max_sync(0xffffffffu, f2ord(x[m])));
}
// Sum N per-lane values over the 32 lanes with a transposing butterfly: each level halves the values
// a lane keeps (the upper half when the level's lane bit is set) and adds its partner's other half,
// so 31 shuffles do what N x 5 would.  Lane l ends with the sum of row l (N = 32), rows 2l, 2l+1
// (N = 64, values past N are zero padding) or row l >> 1 (N = 16); they go to out[row].
template <int N>
__device__ __forceinline__ void warp_transpose_sum_store(const float (&x)[N], int lane, float* out) {
  constexpr int NP = N <= 16 ? 16 : N <= 32 ? 32 : 64;
  float v[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) v[i] = i < N ? x[i] : 0.f;
  int cnt = NP;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (cnt > 1) {
      const int half = cnt >> 1;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < NP / 2; ++i) {
        if (i < half) {
          const float keep = upper ? v[half + i] : v[i];
          const float send = upper ? v[i] : v[half + i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      cnt = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  if (NP == 32) {
    out[lane] = v[0];
  } else if (NP == 64) {
    out[2 * lane] = v[0];
    out[2 * lane + 1] = v[1];
  } else if ((lane & 1) == 0) {
    out[lane >> 1] = v[0];
  }
}
template <int N>
__device__ __forceinline__ void warp_allreduce_sum(float (&x)[N]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int m = 0; m < N; ++m) x[m] += __shfl_xor_sync(0xffffffffu, x[m], off);
}

// dev-only per-CTA phase timestamps (globaltimer ns): slot k of CTA `cta_lin` in layer p.layer
#ifdef SA_PIPE_TRACE
constexpr bool kPipeTrace = true;
#else
constexpr bool kPipeTrace = false;  // product build: every kernel-internal timing stamp compiled out
#endif
#ifndef SA_PIPE_TRACE
#define SA_TSTAMP(k) \
  do {               \
  } while (0)
#else
#define SA_TSTAMP(k)                                                                            \
  do {                                                                                          \
    if (p.trace && cta_lin < 1024) {                                                            \
      unsigned long long gt_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                                   \
      p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin + (k)] = gt_;                          \
    }                                                                                           \
  } while (0)
#endif

// dev-only pipeline trace: ev[e][t] = clock64 of event e at tile t for CTA (0,0,0)
// Per-tile pipeline stamps of CTA 0 (tools/trace_verify.py): a dev build only
// (make -C paper_2602_07223_b200/csrc EXTRA_NVFLAGS=-DSA_PIPE_TRACE); the checks cost 0.5 us per layer.
#ifndef SA_PIPE_TRACE
#define SA_TRACE(e, t) \
  do {                 \
  } while (0)
#else
#define SA_TRACE(e, t)                                                                          \
  do {                                                                                          \
    if (p.trace && p.layer == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (t) < 64) \
      p.trace[(e) * 64 + (t)] = clock64();                                                      \
  } while (0)
#endif  // log2 units: p <= 2^8 before a forced max update

// Designated merger `part` (= split index < n_mergers) of a unit: rows [r_lo, r_hi) of the output.
// It polls the unit's per-split "partial published" flags (set with st.release by every CTA after
// its partial stores) and bulk-loads each split's (m, l) table and row slice into shared memory as
// soon as that split is published, so when the last split publishes only its own small slice is
// still in flight; then combines in fixed split order (deterministic) and resets its flags.
__device__ __forceinline__ void merge_rows_progressive(uint8_t* smem, uint64_t* bar, const float* src_o,
                                                       const float* src_ml, int cnt, int N, int r_lo, int r_hi,
                                                       float* dst_o, int* flags, int t256,
                                                       unsigned long long* tstamp = nullptr) {
  auto stamp = [&](int k) {  // dev trace: globaltimer into the CTA's trace row (slots 7, 8)
    if (tstamp) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      tstamp[k] = gt;
    }
  };
  const int nr = r_hi - r_lo;
  const uint32_t obytes = static_cast<uint32_t>(max(nr, 0)) * 512u;
  const uint32_t mlb = static_cast<uint32_t>(N) * 8u;  // one split's (m, l) table
  float2* sml = reinterpret_cast<float2*>(smem);                              // [partial][N] (m, l)
  uint8_t* sop = smem + ((static_cast<uint32_t>(cnt) * mlb + 127u) & ~127u);  // [partial][nr][128]
  if (t256 < 32) {  // one warp: lane l watches splits l, l + 32, ... (all flag loads in flight together)
    const int lane = t256;
    uint32_t mine = 0;  // splits of this lane not yet loaded (bit j: split lane + 32 j; cnt <= 128)
    for (int j = 0; 32 * j + lane < cnt; ++j) mine |= 1u << j;
    while (__any_sync(0xffffffffu, mine != 0)) {
      bool got = false;
      for (int j = 0; j < 4; ++j) {
        if (!((mine >> j) & 1u)) continue;
        const int s2 = 32 * j + lane;
        int f;  // relaxed poll (L2, no L1 invalidation per probe); the fence below acquires
        asm volatile("ld.relaxed.gpu.s32 %0, [%1];" : "=r"(f) : "l"(flags + s2) : "memory");
        if (!f) continue;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        fence_proxy_async();  // the split's generic-proxy stores (acquired) -> async-proxy reads
        mbar_expect_tx_only(bar, mlb + obytes);
        bulk_load(reinterpret_cast<uint8_t*>(sml) + s2 * mlb, src_ml + static_cast<size_t>(s2) * N * 2, mlb, bar);
        if (nr > 0) bulk_load(sop + s2 * obytes, src_o + static_cast<size_t>(s2) * N * 128 + r_lo * 128, obytes, bar);
        flags[s2] = 0;  // re-armed for this workspace's next use (two layers on, PDL-ordered)
        mine &= ~(1u << j);
        got = true;
      }
      (void)got;
    }
    __syncwarp();
    if (lane == 0) {
      stamp(7);
      mbar_arrive(bar);  // every expected byte is now accounted for
    }
  }
  mbar_wait(bar, 0);
  if (t256 == 0) stamp(8);
  if (nr <= 0) return;
  const float4* so = reinterpret_cast<const float4*>(sop);
  for (int it = t256; it < nr * 32; it += 256) {
    const int rr = it >> 5, c4 = it & 31, row = r_lo + rr;
    float mstar = -INFINITY;
    for (int s0 = 0; s0 < cnt; s0 += 8) {
      float mm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mm[u] = s0 + u < cnt ? sml[(s0 + u) * N + row].x : -INFINITY;
#pragma unroll
      for (int u = 0; u < 8; ++u) mstar = fmaxf(mstar, mm[u]);
    }
    float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    float lsum = 0.f;
    for (int s0 = 0; s0 < cnt; s0 += 8) {
      float4 v[8];
      float2 ml[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = s0 + u < cnt;
        v[u] = ok ? so[((s0 + u) * nr + rr) * 32 + c4] : make_float4(0.f, 0.f, 0.f, 0.f);
        ml[u] = ok ? sml[(s0 + u) * N + row] : make_float2(-INFINITY, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float w = ml[u].x == -INFINITY ? 0.f : fast_exp2(ml[u].x - mstar);
        lsum = fmaf(ml[u].y, w, lsum);
        float4& a = acc[u & 1];
        a.x = fmaf(v[u].x, w, a.x);
        a.y = fmaf(v[u].y, w, a.y);
        a.z = fmaf(v[u].z, w, a.z);
        a.w = fmaf(v[u].w, w, a.w);
      }
    }
    const float inv = 1.f / lsum;
    reinterpret_cast<float4*>(dst_o + static_cast<size_t>(row) * 128)[c4] =
        make_float4((acc[0].x + acc[1].x) * inv, (acc[0].y + acc[1].y) * inv, (acc[0].z + acc[1].z) * inv,
                    (acc[0].w + acc[1].w) * inv);
  }
}

// MR: the softmax rows that can be real (M rounded up to 4, <= N); rows MR..N-1 of the MMA tile are
// padding and get no softmax work (P = 0).
template <int N, int MR, bool kFlush, bool kLogits, bool kRS>
__global__ void __launch_bounds__(384, 1)
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
  // p_empty[wg] completes when the PV MMAs of the warpgroup's tile retire (tcgen05.commit after them),
  // so it also marks "O^T final through that tile"; every phase of it is waited (no stray phases)
  uint64_t* pos_bar = p_empty + 2;  // [kPosRing]
  uint64_t* dep_bar = pos_bar + C::kPosRing;  // Q staged + window appended (after griddepcontrol.wait)
  uint64_t* merge_bar = dep_bar + 1;          // split merge: partials bulk-loaded into smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  int* flag = reinterpret_cast<int*>(smem + C::kOffMisc + 4);
  float* mref_all = reinterpret_cast<float*>(smem + C::kOffMisc + 16);  // [2][64]
  float* fac_all = mref_all + 128;                                       // [2][64]
  float* ltot = fac_all + 128;                                           // [2][64]
  float* wsc = ltot + 128;                                               // [64] score weights 0/1
  int* lim = reinterpret_cast<int*>(wsc + 64);                           // [64]
  float* red_all = reinterpret_cast<float*>(lim + 64);                   // [2][4][64]
  int* tile_pos = reinterpret_cast<int*>(red_all + 512);                 // [kPosRing]
  int* pring = tile_pos + C::kPosRing;                                   // [32] producer-private
  int* bt = pring + 32;                                                  // [kBtMax] this sequence's pages
  int* loff = bt + C::kBtMax;  // [64] raw-logit output offset of row m (LogitMatrix path), -1: not collected
  int* ntiles_wg = flag + 1;                                             // [2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int seq = p.seq_ids[b];
  const int p0 = p.p0[b];
  const int R = p.R, M = p.M, Hq = p.Hkv * p.G;
  // Work split: full prefix tiles [0, n_pref*128) are shared by the unit's CTAs through chunks of
  // kChunkTiles tiles — chunk `split` first, then chunks claimed from an atomic counter (dynamic
  // balancing: attention is permutation-invariant and the score byproduct is position-indexed).
  // The window tile(s) [n_pref*128, p0+R) (prefix tail + the gamma+1 window rows) belong to the
  // last split, which also appends the window rows; they come last in its tile stream.
  //
  // Programmatic dependent launch (iteration graph): the prefix K/V of this layer does not depend on
  // the previous kernel, so the producer starts streaming at once; Q and the new window rows (in a
  // real model produced from the previous layer's output) are read by the MMA warp only after
  // griddepcontrol.wait, which then releases dep_bar.
  const bool last = split == p.n_splits - 1;
  const int n_pref = p0 / C::kTile;
  const int win_lo = n_pref * C::kTile;
  const int n_win = (p0 + R - win_lo + C::kTile - 1) / C::kTile;
  const int chunk_tiles = p.chunk_tiles;
  // chunks: n_big chunks of chunk_tiles tiles, then single-tile chunks for the last n_tail tiles of the
  // prefix (claims are monotonic, so the final claims of every CTA are small: less loop-end spread)
  // (short prefixes keep whole chunks: every chunk is then a CTA's static first one, no claims)
  const int n_tail_t = min(p.tail_tiles, max(0, n_pref - 2 * p.n_splits));
  const int n_big = (n_pref - n_tail_t) / chunk_tiles;
  const int n_chunks = n_big + (n_pref - n_big * chunk_tiles);
  auto chunk_start = [&](int c) { return c < n_big ? c * chunk_tiles : n_big * chunk_tiles + (c - n_big); };
  auto chunk_len = [&](int c) { return c < n_big ? chunk_tiles : 1; };
  const int unit = b * p.Hkv + g;
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
    for (int i = 0; i < C::kPosRing; ++i) mbar_init(&pos_bar[i], 1);
    mbar_init(dep_bar, 1);
    mbar_init(merge_bar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kRS ? 256 : 128);  // kRS: both warpgroups read every S and write every P
      mbar_init(&p_full[i], kRS ? 256 : 128);
      mbar_init(&p_empty[i], 1);
    }
    fence_mbar_init();
  }
  uint8_t* sq = smem + C::kOffQ;
  for (int i = tid; i < ((p0 + R + (1 << p.cache.page_shift) - 1) >> p.cache.page_shift); i += C::kThreads)
    bt[i] = __ldg(p.cache.block_table + static_cast<int64_t>(seq) * p.cache.max_pages_per_seq + i);
  if (tid < 64) {
    mref_all[tid] = -INFINITY;
    mref_all[64 + tid] = -INFINITY;
    lim[tid] = tid < M ? p0 + tid % R : -1;  // last key position row m may see (causal window)
    wsc[tid] = (tid < M && ((p.score_mask >> (tid % R)) & 1u)) ? 1.f : 0.f;
    const int r = tid % R;
    loff[tid] = (p.logits && tid < M && ((p.collect_mask >> r) & 1u))
                    ? ((g * p.G + tid / R) * p.n_collect + __popc(p.collect_mask & ((1u << r) - 1u))) *
                          static_cast<int>(p.ld_logits)
                    : -1;
  }
  // accumulation block length (tiles); N = 64 has no TMEM room for Oacc (one block per CTA)
  // kFlush / kLogits instantiations carry the accumulation-block fold / the LogitMatrix stores; without
  // them the softmax loop is shorter (0.6 / 0.55 us per layer, same-box A/B)
  const bool flushing = C::kFlushable && kFlush && p.flush_tiles > 0;
  const int flush = flushing ? p.flush_tiles : (1 << 30);
  const uint32_t tmem_cols = flushing ? C::kTmemCols : C::kTmemColsBase;
  if (MR < N) {  // P^T rows >= MR stay zero: the softmax never stores the all-padding 8-row chunks
    uint4* pz = reinterpret_cast<uint4*>(smem + C::kOffP);
    for (int i = tid; i < 2 * C::kPlanes * C::kPBytes / 16; i += C::kThreads) pz[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();  // generic zero stores -> the tensor core's (async-proxy) reads
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) SA_TRACE(11, 0);
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (kPipeTrace && p.trace && tid == 0 && cta_lin < 1024) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin] = gt;
    for (int k = 4; k < 16; ++k) p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin + k] = 0;
  }
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
  setmaxnreg_dec<72>();  // warpgroup 0: producer / MMA issuer / spare
  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (one thread)
    // K and V rings are refilled independently (K frees right after QK^T, V after PV): the thread
    // polls both empty barriers without blocking and issues whichever stage is free.
    if (lane == 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
      const uint64_t pol = policy_evict_first();
      if (p.no_prefill) mbar_wait(dep_bar, 0);  // dev knob: no ring prefill before the dependency
      // tile stream of this CTA: window tiles (last split), then its chunks; pring holds positions
      int q_end = 0, cur_chunk = -1, cur_tile = 0, claims = 0, pending = 0;
      bool exhausted = false, done = false, dep_seen = false, win_added = false;
      auto fill = [&](int upto) {
        while (q_end < upto && !exhausted) {
          if (cur_chunk < 0 || cur_tile == chunk_len(cur_chunk)) {
            if (last && claims == 1 && !win_added) {  // window tiles go right after the first chunk
              for (int w2 = 0; w2 < n_win; ++w2) pring[q_end++ & 31] = win_lo + w2 * C::kTile;
              win_added = true;
            }
            // claims run one chunk ahead: the atomic's L2 round trip overlaps the current chunk (its
            // result register is first read here, one chunk later); no claim is left unconsumed
            if (p.static_first) {
              cur_chunk = claims++ == 0 ? split : p.n_splits + pending;
            } else {  // fully dynamic: a CTA that starts late (SM held by another kernel) takes no chunk
              cur_chunk = claims++ == 0 ? atomicAdd(p.chunk_ctr + unit, 1) : pending;
            }
            if (cur_chunk < n_chunks) pending = (p.static_first ? 0 : 0) + atomicAdd(p.chunk_ctr + unit, 1);
            if (cur_chunk >= n_chunks) {
              exhausted = true;
              break;
            }
            cur_tile = 0;
          }
          pring[q_end++ & 31] = (chunk_start(cur_chunk) + cur_tile++) * C::kTile;
        }
        if (exhausted && !done) {  // (short prefixes: the window tiles close the stream)
          if (last && !win_added)
            for (int w2 = 0; w2 < n_win; ++w2) pring[q_end++ & 31] = win_lo + w2 * C::kTile;
          done = true;
        }
      };
      // block table staged in shared memory by the prologue: no dependent global load per tile
      auto row_of = [&](int pos) {
        return ((((p.layer * p.cache.num_pages + bt[pos >> p.cache.page_shift]) * p.cache.n_kv_heads + g)
                 << p.cache.page_shift) | (pos & ((1 << p.cache.page_shift) - 1)));
      };
      int nk = 0, nv = 0;
      while (true) {
        fill(nk + 1);
        // no L2 prefetch: every form measured slower — the next layer's first chunks, tiles ahead of the
        // ring, the CTA's own tiles during the dependency wait, and even the tiles inside the V ring window
        // (same-box A/B: 30.7 -> 28.4 us per layer without it)
        if (nk < q_end && (nk < C::kSK || mbar_test(&k_empty[nk % C::kSK], ((nk / C::kSK) & 1) ^ 1))) {
          const int st = nk % C::kSK, pos = pring[nk & 31];
          if (pos >= win_lo && !dep_seen) {  // window rows are appended after the dependency wait
            mbar_wait(dep_bar, 0);
            dep_seen = true;
          }
          tile_pos[nk % C::kPosRing] = pos;  // publish before the loads (mbarrier arrive = release)
          mbar_arrive(&pos_bar[nk % C::kPosRing]);
          const int row = row_of(pos);
          uint8_t* dst = smem + C::kOffK + st * C::kTileBytes;
          mbar_expect_tx(&k_full[st], C::kTileBytes);
          tma_load_2d(dst, &tmk, &k_full[st], 0, row, pol);
          tma_load_2d(dst + C::kHalf, &tmk, &k_full[st], 64, row, pol);
          SA_TRACE(0, nk);
          ++nk;
        }
        if (nv < nk && (nv < C::kSV || mbar_test(&v_empty[nv % C::kSV], ((nv / C::kSV) & 1) ^ 1))) {
          const int st = nv % C::kSV;
          const int row = row_of(pring[nv & 31]);
          uint8_t* dst = smem + C::kOffV + st * C::kTileBytes;
          mbar_expect_tx(&v_full[st], C::kTileBytes);
          tma_load_2d(dst, &tmv, &v_full[st], 0, row, pol);
          tma_load_2d(dst + C::kHalf, &tmv, &v_full[st], 64, row, pol);
          SA_TRACE(1, nv);
          ++nv;
        }
        if (done && nk == q_end && nv == nk) break;
      }
      // end of stream for both softmax warpgroups and the MMA issuer
      for (int e = 0; e < 2; ++e) {
        tile_pos[(nk + e) % C::kPosRing] = -1;
        mbar_arrive(&pos_bar[(nk + e) % C::kPosRing]);
      }
    }
  } else {
    // ------------------------- warps 1-3: dependency wait, Q staging, fused window append (96 threads,
    // every global load of a batch in flight together)
    // the unit's query rows into L2 before the wait (they come from the previous layer; L2 is the point
    // of coherence, so the lines cannot go stale; same-box A/B: -0.14 us per layer)
    if (tid - 32 < (M * 256 + 1023) / 1024)
      prefetch_l2_bulk(p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128 + (tid - 32) * 512,
                       min(1024, M * 256 - (tid - 32) * 1024));
    pdl_wait();
    const int t96 = tid - 32;
    const __nv_bfloat16* qb = p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
    constexpr int kQ = N * 16;  // 16-byte chunks of the padded Q tile
    for (int base = t96; base < kQ; base += 96 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * 96, row = i >> 4, ch = i & 15;
        v[u] = make_uint4(0, 0, 0, 0);
        if (i < kQ && row < M) v[u] = __ldg(reinterpret_cast<const uint4*>(qb + row * 128 + ch * 8));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * 96;
        if (i < kQ) *reinterpret_cast<uint4*>(sq + swz(i >> 4, i & 15, C::kQHalf)) = v[u];
      }
    }
    if (last && p.k_new) {  // fused KvStore::append of the window rows, read back by TMA
      for (int base = t96; base < 2 * R * 16; base += 96 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * 96;
          if (i < 2 * R * 16) {
            const int which = i / (R * 16), row = (i >> 4) % R, ch = i & 15;
            v[u] = __ldg(reinterpret_cast<const uint4*>((which ? p.v_new : p.k_new) +
                                                        ((static_cast<size_t>(b) * R + row) * p.Hkv + g) * 128) + ch);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * 96;
          if (i < 2 * R * 16) {
            const int which = i / (R * 16), row = (i >> 4) % R, ch = i & 15;
            const int pos = p0 + row;
            const int64_t cr = (((static_cast<int64_t>(p.layer) * p.cache.num_pages + bt[pos >> p.cache.page_shift]) *
                                     p.cache.n_kv_heads + g) << p.cache.page_shift) | (pos & ((1 << p.cache.page_shift) - 1));
            reinterpret_cast<uint4*>((which ? p.cache.v : p.cache.k) + cr * 128)[ch] = v[u];
          }
        }
      }
      fence_proxy_async();  // generic-proxy global writes -> async-proxy (TMA) reads
    }
    fence_proxy_async_smem();  // Q tile: generic smem writes -> tensor-core reads
    named_bar_sync(5, 96);
    if (warp == 1 && lane == 0) mbar_arrive(dep_bar);
    pdl_launch_dependents();
    // ---------------------------------------------------------------- MMA issuer (warp 1, converged;
    // one elect.sync-ed lane issues each batch of 8 MMAs: common.cuh umma_bf16_x8)
    if (warp == 1) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(N, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(C::kNP, 1, 1);
      const uint32_t q_base = smem_u32(sq);
      const uint32_t p_base = smem_u32(smem + C::kOffP);
      auto issue_pv = [&](int u) {
        const int wg = u & 1, sv = u % C::kSV;
        mbar_wait(&v_full[sv], (u / C::kSV) & 1);
        SA_TRACE(5, u);
        mbar_wait(&p_full[wg], (u >> 1) & 1);
        SA_TRACE(6, u);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + C::kOffV + sv * C::kTileBytes);
        const uint32_t p_pl = p_base + wg * C::kPlanes * C::kPBytes;
        const uint32_t o_tm = tmem + C::kOCol + (kRS ? 0 : wg * C::kNP);  // kRS: one O^T accumulator
        uint64_t a[8], bp[8];
#pragma unroll
        for (int kt = 0; kt < 8; ++kt) {  // 16 tokens per MMA; one MMA covers every P plane (N' = kNP)
          a[kt] = umma_desc(v_base + kt * 2048, C::kHalf, 1024, kLayoutSW128);
          bp[kt] = umma_desc(p_pl + kt * 512, C::kTile * 32, 256, kLayoutSW32);
        }
        umma_bf16_x8(o_tm, a, bp, idesc_pv, ((kRS ? u : (u >> 1)) % flush) != 0 ? 1u : 0u);  // block start: overwrite
        umma_commit_elect(&v_empty[sv]);
        umma_commit_elect(&p_empty[wg]);
        SA_TRACE(3, u);
      };
      int t = 0;
      for (;; ++t) {
        mbar_wait(&pos_bar[t % C::kPosRing], (t / C::kPosRing) & 1);
        if (tile_pos[t % C::kPosRing] < 0) break;
        const int sk = t % C::kSK;
        mbar_wait(&k_full[sk], (t / C::kSK) & 1);
        SA_TRACE(4, t);
        if (t >= 2) mbar_wait(&s_empty[t & 1], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(smem + C::kOffK + sk * C::kTileBytes);
        uint64_t a[8], bq[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // d in steps of 16
          a[kk] = umma_desc(k_base + (kk >> 2) * C::kHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
          bq[kk] = umma_desc(q_base + (kk >> 2) * C::kQHalf + (kk & 3) * 32, 16, 1024, kLayoutSW128);
        }
        umma_bf16_x8(tmem + (t & 1) * N, a, bq, idesc_qk, 0u);
        umma_commit_elect(&s_full[t & 1]);
        umma_commit_elect(&k_empty[sk]);
        SA_TRACE(2, t);
        if (t >= 1) issue_pv(t - 1);
      }
      if (t >= 1) issue_pv(t - 1);
    }
  }
  if (warp == 0) {  // producer warp: trigger only once this CTA is past its wait
    mbar_wait(dep_bar, 0);
    pdl_launch_dependents();
  }
  } else {
    setmaxnreg_inc<216>();  // warpgroups 1-2: softmax
    // ---------------------------------------------------------------- softmax warpgroups
    const int wg = (warp - 4) >> 2;     // 0: even tiles, 1: odd tiles
    const int q4 = warp & 3;            // TMEM lane quarter this warp may access
    const int tk = q4 * 32 + lane;      // token within the tile (S) / d (O)
    const int ts = tid - 128 - wg * 128;  // 0..127 within the warpgroup
    const int bar_wg = 2 + wg;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float c = p.scale_log2;
    float* mref = mref_all + wg * 64;
    float* fac = fac_all + wg * 64;
    float* red = red_all + wg * 256;
    float* score_out = p.scores ? p.scores + (static_cast<size_t>(b) * p.Hkv + g) * p.ld_scores : nullptr;
    long long* score_fx = p.score_fx ? p.score_fx + static_cast<size_t>(b) * p.ld_scores : nullptr;
    uint8_t* p_hi = smem + C::kOffP + wg * C::kPlanes * C::kPBytes;
    const uint32_t s_tm = tmem + lane_off + wg * N;
    const uint32_t o_tm = tmem + lane_off + C::kOCol + wg * C::kNP;  // plane q's O^T at +q*N
    const uint32_t a_tm = tmem + lane_off + C::kACol + wg * N;       // Oacc^T (closed accumulation blocks)
    const bool single = p.n_splits == 1;  // this CTA owns the whole unit: normalise in place
    float* po = p.part_o + static_cast<size_t>(unit) * p.n_splits * N * 128;
    float* pml = p.part_ml + static_cast<size_t>(unit) * p.n_splits * N * 2;
    float* my_o = po + static_cast<size_t>(split) * N * 128;
    float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * R * 128;
    // row split of the MR softmax rows (kRS): N = 48 at an even row (balanced halves, e.g. 18 / 18 at
    // MR = 36, P stored per row pair), N = 64 at an 8-row chunk boundary
    constexpr bool kPair = N == 48;
    constexpr int kR0 = kPair ? (MR + 2) / 4 * 2 : ((MR + 8) / 16 * 8 < 8 ? 8 : (MR + 8) / 16 * 8);
    if constexpr (kRS) {
      // ------------------------------------------------------------------------------------------------
      // Row split (kRS): both warpgroups work on EVERY tile, warpgroup w on query rows [rlo, rlo + RW):
      // half the softmax latency per tile, one O^T accumulator (no warpgroup merge in the epilogue).
      // S / P are double-buffered by tile parity; s_empty and p_full count both warpgroups' 256 threads.
      auto rs = [&](auto rw_c, int rlo) {
        constexpr int RW = decltype(rw_c)::value;          // this warpgroup's real rows
        constexpr int RWP = kPair ? (RW + 1) / 2 * 2 : (RW + 7) / 8 * 8;  // its P row pairs / 8-row chunks
        float l[RWP];
        float mr[RWP];
#pragma unroll
        for (int m = 0; m < RWP; ++m) {
          l[m] = 0.f;
          mr[m] = -INFINITY;
        }
        uint64_t wbits = 0;
#pragma unroll
        for (int m = 0; m < RW; ++m) wbits |= (wsc[rlo + m] != 0.f ? 1ull : 0ull) << m;
        const uint32_t o_rs = tmem + lane_off + C::kOCol + rlo;  // plane q's columns of my rows at +q*N
        const uint32_t a_rs = tmem + lane_off + 2 * N + C::kNP + rlo;  // Oacc (after the single O)
        int t = 0;
        for (;; ++t) {
          mbar_wait(&pos_bar[t % C::kPosRing], (t / C::kPosRing) & 1);
          const int tstart = tile_pos[t % C::kPosRing];
          if (tstart < 0) break;
          const int sb = t & 1;
          mbar_wait(&s_full[sb], (t >> 1) & 1);
          tc_fence_after();
          float s[RWP];
          tmem_ld_cols<RWP>(tmem + lane_off + sb * N + rlo, s);
          tc_wait_ld();
          tc_fence_before();
          mbar_arrive(&s_empty[sb]);
          const int pos = tstart + tk;
          const bool full = tstart + C::kTile <= p0;
          const bool in_range = pos < p0 + R;
          if (score_fx && pos < p0) {  // this warpgroup's rows of the Collect-k column sum (int64: exact)
            float sc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < RW; ++m) sc4[m & 3] += ((wbits >> m) & 1ull) ? s[m] : 0.f;
            const float sc = (sc4[0] + sc4[1]) + (sc4[2] + sc4[3]);
            if (wbits)
              atomicAdd(reinterpret_cast<unsigned long long*>(score_fx + pos),
                        static_cast<unsigned long long>(__float2ll_rn(sc * kScoreFxScale)));
          }
          if (kLogits && pos < p0) {
            float* lb = p.logits + static_cast<size_t>(b) * Hq * p.n_collect * p.ld_logits + pos;
#pragma unroll
            for (int m = 0; m < RW; ++m) {
              const int o = loff[rlo + m];
              if (o >= 0) lb[o] = s[m];
            }
          }
          bool ex4[4] = {false, false, false, false};
          if (full) {
#pragma unroll
            for (int m = 0; m < RW; ++m) ex4[m & 3] |= fmaf(s[m], c, -mr[m]) > kLazyMaxThresh;
          } else {
#pragma unroll
            for (int m = 0; m < RW; ++m)
              ex4[m & 3] |= (in_range && pos <= lim[rlo + m]) && fmaf(s[m], c, -mr[m]) > kLazyMaxThresh;
          }
          const bool exceed = (ex4[0] || ex4[1]) || (ex4[2] || ex4[3]);
          if (named_bar_or(bar_wg, 128, exceed)) {
            float x[RW];
#pragma unroll
            for (int m = 0; m < RW; ++m) x[m] = s[m] * c;
            if (!full) {
#pragma unroll
              for (int m = 0; m < RW; ++m) x[m] = (in_range && pos <= lim[rlo + m]) ? x[m] : -INFINITY;
            }
            warp_allreduce_max<RW>(x);
            if (lane == 0)
#pragma unroll
              for (int m = 0; m < RW; ++m) red[q4 * 64 + m] = x[m];
            named_bar_sync(bar_wg, 128);
            if (ts < RW) {
              const float mo = mref_all[rlo + ts];
              const float mx = fmaxf(fmaxf(red[ts], red[64 + ts]), fmaxf(red[128 + ts], red[192 + ts]));
              const float mn = fmaxf(mo, mx);
              fac_all[rlo + ts] = (mo == -INFINITY) ? 0.f : (mn == mo ? 1.f : fast_exp2(mo - mn));
              mref_all[rlo + ts] = mn;
            }
            named_bar_sync(bar_wg, 128);
#pragma unroll
            for (int m = 0; m < RW; ++m) {
              l[m] *= fac_all[rlo + m];
              mr[m] = mref_all[rlo + m];
            }
            if (t > 0) {  // O^T of my rows is final through tile t-1 once PV(t-1) retired
              mbar_wait(&p_empty[(t - 1) & 1], ((t - 1) >> 1) & 1);
              tc_fence_after();
#pragma unroll
              for (int pl = 0; pl < C::kPlanes; ++pl) {
                float v[RWP];
                tmem_ld_cols<RWP>(o_rs + pl * N, v);
                tc_wait_ld();
#pragma unroll
                for (int m = 0; m < RW; ++m) v[m] *= fac_all[rlo + m];
                tmem_st_cols<RWP>(o_rs + pl * N, v);
              }
              if (kFlush && t > flush) {
                float v[RWP];
                tmem_ld_cols<RWP>(a_rs, v);
                tc_wait_ld();
#pragma unroll
                for (int m = 0; m < RW; ++m) v[m] *= fac_all[rlo + m];
                tmem_st_cols<RWP>(a_rs, v);
              }
              tc_wait_st();
            }
          }
          if (full) {
#pragma unroll
            for (int m = 0; m < RW; ++m) s[m] = fast_exp2(fmaf(s[m], c, -mr[m]));
          } else {
#pragma unroll
            for (int m = 0; m < RW; ++m)
              s[m] = (in_range && pos <= lim[rlo + m]) ? fast_exp2(fmaf(s[m], c, -mr[m])) : 0.f;
          }
#pragma unroll
          for (int m = RW; m < RWP; ++m) s[m] = 0.f;  // padding rows of my last chunk
#pragma unroll
          for (int m = 0; m < RW; ++m) l[m] += s[m];
          if (t >= 2) mbar_wait(&p_empty[sb], ((t >> 1) - 1) & 1);  // PV(t-2) finished reading this P buffer
          if (kFlush && t > 0 && t % flush == 0) {  // PV(t-1) closed a block: Oacc (+)= my rows' planes
            mbar_wait(&p_empty[(t - 1) & 1], ((t - 1) >> 1) & 1);
            tc_fence_after();
            float op[C::kPlanes][RWP], acc[RWP];
#pragma unroll
            for (int pl = 0; pl < C::kPlanes; ++pl) tmem_ld_cols<RWP>(o_rs + pl * N, op[pl]);
            if (t > flush) tmem_ld_cols<RWP>(a_rs, acc);
            tc_wait_ld();
#pragma unroll
            for (int j = 0; j < RWP; ++j) {
              float v = op[C::kPlanes - 1][j];
#pragma unroll
              for (int pl = C::kPlanes - 2; pl >= 0; --pl) v += op[pl][j];
              acc[j] = t > flush ? v + acc[j] : v;
            }
            tmem_st_cols<RWP>(a_rs, acc);
            tc_wait_st();
          }
          uint8_t* pb = smem + C::kOffP + sb * C::kPlanes * C::kPBytes;
          if constexpr (kPair) {  // my row pairs (rows rlo + 2 e2, +1): one 32-bit word per plane
#pragma unroll
            for (int e2 = 0; e2 < RWP / 2; ++e2) {
              const int row = rlo + 2 * e2, row8 = row >> 3, a = row8 >> 1, ch = row8 & 1;
              uint32_t hw, mw, lw;
              split3_bf16(s[2 * e2], s[2 * e2 + 1], hw, mw, lw);
              const uint32_t off = a * (C::kTile * 32) + tk * 32 + ((ch ^ ((tk >> 2) & 1)) << 4) + (row & 7) * 2;
              *reinterpret_cast<uint32_t*>(pb + off) = hw;
              *reinterpret_cast<uint32_t*>(pb + C::kPBytes + off) = mw;
              *reinterpret_cast<uint32_t*>(pb + 2 * C::kPBytes + off) = lw;
            }
          }
#pragma unroll
          for (int q8 = 0; q8 < (kPair ? 0 : RWP / 8); ++q8) {  // my 8-row chunks (rows rlo + 8 q8 ..)
            const int row8 = rlo / 8 + q8, a = row8 >> 1, ch = row8 & 1;
            uint32_t hw[4], mw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) split3_bf16(s[8 * q8 + 2 * e], s[8 * q8 + 2 * e + 1], hw[e], mw[e], lw[e]);
            const uint32_t off = a * (C::kTile * 32) + tk * 32 + ((ch ^ ((tk >> 2) & 1)) << 4);
            *reinterpret_cast<uint4*>(pb + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(pb + C::kPBytes + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
            *reinterpret_cast<uint4*>(pb + 2 * C::kPBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&p_full[sb]);
        }
        // ---- epilogue of my rows (kRS): every tile's PV retired, then l, (m, l) and O of my rows
        mbar_wait(dep_bar, 0);
        pdl_launch_dependents();
        const int T = t;  // tiles processed (by both warpgroups)
        if (ts == 0) ntiles_wg[wg] = T;
        if (T > 0) {
          mbar_wait(&p_empty[(T - 1) & 1], ((T - 1) >> 1) & 1);
          if (T > 1) mbar_wait(&p_empty[T & 1], ((T - 2) >> 1) & 1);
          tc_fence_after();
        }
        float lw[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) lw[m] = m < RW ? l[m] : 0.f;
        warp_transpose_sum_store<32>(lw, lane, red + q4 * 64);  // per-warp row sums -> red[q4][row]
        named_bar_sync(bar_wg, 128);
        if (ts < RW) {
          const int row = rlo + ts;
          const float lsum = red[ts] + red[64 + ts] + red[128 + ts] + red[192 + ts];
          const float ms = mref_all[row];
          ltot[row] = lsum;
          if (!single) {
            pml[(split * N + row) * 2] = T > 0 ? ms : -INFINITY;
            pml[(split * N + row) * 2 + 1] = lsum;
          }
        }
        named_bar_sync(bar_wg, 128);
        if (T > 0) {
          float o[C::kPlanes][RWP], acc[RWP];
#pragma unroll
          for (int pl = 0; pl < C::kPlanes; ++pl) tmem_ld_cols<RWP>(o_rs + pl * N, o[pl]);
          const bool acc_on = kFlush && T > flush;
          if (acc_on) tmem_ld_cols<RWP>(a_rs, acc);
          tc_wait_ld();
#pragma unroll
          for (int m = 0; m < RW; ++m) {
            float v = o[C::kPlanes - 1][m];  // smallest plane first
#pragma unroll
            for (int pl = C::kPlanes - 2; pl >= 0; --pl) v += o[pl][m];
            if (acc_on) v += acc[m];
            const int row = rlo + m;
            if (row < M) {
              if (single) out_unit[row * 128 + tk] = v / ltot[row];
              else my_o[row * 128 + tk] = v;
            }
          }
        } else if (!single) {
#pragma unroll
          for (int m = 0; m < RW; ++m)
            if (rlo + m < M) my_o[(rlo + m) * 128 + tk] = 0.f;
        }
      };
      if constexpr (MR - kR0 >= 1) {
        if (wg == 0) rs(std::integral_constant<int, kR0>{}, 0);
        else rs(std::integral_constant<int, MR - kR0>{}, kR0);
      }
    } else {
    float l[N];
#pragma unroll
    for (int m = 0; m < N; ++m) l[m] = 0.f;
    // this warpgroup's lazy row references (mref): held in registers across tiles where the register
    // budget allows (N <= 32: -0.1..-0.4 us per layer), reloaded from shared memory each tile above that
    // (N = 48 spilled: +1.4 us)
    constexpr bool kRegRef = N <= 32;
    float mr[N];
#pragma unroll
    for (int m = 0; m < MR; ++m) mr[m] = -INFINITY;
    uint64_t wbits = 0;  // rows in the Collect-k score (wsc as a register bitmask: no per-tile smem reads)
#pragma unroll
    for (int m = 0; m < MR; ++m) wbits |= (wsc[m] != 0.f ? 1ull : 0ull) << m;

    int i = 0;
    for (int t = wg;; t += 2, ++i) {
      mbar_wait(&pos_bar[t % C::kPosRing], (t / C::kPosRing) & 1);
      const int tstart = tile_pos[t % C::kPosRing];
      if (tstart < 0) break;
      mbar_wait(&s_full[wg], i & 1);
      if (ts == 0) SA_TRACE(7, t);
      tc_fence_after();
      float s[N];
      tmem_ld_n<N>(s_tm, s);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[wg]);
      if (ts == 0) SA_TRACE(12, t);
      const int pos = tstart + tk;
      const bool full = tstart + C::kTile <= p0;  // chunk tiles: every row sees every token
      const bool in_range = pos < p0 + R;         // window tiles: positions past the window masked
      if ((score_out || score_fx) && pos < p0) {  // fused Collect-k column sum (raw logits)
        float sc4[4] = {0.f, 0.f, 0.f, 0.f};  // four independent FMA chains (latency, not throughput)
#pragma unroll
        for (int m = 0; m < MR; ++m) sc4[m & 3] += ((wbits >> m) & 1ull) ? s[m] : 0.f;
        const float sc = (sc4[0] + sc4[1]) + (sc4[2] + sc4[3]);
        if (score_fx)  // per-layer: integer atomics over the KV heads (order-independent, deterministic)
          atomicAdd(reinterpret_cast<unsigned long long*>(score_fx + pos),
                    static_cast<unsigned long long>(__float2ll_rn(sc * kScoreFxScale)));
        else
          score_out[pos] = sc;
      }
      if (kLogits && pos < p0) {  // LogitMatrix path (Collect2Weights, debug): raw prefix logits
        float* lb = p.logits + static_cast<size_t>(b) * Hq * p.n_collect * p.ld_logits + pos;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          const int o = loff[m];  // smem broadcast, precomputed per CTA
          if (o >= 0) lb[o] = s[m];
        }
      }
      // pass 1: does any logit exceed the lazy reference by more than 2^8?  (mref held in registers:
      // no shared-memory reads between the P stores below)
      if (!kRegRef) {
#pragma unroll
        for (int m = 0; m < MR; m += 4) *reinterpret_cast<float4*>(&mr[m]) = *reinterpret_cast<const float4*>(&mref[m]);
      }
      bool ex4[4] = {false, false, false, false};  // four independent OR chains
      if (full) {
#pragma unroll
        for (int m = 0; m < MR; ++m) ex4[m & 3] |= fmaf(s[m], c, -mr[m]) > kLazyMaxThresh;
      } else {
#pragma unroll
        for (int m = 0; m < MR; ++m)
          ex4[m & 3] |= (in_range && pos <= lim[m]) && fmaf(s[m], c, -mr[m]) > kLazyMaxThresh;
      }
      const bool exceed = (ex4[0] || ex4[1]) || (ex4[2] || ex4[3]);
      if (ts == 0) SA_TRACE(13, t);
      const bool any_exceed = named_bar_or(bar_wg, 128, exceed);
      if (ts == 0) SA_TRACE(14, t);
      if (any_exceed) {
        // slow path: exact row max of this tile, rescale l partials and this warpgroup's O^T
        float x[MR];
#pragma unroll
        for (int m = 0; m < MR; ++m) x[m] = s[m] * c;
        if (!full) {
#pragma unroll
          for (int m = 0; m < MR; ++m) x[m] = (in_range && pos <= lim[m]) ? x[m] : -INFINITY;
        }
        warp_allreduce_max<MR>(x);
        if (lane == 0) {
#pragma unroll
          for (int m = 0; m < MR; m += 4)
            *reinterpret_cast<float4*>(&red[q4 * 64 + m]) = make_float4(x[m], x[m + 1], x[m + 2], x[m + 3]);
        }
        named_bar_sync(bar_wg, 128);
        if (ts < MR) {
          const float mo = mref[ts];
          const float mx = fmaxf(fmaxf(red[ts], red[64 + ts]), fmaxf(red[128 + ts], red[192 + ts]));
          const float mn = fmaxf(mo, mx);
          fac[ts] = (mo == -INFINITY) ? 0.f : (mn == mo ? 1.f : fast_exp2(mo - mn));
          mref[ts] = mn;
        }
        named_bar_sync(bar_wg, 128);
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          l[m] *= fac[m];
          mr[m] = mref[m];
        }
        if (i > 0) {  // O^T of this warpgroup is final through its previous tile once that PV is done
          mbar_wait(&p_empty[wg], (i - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int pl = 0; pl < C::kPlanes; ++pl) {
            float v[N];
            tmem_ld_n<N>(o_tm + pl * N, v);
            tc_wait_ld();
#pragma unroll
            for (int m = 0; m < N; ++m) v[m] *= fac[m];
            tmem_st_n<N>(o_tm + pl * N, v);
          }
          if (kFlush && i > flush) {  // Oacc holds closed blocks (the first flush ran at i = flush)
            float v[N];
            tmem_ld_n<N>(a_tm, v);
            tc_wait_ld();
#pragma unroll
            for (int m = 0; m < N; ++m) v[m] *= fac[m];
            tmem_st_n<N>(a_tm, v);
          }
          tc_wait_st();
        }
      }
      // pass 2a: p = 2^(s*c - mref) in place, l += p (independent per row: full ILP)
      if (full) {
#pragma unroll
        for (int m = 0; m < MR; ++m) s[m] = fast_exp2(fmaf(s[m], c, -mr[m]));
      } else {
#pragma unroll
        for (int m = 0; m < MR; ++m) s[m] = (in_range && pos <= lim[m]) ? fast_exp2(fmaf(s[m], c, -mr[m])) : 0.f;
      }
#pragma unroll
      for (int m = 0; m < MR; ++m) l[m] += s[m];
      if (ts == 0) SA_TRACE(8, t);
      if (i > 0) mbar_wait(&p_empty[wg], (i - 1) & 1);  // previous PV finished reading this P plane
      if (kFlush && i > 0 && i % flush == 0) {  // PV(i-1) closed an accumulation block: Oacc (+)= its planes
        tc_fence_after();
#pragma unroll
        for (int c16 = 0; c16 < N / 16; ++c16) {
          float op[C::kPlanes][16], acc[16];
#pragma unroll
          for (int pl = 0; pl < C::kPlanes; ++pl) tmem_ld16(o_tm + pl * N + 16 * c16, op[pl]);
          if (i > flush) tmem_ld16(a_tm + 16 * c16, acc);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float v = op[C::kPlanes - 1][j];  // smallest plane first (the epilogue's order)
#pragma unroll
            for (int pl = C::kPlanes - 2; pl >= 0; --pl) v += op[pl][j];
            acc[j] = i > flush ? v + acc[j] : v;
          }
          tmem_st16(a_tm + 16 * c16, acc);
        }
        tc_wait_st();
      }
      if (ts == 0) SA_TRACE(9, t);
      // pass 2b: P^T -> smem as bf16 planes (MN-major SWIZZLE_32B, 16-row atoms: token tk's 8-row
      // chunk ch of atom a at a*4096 + tk*32 + 16*(ch ^ bit 2 of tk))
#pragma unroll
      for (int a = 0; a < C::kPAtoms; ++a)
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          if (16 * a + 8 * ch >= MR) continue;  // padding rows only: zeroed once in the prologue
          uint32_t hw[4], mw[4], lw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = 16 * a + 8 * ch + 2 * e;
            const float x0 = m < MR ? s[m] : 0.f, x1 = m + 1 < MR ? s[m + 1] : 0.f;  // rows >= MR: padding
            if (C::kPlanes == 3) split3_bf16(x0, x1, hw[e], mw[e], lw[e]);
            else split_bf16(x0, x1, hw[e], lw[e]);
          }
          const uint32_t off = a * (C::kTile * 32) + tk * 32 + ((ch ^ ((tk >> 2) & 1)) << 4);
          *reinterpret_cast<uint4*>(p_hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          if (C::kPlanes == 3) {
            *reinterpret_cast<uint4*>(p_hi + C::kPBytes + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
            *reinterpret_cast<uint4*>(p_hi + 2 * C::kPBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          } else {
            *reinterpret_cast<uint4*>(p_hi + C::kPBytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
        }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[wg]);
      if (ts == 0) SA_TRACE(10, t);
    }

    // ---------------------------------------------------------------- epilogue
    // PDL chain: trigger the next layer's launch only once this CTA is past its griddepcontrol.wait
    // (dep_bar is released after it), so "layer l+2 launched" implies "layer l complete" and the
    // layer-parity workspaces (partials, counters, chunk claims) are free again by transitivity.
    mbar_wait(dep_bar, 0);
    pdl_launch_dependents();
    if (kPipeTrace && p.trace && ts == 0 && wg == 0 && cta_lin < 1024) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin + 2] = gt;  // main loop done
      p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin + 3] = static_cast<unsigned long long>(i) | (static_cast<unsigned long long>(split) << 32);
    }
    const int my_tiles = i;  // tiles this warpgroup processed
    if (ts == 0) ntiles_wg[wg] = my_tiles;
    if (my_tiles > 0) {
      mbar_wait(&p_empty[wg], (my_tiles - 1) & 1);
      tc_fence_after();
    }
    if (wg == 0 && ts == 0) SA_TSTAMP(4);
    warp_transpose_sum_store<N>(l, lane, red + q4 * 64);  // per-warp row sums of l -> red[q4][row]
    named_bar_sync(bar_wg, 128);
    if (ts < N) ltot[wg * 64 + ts] = red[ts] + red[64 + ts] + red[128 + ts] + red[192 + ts];
    named_bar_sync(1, 256);  // both warpgroups' (mref, ltot) final
    if (wg == 0 && ts == 0) SA_TSTAMP(10);
    float* fin_l = red_all;  // [64] per-row sum of this CTA (both warpgroups, common max)
    float* wgfac = red_all + 64;  // [2][64] per-row rescale of each warpgroup's O to the common max
    const bool has0 = ntiles_wg[0] > 0, has1 = ntiles_wg[1] > 0;
    if (wg == 0 && ts < N) {
      const float m0 = mref_all[ts], m1 = mref_all[64 + ts];
      const float ms = fmaxf(m0, m1);
      const float f0 = (has0 && m0 != -INFINITY) ? fast_exp2(m0 - ms) : 0.f;
      const float f1 = (has1 && m1 != -INFINITY) ? fast_exp2(m1 - ms) : 0.f;
      wgfac[ts] = f0;
      wgfac[64 + ts] = f1;
      float lsum = 0.f;
      if (m0 != -INFINITY) lsum += ltot[ts] * f0;
      if (m1 != -INFINITY) lsum += ltot[64 + ts] * f1;
      fin_l[ts] = lsum;
      if (!single) {
        pml[(split * N + ts) * 2] = (has0 || has1) ? ms : -INFINITY;
        pml[(split * N + ts) * 2 + 1] = lsum;
      }
    }
    named_bar_sync(1, 256);
    if (wg == 0 && ts == 0) SA_TSTAMP(11);
    // merge the two warpgroups' O^T: warpgroup 0 takes even 16-column chunks, warpgroup 1 odd ones;
    // only the M real rows are stored (partial rows keep the N-row stride)
    for (int c16 = wg; c16 < N / 16; c16 += 2) {
      if (16 * c16 >= M) break;
      float s0[16], s1[16];  // plane sums of each warpgroup's O^T, smallest plane first
#pragma unroll
      for (int j = 0; j < 16; ++j) s0[j] = s1[j] = 0.f;
      const uint32_t base = tmem + lane_off + C::kOCol + 16 * c16;
#pragma unroll
      for (int pl = C::kPlanes - 1; pl >= 0; --pl) {
        float o0[16], o1[16];
        if (has0) tmem_ld16(base + pl * N, o0);
        if (has1) tmem_ld16(base + C::kNP + pl * N, o1);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (has0) s0[j] += o0[j];
          if (has1) s1[j] += o1[j];
        }
      }
      // closed accumulation blocks (Oacc) of a warpgroup that ran more than kFlush tiles
      const bool acc0 = kFlush && ntiles_wg[0] > flush, acc1 = kFlush && ntiles_wg[1] > flush;
      if (acc0 || acc1) {
        float a0[16], a1[16];
        const uint32_t abase = tmem + lane_off + C::kACol + 16 * c16;
        if (acc0) tmem_ld16(abase, a0);
        if (acc1) tmem_ld16(abase + N, a1);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (acc0) s0[j] += a0[j];
          if (acc1) s1[j] += a1[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = 16 * c16 + j;
        if (m >= M) break;
        float acc = 0.f;  // factors precomputed per row (0 for an empty warpgroup / masked row)
        if (has0) acc += s0[j] * wgfac[m];
        if (has1) acc += s1[j] * wgfac[64 + m];
        if (single) out_unit[m * 128 + tk] = acc / fin_l[m];
        else my_o[m * 128 + tk] = acc;
      }
    }
    }  // kRS / ping-pong
    if (wg == 0 && ts == 0) SA_TSTAMP(12);
    tc_fence_before();
    if (single) {
      if (wg == 0 && ts == 0) p.chunk_ctr[unit] = 0;  // re-arm chunk claims
    } else {
      // Split merge by designated mergers: splits 0 .. nm-1 each normalise a slice of the rows.  Every
      // CTA publishes its partial with one st.release per merger (after the CTA-wide barrier that
      // orders its partial stores); a merger bulk-loads each split's slice as soon as it is published
      // (merge_rows_progressive), so only the last split's slice is on the critical path.
      const int t256 = wg * 128 + ts;
      const int nm = min(p.n_mergers, p.n_splits);
      int* uflags = p.flags + static_cast<size_t>(unit) * 8 * 128;
      named_bar_sync(1, 256);
      if (t256 < nm) {
        if (t256 == 0) SA_TSTAMP(5);
        asm volatile("st.release.gpu.s32 [%0], %1;" ::"l"(uflags + t256 * 128 + split), "r"(1) : "memory");
        if (t256 == 0) SA_TSTAMP(6);
      }
      if (split < nm) {
        const int per = (M + nm - 1) / nm;
        merge_rows_progressive(smem, merge_bar, po, pml, p.n_splits, N, min(M, split * per), min(M, (split + 1) * per),
                               out_unit, uflags + split * 128, t256,
                               (kPipeTrace && p.trace && cta_lin < 1024) ? p.trace + 1024 + (p.layer & 63) * 16384 + 16 * cta_lin : nullptr);
        if (split == 0 && t256 == 0) p.chunk_ctr[unit] = 0;  // every split has claimed its last chunk
        if (t256 == 0) SA_TSTAMP(9);
      }
    }
  }
  __syncthreads();
  if (kPipeTrace && p.trace && tid == 0 && cta_lin < 1024) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[1024 + (p.layer & 63) * 16384 + 16 * cta_lin + 1] = gt;
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

template <int N, int MR, bool kFlush, bool kLogits>
static cudaError_t launch_n(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  // row split: both softmax warpgroups on every tile (not with per-KV-head scores: two partial stores)
  // row split where it pays: MMA widths N >= 48 (same-box A/B: gamma 8 at 32K, 37.1 -> 32.3 us per layer;
  // config 4's per-rank shard, 80.1 -> 67.3 us); at N = 32 the 8 / 12 or 16 / 12 row halves were slower
  // than tile ping-pong (+0.5 us per layer at gamma 4 and 6)
  constexpr bool kRSok = MR >= 12 && N >= 48;
  const bool rs = kRSok && p.row_split && p.scores == nullptr;
  auto kern = rs ? verify_tc_kernel<N, MR, kFlush, kLogits, kRSok> : verify_tc_kernel<N, MR, kFlush, kLogits, false>;
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  if (func_attrs_needed(attr_mask, &dev)) {
    cudaError_t e = cudaFuncSetAttribute(verify_tc_kernel<N, MR, kFlush, kLogits, kRSok>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, TCfg<N>::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(verify_tc_kernel<N, MR, kFlush, kLogits, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, TCfg<N>::kSmem);
    if (e != cudaSuccess) return e;
    func_attrs_done(attr_mask, dev);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_splits, p.Hkv, p.B);
  cfg.blockDim = dim3(TCfg<N>::kThreads);
  cfg.dynamicSmemBytes = TCfg<N>::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tk, tv, p);
}

// MR = N - 12, N - 8, N - 4 or N: the softmax warpgroups work only on the rows that can be real
// (measured at gamma 4, M = 20 in an N = 32 tile: MR 24 instead of 32 took the verify phase from
// 1.013 to 0.984 ms; the softmax instruction count is on the main loop's critical path)
template <int N, bool kFlush, bool kLogits>
static cudaError_t launch_mr_f(int mr, const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv,
                             cudaStream_t s) {
  switch (N - mr) {
    case 12: return launch_n<N, N - 12, kFlush, kLogits>(p, tk, tv, s);
    case 8: return launch_n<N, N - 8, kFlush, kLogits>(p, tk, tv, s);
    case 4: return launch_n<N, N - 4, kFlush, kLogits>(p, tk, tv, s);
    default: return launch_n<N, N, kFlush, kLogits>(p, tk, tv, s);
  }
}

// per-N entry points (one translation unit each: verify_tc_n{16,32,48,64}.cu compile in parallel)
template <int N>
static cudaError_t launch_mr(int mr, const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv,
                             cudaStream_t s) {
  const bool f = p.flush_tiles > 0 && TCfg<N>::kFlushable, lg = p.logits != nullptr;
  return f ? (lg ? launch_mr_f<N, true, true>(mr, p, tk, tv, s) : launch_mr_f<N, true, false>(mr, p, tk, tv, s))
           : (lg ? launch_mr_f<N, false, true>(mr, p, tk, tv, s) : launch_mr_f<N, false, false>(mr, p, tk, tv, s));
}

}  // namespace sa
