// qkv.cu — the model-side producer of the path's inputs: RMSNorm -> fused
// Q/K/V projection -> RoPE, emitting the bf16 q / k_new / v_new buffers the verify and draft kernels
// consume (their fused KvStore::append writes K/V into the cache).
//
// Reference: SPEC-only (the reference ships the weights, not the forward): forward on
// the LayerWeights of weights.hpp:20-30 — h = x / sqrt(mean(x^2) + norm_eps) * attn_norm_gain ("RMS
// normalization", config.hpp:34), q = h wq, k = h wk, v = h wv (wq: d_model x q_dim), then
// apply_rope to every q and k head at the token's absolute position with
// config.rope_theta (config.hpp:32).  Eigen's MatrixXf is column-major, so the reference's wq holds
// exactly the rows of W^T this kernel streams: w_qkv [L][(Hq + 2 Hkv) * 128][d_model] bf16 = the
// per-layer stack of wq^T, wk^T, wv^T (oracle/model.py restates the whole step in float64).
//
// Decode-time projection is weight-streaming: 2..128 tokens against a (Hq+2Hkv)*128 x d_model
// matrix (Llama-3.1-8B shape: 6144 x 4096 bf16 = 50.3 MB per layer), so the bound is HBM and the
// tensor core only has to keep up.  Swap-AB tcgen05: A = a 128-row weight tile (one attention head's
// output features, K-major, TMA SWIZZLE_128B), B = the token tile, D in TMEM [128 lanes][N].  The
// tokens enter as two bf16 planes (hi = bf16(x*g), lo = bf16(x*g - hi)) stacked along N, so the
// product is fp32-accurate although the MMA is bf16 (~2^-17 relative input representation error);
// the 1/rms factor is applied in the epilogue (it commutes with the projection).
//
// Weights are repacked once at sa_qkv_create into [L][head][d_model/64] tiles of 128 x 64 bf16, each
// 16 KB contiguous and already in the UMMA SWIZZLE_128B order, so one CTA's share of a layer is one
// contiguous run read with 1-D bulk copies; the part of the run past the smem ring is prefetched into
// L2 at CTA start.
//
// Grid: stream-K — one CTA per SM, each taking an equal contiguous run of the layer's (head, k-block)
// units (a run touches at most two heads; TMEM accumulators per head, the K-steps rotating over
// independent accumulators).  Weight streaming is bound by the chip's L2->SM rate (~40 GB/s per SM
// with every SM pulling), so every SM must stream: a split-K cluster grid left 3-CTA clusters
// unschedulable past 45 and ran a second wave.  Each CTA writes its per-head partial to global memory;
// the last of a head's contributors reduces them in CTA order (deterministic) and finishes: 1/rms,
// RoPE (cos/sin per token and pair from qkv_prepare), bf16, store.  Two launches per call: qkv_prepare
// (1/rms, the hi/lo token planes, the RoPE table) and qkv_gemm, chained with PDL; the weight tiles of
// the ring are loaded before griddepcontrol.wait (they depend on nothing), so they overlap the previous
// kernel's tail.  Measured (Llama-3.1-8B shape, 5 tokens, 32-layer chain): 24 us per layer = 2.1 TB/s
// of weights; DESIGN.md has the timeline and what bounds it.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "internal.h"

struct sa_qkv {
  int L = 0, Hq = 0, Hkv = 0, D = 0, n_out = 0, nkb = 0, style = 0;
  float eps = 1e-5f;
  double theta = 10000.0;
  __nv_bfloat16* wpack = nullptr;  // [L][heads][nkb][128][64] swizzled 16 KB tiles (owned copy)
  float* gain = nullptr;           // [L][D] (owned copy)
  __nv_bfloat16* xbuf = nullptr;   // [nkb][N][64] swizzled hi/lo token planes (N <= 256)
  float* rbuf = nullptr;           // [128] 1/rms per token
  float2* rope = nullptr;          // [128][64] (cos, sin) per token and RoPE pair
  float* part = nullptr;           // [max grid][2][256][128] split-K partials
  int* counters = nullptr;         // [heads]
  int max_grid = 0;
  unsigned long long* trace = nullptr;  // dev-only (knob "trace")
  int dev_bits = 0;                      // dev-only variant bits (knob "dev")
  int force_tc = 0;                      // dev-only: the tcgen05 stream-K path for every token count
  int device = 0, num_sms = 148;
};

namespace sa {

constexpr int kQkvMaxTokens = 128;
constexpr int kQkvThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int kQkvSmem = 200 * 1024;
constexpr int kWTile = 128 * 64 * 2;  // 16 KB weight tile (128 output features x 64 of d_model)
constexpr int kEpiBytes = 8 * 128 * 4;  // epilogue token-group buffer (end of the ring region)
constexpr int kMaxStages = 12;
constexpr uint32_t kXResMax = 64 * 1024;  // resident token tiles up to this size

struct QkvParams {
  int layer, n_out, nkb, n_tok, rows, NT, N, Hq, Hkv, heads, style;
  float eps;
  double log2_theta;
  const __nv_bfloat16* wpack;
  const float* x;
  const float* gain;
  const int32_t* pos0;
  __nv_bfloat16* xbuf;
  float* rbuf;
  float2* rope;   // [128 tokens][64 pairs] (cos, sin)
  float* part;    // [grid][2][N][128] per-CTA partial accumulators (one per head touched)
  int* counters;  // [heads] arrivals, re-armed by the reducing CTA
  unsigned long long* trace;  // dev-only (SA_QKV_TRACE): [layer][grid][8] globaltimer stamps
  // dev knobs (SA_QKV_DEV, timing experiments only; results are wrong with 2/8/1024/32768): 1 no L2
  // prefetch, 2 skip the MMAs, 4 four stages, 8 no token tiles, 1024 token tiles from a stale buffer,
  // 2048 token tiles per stage even when they fit resident, 4096 at most 4 accumulators, 8192 wait for
  // every preloaded stage before the loop, 16384 no per-iteration stamps, 32768 no refills
  int dev;
  __nv_bfloat16* q;
  __nv_bfloat16* k_new;
  __nv_bfloat16* v_new;
};

// Byte offset of 16-byte chunk c (0..7) of row r in a [rows][64] bf16 tile in SWIZZLE_128B order.
__device__ __forceinline__ uint32_t sw128(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

// One-time repack: w [L][n_out][D] (row = output feature) -> [L][head][kb] swizzled 16 KB tiles.
__global__ void __launch_bounds__(256) qkv_pack(const __nv_bfloat16* w, int n_out, int D, __nv_bfloat16* wpack) {
  const int tile = blockIdx.x;  // (l * heads + h) * nkb + kb
  const int nkb = D / 64, heads = n_out / 128;
  const int kb = tile % nkb, lh = tile / nkb, h = lh % heads, l = lh / heads;
  const __nv_bfloat16* src = w + (static_cast<size_t>(l) * n_out + h * 128) * D + kb * 64;
  uint8_t* dst = reinterpret_cast<uint8_t*>(wpack) + static_cast<size_t>(tile) * 16384;
  for (int i = threadIdx.x; i < 128 * 8; i += 256) {
    const int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(dst + sw128(r, c)) = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(r) * D + c * 8);
  }
}

// One CTA per padded token row: 1/rms and the hi/lo planes of x * gain, swizzled like the B tile.
__global__ void __launch_bounds__(256) qkv_prepare(QkvParams p) {
  // let the projection launch now: it streams its first weight tiles while this kernel waits and runs
  pdl_launch_dependents();
  pdl_wait();  // x is the previous kernel's output; the previous projection's xbuf reads are done
  const int t = blockIdx.x, tid = threadIdx.x;
  const int D = p.nkb * 64;
  const float* xr = p.x + static_cast<size_t>(t) * D;
  const float* g = p.gain + static_cast<size_t>(p.layer) * D;
  const bool live = t < p.n_tok;
  double ss = 0.0;
#pragma unroll 4
  for (int k = tid * 8; k < D; k += 2048) {  // 8 consecutive elements = one 16-byte bf16 chunk
    uint4 hi = make_uint4(0, 0, 0, 0), lo = hi;
    if (live) {
      const float4 x0 = *reinterpret_cast<const float4*>(xr + k), x1 = *reinterpret_cast<const float4*>(xr + k + 4);
      const float4 g0 = *reinterpret_cast<const float4*>(g + k), g1 = *reinterpret_cast<const float4*>(g + k + 4);
      ss += static_cast<double>(x0.x) * x0.x + static_cast<double>(x0.y) * x0.y + static_cast<double>(x0.z) * x0.z +
            static_cast<double>(x0.w) * x0.w + static_cast<double>(x1.x) * x1.x + static_cast<double>(x1.y) * x1.y +
            static_cast<double>(x1.z) * x1.z + static_cast<double>(x1.w) * x1.w;
      split_bf16(x0.x * g0.x, x0.y * g0.y, hi.x, lo.x);
      split_bf16(x0.z * g0.z, x0.w * g0.w, hi.y, lo.y);
      split_bf16(x1.x * g1.x, x1.y * g1.y, hi.z, lo.z);
      split_bf16(x1.z * g1.z, x1.w * g1.w, hi.w, lo.w);
    }
    uint8_t* blk = reinterpret_cast<uint8_t*>(p.xbuf) + static_cast<size_t>(k >> 6) * p.N * 128;
    const int c = (k & 63) >> 3;
    *reinterpret_cast<uint4*>(blk + sw128(t, c)) = hi;
    *reinterpret_cast<uint4*>(blk + sw128(p.NT + t, c)) = lo;
  }
  __shared__ double red[8];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    p.rbuf[t] = live ? static_cast<float>(1.0 / sqrt(s / D + static_cast<double>(p.eps))) : 0.f;
  }
  if (live && tid < 64) {  // RoPE pair j of this token: angle = pos * theta^(-2j/128), reduced in double
    const int b = t / p.rows, r = t - b * p.rows;
    double turns = static_cast<double>(p.pos0[b] + r) * exp2(-p.log2_theta * (2.0 * tid) / 128.0) *
                   0.15915494309189535;
    turns -= floor(turns);
    double sd, cd;
    sincospi(2.0 * turns, &sd, &cd);  // reduced argument: polynomial only, no large-angle path
    p.rope[t * 64 + tid] = make_float2(static_cast<float>(cd), static_cast<float>(sd));
  }
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)), "r"(bytes)
               : "memory");
}

#define QKV_STAMP(k)                                                                     \
  do {                                                                                   \
    if (p.trace) {                                                                       \
      unsigned long long gt_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                            \
      p.trace[(static_cast<size_t>(p.layer) * gridDim.x + blockIdx.x) * 32 + (k)] = gt_; \
    }                                                                                    \
  } while (0)

// First / one-past-last unit ((head, k-block) pair, head-major) of CTA c among n for U units.
__device__ __forceinline__ int unit_begin(int c, int U, int n) { return static_cast<int>(static_cast<int64_t>(c) * U / n); }

__global__ void __launch_bounds__(kQkvThreads, 1) qkv_gemm(QkvParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = p.N, NT = p.NT, nkb = p.nkb, n = gridDim.x, cta = blockIdx.x;
  const int U = p.heads * nkb;
  const int u0 = unit_begin(cta, U, n), u1 = unit_begin(cta + 1, U, n), nk = u1 - u0;
  const int head0 = u0 / nkb, nseg = (u1 - 1) / nkb - head0 + 1;  // heads touched (1 or 2)
  // Token tiles: each bulk copy costs about as much of the SM's copy stream as a 16 KB weight tile,
  // so when the CTA's whole run of token tiles fits (xres) it is loaded with one copy per head
  // segment right after the dependency wait and stays resident; otherwise each stage carries one.
  const uint32_t xbytes = N * 128;
  const bool xres = static_cast<uint32_t>(nk) * xbytes <= kXResMax && !(p.dev & 2048);
  const uint32_t stage_bytes = kWTile + (xres ? 0u : xbytes);
  const uint32_t tx_bytes = (p.dev & 8) || xres ? kWTile : stage_bytes;  // dev 8: X tiles not loaded
  const int ring = kQkvSmem - 1024 - 512;
  const int ring_w = (ring - kEpiBytes - (xres ? nk * static_cast<int>(xbytes) : 0)) & ~1023;
  uint8_t* xsm = smem + ring_w;  // resident token tiles [nk][N][64] (1 KB aligned for SWIZZLE_128B)
  const int S = min((p.dev & 4) ? 4 : kMaxStages, static_cast<int>(ring_w / stage_bytes));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ring);
  uint64_t* empty = full + kMaxStages;
  uint64_t* acc_bar = empty + kMaxStages;  // [2]
  uint64_t* x_bar = acc_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_bar + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  // independent accumulators per head segment: consecutive MMAs into one accumulator serialise on the
  // MMA latency, which dominates at small N, so the K=16 steps rotate over nacc accumulators
  const int nacc = (p.dev & 4096) ? (N <= 64 ? 4 : N <= 128 ? 2 : 1) : max(1, min(16, 256 / N));
  const int acols = 2 * nacc * N;
  const uint32_t tcols = acols <= 32 ? 32 : acols <= 64 ? 64 : acols <= 128 ? 128 : acols <= 256 ? 256 : 512;

  if (tid == 0) {
    QKV_STAMP(0);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&acc_bar[0], 1);
    mbar_init(&acc_bar[1], 1);
    mbar_init(x_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents (the next layer's prepare, or attention) do all their reads after griddepcontrol.wait
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ bulk-copy producer
      // this CTA's units are one contiguous run of the packed weights
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wpack) +
                            (static_cast<size_t>(p.layer) * U + u0) * kWTile;
      auto xsrc = [&](int it) {
        const uint8_t* xb = (p.dev & 1024) ? reinterpret_cast<const uint8_t*>(p.wpack)  // dev: stale source
                                           : reinterpret_cast<const uint8_t*>(p.xbuf);
        return xb + static_cast<size_t>((u0 + it) % nkb) * N * 128;
      };
      const int pre = min(S, nk);
      for (int it = 0; it < pre; ++it) {  // weights do not depend on the previous kernel
        mbar_expect_tx(&full[it], tx_bytes);
        bulk_load(smem + it * stage_bytes, wsrc + static_cast<size_t>(it) * kWTile, kWTile, &full[it]);
      }
      if (nk > pre && !(p.dev & 1)) bulk_prefetch_l2(wsrc + static_cast<size_t>(pre) * kWTile, (nk - pre) * kWTile);
      pdl_wait();
      QKV_STAMP(1);
      QKV_STAMP(11);
      if (xres) {
        const int n0 = min(nk, nkb - u0 % nkb);  // units of the first head segment (contiguous k-blocks)
        mbar_expect_tx(x_bar, nk * xbytes);
        bulk_load(xsm, xsrc(0), n0 * xbytes, x_bar);
        if (nk > n0) bulk_load(xsm + n0 * xbytes, xsrc(n0), (nk - n0) * xbytes, x_bar);
      } else if (!(p.dev & 8)) {
        for (int it = 0; it < pre; ++it) bulk_load(smem + it * stage_bytes + kWTile, xsrc(it), xbytes, &full[it]);
      }
      for (int it = pre; it < ((p.dev & 32768) ? pre : nk); ++it) {  // dev 32768: no refills
        const int st = it % S;
        mbar_wait(&empty[st], ((it / S) - 1) & 1);
        mbar_expect_tx(&full[st], tx_bytes);
        bulk_load(smem + st * stage_bytes, wsrc + static_cast<size_t>(it) * kWTile, kWTile, &full[st]);
        if (!xres && !(p.dev & 8)) bulk_load(smem + st * stage_bytes + kWTile, xsrc(it), xbytes, &full[st]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {  // --------------------------------------- MMA issuer: the whole warp loops,
    // waits are warp-wide and lane 0 issues the tcgen05 instructions
    const uint32_t idesc = umma_idesc_bf16(N, 0, 0);
    if (xres) mbar_wait(x_bar, 0);
    if (p.dev & 8192) {  // dev: wait until every preloaded stage landed, then time the loop over them
      for (int i = 0; i < min(S, nk); ++i) mbar_wait(&full[i], 0);
      if (lane == 0) QKV_STAMP(12);
    }
    const int nk_mma = (p.dev & 32768) ? min(S, nk) : nk;
    const int n0 = min(nk, nkb - u0 % nkb);  // units of the first head segment
    int st = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nk_mma; ++it) {
      const int seg = it < n0 ? 0 : 1, seg_it = it < n0 ? it : it - n0;
      mbar_wait(&full[st], phase);
      tc_fence_after();
      if (lane == 0) {
        if (it == 0) QKV_STAMP(2);
        if (it < 16 && !(p.dev & 16384)) QKV_STAMP(16 + it);  // dev: per-iteration issue times
        if (it == S - 1) QKV_STAMP(8);
        if (it == S) QKV_STAMP(9);
        if (it == (S + nk) / 2) QKV_STAMP(10);
        const uint32_t a_base = smem_u32(smem + st * stage_bytes);
        const uint32_t b_base = xres ? smem_u32(xsm + it * xbytes) : a_base + kWTile;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int m = seg_it * 4 + kk;  // MMA index within the segment: accumulator m % nacc
          if (!(p.dev & 2))
            umma_bf16(tmem + (seg * nacc + (m & (nacc - 1))) * N, umma_desc(a_base + kk * 32, 16, 1024, kLayoutSW128),
                      umma_desc(b_base + kk * 32, 16, 1024, kLayoutSW128), idesc, m >= nacc ? 1u : 0u);
        }
        umma_commit(&empty[st]);
        if (it + 1 == nk || it + 1 == n0) umma_commit(&acc_bar[seg]);
      }
      __syncwarp();
      if (++st == S) {
        st = 0;
        phase ^= 1u;
      }
    }
    if (lane == 0) {
      if ((p.dev & 32768) && nk_mma < nk) {  // dev: release the epilogue (results meaningless)
        umma_commit(&acc_bar[0]);
        if (nseg > 1) umma_commit(&acc_bar[1]);
      }
      QKV_STAMP(3);
    }
    __syncwarp();
  } else {  // ------------------------------------------------ epilogue, warps 2-5 (128 threads)
    pdl_wait();  // 1/rms (rbuf), positions and the head counters are read below
    const int quarter = warp & 3, row = quarter * 32 + lane, et = tid - 64;
    const int kind_q = p.Hq, kind_k = p.Hq + p.Hkv;
    int pair, partner;
    if (p.style == 0) {  // half-split (rotate_half): (i, i+64)
      pair = row & 63;
      partner = row ^ 64;
    } else {  // interleaved (RoFormer): (2j, 2j+1)
      pair = row >> 1;
      partner = row ^ 1;
    }
    const bool first_of_pair = p.style == 0 ? row < 64 : (row & 1) == 0;
    float* ys = reinterpret_cast<float*>(smem + ring - kEpiBytes);  // [8][128] token group
    for (int seg = 0; seg < nseg; ++seg) {
      const int head = head0 + seg;
      mbar_wait(&acc_bar[seg], 0);
      if (seg == 0 && et == 0) QKV_STAMP(4);
      tc_fence_after();
      float* mine = p.part + (static_cast<size_t>(cta) * 2 + seg) * N * 128;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + seg * nacc * N;
      const int seg_units = seg == 0 ? min(nk, nkb - u0 % nkb) : nk - (nkb - u0 % nkb);
      const int used = min(nacc, 4 * seg_units);  // accumulators this segment wrote
      for (int c = 0; c < N; c += 16) {
        float v[16], w[16];
        tmem_ld16(lane_base + c, v);
        for (int a = 1; a < used; ++a) {  // fixed order: deterministic
          tmem_ld16(lane_base + a * N + c, w);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
        }
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) mine[(c + j) * 128 + row] = v[j];
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (et == 0) {
        const int hu0 = head * nkb, hu1 = hu0 + nkb;
        int c0 = static_cast<int>(static_cast<int64_t>(hu0) * n / U);
        while (c0 > 0 && unit_begin(c0, U, n) > hu0) --c0;
        while (unit_begin(c0 + 1, U, n) <= hu0) ++c0;
        int c1 = c0;
        while (c1 + 1 < n && unit_begin(c1 + 1, U, n) < hu1) ++c1;
        const int contributors = c1 - c0 + 1;
        const int prev = atomicAdd(p.counters + head, 1);
        *last_flag = prev == contributors - 1 ? c0 : -1;
        if (prev == contributors - 1) p.counters[head] = 0;  // re-armed for the next call
      }
      named_bar_sync(1, 128);
      const int c0 = *last_flag;
      named_bar_sync(1, 128);
      if (et == 0) QKV_STAMP(5);
      if (c0 < 0) continue;
      __threadfence();
      // last arrival: reduce every contributor's partial in CTA order (deterministic), then finish.
      // 8 tokens x 4 contributors of loads are issued before any is used (one L2 round trip per
      // group: under the next layer's weight stream an L2 round trip costs ~1 us).
      const int hu1 = (head + 1) * nkb;
      const int kind = head < kind_q ? 0 : head < kind_k ? 1 : 2;
      int n_c = 0;
      while (c0 + n_c < n && unit_begin(c0 + n_c, U, n) < hu1) ++n_c;
      for (int g0 = 0; g0 < p.n_tok; g0 += 8) {
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int ci = 0; ci < n_c; ci += 4) {
          float v[4][8][2];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = c0 + ci + cc;
            const bool ok = ci + cc < n_c;
            const int cseg = ok && unit_begin(c, U, n) / nkb != head ? 1 : 0;
            const float* src = p.part + (static_cast<size_t>(ok ? c : c0) * 2 + cseg) * N * 128 + row;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int t = g0 + j;
              v[cc][j][0] = ok && t < p.n_tok ? __ldcg(src + t * 128) : 0.f;
              v[cc][j][1] = ok && t < p.n_tok ? __ldcg(src + (NT + t) * 128) : 0.f;
            }
          }
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += v[cc][j][0] + v[cc][j][1];
        }
        float rs[8];
        float2 csn[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int t = min(g0 + j, p.n_tok - 1);
            rs[j] = __ldcg(p.rbuf + t);
            csn[j] = kind < 2 ? __ldcg(p.rope + t * 64 + pair) : make_float2(1.f, 0.f);
          }
#pragma unroll
        for (int j = 0; j < 8; ++j) ys[j * 128 + row] = acc[j] * rs[j];
        named_bar_sync(1, 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int t = g0 + j;
          if (t >= p.n_tok) break;
          const int b = t / p.rows, r = t - b * p.rows;
          float y = ys[j * 128 + row];
          if (kind < 2) {
            const float yp = ys[j * 128 + partner];
            y = first_of_pair ? __fsub_rn(__fmul_rn(y, csn[j].x), __fmul_rn(yp, csn[j].y))
                              : __fadd_rn(__fmul_rn(y, csn[j].x), __fmul_rn(yp, csn[j].y));
          }
          const __nv_bfloat16 o = __float2bfloat16_rn(y);
          if (kind == 0)
            p.q[((static_cast<size_t>(b) * p.Hq + head) * p.rows + r) * 128 + row] = o;
          else
            (kind == 1 ? p.k_new : p.v_new)[((static_cast<size_t>(b) * p.rows + r) * p.Hkv + head - kind_q -
                                             (kind == 2 ? p.Hkv : 0)) * 128 + row] = o;
        }
        named_bar_sync(1, 128);
      }
      if (et == 0) QKV_STAMP(6);
    }
  }
  __syncthreads();
  if (tid == 0) QKV_STAMP(7);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}


// ---------------------------------------------------------------------------------------------
// Decode-size producer (<= 8 tokens): one fused launch on mma.sync instead of tcgen05.
//
// Measured on this chip: a tcgen05.mma instruction (M = 128, K = 16) costs ~78 ns whatever N is, so
// with 2 x 8 token columns the swap-AB projection is bound by the instruction count (~0.39 us per
// 16 KB weight tile) and needs split-K across CTAs plus a separate prepare kernel.  For <= 8 tokens
// the warp-level m16n8k16 MMA (A = 16 weight rows x 16 of d_model, B = the 8 token columns as bf16
// hi / lo planes) does the same fp32-accurate product at a fraction of the tensor time, and every
// CTA owns whole output rows over the full d_model, so there is no split-K reduction and no second
// launch:
//   * CTA c owns RoPE pairs [c*P/grid, (c+1)*P/grid) (P = n_out / 2; both rows of a pair, so the
//     rotation happens in registers), in 16-row tiles: rows 0-7 = first rows of 8 pairs, 8-15 = their
//     partners — exactly the C-fragment rows gid / gid+8 of one lane;
//   * warp w owns the 32-wide k-blocks w, w+16, ... of d_model; the 16-byte chunk a lane loads
//     (8 consecutive k of one weight row, straight from the packed SWIZZLE_128B tiles) IS its A
//     fragment of two k16 steps once k is permuted inside the block (A and B use the same
//     permutation: logical k 2t4+e / 2t4+8+e of step s = physical 8t4+4s+e / 8t4+4s+2+e);
//   * x * gain is staged once per CTA in shared memory (fp32, padded rows), and 1/rms (double sum of
//     squares, like qkv_prepare) comes from the same pass; B fragments are split to hi / lo per block;
//   * the 16 warps' partial C fragments are summed in warp order through shared memory
//     (deterministic), then the tile's warp applies 1/rms and RoPE (fp32, angle reduced in double as in
//     qkv_prepare) and stores bf16.
// Pre-dependency: the CTA's weight rows are prefetched into L2 (they depend on nothing).
// split3_bf16 (common.cuh): (a, b) -> three bf16 planes, a ~= hi + mid + lo

constexpr int kGemvThreads = 512;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kGemvTiles = 3;  // 16-row tiles per CTA (24 RoPE pairs; Llama-3.1-8B: 3072 pairs / 148 CTAs)

__global__ void __launch_bounds__(kGemvThreads, 1) qkv_gemv(QkvParams p) {
  extern __shared__ __align__(16) float gsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gid = lane >> 2, t4 = lane & 3;
  const int D = p.nkb * 64, T = p.n_tok;
  const int xs_ld = D + 4;                       // padded fp32 row (conflict-free LDS.128 per gid)
  float* xs = gsm;                               // [T][xs_ld] x * gain
  float* red = xs + T * xs_ld;                   // [kGemvWarps][kGemvTiles][32][4] partial C fragments
  __shared__ double ssq[kGemvWarps][8];
  const int P = p.n_out / 2, grid = gridDim.x;
  const int pr0 = static_cast<int>(static_cast<int64_t>(blockIdx.x) * P / grid);
  const int pr1 = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * P / grid);
  // physical weight row (0..n_out) of tile row rr (0..15) of tile t; -1 if past the CTA's pairs
  auto row_of = [&](int t, int rr) {
    const int pp = pr0 + t * 8 + (rr & 7);
    if (pp >= pr1) return -1;
    const int h = pp >> 6, j = pp & 63;
    const int first = p.style == 0 ? j : 2 * j, second = p.style == 0 ? j + 64 : 2 * j + 1;
    return h * 128 + (rr < 8 ? first : second);
  };
  const size_t layer_base = static_cast<size_t>(p.layer) * p.heads * p.nkb;
  // address of the 16-byte chunk holding k = 8c .. 8c+7 of weight row `row` in the packed tiles
  auto wchunk = [&](int row, int c) {
    const int h = row >> 7, rr = row & 127, kt = c >> 3;
    return reinterpret_cast<const uint4*>(p.wpack + ((layer_base + static_cast<size_t>(h) * p.nkb + kt) * 128 + rr) * 64) +
           ((c & 7) ^ (rr & 7));
  };
  float acc[kGemvTiles][4];
#pragma unroll
  for (int t = 0; t < kGemvTiles; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  int rowA[kGemvTiles], rowB[kGemvTiles];
#pragma unroll
  for (int t = 0; t < kGemvTiles; ++t) {
    rowA[t] = row_of(t, gid);
    rowB[t] = row_of(t, gid + 8);
  }
  const int nblk = D / 32;
  uint4 wa[2][kGemvTiles], wb[2][kGemvTiles];
  auto load_w = [&](const int buf, int blk) {
    const int c = blk * 4 + t4;
#pragma unroll
    for (int t = 0; t < kGemvTiles; ++t) {
      (buf ? wa[1] : wa[0])[t] = rowA[t] >= 0 ? __ldcs(wchunk(rowA[t], c)) : make_uint4(0, 0, 0, 0);
      (buf ? wb[1] : wb[0])[t] = rowB[t] >= 0 ? __ldcs(wchunk(rowB[t], c)) : make_uint4(0, 0, 0, 0);
    }
  };
  // pre-dependency (weights depend on nothing): the warp's first two k-blocks into registers.  (An L2
  // prefetch of the rest, one 128-byte bulk prefetch per row and k tile, measured slower: 20.9 vs
  // 16.4 us per layer; dev bit 1 turns it on.)
  if (warp < nblk) load_w(0, warp);
  if (warp + kGemvWarps < nblk) load_w(1, warp + kGemvWarps);
  if (p.dev & 1)
    for (int i = tid; i < kGemvTiles * 16 * p.nkb; i += kGemvThreads) {
      const int t = i / (16 * p.nkb), rr = (i / p.nkb) & 15, kt = i % p.nkb;
      const int row = row_of(t, rr);
      if (row >= 0 && kt >= 4)
        bulk_prefetch_l2(p.wpack + ((layer_base + static_cast<size_t>(row >> 7) * p.nkb + kt) * 128 + (row & 127)) * 64,
                         128);
    }
  pdl_wait();  // x and positions are the previous kernel's outputs
  pdl_launch_dependents();
  // each warp stages x * gain for its own k-blocks (no CTA barrier before the main loop) and keeps
  // per-lane partial sums of squares (double, like qkv_prepare) for the epilogue's 1/rms
  const float* g = p.gain + static_cast<size_t>(p.layer) * D;
  double ss[2] = {0.0, 0.0};  // tokens lane/8 and lane/8 + 4
  {
    const int kq = 4 * (lane & 7), t0 = lane >> 3;
    for (int blk = warp; blk < nblk; blk += kGemvWarps) {
      const int k = blk * 32 + kq;
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g + k));
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = t0 + 4 * e;
        if (t < T) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(p.x + static_cast<size_t>(t) * D + k));
          ss[e] += static_cast<double>(xv.x) * xv.x + static_cast<double>(xv.y) * xv.y +
                   static_cast<double>(xv.z) * xv.z + static_cast<double>(xv.w) * xv.w;
          *reinterpret_cast<float4*>(xs + t * xs_ld + k) = make_float4(xv.x * gg.x, xv.y * gg.y, xv.z * gg.z, xv.w * gg.w);
        }
      }
    }
  }
  __syncwarp();
  auto compute = [&](const uint4 (&wA)[kGemvTiles], const uint4 (&wB)[kGemvTiles], int blk) {
    // B fragments of token gid at k = 32 blk + 8 t4 .. + 7 (hi / lo planes)
    const float* xr = xs + gid * xs_ld + blk * 32 + 8 * t4;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 x0 = gid < T ? *reinterpret_cast<const float4*>(xr) : z4;
    const float4 x1 = gid < T ? *reinterpret_cast<const float4*>(xr + 4) : z4;
    // three bf16 planes (hi + mid + lo represent x * gain to ~2^-24): the product is as accurate as
    // an fp32 one, so outputs round like the exact value except within fp32 noise of a tie
    uint32_t hi[4], mid[4], lo[4];
    split3_bf16(x0.x, x0.y, hi[0], mid[0], lo[0]);
    split3_bf16(x0.z, x0.w, hi[1], mid[1], lo[1]);
    split3_bf16(x1.x, x1.y, hi[2], mid[2], lo[2]);
    split3_bf16(x1.z, x1.w, hi[3], mid[3], lo[3]);
#pragma unroll
    for (int t = 0; t < kGemvTiles; ++t) {
      const uint32_t a0[4] = {wA[t].x, wB[t].x, wA[t].y, wB[t].y}, a1[4] = {wA[t].z, wB[t].z, wA[t].w, wB[t].w};
      mma_bf16(acc[t], a0, lo[0], lo[1]);
      mma_bf16(acc[t], a1, lo[2], lo[3]);
      mma_bf16(acc[t], a0, mid[0], mid[1]);
      mma_bf16(acc[t], a1, mid[2], mid[3]);
      mma_bf16(acc[t], a0, hi[0], hi[1]);
      mma_bf16(acc[t], a1, hi[2], hi[3]);
    }
  };
  // two register buffers with compile-time indices (unrolled by two blocks); blocks 0 and 1 of the
  // warp were loaded before the dependency wait
  for (int blk = warp; blk < nblk; blk += 2 * kGemvWarps) {
    const bool has1 = blk + kGemvWarps < nblk;
    compute(wa[0], wb[0], blk);
    if (blk + 2 * kGemvWarps < nblk) load_w(0, blk + 2 * kGemvWarps);
    if (has1) {
      compute(wa[1], wb[1], blk + kGemvWarps);
      if (blk + 3 * kGemvWarps < nblk) load_w(1, blk + 3 * kGemvWarps);
    }
  }
  // per-token sums of squares: lanes of the same token (lane / 8) reduce, then warps via shared memory
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) ss[e] += __shfl_xor_sync(0xffffffffu, ss[e], off);
    if ((lane & 7) == 0) ssq[warp][(lane >> 3) + 4 * e] = ss[e];
  }
#pragma unroll
  for (int t = 0; t < kGemvTiles; ++t)
    *reinterpret_cast<float4*>(red + ((warp * kGemvTiles + t) * 32 + lane) * 4) =
        make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
  __syncthreads();
  if (warp >= kGemvTiles) return;
  // epilogue: warp t finishes tile t — sum the warps' partials in order, 1/rms, RoPE, bf16 stores
  const int t = warp;
  if (rowA[t] < 0) return;
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  for (int w = 0; w < kGemvWarps; ++w) {
    const float4 v = *reinterpret_cast<const float4*>(red + ((w * kGemvTiles + t) * 32 + lane) * 4);
    c[0] += v.x;
    c[1] += v.y;
    c[2] += v.z;
    c[3] += v.w;
  }
  const int head = rowA[t] >> 7, dA = rowA[t] & 127, dB = rowB[t] & 127;
  const int kind_q = p.Hq, kind_k = p.Hq + p.Hkv;
  const int kind = head < kind_q ? 0 : head < kind_k ? 1 : 2;
  const int j = p.style == 0 ? dA : dA >> 1;  // RoPE pair of this row pair
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int tok = 2 * t4 + e;
    if (tok >= T) break;
    double s2 = 0.0;  // 1/rms of this token (warp-order sum: deterministic)
    for (int w = 0; w < kGemvWarps; ++w) s2 += ssq[w][tok];
    const float rs = static_cast<float>(1.0 / sqrt(s2 / D + static_cast<double>(p.eps)));
    float yA = c[e] * rs, yB = c[2 + e] * rs;
    const int b = tok / p.rows, r = tok - b * p.rows;
    if (kind < 2) {
      double turns = static_cast<double>(p.pos0[b] + r) * exp2(-p.log2_theta * (2.0 * j) / 128.0) * 0.15915494309189535;
      turns -= floor(turns);
      double sd, cd;
      sincospi(2.0 * turns, &sd, &cd);
      const float cs = static_cast<float>(cd), sn = static_cast<float>(sd);
      const float nA = __fsub_rn(__fmul_rn(yA, cs), __fmul_rn(yB, sn));
      const float nB = __fadd_rn(__fmul_rn(yB, cs), __fmul_rn(yA, sn));
      yA = nA;
      yB = nB;
    }
    __nv_bfloat16* dst;
    if (kind == 0)
      dst = p.q + ((static_cast<size_t>(b) * p.Hq + head) * p.rows + r) * 128;
    else
      dst = (kind == 1 ? p.k_new : p.v_new) +
            ((static_cast<size_t>(b) * p.rows + r) * p.Hkv + head - kind_q - (kind == 2 ? p.Hkv : 0)) * 128;
    dst[dA] = __float2bfloat16_rn(yA);
    dst[dB] = __float2bfloat16_rn(yB);
  }
}

size_t qkv_gemv_smem(int D, int T) {
  return (static_cast<size_t>(T) * (D + 4) + kGemvWarps * kGemvTiles * 32 * 4) * sizeof(float);
}

}  // namespace sa

extern "C" {

SA_API sa_status sa_qkv_create(const void* w_qkv, const float* attn_norm_gain, int32_t n_layers, int32_t d_model,
                               int32_t n_q_heads, int32_t n_kv_heads, double norm_eps, double rope_theta,
                               int32_t rope_style, sa_qkv** out) {
  if (!w_qkv || !attn_norm_gain || !out) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (n_layers < 1 || n_kv_heads < 1 || n_q_heads < 1 || n_q_heads % n_kv_heads != 0)
    return sa::fail(SA_INVALID_ARGUMENT, "ModelConfig: n_kv_heads must divide n_q_heads");
  if (d_model < 64 || d_model % 64 != 0) return sa::fail(SA_INVALID_ARGUMENT, "qkv: d_model must be a multiple of 64");
  if (!(norm_eps > 0.0) || !(rope_theta > 0.0)) return sa::fail(SA_INVALID_ARGUMENT, "ModelConfig: norm_eps, rope_theta");
  if (rope_style != 0 && rope_style != 1) return sa::fail(SA_INVALID_ARGUMENT, "qkv: rope_style is 0 or 1");
  auto* h = new sa_qkv();
  h->L = n_layers;
  h->Hq = n_q_heads;
  h->Hkv = n_kv_heads;
  h->D = d_model;
  h->n_out = (n_q_heads + 2 * n_kv_heads) * 128;
  h->nkb = d_model / 64;
  h->style = rope_style;
  h->eps = static_cast<float>(norm_eps);
  h->theta = rope_theta;
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  const size_t tiles = static_cast<size_t>(n_layers) * (n_q_heads + 2 * n_kv_heads) * h->nkb;
  cudaError_t e = cudaMalloc(&h->wpack, tiles * sa::kWTile);
  if (e == cudaSuccess) e = cudaMalloc(&h->gain, static_cast<size_t>(n_layers) * d_model * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&h->xbuf, static_cast<size_t>(h->nkb) * 2 * sa::kQkvMaxTokens * 64 * 2);
  if (e == cudaSuccess) e = cudaMalloc(&h->rbuf, sa::kQkvMaxTokens * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&h->rope, sa::kQkvMaxTokens * 64 * sizeof(float2));
  const int heads = n_q_heads + 2 * n_kv_heads;
  h->max_grid = std::max(heads, std::min(h->num_sms, heads * h->nkb));
  if (e == cudaSuccess)
    e = cudaMalloc(&h->part, static_cast<size_t>(h->max_grid) * 2 * 2 * sa::kQkvMaxTokens * 128 * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&h->counters, heads * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(h->counters, 0, heads * sizeof(int));
  if (e == cudaSuccess)
    e = cudaMemcpy(h->gain, attn_norm_gain, static_cast<size_t>(n_layers) * d_model * sizeof(float),
                   cudaMemcpyDefault);
  if (e == cudaSuccess) {
    sa::qkv_pack<<<static_cast<unsigned>(tiles), 256>>>(static_cast<const __nv_bfloat16*>(w_qkv), h->n_out, d_model,
                                                         h->wpack);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    sa_qkv_destroy(h);
    return sa::cuda_fail(e, "qkv create");
  }
  *out = h;
  return SA_OK;
}

SA_API sa_status sa_qkv_dev_set_knob(sa_qkv* h, const char* name, int64_t value) {
  if (!h || !name) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  const std::string n(name);
  if (n == "dev") {
    h->dev_bits = static_cast<int>(value);
  } else if (n == "impl_tc") {
    h->force_tc = value ? 1 : 0;
  } else if (n == "trace") {
    if (value && !h->trace) {
      const size_t bytes = static_cast<size_t>(h->L) * h->max_grid * 32 * 8;
      SA_CUDA_CHECK(cudaMalloc(&h->trace, bytes));
      SA_CUDA_CHECK(cudaMemset(h->trace, 0, bytes));
    }
  } else {
    return sa::fail(SA_INVALID_ARGUMENT, "unknown dev knob '" + n + "'");
  }
  return SA_OK;
}

SA_API sa_status sa_qkv_destroy(sa_qkv* h) {
  if (!h) return SA_OK;
  if (h->trace) {  // dev-only: dump the stamps of the last call per layer
    std::vector<unsigned long long> t(static_cast<size_t>(h->L) * h->max_grid * 32);
    if (cudaMemcpy(t.data(), h->trace, t.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
      if (FILE* f = std::fopen("/tmp/sa_qkv_trace.bin", "wb")) {
        std::fwrite(t.data(), 8, t.size(), f);
        std::fclose(f);
      }
    }
    cudaFree(h->trace);
  }
  cudaFree(h->wpack);
  cudaFree(h->gain);
  cudaFree(h->xbuf);
  cudaFree(h->rbuf);
  cudaFree(h->rope);
  cudaFree(h->part);
  cudaFree(h->counters);
  delete h;
  return SA_OK;
}

SA_API sa_status sa_qkv_project(sa_qkv* h, int32_t layer, const float* x, const int32_t* positions, int32_t B,
                                int32_t rows, void* q, void* k_new, void* v_new, void* stream) {
  if (!h || !x || !positions || !q || !k_new || !v_new) return sa::fail(SA_INVALID_ARGUMENT, "null argument");
  if (layer < 0 || layer >= h->L) return sa::fail(SA_OUT_OF_RANGE, "qkv: layer out of range");
  if (B < 1 || rows < 1 || B * rows > sa::kQkvMaxTokens)
    return sa::fail(SA_INVALID_ARGUMENT, "qkv: 1 <= B * rows <= 128 tokens per call");
  sa::QkvParams p{};
  p.layer = layer;
  p.n_out = h->n_out;
  p.nkb = h->nkb;
  p.n_tok = B * rows;
  p.rows = rows;
  p.NT = (p.n_tok + 7) / 8 * 8;
  p.N = 2 * p.NT;
  p.Hq = h->Hq;
  p.Hkv = h->Hkv;
  const int heads = h->Hq + 2 * h->Hkv;
  p.heads = heads;
  p.style = h->style;
  p.eps = h->eps;
  p.log2_theta = std::log2(h->theta);
  p.wpack = h->wpack;
  p.x = x;
  p.gain = h->gain;
  p.pos0 = positions;
  p.xbuf = h->xbuf;
  p.rbuf = h->rbuf;
  p.rope = h->rope;
  p.part = h->part;
  p.counters = h->counters;
  p.trace = h->trace;
  p.dev = h->dev_bits;
  p.q = static_cast<__nv_bfloat16*>(q);
  p.k_new = static_cast<__nv_bfloat16*>(k_new);
  p.v_new = static_cast<__nv_bfloat16*>(v_new);
  auto s = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute pdl1[1];
  pdl1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl1[0].val.programmaticStreamSerializationAllowed = 1;
  const bool force_tc = h->force_tc != 0;
  const size_t gsmem = sa::qkv_gemv_smem(h->D, p.n_tok);
  if (p.n_tok <= 8 && gsmem <= 200 * 1024 && !force_tc) {  // decode sizes: one fused mma.sync launch
    static std::atomic<uint64_t> gattr{0};
    int gdev = 0;
    if (sa::func_attrs_needed(gattr, &gdev)) {
      SA_CUDA_CHECK(cudaFuncSetAttribute(sa::qkv_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      sa::func_attrs_done(gattr, gdev);
    }
    const int P = h->n_out / 2;
    cudaLaunchConfig_t cg{};
    cg.gridDim = dim3(std::max((P + sa::kGemvTiles * 8 - 1) / (sa::kGemvTiles * 8), std::min(h->num_sms, P)));
    cg.blockDim = dim3(sa::kGemvThreads);
    cg.dynamicSmemBytes = gsmem;
    cg.stream = s;
    cg.attrs = pdl1;
    cg.numAttrs = 1;
    SA_CUDA_CHECK(cudaLaunchKernelEx(&cg, sa::qkv_gemv, p));
    return SA_OK;
  }
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  if (sa::func_attrs_needed(attr_mask, &dev)) {
    SA_CUDA_CHECK(cudaFuncSetAttribute(sa::qkv_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, sa::kQkvSmem));
    sa::func_attrs_done(attr_mask, dev);
  }
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t c1{};
  c1.gridDim = dim3(p.NT);
  c1.blockDim = dim3(256);
  c1.stream = s;
  c1.attrs = pdl;
  c1.numAttrs = 1;
  SA_CUDA_CHECK(cudaLaunchKernelEx(&c1, sa::qkv_prepare, p));
  cudaLaunchConfig_t c2{};
  c2.gridDim = dim3(h->max_grid);  // stream-K: every SM takes an equal run of (head, k-block) units
  c2.blockDim = dim3(sa::kQkvThreads);
  c2.dynamicSmemBytes = sa::kQkvSmem;
  c2.stream = s;
  c2.attrs = pdl;
  c2.numAttrs = 1;
  SA_CUDA_CHECK(cudaLaunchKernelEx(&c2, sa::qkv_gemm, p));
  return SA_OK;
}

}  // extern "C"
