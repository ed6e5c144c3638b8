// draft.cu — sparse draft attention: index gather fused with attention (+ fused KV append).
//
// Reference: KvStore::gather (kv_store.cpp:67-88) followed by attend (attention.cpp:70-76) over
// [K_T ; K_tail], the SPEC draft-forward key set T ∪ {positions >= draft window start}
// (SPEC.md:385,447).  The reference materialises the gathered K/V copies; here each CTA gathers
// its slice of the virtual key list T[0..k) ++ [p0, p0+step) straight into shared memory with
// TMA tile::gather4 (4 rows x 64 columns per instruction) in the swizzled layout the mma.sync
// flash step reads, for the G q-heads of its KV head (one 16-row tile).
//
// Grid (CS x n_sub, Hkv, B) launched as clusters of CS CTAs: the CS splits of one cluster merge their
// partial (max, sum, O) through distributed shared memory; with n_sub > 1 clusters per (sequence, KV
// head) the clusters' merged slices are combined once more through global memory (two-level merge).
//
// Programmatic dependent launch: the selected prefix rows (T from the select kernel, positions
// < p0, never written during the draft phase) are gathered BEFORE griddepcontrol.wait, overlapping
// the previous layer's kernel; the query, the tail rows and this step's new row (which a real model
// produces in the previous layer) are read after it.
#include "attn_core.cuh"
#include <algorithm>
#include <map>
#include <mutex>

#include "internal.h"

namespace sa {

// Swap-AB mma.sync flash step for <= 8 query rows (the G q-heads of one KV head):
//   S^T(16 tok x 8 rows) = K(16x128) Q^T            8 x mma.m16n8k16 per 16 tokens
//   O^T(128 d x 8 rows) += V^T(128 x 16 tok) P^T      8 d-blocks x (hi, mid, lo) = 24 mma per 16 tokens
// Thread (gid = lane/4, t4 = lane%4) holds S^T for tokens gid / gid+8 and query rows 2*t4, 2*t4+1;
// P^T is re-laid out as the B operand with movmatrix (8x8 transpose), so no shared-memory trip.
//
// kPack (G <= 4): the four real query rows use only half of the n8 tile, so the P planes share it:
// B columns 0-3 carry P_hi of rows 0-3 and columns 4-7 P_mid of the same rows (one mma), and a second
// mma adds P_lo into columns 0-3 — 16 instead of 24 PV mma per 16 tokens.  Lanes with t4 >= 2 then
// track the running max of rows 2*t4-4+e (their accumulator columns hold those rows' P_mid terms), and
// finalize() folds columns 4-7 into 0-3.
template <bool kPack>
struct DraftWarp {
  float o[8][4];     // O^T accumulators: d-block jj rows gid / gid+8, query rows 2t4 / 2t4+1
  float m[2], l[2];  // running max (scaled log2) and per-thread partial sums of rows 2t4, 2t4+1
  uint32_t qb[8][2];  // Q^T B-fragments per k16 step of d

  __device__ __forceinline__ void init(const __nv_bfloat16* q_rows, int G, int lane) {
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
    const int gid = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b0 = 0, b1 = 0;
      if (gid < G) {
        b0 = __ldg(reinterpret_cast<const uint32_t*>(q_rows + gid * 128 + kk * 16 + 2 * t4));
        b1 = __ldg(reinterpret_cast<const uint32_t*>(q_rows + gid * 128 + kk * 16 + 8 + 2 * t4));
      }
      qb[kk][0] = b0;
      qb[kk][1] = b1;
    }
  }

  // NB sub-blocks of 16 tokens each (sub-block i: tokens [r0[i], r0[i]+16) of the swizzled K/V tile
  // at k_smem[i] / v_smem[i], the first n_valid[i] valid) in ONE online-softmax step: the QK^T
  // chains of the sub-blocks are independent (ILP), one row-max reduction and one rescale cover them.
  template <int NB>
  __device__ __forceinline__ void step(const uint32_t (&k_smem)[NB], const uint32_t (&v_smem)[NB], uint32_t half,
                                       const int (&r0)[NB], int lane, float c, const int (&n_valid)[NB],
                                       long long* cyc = nullptr) {
    const int gid = lane >> 2, mi = lane >> 3;
    if (cyc) cyc[0] = clock64();
    float s[NB][4];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) {
      const int tok = r0[bi] + (mi & 1) * 8 + (lane & 7);
      float s2[4] = {0.f, 0.f, 0.f, 0.f};  // two accumulator chains halve the dependent mma depth
      s[bi][0] = s[bi][1] = s[bi][2] = s[bi][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        uint32_t a[4], a2[4];
        ldsm_x4(k_smem[bi] + swz(tok, 2 * kk + (mi >> 1), half), a[0], a[1], a[2], a[3]);
        ldsm_x4(k_smem[bi] + swz(tok, 2 * (kk + 1) + (mi >> 1), half), a2[0], a2[1], a2[2], a2[3]);
        mma_bf16(s[bi], a, qb[kk][0], qb[kk][1]);
        mma_bf16(s2, a2, qb[kk + 1][0], qb[kk + 1][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s[bi][i] += s2[i];
      if (gid >= n_valid[bi]) s[bi][0] = s[bi][1] = -INFINITY;
      if (gid + 8 >= n_valid[bi]) s[bi][2] = s[bi][3] = -INFINITY;
    }
    if (cyc) {  // dev timing: S landed
      asm volatile("" ::"f"(s[NB - 1][0]), "f"(s[0][3]));
      cyc[1] = clock64();
    }
    // per query row (2t4 + e): max over the NB x 16 tokens (in-thread, then 8 gid lanes)
    float tmax[2] = {fmaxf(s[0][0], s[0][2]), fmaxf(s[0][1], s[0][3])};
#pragma unroll
    for (int bi = 1; bi < NB; ++bi) {
      tmax[0] = fmaxf(tmax[0], fmaxf(s[bi][0], s[bi][2]));
      tmax[1] = fmaxf(tmax[1], fmaxf(s[bi][1], s[bi][3]));
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      tmax[0] = fmaxf(tmax[0], __shfl_xor_sync(0xffffffffu, tmax[0], off));
      tmax[1] = fmaxf(tmax[1], __shfl_xor_sync(0xffffffffu, tmax[1], off));
    }
    if (kPack) {  // lanes t4 >= 2 follow rows 2*t4-4+e (the P_mid columns they accumulate)
      const float x0 = __shfl_xor_sync(0xffffffffu, tmax[0], 2), x1 = __shfl_xor_sync(0xffffffffu, tmax[1], 2);
      if ((lane & 3) >= 2) {
        tmax[0] = x0;
        tmax[1] = x1;
      }
    }
    float mnew[2];
    bool grow = false;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      mnew[e] = fmaxf(m[e], tmax[e] * c);
      grow |= mnew[e] > m[e];
    }
    if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float f = (mnew[e] == -INFINITY || m[e] == mnew[e]) ? 1.f : fast_exp2(m[e] - mnew[e]);
        l[e] *= f;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          o[jj][e] *= f;
          o[jj][2 + e] *= f;
        }
        m[e] = mnew[e];
      }
    }
    const float b0 = m[0] == -INFINITY ? 0.f : m[0], b1 = m[1] == -INFINITY ? 0.f : m[1];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) {
      const float p0 = fast_exp2(fmaf(s[bi][0], c, -b0)), p1 = fast_exp2(fmaf(s[bi][1], c, -b1));
      const float p2 = fast_exp2(fmaf(s[bi][2], c, -b0)), p3 = fast_exp2(fmaf(s[bi][3], c, -b1));
      l[0] += p0 + p2;
      l[1] += p1 + p3;
      // P = hi + mid + lo bf16 planes (~2^-27 relative: the tau = 1e-3 elementwise bar of SURVEY §8c)
      uint32_t h01, m01, l01, h23, m23, l23;
      split3_bf16(p0, p1, h01, m01, l01);  // token gid,   rows 2t4, 2t4+1
      split3_bf16(p2, p3, h23, m23, l23);  // token gid+8
      // B fragments of P^T (k = tokens, n = rows): 8x8 transposes of the two token halves
      uint32_t bh0 = movmatrix_trans(h01), bh1 = movmatrix_trans(h23);
      const uint32_t bm0 = movmatrix_trans(m01), bm1 = movmatrix_trans(m23);
      uint32_t bl0 = movmatrix_trans(l01), bl1 = movmatrix_trans(l23);
      if (kPack) {  // columns 4-7 <- P_mid of rows 0-3 (held by lane ^ 16 after the transpose); P_lo: 0-3
        const uint32_t x0 = __shfl_xor_sync(0xffffffffu, bm0, 16), x1 = __shfl_xor_sync(0xffffffffu, bm1, 16);
        if (gid >= 4) {
          bh0 = x0;
          bh1 = x1;
          bl0 = bl1 = 0u;
        }
      }
      const int tok = r0[bi] + (mi >> 1) * 8 + (lane & 7);
      if (cyc && bi == 0) {  // dev timing: P fragments of the first sub-block ready
        asm volatile("" ::"r"(bh0), "r"(bl1));
        cyc[2] = clock64();
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {  // one V fragment load serves the three P planes
        uint32_t a[4];
        ldsm_x4_t(v_smem[bi] + swz(tok, 2 * jj + (mi & 1), half), a[0], a[1], a[2], a[3]);
        mma_bf16(o[jj], a, bh0, bh1);
        if (!kPack) mma_bf16(o[jj], a, bm0, bm1);
        mma_bf16(o[jj], a, bl0, bl1);
      }
    }
    if (cyc) {  // dev timing: PV accumulators landed
      asm volatile("" ::"f"(o[7][3]), "f"(o[0][0]));
      cyc[3] = clock64();
    }
  }

  __device__ __forceinline__ void finalize() {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) l[e] += __shfl_xor_sync(0xffffffffu, l[e], off);
    if (kPack)  // fold the P_mid columns 4-7 into rows 0-3 (lanes t4 < 2)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[jj][i] += __shfl_xor_sync(0xffffffffu, o[jj][i], 2);
  }
};

struct DCfg {
  static constexpr int kTile = 64;
  static constexpr int kMaxTiles = 3;   // resident tiles per round (192 keys)
  static constexpr int kMaxThreads = 256;  // 8 warps (two CTAs per SM: <= 128 registers per thread)
  static constexpr int kMaxWarps = kMaxThreads / 32;
  static constexpr int kMaxCS = 16;
  static constexpr int kHalf = kTile * 128;
  static constexpr int kTileBytes = 2 * kHalf;
  static constexpr int kOffV = kMaxTiles * kTileBytes;
  static constexpr int kPartFloats = 8 * 128 + 16;  // CTA partial: O[8 rows][128], m[8], l[8]
  static constexpr int kOffPart = 2 * kMaxTiles * kTileBytes;
  static constexpr int kOffRow = kOffPart + kPartFloats * 4;      // int64 source rows of the round
  static constexpr int kRowRounds = 3;  // rounds whose source rows are resolved before the dependency wait
  static constexpr int kOffRecv = kOffRow + kRowRounds * kMaxTiles * kTile * 8;  // merge inbox [kMaxCS][kRecvFloats]
  static constexpr int kRecvFloats = 8 * 128 / 1 + 16;            // worst case (CS = 1) slice + (m, l)
  static constexpr int kRecvPerSender = 64 + 16;                  // CS = 16, G = 8: 64-float slice + (m, l)
  static constexpr int kRecvBytes = kMaxCS * kRecvPerSender * 4 > kRecvFloats * 4 ? kMaxCS * kRecvPerSender * 4
                                                                                  : kRecvFloats * 4;
  static constexpr int kOffBar = kOffRecv + kRecvBytes;
  static constexpr int kOffGBar = kOffBar + 16;  // row-gather mbarriers, one per round buffer
  static constexpr int kOffNew = kOffBar + 32;   // this step's new K / V row (32 x 16 B), staged
  static constexpr int kSmem = kOffNew + 512 + 1024;
  // streaming mode (chunks of several rounds): a second K/V buffer after everything else, so round
  // r+1 is gathered while round r is computed (one CTA per SM)
  static constexpr int kOffBuf1 = (kOffNew + 512 + 1023) / 1024 * 1024;
  static constexpr int kOffBt = kOffBuf1 + 2 * kMaxTiles * kTileBytes;  // streaming: block table in smem
  static constexpr int kBtMax = 2048;
  static constexpr int kSmemStream = kOffBt + kBtMax * 4 + 1024;
  static_assert(kMaxWarps * 8 * 132 * 4 <= kOffPart, "warp partials must fit in the tile buffers");
  static_assert(kMaxTiles * kTile * 8 >= kMaxWarps * 16 * 4, "warp (m, l) table fits the row-source area");
  static_assert(kSmem <= 113 * 1024, "two CTAs per SM: the next PDL launch co-resides");
  static_assert(kSmemStream <= 227 * 1024, "streaming mode fits one CTA per SM");
};

// Per-CTA phase stamps (tools/trace_draft.py): dev builds only (-DSA_PIPE_TRACE); the checks cost
// ~0.1 us per launch in the product build.
__device__ __forceinline__ void dtrace(const DraftParams& p, int phase) {
#ifndef SA_PIPE_TRACE
  return;
#endif
  if (p.trace && threadIdx.x == 0) {
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (cta < 512) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      const size_t launch = static_cast<size_t>((p.step - 1) & 7) * 64 + (p.layer & 63);
      p.trace[(launch * 512 + cta) * 16 + phase] = gt;
      if (phase == 0) {  // slot 15: the SM this CTA runs on
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[(launch * 512 + cta) * 16 + 15] = smid;
      }
    }
  }
}

// Grid (CS, Hkv, B) in clusters of CS CTAs: CTA `split` of a (sequence, KV head) owns rows
// [split*chunk, (split+1)*chunk) of the virtual key list T[0..k) ++ [p0, p0+draft_off+step).
//
// Before griddepcontrol.wait (overlapping the previous launch, two CTAs per SM): every row that
// already exists — the selected prefix rows and the tail rows appended by earlier draft steps —
// is resolved (index + block-table loads) and gathered into shared memory with 16-byte cp.async.
// After the wait: the query and this step's new row (produced by the previous layer in a real
// model), the fused append, then the mma.sync flash step over the resident rows.
//
// Merge without a global round trip and without a second cluster barrier: CTA r owns output slice r
// of the G x 128 outputs; every CTA pushes its partial slices and (m, l) into the owners' inboxes
// with st.async (remote shared-memory stores completing as transaction bytes on the owner's
// mbarrier), and each owner combines its slice once its inbox is full.
// kMode 0: one round of <= 192 rows per CTA, two CTAs per SM (config 2: the round loop compiles away);
// 1: several rounds, two CTAs per SM; 2: streaming (double-buffered rounds, one CTA per SM)
template <int kMode, bool kPack>
__global__ void __launch_bounds__(DCfg::kMaxThreads, kMode == 2 ? 1 : 2) draft_kernel(const __grid_constant__ DraftParams p) {
  constexpr bool kStream = kMode == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* part = reinterpret_cast<float*>(smem + DCfg::kOffPart);
  float* inbox = reinterpret_cast<float*>(smem + DCfg::kOffRecv);
  uint64_t* inbox_bar = reinterpret_cast<uint64_t*>(smem + DCfg::kOffBar);
  uint64_t* gbar = reinterpret_cast<uint64_t*>(smem + DCfg::kOffGBar);  // [buffer]: a round's rows landed
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  const int g = blockIdx.y, b = blockIdx.z;
  const int CS = p.n_splits;          // CTAs per cluster
  const int split = blockIdx.x % CS;  // rank in the cluster
  const int sub = blockIdx.x / CS, n_sub = gridDim.x / CS;  // clusters per unit (two-level merge if > 1)
  const int seq = p.seq_ids[b];
  const int p0 = p.p0[b];
  const int j = p.step;
  const int set = p.n_sets == 1 ? 0 : g;
  const int k = p.k_act[b * p.n_sets + set];
  const int32_t* T = p.idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  const int tail = p.draft_off + j;  // tail rows [p0, p0 + tail): committed verify rows, then this chain's
  const int m_total = k + tail;
  const int v_begin = blockIdx.x * p.chunk;
  const int v_end = min(m_total, v_begin + p.chunk);
  const int n = max(0, v_end - v_begin);
  const int Hq = p.Hkv * p.G;
  const int new_pos = p0 + tail - 1;
  const int new_v = k + tail - 1;  // virtual index of this step's new row
  // rows written by earlier draft steps of this layer come from launches >= 2 back in the PDL
  // chain, complete once this grid runs (every earlier CTA passed its own wait before triggering)
  const bool old_tail_ready = p.cache.n_layers >= 2;
  // output slices: CTA r owns outputs [r*per, min(G*128, (r+1)*per)), per a multiple of 4
  const int n_out = p.G * 128;
  const int per = ((n_out + CS - 1) / CS + 3) & ~3;
  const int my_lo = min(n_out, split * per), my_hi = min(n_out, my_lo + per);
  const int rstride = per + 16;  // inbox floats per sender
  dtrace(p, 0);
  if (tid == 0) {
    mbar_init(inbox_bar, 1);
    mbar_init(gbar, 1);
    mbar_init(gbar + 1, 1);
    fence_mbar_init();
  }
  cluster_arrive_release();  // inbox barriers initialised (waited on just before the pushes)

  int64_t* src_row = reinterpret_cast<int64_t*>(smem + DCfg::kOffRow);  // -1: new row (k_new), -2: zero fill
  // pre: true -> rows that exist before this launch (gathered ahead of the dependency wait)
  auto is_pre = [&](int v) { return v < k || (v == new_v ? !p.k_new : old_tail_ready); };
  auto resolve = [&](int r0, int rows, bool pre_pass, int64_t* src_row) {
    for (int r = tid; r < rows; r += nthr) {
      const int v = v_begin + r0 + r;
      if (v >= v_end) {  // zero fill: known before the dependency
        if (pre_pass) src_row[r] = -2;
        continue;
      }
      if (is_pre(v) != pre_pass) continue;
      const bool is_tail = v >= k;
      const int pos = is_tail ? p0 + (v - k) : __ldg(T + v);
      src_row[r] = (p.k_new && pos == new_pos) ? -1 : cache_row(p.cache, seq, p.layer, g, pos);
    }
  };
  // TMA row gather (tile::gather4): per group of 4 rows, K and V x two 64-column halves, each one
  // instruction writing 4 x 128 bytes in the 128-byte-swizzled tile layout the flash step reads;
  // completion counted on the buffer's mbarrier (the round's bytes are expected up front).  A group
  // goes in the pass (before / after the dependency wait) of its rows; zero-fill rows and this
  // step's new row (out-of-range coordinates: zero-filled, the new row stored from registers once
  // its round has landed) fit either.  `all`: every group (rounds issued after the wait).
  auto gather = [&](int r0, int rows, bool pre_pass, int buf, const int64_t* src_row, bool all) {
    const uint32_t base = smem_u32(buf ? smem + DCfg::kOffBuf1 : smem);
    const uint32_t bar = smem_u32(gbar + buf);
    for (int i = tid; i < rows; i += nthr) {  // rows (a multiple of 16) = groups x 4 instructions
      const int r = (i >> 2) * 4, op = i & 3;  // op bit 0: column half, bit 1: V
      int y[4];
      bool pre = true;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v = v_begin + r0 + r + j;
        y[j] = -1;
        if (v >= v_end || (p.k_new && v == new_v)) continue;
        pre = pre && is_pre(v);
        y[j] = static_cast<int>(src_row[r + j]);  // < 0 (new row / zero fill): out of range
      }
      if (!all && pre != pre_pass) continue;
      const uint32_t dst = base + ((op & 2) ? DCfg::kOffV : 0) + (r >> 6) * DCfg::kTileBytes + (op & 1) * DCfg::kHalf +
                           (r & 63) * 128;
      tma_gather4(dst, (op & 2) ? &p.tmv : &p.tmk, bar, (op & 1) * 64, y[0], y[1], y[2], y[3]);
    }
  };

  constexpr int kRoundRows = DCfg::kMaxTiles * DCfg::kTile;
  const int n_rounds = kMode == 0 ? 1 : max(1, (n + kRoundRows - 1) / kRoundRows);
  // two-CTA-per-SM mode with several rounds (a few units, large k): every round's pre-existing source
  // rows are resolved before the dependency wait (own src_row area per round) and the rows of rounds
  // >= 1 are prefetched into L2, so a later round costs one L2 gather instead of index + block-table
  // + HBM round trips after the previous round's compute
  const bool early = !kStream && n_rounds > 1 && n_rounds <= DCfg::kRowRounds;
  auto round_src = [&](int round) { return early ? src_row + round * kRoundRows : src_row; };
  auto round_pad = [&](int round) { return (min(kRoundRows, n - round * kRoundRows) + 15) & ~15; };
  {  // round 0, pre-existing rows: independent of the previous kernel
    const int rows0 = (min(kRoundRows, n) + 15) & ~15;
    resolve(0, rows0, true, src_row);
    if (early)
      for (int rd = 1; rd < n_rounds; ++rd) resolve(rd * kRoundRows, round_pad(rd), true, round_src(rd));
    if (tid == 0) mbar_expect_tx(gbar, static_cast<uint32_t>(rows0) * 512u);  // round 0: K + V, 256 B each
    __syncthreads();
    gather(0, rows0, true, 0, src_row, false);
    if (early)  // later rounds' rows into L2 (measured: k = 4096, 8.85 -> 8.75 us per launch)
      for (int rd = 1; rd < n_rounds; ++rd) {
        const int64_t* sr = round_src(rd);
        const int rp = round_pad(rd);
        for (int i = tid; i < 2 * rp; i += nthr) {
          const int64_t row = sr[i >> 1];
          if (row >= 0 && is_pre(v_begin + rd * kRoundRows + (i >> 1)))
            prefetch_l2_bulk(((i & 1) ? p.cache.v : p.cache.k) + row * 128, 256);
        }
      }
  }
  pdl_wait();  // previous layer complete: q and this step's new row are valid
  pdl_launch_dependents();
  dtrace(p, 1);
  // post-wait rows of round 0: this step's new row (straight from k_new/v_new, one warp, no
  // barrier) — its round trip overlaps the query loads below; the general path only when earlier
  // steps' rows may still be in flight (a one-layer chain)
  const int rows0_pad = (min(kRoundRows, n) + 15) & ~15;
  // this step's new row, one 16-byte chunk per lane of the last warp (K: lanes 0-15, V: 16-31),
  // staged in shared memory until its round's gather has landed (its TMA slot is zero-filled)
  const bool has_new = p.k_new && warp == nwarps - 1 && new_v >= v_begin && new_v < v_end;
  const int new_round = (new_v - v_begin) / kRoundRows;
  if (has_new) {
    cp_async_16(smem + DCfg::kOffNew + lane * 16,
                (lane < 16 ? p.k_new : p.v_new) + (static_cast<size_t>(b) * p.Hkv + g) * 128 + (lane & 15) * 8, 16);
    cp_async_commit();
  }
  if (!old_tail_ready) {
    __syncthreads();  // src_row of the pre pass consumed by every thread
    resolve(0, rows0_pad, false, src_row);
    __syncthreads();
    gather(0, rows0_pad, false, 0, src_row, false);
  }
  // streaming mode: the sequence's block table staged in shared memory and each thread's T entry of
  // the next round loaded one round ahead, so resolving a round's source rows costs no dependent
  // global round trip between two rounds' compute
  int* bt_s = reinterpret_cast<int*>(smem + DCfg::kOffBt);
  const int n_pages_seq = ((p0 + tail) >> p.cache.page_shift) + 1;
  const bool bt_smem = kStream && n_pages_seq <= DCfg::kBtMax;
  int tq = 0;
  if (kStream) {
    if (bt_smem)
      for (int i = tid; i < n_pages_seq; i += nthr)
        bt_s[i] = __ldg(p.cache.block_table + static_cast<int64_t>(seq) * p.cache.max_pages_per_seq + i);
    const int v2 = v_begin + kRoundRows + tid;
    if (tid < kRoundRows && v2 < min(v_end, k)) tq = __ldg(T + v2);
  }
  long long cyc[4] = {0, 0, 0, 0};  // dev timing of warp 0's first step (trace knob)
  DraftWarp<kPack> w;
  w.init(p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * 128, p.G, lane);
#ifdef SA_PIPE_TRACE
  if (p.trace) {  // dev: stamp 10 once this thread's query fragments have landed
    asm volatile("" ::"r"(w.qb[7][1]), "r"(w.qb[0][0]));
    dtrace(p, 10);
  }
#endif
  const bool dbuf = kStream && n_rounds > 1;  // double-buffered rounds (streaming mode)
  auto issue_round = [&](int round, int buf) {  // every row of a later round (after the wait)
    const int rr0 = round * kRoundRows;
    const int rp = (min(kRoundRows, n - rr0) + 15) & ~15;
    __syncthreads();  // buffer `buf` and src_row free
    int64_t* sr = round_src(round);
    if (kStream) {
      if (tid < rp) {
        const int v = v_begin + rr0 + tid;
        int64_t row = -2;
        if (v < v_end) {
          const int pos = v < k ? tq : p0 + (v - k);
          if (p.k_new && pos == new_pos) {
            row = -1;
          } else {
            const int page = bt_smem ? bt_s[pos >> p.cache.page_shift]
                                     : __ldg(p.cache.block_table + static_cast<int64_t>(seq) * p.cache.max_pages_per_seq +
                                             (pos >> p.cache.page_shift));
            row = ((((int64_t)p.layer * p.cache.num_pages + page) * p.cache.n_kv_heads + g) << p.cache.page_shift) +
                  (pos & ((1 << p.cache.page_shift) - 1));
          }
        }
        sr[tid] = row;
      }
      const int v2 = v_begin + rr0 + kRoundRows + tid;  // the next round's T entry, one round ahead
      tq = (tid < kRoundRows && v2 < min(v_end, k)) ? __ldg(T + v2) : 0;
    } else {
      if (!early) resolve(rr0, rp, true, sr);
      resolve(rr0, rp, false, sr);
    }
    if (tid == 0) mbar_expect_tx(gbar + buf, static_cast<uint32_t>(rp) * 512u);
    __syncthreads();
    fence_proxy_async_smem();  // the buffer's previous round, read by ldmatrix, before the async-proxy writes
    gather(rr0, rp, true, buf, sr, true);
  };
  if (dbuf) issue_round(1, 1);
  for (int round = 0; round < n_rounds; ++round) {
    const int r0 = round * kRoundRows;
    const int rows = min(kRoundRows, n - r0);
    const int rows_pad = (rows + 15) & ~15;
    const int buf = dbuf ? (round & 1) : 0;
    if (!dbuf && round > 0) issue_round(round, 0);
    mbar_wait(gbar + buf, dbuf ? ((round >> 1) & 1) : (round & 1));  // this round landed (the next in flight)
    if (has_new && new_round == round) {
      const int r = new_v - v_begin - r0;
      const uint32_t off = (r >> 6) * DCfg::kTileBytes + swz(r & 63, lane & 15, DCfg::kHalf);
      cp_async_wait_all();  // each lane reads back its own chunk
      *reinterpret_cast<uint4*>((buf ? smem + DCfg::kOffBuf1 : smem) + (lane < 16 ? 0 : DCfg::kOffV) + off) =
          *reinterpret_cast<const uint4*>(smem + DCfg::kOffNew + lane * 16);
    }
    __syncthreads();
    dtrace(p, 2);
    const int n_sub = rows_pad >> 4;
    // warp w takes sub-blocks w, w + nwarps, ...; two at a time in one softmax step
    const uint32_t kb = smem_u32(buf ? smem + DCfg::kOffBuf1 : smem), vb = kb + DCfg::kOffV;
    for (int sb = warp; sb < n_sub; sb += 2 * nwarps) {
      const int sb2 = sb + nwarps;
      const int nv0 = min(16, n - (r0 + sb * 16));
      if (sb2 < n_sub) {
        const uint32_t ks[2] = {kb + (sb >> 2) * DCfg::kTileBytes, kb + (sb2 >> 2) * DCfg::kTileBytes};
        const uint32_t vs[2] = {vb + (sb >> 2) * DCfg::kTileBytes, vb + (sb2 >> 2) * DCfg::kTileBytes};
        const int rr[2] = {(sb & 3) * 16, (sb2 & 3) * 16};
        const int nv[2] = {nv0, min(16, n - (r0 + sb2 * 16))};
#ifdef SA_PIPE_TRACE  // dev build: warp 0's step phases in cycles (tools/trace_draft.py)
        w.step<2>(ks, vs, DCfg::kHalf, rr, lane, p.scale_log2, nv, (p.trace && tid == 0) ? cyc : nullptr);
#else
        w.step<2>(ks, vs, DCfg::kHalf, rr, lane, p.scale_log2, nv);
#endif
      } else {
        const uint32_t ks[1] = {kb + (sb >> 2) * DCfg::kTileBytes};
        const uint32_t vs[1] = {vb + (sb >> 2) * DCfg::kTileBytes};
        const int rr[1] = {(sb & 3) * 16};
        const int nv[1] = {nv0};
        w.step<1>(ks, vs, DCfg::kHalf, rr, lane, p.scale_log2, nv);
      }
    }
    if (dbuf && round + 2 < n_rounds) issue_round(round + 2, buf);
  }
  w.finalize();
  dtrace(p, 3);
#ifdef SA_PIPE_TRACE
  if (p.trace && tid == 0 && warp == 0) {  // dev: step<2> phases of warp 0 in cycles -> slots 11-13
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const size_t launch = static_cast<size_t>((p.step - 1) & 7) * 64 + (p.layer & 63);
    if (cta < 512)
      for (int k2 = 0; k2 < 3; ++k2) p.trace[(launch * 512 + cta) * 16 + 11 + k2] = cyc[k2 + 1] - cyc[k2];
  }
#endif

  // in-CTA merge of the warps' partials (only the G real query rows), fused with the push: every
  // warp stores its raw O fragments and (m, l); after one barrier each thread rescales the warps'
  // float4 groups of its output to the CTA-wide row max, sums them in warp order (deterministic)
  // and pushes the result straight into the owner's inbox with st.async; the first thread of each
  // row also pushes the row's (m*, l*).
  constexpr int kWs = 132;  // padded row stride of a warp partial (floats): conflict-free stores
  float* wps = reinterpret_cast<float*>(smem);             // [nwarps][G][kWs] raw partials
  float* wml = reinterpret_cast<float*>(smem + DCfg::kOffRow);  // [kMaxWarps][16]: m[8], l[8]
  __syncthreads();  // every warp done reading K/V tiles (wps aliases them) and src_row
  dtrace(p, 8);
  const int gid = lane >> 2, t4 = lane & 3;
  {
    float* wp = wps + warp * (p.G * kWs);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int row = 2 * t4 + e;
      if (row < p.G) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          wp[row * kWs + 16 * jj + gid] = w.o[jj][e];
          wp[row * kWs + 16 * jj + gid + 8] = w.o[jj][2 + e];
        }
        if (gid == 0) {
          wml[warp * 16 + row] = w.m[e];
          wml[warp * 16 + 8 + row] = w.l[e];
        }
      }
    }
  }
  __syncthreads();
  dtrace(p, 5);
  cluster_wait_acquire();  // every owner's inbox barrier is initialised
  // a one-CTA "cluster" (streaming mode, cs = 1) writes its inbox with plain shared stores: st.async
  // needs a real cluster (compute-sanitizer memcheck)
  const bool solo = CS == 1;
  if (tid == 0 && !solo) {
    const int my_vals = my_hi - my_lo;
    mbar_arrive_expect_tx(inbox_bar, static_cast<uint32_t>(CS) * (my_vals + 2 * p.G) * 4u);
  }
  const uint32_t inbox_addr = smem_u32(inbox), bar_addr = smem_u32(inbox_bar);
  // the CTA's per-row (m*, l*) to every owner, by the last warp: lane 8*r + q holds warp q's (m, l) of
  // row base + r; three xor levels give the row max and the rescaled sum (fixed tree order:
  // deterministic), then lane 8*r + j pushes the (m*, l*) pair of its row to owners j and j + 8
  if (warp == nwarps - 1) {
    for (int base = 0; base < p.G; base += 4) {
      const int row = base + (lane >> 3), q = lane & 7;
      const bool ok = row < p.G && q < nwarps;
      const float mq = ok ? wml[q * 16 + row] : -INFINITY;
      float ms = mq;
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, off));
      float ls = (ok && mq != -INFINITY) ? wml[q * 16 + 8 + row] * fast_exp2(mq - ms) : 0.f;
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
      if (row < p.G && solo && q == 0) {
        inbox[per + 2 * row] = ms;
        inbox[per + 2 * row + 1] = ls;
      } else if (row < p.G && !solo) {
        for (int o = q; o < CS; o += 8)
          st_async_v2(mapa_shared(inbox_addr + (split * rstride + per + 2 * row) * 4, o), ms, ls,
                      mapa_shared(bar_addr, o));
      }
    }
  }
  for (int q4 = tid; q4 < n_out / 4; q4 += nthr) {
    const int e = q4 * 4, row = e >> 7, col = e & 127;
    float mq[DCfg::kMaxWarps];
#pragma unroll
    for (int q = 0; q < DCfg::kMaxWarps; ++q) mq[q] = q < nwarps ? wml[q * 16 + row] : -INFINITY;
    float mstar = -INFINITY;
#pragma unroll
    for (int q = 0; q < DCfg::kMaxWarps; ++q) mstar = fmaxf(mstar, mq[q]);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < DCfg::kMaxWarps; ++q) {  // fixed warp order: deterministic
      if (q < nwarps) {
        const float f = mq[q] == -INFINITY ? 0.f : fast_exp2(mq[q] - mstar);
        const float4 x = *reinterpret_cast<const float4*>(wps + (q * p.G + row) * kWs + col);
        v.x += x.x * f;
        v.y += x.y * f;
        v.z += x.z * f;
        v.w += x.w * f;
      }
    }
    const int owner = e / per;
    if (solo)
      *reinterpret_cast<float4*>(inbox + e) = v;
    else
      st_async_v4(mapa_shared(inbox_addr + (split * rstride + (e - owner * per)) * 4, owner), v,
                  mapa_shared(bar_addr, owner));
  }
  // fused append of this step's provisional row (KvStore::append, kv_store.cpp:39-45), off the
  // critical path: this launch reads the row from k_new / v_new; later steps of this layer gather it
  // from the cache either before their own dependency wait (launches >= L back, complete) or after it
  if (blockIdx.x == gridDim.x - 1 && p.k_new && tid < 32) {
    const int which = tid >> 4, ch = tid & 15;
    const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + (static_cast<size_t>(b) * p.Hkv + g) * 128;
    const int64_t row = cache_row(p.cache, seq, p.layer, g, new_pos);
    __nv_bfloat16* dst = (which ? p.cache.v : p.cache.k) + row * 128;
    reinterpret_cast<uint4*>(dst)[ch] = __ldg(reinterpret_cast<const uint4*>(src) + ch);
  }
  // combine my slice once every sender's contribution has landed
  dtrace(p, 6);
  if (solo)
    __syncthreads();
  else
    mbar_wait_cluster(inbox_bar, 0);
  dtrace(p, 7);
  float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * 128;
  // two-level merge (n_sub clusters per unit): each cluster's owner r stores its merged slice
  // (unnormalised, relative to the slice rows' max) and the (m, l) of its rows; the last of the
  // unit's n_sub owners of slice r to arrive combines them in cluster order (deterministic)
  const size_t ubase = (static_cast<size_t>(b) * p.Hkv + g) * n_sub;
  float* lvl_o = p.part_o + ubase * n_out;                       // [unit][sub][G*128]
  float* lvl_ml = p.part_ml + (ubase * CS + split) * 16;         // [unit][sub][CS][8 rows][2]
  const size_t lvl_ml_sub = static_cast<size_t>(CS) * 16;
  for (int e = my_lo + tid; e < my_hi; e += nthr) {
    const int row = e >> 7, off = e - my_lo;
    float ms[DCfg::kMaxCS], ls[DCfg::kMaxCS], os[DCfg::kMaxCS];  // all inbox loads in flight together
#pragma unroll
    for (int s2 = 0; s2 < DCfg::kMaxCS; ++s2) {
      const bool ok = s2 < CS;
      ms[s2] = ok ? inbox[s2 * rstride + per + 2 * row] : -INFINITY;
      ls[s2] = ok ? inbox[s2 * rstride + per + 2 * row + 1] : 0.f;
      os[s2] = ok ? inbox[s2 * rstride + off] : 0.f;
    }
    float mstar = -INFINITY;
#pragma unroll
    for (int s2 = 0; s2 < DCfg::kMaxCS; ++s2) mstar = fmaxf(mstar, ms[s2]);
    float acc = 0.f, lsum = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < DCfg::kMaxCS; ++s2) {
      const float f = ms[s2] == -INFINITY ? 0.f : fast_exp2(ms[s2] - mstar);
      acc += os[s2] * f;
      lsum += ls[s2] * f;
    }
    if (n_sub == 1) {
      out_unit[e] = acc / lsum;
    } else {
      lvl_o[static_cast<size_t>(sub) * n_out + e] = acc;
      if (e == my_lo || (e & 127) == 0) {
        lvl_ml[sub * lvl_ml_sub + 2 * row] = mstar;
        lvl_ml[sub * lvl_ml_sub + 2 * row + 1] = lsum;
      }
    }
  }
  if (n_sub > 1) {
    int* cnt = p.counters + (static_cast<size_t>(b) * p.Hkv + g) * DCfg::kMaxCS + split;
    __syncthreads();
    int prev = 0;
    if (tid == 0) {
      __threadfence();
      prev = atomicAdd(cnt, 1);
    }
    if (!__syncthreads_or(tid == 0 && prev == n_sub - 1)) return;
    __threadfence();
    for (int e = my_lo + tid; e < my_hi; e += nthr) {
      const int row = e >> 7;
      float mstar = -INFINITY;
      for (int s2 = 0; s2 < n_sub; ++s2) mstar = fmaxf(mstar, __ldcg(lvl_ml + s2 * lvl_ml_sub + 2 * row));
      float acc = 0.f, lsum = 0.f;
      for (int s2 = 0; s2 < n_sub; ++s2) {  // cluster order: deterministic
        const float m2 = __ldcg(lvl_ml + s2 * lvl_ml_sub + 2 * row);
        const float f = m2 == -INFINITY ? 0.f : fast_exp2(m2 - mstar);
        acc += __ldcg(lvl_o + static_cast<size_t>(s2) * n_out + e) * f;
        lsum += __ldcg(lvl_ml + s2 * lvl_ml_sub + 2 * row + 1) * f;
      }
      out_unit[e] = acc / lsum;
    }
    if (tid == 0) *cnt = 0;  // re-armed for the next launch (which reads it after its dependency wait)
  }
  dtrace(p, 4);
}

template <int kMode, bool kPack>
static cudaError_t draft_set_attrs_one() {
  constexpr bool kStream = kMode == 2;
  cudaError_t e = cudaFuncSetAttribute(draft_kernel<kMode, kPack>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kStream ? DCfg::kSmemStream : DCfg::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(draft_kernel<kMode, kPack>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

static cudaError_t draft_set_attrs() {
  static std::atomic<uint64_t> attr_mask{0};
  int dev = 0;
  if (func_attrs_needed(attr_mask, &dev)) {
    cudaError_t e = draft_set_attrs_one<0, false>();
    if (e == cudaSuccess) e = draft_set_attrs_one<0, true>();
    if (e == cudaSuccess) e = draft_set_attrs_one<1, false>();
    if (e == cudaSuccess) e = draft_set_attrs_one<1, true>();
    if (e == cudaSuccess) e = draft_set_attrs_one<2, false>();
    if (e == cudaSuccess) e = draft_set_attrs_one<2, true>();
    if (e != cudaSuccess) return e;
    func_attrs_done(attr_mask, dev);
  }
  return cudaSuccess;
}

// How many clusters of `cs` CTAs (full 8-warp blocks) the device runs at once in the given mode:
// clusters must fit inside one GPC, so on 148 SMs e.g. eight 16-CTA clusters of the one-CTA-per-SM
// streaming mode do NOT all fit and a second wave would follow.  Cached per (device, mode, cs).
int draft_max_active_clusters(int stream, int cs) {
  static std::mutex mu;
  static std::map<int, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  const int key = (dev * 2 + (stream ? 1 : 0)) * 64 + cs;
  std::lock_guard<std::mutex> lk(mu);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  int n = 0;
  if (draft_set_attrs() == cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(DCfg::kMaxThreads);
    cfg.dynamicSmemBytes = stream ? DCfg::kSmemStream : DCfg::kSmem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if ((stream ? cudaOccupancyMaxActiveClusters(&n, draft_kernel<2, false>, &cfg)
                : cudaOccupancyMaxActiveClusters(&n, draft_kernel<1, false>, &cfg)) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
  }
  memo[key] = n;
  return n;
}

cudaError_t launch_draft(const DraftParams& p, cudaStream_t s) {
  if (cudaError_t e = draft_set_attrs()) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_splits * p.n_sub, p.Hkv, p.B);
  // one warp per 16-row sub-block of the CTA's chunk (<= 9 warps, two CTAs per SM)
  cfg.blockDim = dim3(32 * std::min(DCfg::kMaxWarps, std::max(1, (std::min(p.chunk, DCfg::kMaxTiles * DCfg::kTile) + 15) / 16)));
  cfg.dynamicSmemBytes = p.stream ? DCfg::kSmemStream : DCfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[3];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = p.n_splits;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  // spread: the CTAs of a cluster on distinct SMs (the default policy packs two CTAs of one launch on
  // an SM when a GPC hosts two clusters, and those CTAs compute ~1 us slower: the launch's straggler)
  attrs[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
  attrs[1].val.clusterSchedulingPolicyPreference = static_cast<cudaClusterSchedulingPolicy>(p.cluster_policy);
  attrs[2].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[2].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = p.use_pdl ? 3 : 2;
  const bool pack = p.G <= 4;  // P_hi | P_mid share one n8 tile (DraftWarp<true>)
  if (p.stream)
    return pack ? cudaLaunchKernelEx(&cfg, draft_kernel<2, true>, p) : cudaLaunchKernelEx(&cfg, draft_kernel<2, false>, p);
  if (p.chunk <= DCfg::kMaxTiles * DCfg::kTile)  // one round per CTA
    return pack ? cudaLaunchKernelEx(&cfg, draft_kernel<0, true>, p) : cudaLaunchKernelEx(&cfg, draft_kernel<0, false>, p);
  return pack ? cudaLaunchKernelEx(&cfg, draft_kernel<1, true>, p) : cudaLaunchKernelEx(&cfg, draft_kernel<1, false>, p);
}

int draft_max_splits() { return DCfg::kMaxCS; }
int draft_round_rows() { return DCfg::kMaxTiles * DCfg::kTile; }

}  // namespace sa
