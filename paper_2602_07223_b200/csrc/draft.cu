// draft.cu — sparse draft attention: index gather fused with attention (+ fused KV append).
//
// Reference: KvStore::gather (kv_store.cpp:67-88) followed by attend (attention.cpp:70-76) over
// [K_T ; K_tail], the SPEC draft-forward key set T ∪ {positions >= draft window start}
// (SPEC.md:385,447).  The reference materialises the gathered K/V copies; here each CTA
// gathers its slice of the virtual key list straight into shared memory with 16-byte cp.async
// (warp-coalesced: 16 lanes per 256-byte row) in the same swizzled layout the TMA path produces,
// then runs the shared mma.sync flash step for the G q-heads of the KV head (one 16-row tile).
//
// Grid (n_splits, Hkv, B): split s covers virtual keys [s*chunk, (s+1)*chunk) of
// T[0..k) ++ [p0, p0+step); the last-arriving CTA merges the splits.
#include "attn_core.cuh"
#include "internal.h"

namespace sa {

struct DCfg {
  static constexpr int kTile = 64;
  static constexpr int kMaxTiles = 2;  // chunk <= 128 keys per CTA
  static constexpr int kThreads = 128;
  static constexpr int kHalf = kTile * 128;
  static constexpr int kTileBytes = 2 * kHalf;
  static constexpr int kOffV = kMaxTiles * kTileBytes;
  static constexpr int kOffQ = 2 * kMaxTiles * kTileBytes;
  static constexpr int kQHalf = 16 * 128;
  static constexpr int kOffMisc = kOffQ + 2 * kQHalf;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static constexpr int kMaxSplits = 192;
  static_assert(4 * kWpFloats * 4 <= kOffQ && kMaxSplits * 16 * 8 <= kOffQ, "epilogue scratch must fit");
};

__global__ void __launch_bounds__(DCfg::kThreads) draft_kernel(const DraftParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  int* misc = reinterpret_cast<int*>(smem + DCfg::kOffMisc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int seq = p.seq_ids[b];
  const int p0 = p.p0[b];
  const int j = p.step;
  const int set = p.n_sets == 1 ? 0 : g;
  const int k = p.k_act[b * p.n_sets + set];
  const int32_t* T = p.idx + (static_cast<size_t>(b) * p.n_sets + set) * p.k_cap;
  const int m_total = k + j;
  const int v_begin = split * p.chunk;
  const int v_end = min(m_total, v_begin + p.chunk);
  const int n = max(0, v_end - v_begin);
  const int n_tiles = ceil_div(n, DCfg::kTile);
  const int Hq = p.Hkv * p.G;
  const int new_pos = p0 + j - 1;

  // Gather K/V rows of the virtual key list into swizzled smem tiles (zero-fill past the end).
  for (int i = tid; i < n_tiles * DCfg::kTile * 16; i += DCfg::kThreads) {
    const int r = i >> 4, ch = i & 15, tile = r >> 6, rr = r & 63;
    const uint32_t off = tile * DCfg::kTileBytes + swz(rr, ch, DCfg::kHalf);
    const int v = v_begin + r;
    const __nv_bfloat16 *sk = p.cache.k, *sv = p.cache.v;
    int bytes = 0;
    if (v < v_end) {
      const int pos = v < k ? __ldg(T + v) : p0 + (v - k);
      if (p.k_new && pos == new_pos) {
        sk = p.k_new + (static_cast<size_t>(b) * p.Hkv + g) * 128 + ch * 8;
        sv = p.v_new + (static_cast<size_t>(b) * p.Hkv + g) * 128 + ch * 8;
      } else {
        const int64_t row = cache_row(p.cache, seq, p.layer, g, pos);
        sk = p.cache.k + row * 128 + ch * 8;
        sv = p.cache.v + row * 128 + ch * 8;
      }
      bytes = 16;
    }
    cp_async_16(smem + off, sk, bytes);
    cp_async_16(smem + DCfg::kOffV + off, sv, bytes);
  }
  cp_async_commit();
  // Q rows of the G heads (one 16-row tile, zero-padded).
  uint8_t* sq = smem + DCfg::kOffQ;
  const __nv_bfloat16* qb = p.q + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * 128;
  for (int i = tid; i < 16 * 16; i += DCfg::kThreads) {
    const int row = i >> 4, ch = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < p.G) v = __ldg(reinterpret_cast<const uint4*>(qb + row * 128 + ch * 8));
    *reinterpret_cast<uint4*>(sq + swz(row, ch, DCfg::kQHalf)) = v;
  }
  // Fused append of this step's provisional row (KvStore::append, kv_store.cpp:39-45).
  if (split == 0 && p.k_new && tid < 32) {
    const int which = tid >> 4, ch = tid & 15;
    const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + (static_cast<size_t>(b) * p.Hkv + g) * 128;
    const int64_t row = cache_row(p.cache, seq, p.layer, g, new_pos);
    __nv_bfloat16* dst = (which ? p.cache.v : p.cache.k) + row * 128;
    reinterpret_cast<uint4*>(dst)[ch] = __ldg(reinterpret_cast<const uint4*>(src) + ch);
  }
  cp_async_wait_all();
  __syncthreads();

  WarpAttn w;
  w.init();
  w.load_q(smem_u32(sq), DCfg::kQHalf, 0, lane);
  const int t4 = lane & 3;
  for (int t = 0; t < n_tiles; ++t) {
    const uint32_t kt = smem_u32(smem + t * DCfg::kTileBytes);
    const uint32_t vt = smem_u32(smem + DCfg::kOffV + t * DCfg::kTileBytes);
    const int r0 = warp * 16;
    if (t * DCfg::kTile + r0 >= n) break;
    float s[2][4];
    w.qk(kt, DCfg::kHalf, r0, lane, s);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (t * DCfg::kTile + r0 + 8 * nt + 2 * t4 + (e & 1) >= n) s[nt][e] = -INFINITY;
    w.softmax_pv(s, vt, DCfg::kHalf, r0, lane, p.scale_log2);
  }
  w.finalize_l();

  __syncthreads();
  float* wps = reinterpret_cast<float*>(smem);
  store_warp_partial(w, wps + warp * kWpFloats, lane);
  __syncthreads();
  const int unit = b * p.Hkv + g;
  float* po = p.part_o + static_cast<size_t>(unit) * p.n_splits * 16 * 128;
  float* pml = p.part_ml + static_cast<size_t>(unit) * p.n_splits * 16 * 2;
  cta_partial_to_global<1, 4>(wps, po + static_cast<size_t>(split) * 16 * 128,
                              pml + static_cast<size_t>(split) * 16 * 2, tid, DCfg::kThreads);
  float* out_unit = p.out + (static_cast<size_t>(b) * Hq + static_cast<size_t>(g) * p.G) * 128;
  combine_splits(po, pml, p.n_splits, 16, p.G, p.counters + unit, misc, wps, tid, DCfg::kThreads, 1,
                 [&](int row) { return out_unit + static_cast<size_t>(row) * 128; });
}

cudaError_t launch_draft(const DraftParams& p, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(draft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DCfg::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(p.n_splits, p.Hkv, p.B);
  draft_kernel<<<grid, DCfg::kThreads, DCfg::kSmem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace sa
