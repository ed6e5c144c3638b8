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
// Grid: (splits, heads) with the splits of one head forming a thread-block cluster over d_model
// (split-K, ~148 CTAs streaming at once); the partial tiles are reduced in a fixed order through
// DSMEM (deterministic), each CTA of the cluster finishing a slice of the tokens: scale, RoPE,
// bf16, store.  Weight tiles are streamed before griddepcontrol.wait (they do not depend on the
// previous kernel), so under PDL the weight stream overlaps the previous kernel's tail.
#include <cmath>

#include "internal.h"

struct sa_qkv {
  int L = 0, Hq = 0, Hkv = 0, D = 0, n_out = 0, nkb = 0, style = 0;
  float eps = 1e-5f;
  double theta = 10000.0;
  const __nv_bfloat16* w = nullptr;  // [L][n_out][D] (caller-owned device memory)
  const float* gain = nullptr;       // [L][D]
  __nv_bfloat16* xbuf = nullptr;     // [nkb][N][64] hi/lo token planes (N <= 256)
  float* rbuf = nullptr;             // [128] 1/rms per token
  CUtensorMap tmap_w{}, tmap_x{};
  int device = 0, num_sms = 148;
};

namespace sa {

constexpr int kQkvMaxTokens = 128;
constexpr int kQkvThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int kQkvSmem = 200 * 1024;
constexpr int kWTile = 128 * 64 * 2;  // 16 KB weight tile (128 output features x 64 of d_model)

struct QkvParams {
  int layer, n_out, nkb, n_tok, rows, NT, N, Hq, Hkv, splits, style;
  float eps;
  double log2_theta;
  const __nv_bfloat16* w;
  const float* x;
  const float* gain;
  const int32_t* pos0;
  __nv_bfloat16* xbuf;
  float* rbuf;
  __nv_bfloat16* q;
  __nv_bfloat16* k_new;
  __nv_bfloat16* v_new;
};

// One CTA per padded token row: 1/rms and the hi/lo planes of x * gain in the TMA tile layout.
__global__ void __launch_bounds__(256) qkv_prepare(QkvParams p) {
  pdl_wait();  // x is the previous kernel's output; the previous projection's xbuf reads are done
  const int t = blockIdx.x, tid = threadIdx.x;
  const int D = p.nkb * 64;
  const float* xr = p.x + static_cast<size_t>(t) * D;
  const float* g = p.gain + static_cast<size_t>(p.layer) * D;
  const bool live = t < p.n_tok;
  double ss = 0.0;
  for (int k = tid * 2; k < D; k += 512) {
    uint32_t hi2 = 0, lo2 = 0;
    if (live) {
      const float2 xv = *reinterpret_cast<const float2*>(xr + k);
      const float2 gv = *reinterpret_cast<const float2*>(g + k);
      ss += static_cast<double>(xv.x) * xv.x + static_cast<double>(xv.y) * xv.y;
      split_bf16(xv.x * gv.x, xv.y * gv.y, hi2, lo2);
    }
    __nv_bfloat16* dst = p.xbuf + (static_cast<size_t>(k >> 6) * p.N + t) * 64 + (k & 63);
    *reinterpret_cast<uint32_t*>(dst) = hi2;
    *reinterpret_cast<uint32_t*>(dst + static_cast<size_t>(p.NT) * 64) = lo2;
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
  __syncthreads();
  pdl_launch_dependents();
}

__global__ void __launch_bounds__(kQkvThreads, 1) qkv_gemm(const __grid_constant__ CUtensorMap tmw,
                                                            const __grid_constant__ CUtensorMap tmx, QkvParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x, head = blockIdx.y;
  const int N = p.N, NT = p.NT;
  const uint32_t stage_bytes = kWTile + N * 128;
  const int ring = kQkvSmem - 1024 - 256;
  const int S = min(8, static_cast<int>(ring / stage_bytes));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ring);
  uint64_t* empty = full + 8;
  uint64_t* acc_bar = empty + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_bar + 1);
  float* part = reinterpret_cast<float*>(smem);                   // [N][128] (after the mainloop)
  float* fin = part + static_cast<size_t>(N) * 128;               // [slice][128]
  const int kb0 = split * p.nkb / p.splits, kb1 = (split + 1) * p.nkb / p.splits, nk = kb1 - kb0;
  const uint32_t tcols = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_bar, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmw);
    tma_prefetch_desc(&tmx);
  }
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      const uint64_t pol = policy_evict_first(), pol_x = policy_evict_last();
      const int wrow = p.layer * p.n_out + head * 128;
      const int pre = min(S, nk);
      for (int it = 0; it < pre; ++it) {  // weights do not depend on the previous kernel
        mbar_expect_tx(&full[it], stage_bytes);
        tma_load_2d(smem + it * stage_bytes, &tmw, &full[it], (kb0 + it) * 64, wrow, pol);
      }
      pdl_wait();
      auto load_x = [&](int it, int st) {
        uint8_t* dst = smem + st * stage_bytes + kWTile;
        for (int r = 0; r < N; r += 16) tma_load_2d(dst + r * 128, &tmx, &full[st], 0, (kb0 + it) * N + r, pol_x);
      };
      for (int it = 0; it < pre; ++it) load_x(it, it);
      for (int it = pre; it < nk; ++it) {
        const int st = it % S;
        mbar_wait(&empty[st], ((it / S) - 1) & 1);
        mbar_expect_tx(&full[st], stage_bytes);
        tma_load_2d(smem + st * stage_bytes, &tmw, &full[st], (kb0 + it) * 64, wrow, pol);
        load_x(it, st);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      const uint32_t idesc = umma_idesc_bf16(N, 0, 0);
      for (int it = 0; it < nk; ++it) {
        const int st = it % S;
        mbar_wait(&full[st], (it / S) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem + st * stage_bytes), b_base = a_base + kWTile;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, umma_desc(a_base + kk * 32, 16, 1024, kLayoutSW128),
                    umma_desc(b_base + kk * 32, 16, 1024, kLayoutSW128), idesc, (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[st]);
      }
      umma_commit(acc_bar);
    }
    __syncwarp();
  } else {  // ------------------------------------------------------------ epilogue, warps 2-5
    pdl_wait();  // 1/rms (rbuf) and the positions are read below
    const int quarter = warp & 3, row = quarter * 32 + lane;
    mbar_wait(acc_bar, 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c, v);
      tc_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) part[(c + j) * 128 + row] = v[j];
    }
  }
  tc_fence_before();
  cluster_sync_all();  // every split's partial tile is in its shared memory

  const int t0 = split * p.n_tok / p.splits, t1 = (split + 1) * p.n_tok / p.splits;
  if (warp >= 2) {
    const int row = (warp & 3) * 32 + lane;
    const uint32_t part_addr = smem_u32(part);
    for (int t = t0; t < t1; ++t) {
      float hi = 0.f, lo = 0.f;
      for (int c = 0; c < p.splits; ++c) {  // fixed order over the splits: deterministic
        const uint32_t base = mapa_shared(part_addr, c);
        hi += ld_dsmem_f32(base + (t * 128 + row) * 4);
        lo += ld_dsmem_f32(base + ((NT + t) * 128 + row) * 4);
      }
      fin[(t - t0) * 128 + row] = (hi + lo) * p.rbuf[t];
    }
    named_bar_sync(1, 128);
    const int kind = head < p.Hq ? 0 : head < p.Hq + p.Hkv ? 1 : 2;  // q / k / v head
    int pair, partner;
    if (p.style == 0) {  // half-split (rotate_half): (i, i+64)
      pair = row & 63;
      partner = row ^ 64;
    } else {  // interleaved (RoFormer): (2j, 2j+1)
      pair = row >> 1;
      partner = row ^ 1;
    }
    const bool first = p.style == 0 ? row < 64 : (row & 1) == 0;
    const double inv_freq = exp2(-p.log2_theta * (2.0 * pair) / 128.0);
    for (int t = t0; t < t1; ++t) {
      const int b = t / p.rows, r = t - b * p.rows;
      float y = fin[(t - t0) * 128 + row];
      if (kind < 2) {
        const double ang = static_cast<double>(p.pos0[b] + r) * inv_freq;
        const float cs = static_cast<float>(cos(ang)), sn = static_cast<float>(sin(ang));
        const float yp = fin[(t - t0) * 128 + partner];
        y = first ? __fsub_rn(__fmul_rn(y, cs), __fmul_rn(yp, sn)) : __fadd_rn(__fmul_rn(y, cs), __fmul_rn(yp, sn));
      }
      const __nv_bfloat16 o = __float2bfloat16_rn(y);
      if (kind == 0)
        p.q[((static_cast<size_t>(b) * p.Hq + head) * p.rows + r) * 128 + row] = o;
      else
        (kind == 1 ? p.k_new : p.v_new)[((static_cast<size_t>(b) * p.rows + r) * p.Hkv + head - p.Hq -
                                         (kind == 2 ? p.Hkv : 0)) * 128 + row] = o;
    }
  }
  __syncthreads();
  pdl_launch_dependents();
  cluster_sync_all();  // peers have finished reading this CTA's partial tile
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
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
  h->w = static_cast<const __nv_bfloat16*>(w_qkv);
  h->gain = attn_norm_gain;
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  cudaError_t e = cudaMalloc(&h->xbuf, static_cast<size_t>(h->nkb) * 2 * sa::kQkvMaxTokens * 64 * 2);
  if (e == cudaSuccess) e = cudaMalloc(&h->rbuf, sa::kQkvMaxTokens * sizeof(float));
  if (e != cudaSuccess) {
    sa_qkv_destroy(h);
    return sa::cuda_fail(e, "qkv buffers");
  }
  std::string err;
  if (!sa::encode_tensor_map_2d(&h->tmap_w, const_cast<__nv_bfloat16*>(h->w), static_cast<uint64_t>(d_model),
                                static_cast<uint64_t>(n_layers) * h->n_out, 128, &err) ||
      !sa::encode_tensor_map_2d(&h->tmap_x, h->xbuf, 64, static_cast<uint64_t>(h->nkb) * 2 * sa::kQkvMaxTokens, 16,
                                &err)) {
    sa_qkv_destroy(h);
    return sa::fail(SA_CUDA_ERROR, err);
  }
  *out = h;
  return SA_OK;
}

SA_API sa_status sa_qkv_destroy(sa_qkv* h) {
  if (!h) return SA_OK;
  cudaFree(h->xbuf);
  cudaFree(h->rbuf);
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
  p.splits = std::max(1, std::min({h->num_sms / heads, 8, h->nkb}));
  p.style = h->style;
  p.eps = h->eps;
  p.log2_theta = std::log2(h->theta);
  p.w = h->w;
  p.x = x;
  p.gain = h->gain;
  p.pos0 = positions;
  p.xbuf = h->xbuf;
  p.rbuf = h->rbuf;
  p.q = static_cast<__nv_bfloat16*>(q);
  p.k_new = static_cast<__nv_bfloat16*>(k_new);
  p.v_new = static_cast<__nv_bfloat16*>(v_new);
  // the epilogue overlays [N][128] partials + the token slice on the (drained) stage ring
  const int slice = (p.n_tok + p.splits - 1) / p.splits;
  if ((p.N + slice) * 128 * 4 > sa::kQkvSmem - 1024 - 256) return sa::fail(SA_INVALID_ARGUMENT, "qkv: too many tokens");
  auto s = static_cast<cudaStream_t>(stream);
  static bool attr_set = false;
  if (!attr_set) {
    SA_CUDA_CHECK(cudaFuncSetAttribute(sa::qkv_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, sa::kQkvSmem));
    attr_set = true;
  }
  cudaLaunchAttribute pdl[2];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t c1{};
  c1.gridDim = dim3(p.NT);
  c1.blockDim = dim3(256);
  c1.stream = s;
  c1.attrs = pdl;
  c1.numAttrs = 1;
  SA_CUDA_CHECK(cudaLaunchKernelEx(&c1, sa::qkv_prepare, p));
  pdl[1].id = cudaLaunchAttributeClusterDimension;
  pdl[1].val.clusterDim.x = p.splits;
  pdl[1].val.clusterDim.y = 1;
  pdl[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t c2{};
  c2.gridDim = dim3(p.splits, heads);
  c2.blockDim = dim3(sa::kQkvThreads);
  c2.dynamicSmemBytes = sa::kQkvSmem;
  c2.stream = s;
  c2.attrs = pdl;
  c2.numAttrs = 2;
  SA_CUDA_CHECK(cudaLaunchKernelEx(&c2, sa::qkv_gemm, h->tmap_w, h->tmap_x, p));
  return SA_OK;
}

}  // extern "C"
