// Dev microbenchmark: TMA streaming bandwidth on B200 for the verify kernel's access patterns.
//   mode 0: 2-D tensor map over [rows][128] bf16 (256 B pitch), two 64-col SWIZZLE_128B boxes per
//           128-row tile (the current verify layout: each box reads 128 B of every 256 B row)
//   mode 1: same bytes, tensor map over [rows*2][64] (128 B pitch): each box is 16 KB contiguous
//   mode 2: 1-D cp.async.bulk of 32 KB contiguous per tile
// Each CTA streams `tiles` consecutive 32 KB tiles through a `stages`-deep ring; consumers only
// wait and release.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_stream tools/microbench/tma_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                   su32(dst)),
               "l"(m), "r"(su32(bar)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

constexpr int kTileBytes = 32768;

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap m0,
                                                         const __grid_constant__ CUtensorMap m1, const char* base,
                                                         int mode, int tiles_per_cta, int stages, int64_t total_tiles, int64_t off_tiles,
                                                         unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kTileBytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tiles_per_cta;
  if (threadIdx.x == 0) {
    for (int i = 0; i < tiles_per_cta; ++i) {
      const int s = i % stages;
      if (i >= stages) wait(&empty[s], ((i / stages) - 1) & 1);
      char* dst = smem + s * kTileBytes;
      const int64_t tile = (off_tiles + t0 + i) % total_tiles;
      expect_tx(&full[s], kTileBytes);
      if (mode == 0) {
        const int row = static_cast<int>(tile * 128);
        tma2d(dst, &m0, &full[s], 0, row);
        tma2d(dst + 16384, &m0, &full[s], 64, row);
      } else if (mode == 1) {
        const int row = static_cast<int>(tile * 256);
        tma2d(dst, &m1, &full[s], 0, row);
        tma2d(dst + 16384, &m1, &full[s], 0, row + 128);
      } else {
        bulk1d(dst, base + tile * kTileBytes, kTileBytes, &full[s]);
      }
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < tiles_per_cta; ++i) {
      const int s = i % stages;
      wait(&full[s], (i / stages) & 1);
      acc += reinterpret_cast<const unsigned long long*>(smem + s * kTileBytes)[i & 7];
      arrive(&empty[s]);
    }
    if (acc == 0x12345) sink[0] = acc;
  }
}

static CUtensorMap make_map(void* base, uint64_t inner, uint64_t rows, uint64_t pitch) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", r);
  return m;
}

int main() {
  const int64_t bytes = 4LL << 30;  // 4 GiB buffer (32 x a config-2 layer): no L2 reuse
  const int64_t total_tiles = bytes / kTileBytes;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  CUtensorMap m0 = make_map(buf, 128, bytes / 256, 256), m1 = make_map(buf, 64, bytes / 128, 128);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int ctas : {144, 148}) {
    for (int stages : {2, 5, 6}) {
      for (int mode = 0; mode < 3; ++mode) {
        const int tiles_per_cta = static_cast<int>((134LL << 20) / kTileBytes / ctas);  // ~one layer per launch
        const size_t sm = stages * kTileBytes + 2 * stages * 8;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int iters = 20;
        const int64_t per_launch = static_cast<int64_t>(ctas) * tiles_per_cta;
        for (int w = 0; w < 3; ++w)
          stream_kernel<<<ctas, 128, sm>>>(m0, m1, buf, mode, tiles_per_cta, stages, total_tiles, w * per_launch, sink);
        cudaEventRecord(a);
        for (int it = 0; it < iters; ++it)  // successive launches walk through the 4 GiB buffer
          stream_kernel<<<ctas, 128, sm>>>(m0, m1, buf, mode, tiles_per_cta, stages, total_tiles,
                                           (it + 3) * per_launch, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double gb = static_cast<double>(ctas) * tiles_per_cta * kTileBytes * iters / 1e9;
        printf("ctas %d stages %d mode %d: %.1f GB/s (%.2f us per launch)  err=%s\n", ctas, stages, mode,
               gb / (ms / 1e3), ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
