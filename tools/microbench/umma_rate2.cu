// Dev microbenchmark (round 2): tcgen05.mma (kind::f16, M=128, K=16) issue throughput when issued the
// way a production kernel should: warp 0 converged, one elect.sync-ed lane, 8 MMAs per asm block with
// descriptors advanced by immediates (no per-MMA R2UR of freshly computed registers).  Compare with
// umma_rate.cu (a divergent lane-0 loop, ~78 ns per MMA whatever N).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/umma_rate2 tools/microbench/umma_rate2.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) | (static_cast<uint64_t>(64) << 32) |
         (uint64_t{1} << 46) | (uint64_t{2} << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (8u << 24);
}

// 8 MMAs into accumulator columns [acc, acc+n) (accumulate), K steps of 32 bytes along the swizzled row
#define MMA8(ACC, AD, BD, ID)                                                                        \
  asm volatile(                                                                                      \
      "{\n\t.reg .pred e;\n\t.reg .b64 a, b;\n\t"                                                   \
      "elect.sync _|e, 0xffffffff;\n\t"                                                              \
      "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t"                                                         \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"                                 \
      "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"                                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t}" ::"r"(ACC),                  \
      "l"(AD), "l"(BD), "r"(ID)                                                                      \
      : "memory")

__global__ void k(int n, int iters, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t{1023});
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (warp == 0) {
    const uint64_t a = desc(su32(s)), b = desc(su32(s + 32768));
    const uint32_t id = idesc(n);
    __syncwarp();
    const unsigned long long t0 = gt();
    for (int i = 0; i < iters; i += 8) {
      const uint32_t acc = tm + ((i >> 3) % nacc) * n;
      MMA8(acc, a, b, id);
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
        : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(&bar))
                 : "memory");
    const unsigned long long t1 = gt();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  unsigned long long h[148];
  for (int n : {8, 16, 32, 48, 64, 128, 256})
    for (int nacc : {1, 2}) {
      if (n * nacc > 512) continue;
      const int iters = 4096;
      k<<<148, 128, 80 * 1024>>>(n, iters, nacc, d);
      k<<<148, 128, 80 * 1024>>>(n, iters, nacc, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double sum = 0;
      for (int i = 0; i < 148; ++i) sum += h[i];
      const double ns = sum / 148 / iters;
      printf("elect+unrolled N=%3d nacc=%d: %.2f ns per MMA (M128 K16) -> %.1f TFLOP/s chip  err=%s\n", n, nacc, ns,
             2.0 * 128 * 16 * n * 148 / ns / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
