// Dev microbenchmark: issue cadence of back-to-back tcgen05.mma (kind::f16, M=128, K=16, A and B from
// SWIZZLE_128B smem tiles) for several N, with rotating TMEM accumulators, one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/umma_rate tools/microbench/umma_rate.cu
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
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (8u << 24);
}

__global__ void k(int n, int iters, int nacc, int a_tmem, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t{1023});
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0x3c003c00u;
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
    unsigned long long t0 = 0;
    if (lane == 0) {
      const uint32_t a = su32(s), b = su32(s + 16384);
      t0 = gt();
      for (int i = 0; i < iters; ++i) {
        const int kk = i & 3;
        const uint32_t acc = (i % nacc) * n;
        if (a_tmem)  // A from TMEM columns [384, 512) (garbage contents: timing only)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + acc),
              "r"(tm + 384 + kk * 8), "l"(desc(b + kk * 32)), "r"(idesc(n)), "r"(i >= nacc ? 1 : 0)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + acc),
              "l"(desc(a + kk * 32)), "l"(desc(b + kk * 32)), "r"(idesc(n)), "r"(i >= nacc ? 1 : 0)
              : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                       su32(&bar))
                   : "memory");
      out[blockIdx.x] = gt() - t0;
    }
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  unsigned long long h[148];
  for (int at = 0; at < 2; ++at)
  for (int n : {16, 32, 64, 128, 256})
    for (int nacc : {1, 4}) {
      if (n * nacc > (at ? 384 : 512)) continue;
      const int iters = 256;
      k<<<148, 128, 64 * 1024>>>(n, iters, nacc, at, d);
      k<<<148, 128, 64 * 1024>>>(n, iters, nacc, at, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double sum = 0;
      for (int i = 0; i < 148; ++i) sum += h[i];
      const double ns = sum / 148 / iters;
      printf("A=%s N=%3d nacc=%d: %.1f ns per MMA (M128 K16) -> %.2f TFLOP/s chip  err=%s\n", at ? "tmem" : "smem", n, nacc, ns,
             2.0 * 128 * 16 * n * 148 / ns / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
