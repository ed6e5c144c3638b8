// Dev check: tcgen05.mma with the A operand in TMEM (staged from a SWIZZLE_128B smem tile with
// tcgen05.cp.128x256b) gives the same D as A read from shared memory.  M=128, N=32, K=128 (8 steps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_a tools/microbench/tmem_a.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {  // SW128 K-major: LBO 16, SBO 1024
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) | (static_cast<uint64_t>(64) << 32) |
         (uint64_t{1} << 46) | (uint64_t{2} << 61);
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ uint32_t swz(int row, int chunk, uint32_t half_bytes) {
  return (chunk >> 3) * half_bytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

// A: [128 tok][128 dim] bf16 (global, row-major), B: [32 rows][128 dim]; out: D[128][32] twice
__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* Bm, float* out_smem, float* out_tmem) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t{1023});
  uint8_t* sa = s;            // 2 halves x [128][128 B]
  uint8_t* sb = s + 32768;    // 2 halves x [32][128 B]
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 16; i += 128) {  // 16-byte chunks
    const int r = i >> 4, c = i & 15;
    *reinterpret_cast<uint4*>(sa + swz(r, c, 128 * 128)) = reinterpret_cast<const uint4*>(A + r * 128)[c];
  }
  for (int i = tid; i < 32 * 16; i += 128) {
    const int r = i >> 4, c = i & 15;
    *reinterpret_cast<uint4*>(sb + swz(r, c, 32 * 128)) = reinterpret_cast<const uint4*>(Bm + r * 128)[c];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;  // cols [0,32): D smem-A, [32,64): D tmem-A, [64,128): A staged
  if (tid == 0) {
    const uint32_t a = su32(sa), b = su32(sb);
    for (int kk = 0; kk < 8; ++kk) {  // stage A into TMEM: 8 columns (16 bf16) per K step
      const uint64_t ad = desc(a + (kk >> 2) * 16384 + (kk & 3) * 32);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 64 + kk * 8), "l"(ad) : "memory");
    }
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t ad = desc(a + (kk >> 2) * 16384 + (kk & 3) * 32);
      const uint64_t bd = desc(b + (kk >> 2) * 4096 + (kk & 3) * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(ad), "l"(bd),
                   "r"(idesc(32)), "r"(kk > 0 ? 1 : 0)
                   : "memory");
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 32),
                   "r"(tm + 64 + kk * 8), "l"(bd), "r"(idesc(32)), "r"(kk > 0 ? 1 : 0)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 64; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + ((warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (c < 32) out_smem[row * 32 + c] = __uint_as_float(v);
    else out_tmem[row * 32 + c - 32] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
  const int M = 128, N = 32, K = 128;
  __nv_bfloat16 *hA = new __nv_bfloat16[M * K], *hB = new __nv_bfloat16[N * K];
  float* ref = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k2 = 0; k2 < K; ++k2) acc += (double)__bfloat162float(hA[m * K + k2]) * __bfloat162float(hB[n * K + k2]);
      ref[m * N + n] = (float)acc;
    }
  __nv_bfloat16 *dA, *dB;
  float *d1, *d2;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&d1, M * N * 4);
  cudaMalloc(&d2, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 48 * 1024>>>(dA, dB, d1, d2);
  cudaError_t e = cudaDeviceSynchronize();
  float* h1 = new float[M * N];
  float* h2 = new float[M * N];
  cudaMemcpy(h1, d1, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, d2, M * N * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < M * N; ++i) {
    e1 = fmax(e1, fabs(h1[i] - ref[i]));
    e2 = fmax(e2, fabs(h2[i] - ref[i]));
  }
  printf("err=%s  max|D_smemA - ref| = %g   max|D_tmemA - ref| = %g   (D[0][0..3] tmem: %g %g %g %g ref %g %g %g %g)\n",
         cudaGetErrorString(e), e1, e2, h2[0], h2[1], h2[2], h2[3], ref[0], ref[1], ref[2], ref[3]);
  return 0;
}
