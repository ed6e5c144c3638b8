// Dev microbenchmark: cost of an MMA-issuer style loop over already-complete mbarriers
// (try_wait + tcgen05.fence + tcgen05.commit), alone and with other warps parked in try_wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mbar_loop tools/microbench/mbar_loop.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)),
               "r"(ph)
               : "memory");
}

__global__ void k(int mode, unsigned long long* out) {
  __shared__ uint64_t bars[16];
  __shared__ uint64_t never;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&never)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[i])) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0) {
      unsigned long long t0 = gt();
      for (int it = 0; it < 16; ++it) {
        wait(&bars[it], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (mode & 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&never))
                       : "memory");
      }
      unsigned long long t1 = gt();
      out[blockIdx.x] = t1 - t0;
      if (mode & 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&never)) : "memory");
    }
    __syncwarp();
  } else if ((mode & 2) && warp >= 2) {
    wait(&never, 0);  // parked until warp 1 releases it
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  for (int mode = 0; mode < 4; ++mode) {
    k<<<148, 192>>>(mode, d);
    k<<<148, 192>>>(mode, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("mode %d (commit=%d parked_warps=%d): 16 iterations %.1f ns avg  err=%s\n", mode, mode & 1, (mode >> 1) & 1,
           s / 148.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
