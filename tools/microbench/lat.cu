// Dev microbenchmark: dependent-chain latencies on B200 (cycles): mma.sync m16n8k16 bf16, shfl,
// ldmatrix, ex2.approx, LDS.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc) {
  __shared__ __align__(16) unsigned short sm[4096];
  for (int i = threadIdx.x; i < 4096; i += 32) sm[i] = 0x3c00;
  __syncwarp();
  float d[4] = {0, 0, 0, 0};
  unsigned a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u}, b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  long long t1 = clock64();
  float x = d[0];
  for (int i = 0; i < 256; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0f;
  long long t2 = clock64();
  unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 7) * 16;
  unsigned r0 = 0, r1, r2, r3;
  for (int i = 0; i < 256; ++i) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr + (r0 & 16)));
  }
  long long t3 = clock64();
  float y = x;
  for (int i = 0; i < 256; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y));
  long long t4 = clock64();
  unsigned v = threadIdx.x;
  const unsigned* s32 = reinterpret_cast<const unsigned*>(sm);
  for (int i = 0; i < 256; ++i) v = s32[(v & 7) + (i & 1)];
  long long t5 = clock64();
  out[threadIdx.x] = d[0] + x + r0 + r1 + r2 + r3 + y + v;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256; cyc[4] = (t5 - t4) / 256;
  }
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c); k<<<1, 32>>>(o, c); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("latency cycles: mma.sync.m16n8k16 %lld  shfl+fadd %lld  ldmatrix.x4 %lld  ex2 %lld  lds %lld\n", h[0], h[1], h[2], h[3], h[4]);
}
