// Dev microbenchmark: %globaltimer update granularity vs clock64 on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int n = 0;
  long long c0 = clock64();
  while (n < 64) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[n++] = t - prev; prev = t; }
  }
  out[64] = clock64() - c0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 65 * 8);
  k<<<1, 1>>>(d); cudaDeviceSynchronize();
  unsigned long long h[65]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("globaltimer increments (ns):"); for (int i = 0; i < 64; ++i) printf(" %llu", h[i]);
  printf("\ncycles for 64 increments: %llu\n", h[64]);
}
