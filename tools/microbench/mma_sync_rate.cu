// Dev microbenchmark: legacy mma.sync.m16n8k16 (bf16 -> f32) on B200: dependent-chain latency and
// per-SM issue throughput with W warps per CTA (one CTA per SM, 148 CTAs), 8 independent
// accumulator chains per warp.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/msr mma_sync_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void rate(float* out, long long* cyc, int iters) {
  float d[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  unsigned a0 = 0x3c003c00u ^ threadIdx.x, a1 = 0x3c003c00u, a2 = 0x3c003c00u, a3 = 0x3c003c00u;
  unsigned b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CHAINS>
void run(int warps, int iters) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  rate<CHAINS><<<148, 32 * warps>>>(out, cyc, iters);
  rate<CHAINS><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double mmas = static_cast<double>(iters) * CHAINS * warps;
  printf("warps/SM %2d chains %d: %7.2f cycles per MMA per warp (latency if 1 chain), SM rate %.3f MMA/cycle "
         "(%.0f FLOP/cycle/SM)  err=%s\n",
         warps, CHAINS, avg / (static_cast<double>(iters) * CHAINS), mmas / avg, mmas / avg * 4096.0,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1, 4096);
  run<2>(1, 2048);
  run<4>(1, 1024);
  run<8>(1, 512);
  run<8>(4, 512);
  run<8>(8, 512);
  run<8>(16, 512);
  run<4>(32, 512);
  return 0;
}
