// Dev probe: TMA tile::gather4 semantics on B200 (sm_100a) for the draft's row gather.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/g4 gather4_probe.cu -lcuda
// A [1024][128] bf16 tensor (element = row * 128 + col, as a 16-bit pattern) is read with
// gather4 (4 arbitrary rows x 64 columns, SWIZZLE_128B) into rows 4..7 of a 64-row tile half at a
// 512-byte (not 1024-byte) aligned shared address; the probe checks every element against the
// draft's swizzled layout (off = half + r * 128 + ((chunk ^ (r & 7)) * 16)), an out-of-range row
// index (zero fill), and a negative one, for tensor-map boxes {64, 1} and {64, 4}.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

__global__ void probe(const __grid_constant__ CUtensorMap m, uint16_t* out, int r0, int r1, int r2, int r3, int* tx) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0xdeadbeefu;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * 512));
    for (int h = 0; h < 2; ++h) {
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem + h * 8192 + 4 * 128));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(h * 64), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
          : "memory");
    }
  }
  uint32_t done = 0;
  long long spins = 0;
  while (!done && spins < (1ll << 24)) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(b));
    ++spins;
  }
  if (threadIdx.x == 0) *tx = done ? 1 : 0;
  __syncthreads();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(smem)[i];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int R = 1024;
  uint16_t* h = new uint16_t[R * 128];
  for (int i = 0; i < R * 128; ++i) h[i] = static_cast<uint16_t>(i & 0xffff);
  uint16_t *d, *o;
  int* tx;
  cudaMalloc(&d, R * 128 * 2);
  cudaMalloc(&o, 16384);
  cudaMalloc(&tx, 4);
  cudaMemcpy(d, h, R * 128 * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
  const int rows[4] = {5, 900, 1500 /* out of range */, 17};
  for (int box_rows : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {64, %d}: encode %d\n", box_rows, static_cast<int>(r));
    if (r != CUDA_SUCCESS) continue;
    for (int neg = 0; neg < 2; ++neg) {
      const int rr2 = neg ? -3 : rows[2];
      cudaMemset(tx, 0, 4);
      probe<<<1, 128, 16384>>>(m, o, rows[0], rows[1], rr2, rows[3], tx);
      cudaError_t e = cudaDeviceSynchronize();
      uint16_t out[8192];
      int htx = 0;
      cudaMemcpy(out, o, 16384, cudaMemcpyDeviceToHost);
      cudaMemcpy(&htx, tx, 4, cudaMemcpyDeviceToHost);
      int bad = 0, zero_ok = 1, untouched = 0;
      for (int slot = 0; slot < 4; ++slot) {
        const int rr = 4 + slot;
        for (int col = 0; col < 128; ++col) {
          const int chunk = (col & 63) >> 3;
          const int off = (col >= 64 ? 8192 : 0) + rr * 128 + ((chunk ^ (rr & 7)) * 16) + (col & 7) * 2;
          const uint16_t got = out[off / 2];
          if (slot == 2) {
            if (got != 0) zero_ok = 0;
          } else {
            const uint16_t want = static_cast<uint16_t>((rows[slot] * 128 + col) & 0xffff);
            if (got != want) ++bad;
          }
        }
      }
      for (int i = 0; i < 8192; ++i) {
        const int byte = i * 2, hoff = byte % 8192, row = hoff / 128;
        if (row < 4 || row >= 8) untouched += out[i] == 0xbeef || out[i] == 0xdead ? 0 : 1;
      }
      printf("  row2=%d: err=%s complete=%d mismatches=%d zero_fill_ok=%d writes_outside_rows_4_7=%d\n", rr2,
             cudaGetErrorString(e), htx, bad, zero_ok, untouched);
    }
  }
  return 0;
}
