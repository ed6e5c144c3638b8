// Dev: how many thread-block clusters of size c fit at once (cudaOccupancyMaxActiveClusters) for a
// one-CTA-per-SM kernel (200 KB dynamic shared memory, 384 threads) and a two-CTA-per-SM one (100 KB).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1() {}
int main() {
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k1, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {200 * 1024, 100 * 1024}) {
    printf("smem %d KB:", smem / 1024);
    for (int c = 1; c <= 16; ++c) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(c, 1, 1);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = c;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      cfg.attrs = &a;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k1, &cfg);
      printf(" %d:%d%s", c, n, e ? "!" : "");
    }
    printf("\n");
  }
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d\n", pr.multiProcessorCount);
  return 0;
}
