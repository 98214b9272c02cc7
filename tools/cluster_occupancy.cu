// Max co-resident clusters per cluster size for a 1-CTA/SM kernel (~226 KB smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
  const int smem = 226 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c = 1; c <= 16; ++c) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c * 64); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = smem; cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
