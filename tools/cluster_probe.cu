// Resident clusters per width for a 512-thread, one-CTA-per-SM kernel
// (cudaOccupancyMaxActiveClusters), the constraint the select's cluster width
// is chosen against.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl = 1; cl <= 16; ++cl) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cl, 1);
    lc.blockDim = dim3(512);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    lc.attrs = a; lc.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &lc);
    printf("cluster %2d: %3d resident clusters = %3d CTAs (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
  return 0;
}
