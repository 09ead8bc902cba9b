// Probe: max co-resident clusters for cluster sizes 1..16 at 1 CTA/SM (200 KB smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d L2 %d bytes\n", sms, l2);
  for (int cs : {1, 2, 3, 4, 6, 8, 16}) {
    cudaLaunchConfig_t lc = {}; cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    lc.gridDim = dim3(cs * 64); lc.blockDim = dim3(256); lc.dynamicSmemBytes = 200 * 1024; lc.attrs = a; lc.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &lc);
    printf("cluster %2d: max active clusters %d -> %d SMs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
}
