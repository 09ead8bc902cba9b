// Probe: a persistent 1-CTA/SM grid launched with cluster dim 2 and the Blackwell "preferred
// substitute cluster" dim 4 (cudaLaunchAttributePreferredClusterDimension).  Per CTA: blockIdx,
// %cluster_nctarank, %cluster_ctarank, %clusterid.x, %smid and its start time, so we learn
//  * how many CTAs run in 4-CTA clusters and how many in 2-CTA ones,
//  * whether a 4-CTA cluster is always blocks 4i..4i+3 with ctarank == blockIdx % 4,
//  * whether the whole grid is co-resident (start times within a few us).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(int* out, unsigned long long* t) {
  extern __shared__ int s[];
  uint32_t n, r, cid, sm;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) {
    t[blockIdx.x] = gtime();
    out[4 * blockIdx.x + 0] = n;
    out[4 * blockIdx.x + 1] = r;
    out[4 * blockIdx.x + 2] = cid;
    out[4 * blockIdx.x + 3] = sm;
    s[0] = sm;
    const uint64_t t0 = gtime();
    while (gtime() - t0 < 200000) {}
  }
  asm volatile("barrier.cluster.arrive; barrier.cluster.wait;" ::: "memory");
}
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d; unsigned long long* dt;
  cudaMalloc(&d, 4 * sizeof(int) * sms); cudaMalloc(&dt, sizeof(unsigned long long) * sms);
  for (int rep = 0; rep < 3; ++rep) {
    cudaLaunchConfig_t lc = {}; cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributePreferredClusterDimension; a[1].val.preferredClusterDim.x = 4;
    a[1].val.preferredClusterDim.y = 1; a[1].val.preferredClusterDim.z = 1;
    lc.gridDim = dim3(sms); lc.blockDim = dim3(128); lc.dynamicSmemBytes = smem; lc.attrs = a; lc.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&lc, k, d, dt);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    int h[4 * 160]; unsigned long long ht[160];
    cudaMemcpy(h, d, 4 * sizeof(int) * sms, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht, dt, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    int n4 = 0, n2 = 0, misaligned = 0;
    unsigned long long tmin = ~0ull, tmax = 0;
    for (int b = 0; b < sms; ++b) {
      if (h[4 * b] == 4) ++n4; else if (h[4 * b] == 2) ++n2;
      if (h[4 * b + 1] != b % h[4 * b]) ++misaligned;
      if (ht[b] < tmin) tmin = ht[b];
      if (ht[b] > tmax) tmax = ht[b];
    }
    printf("rep %d: CTAs in 4-clusters %d, in 2-clusters %d, ctarank != blockIdx %% n: %d, start spread %.1f us\n",
           rep, n4, n2, misaligned, (tmax - tmin) / 1e3);
    if (rep == 0)
      for (int b = 0; b < sms; ++b)
        printf("  blk %3d n %d rank %d cid %3d sm %3d dt %.1f\n", b, h[4 * b], h[4 * b + 1], h[4 * b + 2], h[4 * b + 3],
               (ht[b] - tmin) / 1e3);
  }
  return 0;
}
