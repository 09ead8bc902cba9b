// Probe: how fast can one SM push bytes out to global memory (L2), and how does that scale
// with the number of SMs doing it at once?  Each CTA (one per SM, `nsm` CTAs) writes
// `rounds` x 64 KB from its shared memory to its own region of a global buffer by
//   mode 0: cp.async.bulk (1-D bulk copy smem -> global), 4 KB per op
//   mode 1: cp.reduce.async.bulk .add.f32 (1-D bulk reduce-add), 4 KB per op
//   mode 2: st.global.v4 from registers, fully coalesced (512 B per warp instruction)
//   mode 3: cp.async.bulk, 16 KB per op
//   mode 4: the other direction for comparison: cp.async.bulk global -> smem, 4 KB per op,
//           64 KB in flight per round (mbarrier complete_tx)
// and times the store phase with clock64 (issue of the first op .. all ops complete).
// Reports bytes per SM clock per SM and the aggregate GB/s.  Regions are L2-resident when
// nsm x rounds x 64 KB fits (it does for the sizes used), so this measures the SM -> L2 path.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256, 1) k(float* out, int rounds, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(128) float s[];
  const int n = 64 * 1024 / 4;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = 1.0f + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  float* region = out + static_cast<size_t>(blockIdx.x) * rounds * n;
  const uint32_t sbase = smem_u32(s);
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (mode == 2) {
    const float4* src = reinterpret_cast<const float4*>(s);
    for (int r = 0; r < rounds; ++r) {
      float4* dst = reinterpret_cast<float4*>(region + static_cast<size_t>(r) * n);
#pragma unroll 4
      for (int i = threadIdx.x; i < n / 4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
  } else if (mode == 4) {
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = smem_u32(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int r = 0; r < rounds; ++r) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(64 * 1024) : "memory");
        for (int c = 0; c < 16; ++c) {
          const char* g = reinterpret_cast<const char*>(region + static_cast<size_t>(r) * n) + c * 4096;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(sbase + c * 4096), "l"(g), "r"(4096), "r"(b) : "memory");
        }
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(b), "r"(r & 1) : "memory");
      }
    }
  } else if (threadIdx.x < 32) {
    const int chunk = mode == 3 ? 16384 : 4096;
    const int per_warp = 64 * 1024 / chunk / 1;   // warp 0 issues everything
    if (threadIdx.x == 0) {
      for (int r = 0; r < rounds; ++r)
        for (int c = 0; c < per_warp; ++c) {
          char* g = reinterpret_cast<char*>(region + static_cast<size_t>(r) * n) + c * chunk;
          const uint32_t sa = sbase + c * chunk;
          if (mode == 1)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                         :: "l"(g), "r"(sa), "r"(chunk) : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(g), "r"(sa), "r"(chunk) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int smem = 64 * 1024 + 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // rounds per CTA: 8 (148 x 512 KB = 74 MB, L2-resident) or more from argv[1] (e.g. 64:
  // 606 MB, so every line of a pass was evicted since the previous one: DRAM-resident)
  const int rounds = argc > 1 ? atoi(argv[1]) : 8;
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, static_cast<size_t>(sms) * rounds * 64 * 1024);
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"bulk copy 4KB", "bulk reduce-add f32 4KB", "st.global.v4 (256 thr)", "bulk copy 16KB",
                         "bulk LOAD 4KB (64KB/round)"};
  for (int mode : {0, 1, 2, 3, 4})
    for (int nsm : {1, 8, 37, 74, 148}) {
      for (int w = 0; w < 2; ++w) k<<<nsm, 256, smem>>>(out, rounds, mode, cyc);
      cudaEventRecord(e0);
      const int reps = 5;
      for (int w = 0; w < reps; ++w) k<<<nsm, 256, smem>>>(out, rounds, mode, cyc);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> h(nsm);
      cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      const double bytes = rounds * 64.0 * 1024;
      printf("%-26s nsm %3d: median %.1f B/clk/SM (min %.1f, max %.1f), kernel %.2f us, aggregate %.0f GB/s\n",
             names[mode], nsm, bytes / h[nsm / 2], bytes / h[nsm - 1], bytes / h[0], ms * 1000 / reps,
             nsm * bytes / (ms * 1e-3 / reps) / 1e9);
    }
  return 0;
}
