// Probe (diagnostic, not a product component): does an SM see each L2 line at a "near" or
// "far" latency, and does repeated access from a far SM make a line near (a copy in the
// requester's die)?  One CTA per SM; thread 0 times dependent ld.global.cg loads (L2, not L1)
// of NADDR lines, 2 KB apart, with clock64, several passes after a warm-up pass.
//   out: per SM (by %smid): the minimum latency per address over the passes, and the
//   latency of the first and the last pass, so a line that turns near after the first far
//   access shows up as first >> last.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/probe_l2_dies.cu -o probe_l2_dies
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int NADDR = 64;
constexpr int PASSES = 8;

__global__ void probe(const uint32_t* __restrict__ buf, uint32_t* lat_first, uint32_t* lat_last, uint32_t* lat_min,
                      int* smid_of_block) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x != 0) return;
  smid_of_block[blockIdx.x] = static_cast<int>(smid);
  // the chain: buf[i * 512] holds the index of the next line (stride 2 KB); a dependent chain
  // keeps one load in flight, so each timed load is one L2 round trip
  uint32_t mins[NADDR];
  for (int a = 0; a < NADDR; ++a) mins[a] = 0xffffffffu;
  uint32_t idx = 0;
  for (int pass = 0; pass <= PASSES; ++pass) {
    for (int a = 0; a < NADDR; ++a) {
      const uint32_t* p = buf + static_cast<size_t>(a) * 512;
      long long t0, t1;
      uint32_t v;
      // (asm volatile statements keep their order; the add waits for the load on the
      // scoreboard, and the clock read issues after it)
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
      asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p + (idx & 1)) : "memory");
      asm volatile("add.u32 %0, %0, %1;" : "+r"(idx) : "r"(v) : "memory");
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
      const uint32_t dt = static_cast<uint32_t>(t1 - t0);
      if (pass == 1) lat_first[smid * NADDR + a] = dt;
      if (pass == PASSES) lat_last[smid * NADDR + a] = dt;
      if (pass >= 1 && dt < mins[a]) mins[a] = dt;
    }
  }
  for (int a = 0; a < NADDR; ++a) lat_min[smid * NADDR + a] = mins[a] + (idx == 0xdeadbeefu);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* buf;
  cudaMalloc(&buf, NADDR * 2048);
  cudaMemset(buf, 0, NADDR * 2048);
  uint32_t *lf, *ll, *lm;
  int* sm_of;
  const size_t n = static_cast<size_t>(256) * NADDR;
  cudaMalloc(&lf, n * 4); cudaMalloc(&ll, n * 4); cudaMalloc(&lm, n * 4); cudaMalloc(&sm_of, 1024 * 4);
  cudaMemset(lm, 0, n * 4);
  // one block per SM: tiny blocks would pile several on one SM, so ask for most of the smem
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<sms, 32, 200 * 1024>>>(buf, lf, ll, lm, sm_of);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<uint32_t> hf(n), hl(n), hm(n);
  cudaMemcpy(hf.data(), lf, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hl.data(), ll, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hm.data(), lm, n * 4, cudaMemcpyDeviceToHost);
  printf("# sms %d naddr %d passes %d: per SM: min latency per address (cycles)\n", sms, NADDR, PASSES);
  for (int s = 0; s < 256; ++s) {
    if (hm[s * NADDR] == 0) continue;
    printf("sm %3d min:", s);
    for (int a = 0; a < NADDR; ++a) printf(" %u", hm[s * NADDR + a]);
    printf("\nsm %3d first:", s);
    for (int a = 0; a < NADDR; ++a) printf(" %u", hf[s * NADDR + a]);
    printf("\nsm %3d last:", s);
    for (int a = 0; a < NADDR; ++a) printf(" %u", hl[s * NADDR + a]);
    printf("\n");
  }
  return 0;
}
