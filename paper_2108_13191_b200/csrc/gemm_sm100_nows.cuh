// gemm_sm100_nows.cuh -- ABLATION ONLY (the paper's fig:gradual-opts P:951-965):
// the same C[M][N] += A[M][K] . B[K][N] with NO warp specialisation, for the ablation row
// "non-warp-specialised" (option warp_specialize = -1).  Never picked by the product.
//
// Structure (the Ampere-era design of the paper's Algorithm 1, Sec. 3.5
// and Sec. 3.9, transcribed to tcgen05/TMA without the B200-specific split of roles):
//   * one 128 x 128 C tile per CTA, non-persistent grid (one thread block per tile);
//   * ONE thread runs the k-loop as a multistage software pipeline (ring_stages - 1 k-blocks
//     in flight): at k-block kb it refills the stage k-block kb - 1 used once kb - 1's MMAs
//     have read it, waits for kb's data and issues kb's MMAs -- loads, MMAs and their
//     completions are serialised in one instruction stream;
//   * the epilogue starts after the mainloop (no overlap with the next tile's MMAs): every
//     thread reads one accumulator row from TMEM, adds C_in loaded straight from global
//     memory and stores its row with plain element stores (no TMA, no smem staging).
// K-chunk promotion into F32 registers as in gemm_sm100.cuh (R4), so results stay
// within the F32 bar at any K.
#pragma once
#include <cuda_fp16.h>
#include "gemm_sm100.cuh"

namespace g16 {

struct NwsCfg {
  static constexpr int BM = 128, BN = 128, BK = 64, UMMA_K = 16;
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = BM * BK * 2;          // 16 KB
  static constexpr int B_ATOM_BYTES = 64 * BK * 2;     // 8 KB: 64 columns x 64 k
  static constexpr int B_BYTES = BN * BK * 2;          // 16 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_BAR = STAGES * STAGE_BYTES;
  static constexpr int NBAR = 2 * STAGES + 1;          // full[S], empty[S], acc_full
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static constexpr int THREADS = 128;
  static constexpr int TMEM_COLS = 128;
};

template <bool OUT_F16>
__global__ void __launch_bounds__(128, 1)
gemm_f16_sm100_nows_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                           const __grid_constant__ CUtensorMap /*tm_c: unused, plain stores*/,
                           const __grid_constant__ GemmParams p, const __grid_constant__ PeerMaps /*unused*/,
                           const __grid_constant__ CUtensorMap /*unused*/) {
  using Cfg = NwsCfg;
  constexpr int BK = Cfg::BK;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base + Cfg::OFF_A, sB = base + Cfg::OFF_B;
  const uint32_t bar0 = base + Cfg::OFF_BAR;
  const uint32_t full_bar = bar0, empty_bar = bar0 + 8 * Cfg::STAGES, accf_bar = bar0 + 16 * Cfg::STAGES;
  const uint32_t tmem_slot = bar0 + 8 * Cfg::NBAR;
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int RS = p.ring_stages;
  if (threadIdx.x == 0) {
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    mbar_init(accf_bar, 1);
    fence_mbarrier_init();
  }
  if (warp == 0) tmem_alloc<1>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");
  griddep_wait();

  const int tm = static_cast<int>(blockIdx.x) / p.tiles_n, tn = static_cast<int>(blockIdx.x) % p.tiles_n;
  const int KB = p.k_blocks;
  const uint64_t pol = policy_evict_normal();
  const uint32_t idesc = idesc_f16_f32acc<128, 128>() | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
  auto load = [&](int kb) {   // (thread 0) k-block kb into stage kb % RS
    const int s = kb % RS;
    mbar_arrive_expect_tx(full_bar + 8 * s, Cfg::STAGE_BYTES);
    tma_load_2d_hint(sA + s * Cfg::A_BYTES, &tm_a, kb * BK, tm * Cfg::BM, full_bar + 8 * s, pol);
    for (int h = 0; h < Cfg::BN / 64; ++h)
      tma_load_2d_hint(sB + s * Cfg::B_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, tn * Cfg::BN + 64 * h, kb * BK,
                       full_bar + 8 * s, pol);
  };
  float racc[Cfg::BN];
  const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
  int acc_phase = 0;
  for (int kb0 = 0; kb0 < KB; kb0 += p.kb_per_chunk) {
    const int kb1 = min(kb0 + p.kb_per_chunk, KB);
    if (threadIdx.x == 0) {
      // ---- the whole pipeline of this K chunk in one thread (a multistage software pipeline
      // as on Ampere, Sec. 3.5): RS - 1 k-blocks in flight; at k-block kb the stage k-block
      // kb - 1 used is refilled with kb + RS - 1 once kb - 1's MMAs have read it
      for (int kb = kb0; kb < min(kb0 + RS - 1, kb1); ++kb) load(kb);
      for (int kb = kb0; kb < kb1; ++kb) {
        if (kb + RS - 1 < kb1) {
          if (kb > kb0) mbar_wait(empty_bar + 8 * ((kb - 1) % RS), static_cast<uint32_t>(((kb - 1) / RS) & 1));
          load(kb + RS - 1);
        }
        const int s = kb % RS;
        mbar_wait(full_bar + 8 * s, static_cast<uint32_t>((kb / RS) & 1));
        tc_fence_after();
        for (int k = 0; k < BK / Cfg::UMMA_K; ++k)
          umma_f16<1>(tmem_base, desc_sw128(sA + s * Cfg::A_BYTES + 32 * k, 16, 1024),
                      desc_sw128(sB + s * Cfg::B_BYTES + 2048 * k, Cfg::B_ATOM_BYTES, 1024), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(empty_bar + 8 * s);
      }
      umma_commit(accf_bar);
    }
    // ---- every thread: promote this chunk into F32 registers (its accumulator row)
    mbar_wait(accf_bar, static_cast<uint32_t>(acc_phase));
    acc_phase ^= 1;
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < Cfg::BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_row + 32 * c, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        racc[32 * c + j] = kb0 == 0 ? __uint_as_float(v[j]) : __fadd_rn(racc[32 * c + j], __uint_as_float(v[j]));
    }
    tc_fence_before();
    __syncthreads();   // TMEM read by all before the next chunk overwrites it
    tc_fence_after();
  }
  // ---- C_out = C_in + acc: each thread its row, plain global loads and stores
  const int row = tm * Cfg::BM + static_cast<int>(threadIdx.x);
  if (row < p.M) {
    const int col0 = tn * Cfg::BN;
    if constexpr (!OUT_F16) {
      float* crow = static_cast<float*>(p.c_ptr) + static_cast<long long>(row) * p.ldc;
#pragma unroll
      for (int j = 0; j < Cfg::BN; ++j) {
        const int col = col0 + j;
        if (col < p.N) crow[col] = (p.beta0 ? 0.f : crow[col]) + racc[j];
      }
    } else {
      __half* crow = static_cast<__half*>(p.c_ptr) + static_cast<long long>(row) * p.ldc;
#pragma unroll
      for (int j = 0; j < Cfg::BN; ++j) {
        const int col = col0 + j;
        if (col < p.N) crow[col] = __float2half_rn((p.beta0 ? 0.f : __half2float(crow[col])) + racc[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace g16
