// gemm_sm100.cuh -- the persistent, warp-specialised sm_100a kernel for
//     C[M][N] += A[M][K] . B[K][N]        (A, B binary16, row-major; C F32 or F16)
// PAPER.md Sec. 4 P:908-909 ("C = AB + C ... row-major"), Algorithm 1
// P:363-398 (two-level tiled tensor-core matmul), re-designed for B200:
//
//  paper (Ampere, WMMA)                        here (sm_100a)
//  -------------------------------------------  ---------------------------------------------
//  block tile tbm x tbn x tbk in smem (A3,A4)   CTA-pair tile (128*CG) x BN x 64, TMA-loaded
//  padded smem leading dim (Sec 3.3)     128B hardware swizzle (TMA + UMMA descriptors)
//  warp tiles + WMMA 16x16x16 (Sec 3.4)         one thread issues tcgen05.mma M=128*CG,N=BN,K=16
//  C in registers, hoisted          accumulator in TMEM for the whole K loop
//  1-stage k-loop split (Sec 3.5)    STAGES-deep mbarrier ring (full/empty)
//  __syncthreads around copies (Sec 3.6)        per-stage mbarriers + tcgen05.commit
//  128-bit vector global->smem copies (3.7)     cp.async.bulk.tensor boxes of 8-16 KB
//  one thread block per C tile (Sec 3.9)        persistent clusters, grouped raster schedule
//  C stored once per warp tile      epilogue warps: TMEM -> regs (+C_in) -> smem
//                                               -> TMA store, overlapped with the next tile's
//                                               mainloop through a double-buffered TMEM acc
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (pair leader only),
// w2 TMEM allocator, w3 idle, w4..w7 epilogue (warp w reads TMEM lanes 32*(w%4)..).
#pragma once
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"

namespace g16 {

struct GemmParams {
  int M, N, K;
  int tiles_m, tiles_n, num_tiles;  // tiles of (128*CG) x BN
  int k_blocks;                     // ceil(K / 64)
  int group_m;                      // raster group height in tiles
  int c_ragged;                     // N * sizeof(C) % 16 != 0: TMA stores would write a
                                    // whole 16-byte granule past column N-1, so the chunk
                                    // holding column N-1 is stored element-wise instead
  void* c_ptr;                      // C base (used only by that ragged-N store path)
  long long ldc;                    // C leading dimension in elements
};

template <int CG_, int BN_, int STAGES_, bool OUT_F16_>
struct KCfg {
  static constexpr int CG = CG_;            // CTAs per MMA (cta_group)
  static constexpr int BN = BN_;            // UMMA N (tile columns)
  static constexpr int STAGES = STAGES_;
  static constexpr bool OUT_F16 = OUT_F16_;
  static constexpr int BM = 128;            // rows per CTA (TMEM lanes)
  static constexpr int BK = 64;             // K per stage = one 128B swizzle span of F16
  static constexpr int UMMA_K = 16;
  static constexpr int BN_CTA = BN / CG;    // B columns staged per CTA
  static_assert(BN_CTA % 64 == 0, "B is staged in 64-column (128 B) swizzle atoms");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
  static constexpr int A_BYTES = BM * BK * 2;         // 16 KB
  static constexpr int B_ATOM_BYTES = 64 * BK * 2;    // 64 cols x 64 k = 8 KB
  static constexpr int B_BYTES = BN_CTA * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_COLS = BN;                 // one accumulator buffer
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int CW = OUT_F16 ? 64 : 32;        // epilogue chunk width (128 B of C)
  static constexpr int NCHUNK = BN / CW;
  static constexpr int EPI_WARPS = 4;
  static constexpr int EPI_SLOTS = 2;
  static constexpr int EPI_BUF = 32 * 128;            // 32 rows x 128 B
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_E = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_E + EPI_WARPS * EPI_SLOTS * EPI_BUF;
  // barriers: full[S], empty[S], acc_full[2], acc_empty[2], epi[4][2], tmem slot
  static constexpr int NBAR = 2 * STAGES + 4 + EPI_WARPS * EPI_SLOTS;
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static constexpr int THREADS = 256;
};

// UMMA shared-memory descriptor, SWIZZLE_128B layout (sm_100 "version 1").
// bits [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1,
// [49,52) base offset=0, [61,64) layout=2 (128B swizzle).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// UMMA instruction descriptor, kind::f16: D F32, A/B F16, A K-major, B MN-major.
template <int M, int N>
__device__ __forceinline__ constexpr uint32_t idesc_f16_f32acc() {
  return (1u << 4)                          // c_format = F32
         | (0u << 7) | (0u << 10)           // a_format = b_format = F16
         | (0u << 15)                       // A K-major (row-major A: K contiguous)
         | (1u << 16)                       // B MN-major (row-major B: N contiguous)
         | (static_cast<uint32_t>(N >> 3) << 17)
         | (static_cast<uint32_t>(M >> 4) << 24);
}

// Grouped raster: consecutive tile ids walk `group_m` tile-rows of one column
// strip before moving right, so co-resident clusters share A and B tiles in L2.
__device__ __forceinline__ void tile_coords(int tile, const GemmParams& p, int& tm, int& tn) {
  const int per_group = p.group_m * p.tiles_n;
  const int g = tile / per_group;
  const int first = g * p.group_m;
  const int gs = min(p.tiles_m - first, p.group_m);
  const int local = tile - g * per_group;
  tm = first + local % gs;
  tn = local / gs;
}

template <class Cfg>
__global__ void __launch_bounds__(256, 1)
gemm_f16_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_c,
                      const GemmParams p) {
  constexpr int CG = Cfg::CG, BN = Cfg::BN, STAGES = Cfg::STAGES, BM = Cfg::BM, BK = Cfg::BK;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base + Cfg::OFF_A;
  const uint32_t sB = base + Cfg::OFF_B;
  const uint32_t sE = base + Cfg::OFF_E;
  const uint32_t bar0 = base + Cfg::OFF_BAR;
  const uint32_t full_bar = bar0;
  const uint32_t empty_bar = bar0 + 8 * STAGES;
  const uint32_t accf_bar = bar0 + 16 * STAGES;
  const uint32_t acce_bar = accf_bar + 16;
  const uint32_t epi_bar = acce_bar + 16;
  const uint32_t tmem_slot = bar0 + 8 * Cfg::NBAR;

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_c);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf_bar + 8 * b, 1);
      mbar_init(acce_bar + 8 * b, Cfg::EPI_WARPS * CG);
    }
    for (int i = 0; i < Cfg::EPI_WARPS * Cfg::EPI_SLOTS; ++i) mbar_init(epi_bar + 8 * i, 1);
    fence_mbarrier_init();
  }
  if (warp == 2) tmem_alloc<CG>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");

  const int cluster = static_cast<int>(blockIdx.x) / CG;
  const int nclusters = static_cast<int>(gridDim.x) / CG;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint32_t full_leader = (CG == 2) ? mapa_shared(full_bar, 0) : full_bar;
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
        int tm, tn;
        tile_coords(tile, p, tm, tn);
        const int a_row = tm * BM * CG + static_cast<int>(rank) * BM;
        const int b_col = tn * BN + static_cast<int>(rank) * Cfg::BN_CTA;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty_bar + 8 * stage, phase ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(full_bar + 8 * stage, Cfg::STAGE_BYTES * CG);
          const uint32_t fb = full_leader + 8 * stage;
          const uint32_t a_dst = sA + stage * Cfg::A_BYTES;
          const uint32_t b_dst = sB + stage * Cfg::B_BYTES;
          if constexpr (CG == 2) {
            tma_load_2d_pair(a_dst, &tm_a, kb * BK, a_row, fb);
#pragma unroll
            for (int h = 0; h < Cfg::BN_CTA / 64; ++h)
              tma_load_2d_pair(b_dst + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h, kb * BK, fb);
          } else {
            tma_load_2d(a_dst, &tm_a, kb * BK, a_row, fb);
#pragma unroll
            for (int h = 0; h < Cfg::BN_CTA / 64; ++h)
              tma_load_2d(b_dst + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h, kb * BK, fb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair leader) =====================
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32acc<BM * CG, BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
        mbar_wait_cluster(acce_bar + 8 * acc, acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(full_bar + 8 * stage, phase);
          tc_fence_after();
          const uint32_t a_s = sA + stage * Cfg::A_BYTES;
          const uint32_t b_s = sB + stage * Cfg::B_BYTES;
#pragma unroll
          for (int k = 0; k < BK / Cfg::UMMA_K; ++k) {
            // A (K-major): advance 16 elements = 32 B inside the 128B swizzle row.
            const uint64_t adesc = desc_sw128(a_s + 32 * k, 16, 1024);
            // B (MN-major): advance 16 k-rows = 2 swizzle atoms of 8 rows x 128 B;
            // 64-column groups are B_ATOM_BYTES apart (LBO), 8-row groups 1 KB (SBO).
            const uint64_t bdesc = desc_sw128(b_s + 2048 * k, Cfg::B_ATOM_BYTES, 1024);
            umma_f16<CG>(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          if constexpr (CG == 2) umma_commit_pair(empty_bar + 8 * stage, 0x3);
          else umma_commit(empty_bar + 8 * stage);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        if constexpr (CG == 2) umma_commit_pair(accf_bar + 8 * acc, 0x3);
        else umma_commit(accf_bar + 8 * acc);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue warps =====================
    const uint32_t ew = warp - 4;          // == warp % 4: TMEM lane quadrant
    const uint32_t q = warp & 3;
    const uint32_t ebuf0 = sE + ew * Cfg::EPI_SLOTS * Cfg::EPI_BUF;
    const uint32_t ebar0 = epi_bar + 8 * Cfg::EPI_SLOTS * ew;
    const uint32_t acce_leader = (CG == 2) ? mapa_shared(acce_bar, 0) : acce_bar;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t chunk_ctr = 0;
    uint32_t slot_phase = 0;  // bit s = parity to wait for on slot s
    for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
      int tm, tn;
      tile_coords(tile, p, tm, tn);
      const int row0 = tm * BM * CG + static_cast<int>(rank) * BM + static_cast<int>(q) * 32;
      const int col0 = tn * BN;
      if (lane == 0) {
#pragma unroll 1
        for (int c = 0; c < Cfg::NCHUNK; ++c) tma_prefetch_l2_2d(&tm_c, col0 + c * Cfg::CW, row0);
      }
      mbar_wait(accf_bar + 8 * acc, acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
#pragma unroll 1
      for (int c = 0; c < Cfg::NCHUNK; ++c) {
        const uint32_t slot = chunk_ctr & 1u;
        const uint32_t sbuf = ebuf0 + slot * Cfg::EPI_BUF;
        const uint32_t sbar = ebar0 + 8 * slot;
        if (lane == 0) {
          bulk_wait_group_read<1>();   // the store that last used this slot has read it
          mbar_arrive_expect_tx(sbar, Cfg::EPI_BUF);
          tma_load_2d(sbuf, &tm_c, col0 + c * Cfg::CW, row0, sbar);
        }
        __syncwarp();
        uint32_t v0[32];
        uint32_t v1[32];
        tmem_ld_32x32b_x32(t_row + c * Cfg::CW, v0);
        if constexpr (Cfg::OUT_F16) tmem_ld_32x32b_x32(t_row + c * Cfg::CW + 32, v1);
        tmem_wait_ld();
        if (c == Cfg::NCHUNK - 1) {
          // accumulator buffer fully read into registers: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(acce_leader + 8 * acc);
            else mbar_arrive(acce_bar + 8 * acc);
          }
        }
        mbar_wait(sbar, (slot_phase >> slot) & 1u);
        slot_phase ^= (1u << slot);
        // Row `lane` of the 32x128B box; 16-byte unit j sits at j ^ (row % 8) (128B swizzle).
        const uint32_t row_addr = sbuf + lane * 128u;
        const bool manual = p.c_ragged && (col0 + (c + 1) * Cfg::CW > p.N);
        const int grow = row0 + static_cast<int>(lane);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t addr = row_addr + ((static_cast<uint32_t>(j) ^ (lane & 7u)) << 4);
          if constexpr (!Cfg::OUT_F16) {
            const float4 ci = lds128(addr);
            const float o0 = ci.x + __uint_as_float(v0[4 * j + 0]), o1 = ci.y + __uint_as_float(v0[4 * j + 1]);
            const float o2 = ci.z + __uint_as_float(v0[4 * j + 2]), o3 = ci.w + __uint_as_float(v0[4 * j + 3]);
            if (!manual) {
              sts128(addr, o0, o1, o2, o3);
            } else if (grow < p.M) {
              float* dst = static_cast<float*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc;
              const int cb = col0 + c * Cfg::CW + 4 * j;
              const float o[4] = {o0, o1, o2, o3};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (cb + e < p.N) dst[cb + e] = o[e];
            }
          } else {
            const uint4 ci = lds128u(addr);
            const uint32_t* src = (j < 4) ? &v0[8 * j] : &v1[8 * (j - 4)];
            const float2 c0 = f16x2_to_f32(ci.x), c1 = f16x2_to_f32(ci.y);
            const float2 c2 = f16x2_to_f32(ci.z), c3 = f16x2_to_f32(ci.w);
            const uint32_t o0 = cvt_f16x2_rn(c0.x + __uint_as_float(src[0]), c0.y + __uint_as_float(src[1]));
            const uint32_t o1 = cvt_f16x2_rn(c1.x + __uint_as_float(src[2]), c1.y + __uint_as_float(src[3]));
            const uint32_t o2 = cvt_f16x2_rn(c2.x + __uint_as_float(src[4]), c2.y + __uint_as_float(src[5]));
            const uint32_t o3 = cvt_f16x2_rn(c3.x + __uint_as_float(src[6]), c3.y + __uint_as_float(src[7]));
            if (!manual) {
              sts128u(addr, o0, o1, o2, o3);
            } else if (grow < p.M) {
              uint16_t* dst = static_cast<uint16_t*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc;
              const int cb = col0 + c * Cfg::CW + 8 * j;
              const uint32_t o[4] = {o0, o1, o2, o3};
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (cb + e < p.N) dst[cb + e] = static_cast<uint16_t>(o[e >> 1] >> (16 * (e & 1)));
            }
          }
        }
        if (!manual) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_c, col0 + c * Cfg::CW, row0, sbuf);
            bulk_commit_group();
          }
        } else {
          __syncwarp();
        }
        ++chunk_ctr;
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    if (lane == 0) bulk_wait_group<0>();
  }

  // ===================== teardown =====================
  __syncwarp();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace g16
