// gemm_sm100_wide.cuh -- the F16-output kernel with a 256 x 512 CTA-pair tile
// (GEMM_CFG_PAIR_256x512), for the same operation as gemm_sm100.cuh:
//     C[M][N] += A[M][K] . B[K][N]        (A, B binary16, row-major; C binary16)
// PAPER.md Sec. 4.2 P:967-996 (F16 accumulate/output mode), Algorithm 1 P:363-398.
//
// Why a second kernel (DESIGN.md section 13 item 1, profiles/r01/findings.md
// section 2): the B200 runs this GEMM power-capped, and operand traffic from L2
// into shared memory is the largest power consumer the kernel controls.  A
// 256 x 512 pair tile moves 25 % fewer operand bytes per FLOP than 256 x 256
// (each CTA stages 128 rows of A and 256 columns of B per k-block for
// 128 x 512 outputs, instead of 128 + 128 for 128 x 256).  Measured: the SM
// clock under the power cap rises ~12-17 % (profiles/r01/wide_tile.md).
//
// The price is TMEM: one 128-lane x 512-column F32 accumulator fills all of it,
// so there is no second buffer and no K-chunk promotion.  Both are affordable
// only in the F16 mode:
//  * accuracy: one TMEM chain over the whole K truncates at ~1.2e-6 relative
//    error per 1024 of K (R4), ~2e-5 at K = 16384 -- two orders under
//    the F16 mode's 2e-3 bar, whose error is the final RNE rounding (~2e-4);
//  * overlap: the epilogue loads the tile's C_in into registers (packed F16,
//    128 registers per thread) while the tile's MMAs run, so after the last MMA
//    it only has to read TMEM, add and round in registers, and hand TMEM back.
//    The stores of C_out then overlap the next tile's mainloop.  With F32 C the
//    same tile would need 256 registers per thread, so F32 stays on
//    gemm_sm100.cuh.
//  * the remaining TMEM hand-over is split in two halves h0 = columns [0,256)
//    and h1 = [256,512) (one UMMA each): the last SPLIT k-blocks of a tile issue
//    all their h0 MMAs before their h1 MMAs, so the epilogue drains h0 while the
//    tensor core finishes h1; and the first SPLIT k-blocks of the next tile issue
//    h0 MMAs as soon as h0 is free, while h1 is still being drained.  The drain
//    then hides almost entirely behind MMAs (per-tile traces in wide_tile.md).
//
// Roles (352 threads) as in gemm_sm100.cuh: w0..w7 epilogue, w8 TMA producer,
// w9 MMA issuer (pair leader), w10 TMEM allocator.  Epilogue warp w reads TMEM
// lanes 32*(w%4).. (hardware quadrant rule) and, of each half h, the 128
// accumulator columns [256 h + 128 (w/4), +128).
#pragma once
#include "gemm_sm100.cuh"

namespace g16 {

template <int STAGES_>
struct WCfg {
  static constexpr int CG = 2;
  static constexpr int BN = 512;             // pair tile columns = 2 UMMAs of N = 256
  static constexpr int UMMA_N = 256;
  static constexpr int STAGES = STAGES_;
  static constexpr int BM = 128;             // rows per CTA
  static constexpr int BK = 64;              // one 128 B swizzle span of F16
  static constexpr int UMMA_K = 16;
  static constexpr int A_BYTES = BM * BK * 2;            // 16 KB
  static constexpr int B_ATOM_BYTES = 64 * BK * 2;       // 64 columns x 64 k = 8 KB
  static constexpr int B_HALF_BYTES = 2 * B_ATOM_BYTES;  // this CTA's 128 columns of one UMMA
  static constexpr int B_BYTES = 2 * B_HALF_BYTES;       // 32 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KB
  static constexpr int TMEM_COLS = 512;
  static constexpr int EPI_WARPS = 8;
  static constexpr int CPH = 128;            // accumulator columns per epilogue warp per half
  static constexpr int CPW = 2 * CPH;        // ... per tile
  static constexpr int CW = 64;              // output chunk: 32 rows x 64 F16 = 32 x 128 B
  static constexpr int NOUT = CPW / CW;      // 4 chunks per warp per tile
  static constexpr int EPI_BUF = 32 * 128;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_E = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_E + EPI_WARPS * EPI_BUF;
  // barriers: full[S], empty[S], acc_full[2 halves], acc_empty[2 halves], epi[8]; then the TMEM slot
  static constexpr int NBAR = 2 * STAGES + 4 + EPI_WARPS;
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static constexpr int THREADS = 352;
  static constexpr int W_PRODUCER = 8, W_MMA = 9, W_ALLOC = 10;
};

// Global column of local column L (0..255) of epilogue warp group g (= w / 4) in tile column tn.
__device__ __forceinline__ int wide_col(int tn, int g, int L) { return tn * 512 + (L >> 7) * 256 + 128 * g + (L & 127); }

// EXT = false: plain C += A.B (and beta = 0, BF16 inputs); EXT = true: any of bias,
// ReLU, accum_f16 -- a separate instantiation, so the per-element option code
// costs the plain kernel neither instructions nor registers in the drain.
template <class Cfg, bool EXT>
__global__ void __launch_bounds__(352, 1)
gemm_f16_sm100_wide_kernel(const __grid_constant__ CUtensorMap tm_a,
                           const __grid_constant__ CUtensorMap tm_b,
                           const __grid_constant__ CUtensorMap tm_c,
                           const __grid_constant__ GemmParams p,
                           const __grid_constant__ PeerMaps /*unused: no fused gather here*/,
                           const __grid_constant__ CUtensorMap /*unused: no C_in prefetch map*/) {
  constexpr int STAGES = Cfg::STAGES, BM = Cfg::BM, BK = Cfg::BK;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base + Cfg::OFF_A;
  const uint32_t sB = base + Cfg::OFF_B;
  const uint32_t sE = base + Cfg::OFF_E;
  const uint32_t bar0 = base + Cfg::OFF_BAR;
  const uint32_t full_bar = bar0;
  const uint32_t empty_bar = bar0 + 8 * STAGES;
  const uint32_t accf_bar = bar0 + 16 * STAGES;   // [h]
  const uint32_t acce_bar = accf_bar + 16;        // [h]
  const uint32_t epi_bar = acce_bar + 16;
  const uint32_t tmem_slot = bar0 + 8 * Cfg::NBAR;

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();

  if (warp == Cfg::W_PRODUCER && lane == 0) {
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_c);
  }
  if (warp == Cfg::W_MMA && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(accf_bar + 8 * h, 1);
      mbar_init(acce_bar + 8 * h, Cfg::EPI_WARPS * 2);
    }
    for (int i = 0; i < Cfg::EPI_WARPS; ++i) mbar_init(epi_bar + 8 * i, 1);
    fence_mbarrier_init();
  }
  if (warp == Cfg::W_ALLOC) tmem_alloc<2>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");
  tmem_base = __shfl_sync(0xffffffffu, tmem_base, 0);   // (warp-uniform)
  griddep_wait();   // PDL: nothing above touched global memory

  const int cluster = static_cast<int>(blockIdx.x) / 2;
  const int nclusters = static_cast<int>(gridDim.x) / 2;

  if (warp == Cfg::W_PRODUCER) {
    // ===================== TMA producer =====================
    // (the whole warp runs the loop: warp-uniform TMA operands; the elected lane issues)
    {
      const bool leader = elect_one();
      const uint32_t full_leader = mapa_shared(full_bar, 0);
      const uint64_t pol_a = p.l2_hints ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_b = policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
        int tm, tn;
        tile_coords(tile, p, tm, tn);
        const int a_row = tm * BM * 2 + static_cast<int>(rank) * BM;
        // UMMA h covers columns [512 tn + 256 h, +256); CTA r stages its 128-column half
        const int b_col = tn * Cfg::BN + static_cast<int>(rank) * 128;
        if (tile + nclusters >= p.num_tiles && leader) griddep_launch_dependents();
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty_bar + 8 * stage, phase ^ 1u);
          if (leader) {
          if (rank == 0) mbar_arrive_expect_tx(full_bar + 8 * stage, Cfg::STAGE_BYTES * 2);
          const uint32_t fb = full_leader + 8 * stage;
          const uint32_t a_dst = sA + stage * Cfg::A_BYTES;
          const uint32_t b_dst = sB + stage * Cfg::B_BYTES;
          const int kc = kb * BK;
          tma_load_2d_pair_hint(a_dst, &tm_a, kc, a_row, fb, pol_a);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int t = 0; t < 2; ++t)
              tma_load_2d_pair_hint(b_dst + h * Cfg::B_HALF_BYTES + t * Cfg::B_ATOM_BYTES, &tm_b,
                                    b_col + h * Cfg::UMMA_N + 64 * t, kc, fb, pol_b);
          }   // leader
          __syncwarp();
          if (++stage == p.ring_stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == Cfg::W_MMA) {
    // ===================== MMA issuer (pair leader) =====================
    // the whole warp runs the loop (uniform control flow and operands); the elected lane issues
    if (rank == 0) {
      const bool leader = elect_one();
      const uint32_t idesc = (idesc_f16_f32acc<256, 256>() & (p.accum_f16 ? ~(3u << 4) : ~0u)) |
                             (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      // the 4 K=16 UMMAs of one k-block for accumulator half h
      auto mma_half = [&](int stage, int h, bool first) {
        const uint32_t a_s = sA + stage * Cfg::A_BYTES;
        const uint32_t b_s = sB + stage * Cfg::B_BYTES + h * Cfg::B_HALF_BYTES;
#pragma unroll
        for (int k = 0; k < BK / Cfg::UMMA_K; ++k)
          if (leader) umma_f16<2>(tmem_base + static_cast<uint32_t>(h * Cfg::UMMA_N), desc_sw128(a_s + 32 * k, 16, 1024),
                      desc_sw128(b_s + 2048 * k, Cfg::B_ATOM_BYTES, 1024), idesc, (first && k == 0) ? 0u : 1u);
      };
      // split k-blocks per tile end: ring_stages - 1 leaves one stage for the next tile's
      // first load (all 4 stages measured equal within noise, +1 % / -0.2 %)
      const int split_max = p.ring_stages > 1 ? p.ring_stages - 1 : 1;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_phase = 0;
      int it = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters, ++it) {
        const bool tr = p.trace != nullptr && blockIdx.x == 0 && leader && it < 60;
        uint64_t clk0 = 0;
        if (tr) {
          p.trace[8 * it + 0] = globaltimer_ns();
          clk0 = clock64();
        }
        const int head = min(split_max, p.k_blocks);              // split k-blocks at the start
        const int tail = min(split_max, p.k_blocks - head);       // ... and at the end
        // ---- head: h0 MMAs as soon as the epilogue has drained h0, then h1
        mbar_wait(acce_bar, acc_phase ^ 1u);
        tc_fence_after();
        if (tr) p.trace[8 * it + 1] = globaltimer_ns();
        {
          int s = stage;
          uint32_t ph = phase;
          for (int i = 0; i < head; ++i) {
            mbar_wait(full_bar + 8 * s, ph);
            tc_fence_after();
            mma_half(s, 0, i == 0);
            if (++s == p.ring_stages) { s = 0; ph ^= 1u; }
          }
          if (tail == 0 && leader) umma_commit_pair(accf_bar, 0x3);
          mbar_wait(acce_bar + 8, acc_phase ^ 1u);
          tc_fence_after();
          for (int i = 0; i < head; ++i) {
            mma_half(stage, 1, i == 0);
            if (leader) umma_commit_pair(empty_bar + 8 * stage, 0x3);
            if (++stage == p.ring_stages) { stage = 0; phase ^= 1u; }
          }
          if (tail == 0 && leader) umma_commit_pair(accf_bar + 8, 0x3);
        }
        // ---- middle: both halves per k-block
        for (int kb = head; kb < p.k_blocks - tail; ++kb) {
          mbar_wait(full_bar + 8 * stage, phase);
          tc_fence_after();
          mma_half(stage, 0, false);
          mma_half(stage, 1, false);
          if (leader) umma_commit_pair(empty_bar + 8 * stage, 0x3);
          if (++stage == p.ring_stages) { stage = 0; phase ^= 1u; }
        }
        // ---- tail: all h0 MMAs, hand h0 to the epilogue, then the h1 MMAs
        if (tail > 0) {
          int s = stage;
          uint32_t ph = phase;
          for (int i = 0; i < tail; ++i) {
            mbar_wait(full_bar + 8 * s, ph);
            tc_fence_after();
            mma_half(s, 0, false);
            if (++s == p.ring_stages) { s = 0; ph ^= 1u; }
          }
          if (leader) umma_commit_pair(accf_bar, 0x3);
          for (int i = 0; i < tail; ++i) {
            mma_half(stage, 1, false);
            if (leader) umma_commit_pair(empty_bar + 8 * stage, 0x3);
            if (++stage == p.ring_stages) { stage = 0; phase ^= 1u; }
          }
          if (leader) umma_commit_pair(accf_bar + 8, 0x3);
        }
        if (tr) {
          p.trace[8 * it + 2] = globaltimer_ns();
          p.trace[8 * it + 7] = clock64() - clk0;   // SM cycles of this tile (MMA warp)
        }
        acc_phase ^= 1u;
      }
    }
  } else if (warp < Cfg::EPI_WARPS) {
    // ===================== epilogue warps =====================
    const uint32_t q = warp & 3;                   // TMEM lane quadrant
    const int grp = static_cast<int>(warp >> 2);   // column group within each half
    const uint32_t ebuf = sE + warp * Cfg::EPI_BUF;
    const uint32_t ebar = epi_bar + 8 * warp;
    const uint32_t acce_leader = mapa_shared(acce_bar, 0);
    const uint64_t pol_c = p.l2_hints ? policy_evict_first() : policy_evict_normal();
    const bool load_c = !p.beta0;
    uint32_t acc_phase = 0;
    uint32_t ebar_phase = 0;
    // this thread's row of the warp's 32 x 256 region (local column L -> wide_col):
    // C_in, then C_out, as packed F16x2; cv[i] holds local columns 2i, 2i+1
    uint32_t cv[Cfg::CPW / 2];
    int it = 0;
    for (int tile = cluster; tile < p.num_tiles; tile += nclusters, ++it) {
      const bool tr = p.trace != nullptr && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 60;
      if (tr) p.trace[8 * it + 3] = globaltimer_ns();
      int tm, tn;
      tile_coords(tile, p, tm, tn);
      const int row0 = tm * BM * 2 + static_cast<int>(rank) * BM + static_cast<int>(q) * 32;
      // ---- C_in -> registers while this tile's MMAs run (one 4 KB staging slot per warp)
      if (load_c) {
#pragma unroll
        for (int c = 0; c < Cfg::NOUT; ++c) {
          if (lane == 0) {
            bulk_wait_group_read<0>();   // the previous store out of the slot has read it
            mbar_arrive_expect_tx(ebar, 32 * 128);
            tma_load_2d_hint(ebuf, &tm_c, wide_col(tn, grp, c * Cfg::CW), row0, ebar, pol_c);
          }
          mbar_wait(ebar, ebar_phase);
          ebar_phase ^= 1u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 v = lds128u(ebuf + swz<128>(lane, static_cast<uint32_t>(j)));
            cv[32 * c + 4 * j + 0] = v.x;
            cv[32 * c + 4 * j + 1] = v.y;
            cv[32 * c + 4 * j + 2] = v.z;
            cv[32 * c + 4 * j + 3] = v.w;
          }
          fence_proxy_async_smem();   // generic reads before the next async-proxy write
          __syncwarp();
        }
      } else {
#pragma unroll
        for (int i = 0; i < Cfg::CPW / 2; ++i) cv[i] = 0u;
      }
      // ---- bias: this warp's 2 x 128 columns staged once per tile in its (now idle) staging
      // slot, so the drain below reads them from shared memory (broadcast) instead of issuing
      // a global load per element pair while the MMA may be waiting for the TMEM half
      if constexpr (EXT) {
        if (p.bias != nullptr) {
          if (lane == 0 && !load_c) bulk_wait_group_read<0>();   // the previous tile's last store
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 bb = load_bias4(p.bias, wide_col(tn, grp, h * Cfg::CPH + 4 * static_cast<int>(lane)), p.N);
            sts128(ebuf + static_cast<uint32_t>(h * Cfg::CPH * 4) + 16u * lane, bb.x, bb.y, bb.z, bb.w);
          }
          __syncwarp();
        }
      }
      // ---- the accumulator, half by half: TMEM -> registers, + C_in (+ bias, relu),
      // one RNE rounding; each half goes back to the MMA warp as soon as it is read
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mbar_wait(accf_bar + 8 * h, acc_phase);
        tc_fence_after();
        if (tr && h == 0) p.trace[8 * it + 4] = globaltimer_ns();
        const uint32_t t_row = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(h * Cfg::UMMA_N + grp * Cfg::CPH);
        uint32_t* cvh = cv + h * (Cfg::CPH / 2);
        if constexpr (!EXT) {
          // plain C += A.B: the MMAs may wait for this loop, so it is kept short:
          // 5 instructions per output pair, no per-element option tests
#pragma unroll
          for (int c = 0; c < Cfg::CPH / 16; ++c) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(t_row + 16 * c, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 ci = f16x2_to_f32(cvh[8 * c + j]);
              cvh[8 * c + j] = cvt_f16x2_rn(ci.x + __uint_as_float(v[2 * j]), ci.y + __uint_as_float(v[2 * j + 1]));
            }
          }
        } else {
#pragma unroll   // (cv must be indexed by constants: a rolled loop would move it to local memory)
          for (int c = 0; c < Cfg::CPH / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + 32 * c, v);
            tmem_wait_ld();
            if (p.accum_f16) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(f16x2_to_f32(v[j]).x);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float2 ci = f16x2_to_f32(cvh[16 * c + j]);
              float o0 = ci.x + __uint_as_float(v[2 * j]);
              float o1 = ci.y + __uint_as_float(v[2 * j + 1]);
              if (p.bias != nullptr) {   // (staged above; columns past N hold 0)
                const float2 bb = lds64f(ebuf + static_cast<uint32_t>(4 * (h * Cfg::CPH + 32 * c + 2 * j)));
                o0 += bb.x;
                o1 += bb.y;
              }
              if (p.relu) {
                o0 = relu_keep_nan(o0);
                o1 = relu_keep_nan(o1);
              }
              cvh[16 * c + j] = cvt_f16x2_rn(o0, o1);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acce_leader + 8 * h);   // TMEM half h free for the next tile
      }
      acc_phase ^= 1u;
      if (tr) p.trace[8 * it + 5] = globaltimer_ns();
      // ---- C_out: registers -> swizzled staging -> TMA store (overlaps the next mainloop).
      // Last tile: every MMA of the pair has completed (both halves' barriers), so the
      // operand ring is idle -- stage all NOUT chunks there and store them back to back
      // (static_assert below: 8 warps x NOUT x 4 KB fit in the ring)
      static_assert(Cfg::EPI_WARPS * Cfg::NOUT * Cfg::EPI_BUF <= Cfg::STAGES * Cfg::STAGE_BYTES, "tail ring");
      const bool ring = p.tail_ring && tile + nclusters >= p.num_tiles;
      if (ring) fence_proxy_async_smem();
      const int grow = row0 + static_cast<int>(lane);
#pragma unroll
      for (int c = 0; c < Cfg::NOUT; ++c) {
        const int ccol = wide_col(tn, grp, c * Cfg::CW);
        if (ccol >= p.N) break;   // warp-uniform; chunk columns increase with c
        const uint32_t sbuf = ring ? sA + (warp * Cfg::NOUT + c) * Cfg::EPI_BUF : ebuf;
        if (lane == 0 && !ring) bulk_wait_group_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          sts128u(sbuf + swz<128>(lane, static_cast<uint32_t>(j)), cv[32 * c + 4 * j + 0], cv[32 * c + 4 * j + 1],
                  cv[32 * c + 4 * j + 2], cv[32 * c + 4 * j + 3]);
        const bool manual = p.c_ragged && (ccol + Cfg::CW > p.N);
        if (!manual) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d_hint(&tm_c, ccol, row0, sbuf, pol_c);
            bulk_commit_group();
          }
        } else {
          // ragged N edge (N * 2 % 16 != 0): element-wise stores of this thread's
          // row, read back from the staged chunk, clipped at column N
          __syncwarp();
          if (grow < p.M) {
            uint16_t* dst = static_cast<uint16_t*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc;
#pragma unroll 1
            for (int j = 0; j < 8; ++j) {
              const uint4 v = lds128u(sbuf + swz<128>(lane, static_cast<uint32_t>(j)));
              const uint32_t o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (ccol + 8 * j + e < p.N) dst[ccol + 8 * j + e] = static_cast<uint16_t>(o[e >> 1] >> (16 * (e & 1)));
            }
          }
        }
      }
      __syncwarp();
      if (tr) p.trace[8 * it + 6] = globaltimer_ns();
    }
    if (lane == 0) bulk_wait_group<0>();
  }

  // ===================== teardown =====================
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == Cfg::W_ALLOC) {
    tc_fence_after();
    tmem_dealloc<2>(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace g16
