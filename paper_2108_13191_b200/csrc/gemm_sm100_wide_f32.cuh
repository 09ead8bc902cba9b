// gemm_sm100_wide_f32.cuh -- the 256 x 512 CTA-pair tile for F32 C (GEMM_CFG_PAIR_256x512
// with GEMM_ACC_F32), for the same operation as gemm_sm100.cuh:
//     C[M][N] += A[M][K] . B[K][N]        (A, B binary16 or bfloat16, row-major; C float)
// PAPER.md Sec. 4.1 P:924-949 (F16 inputs, F32 accumulate/output), Algorithm 1 P:363-398;
// the block tile that maximises operand reuse, Sec. 3.2 P:440-452.
//
// Why (profiles/r01/findings.md sections 1-2): the B200 runs this GEMM
// power-capped and operand traffic from L2 into shared memory is the largest power cost the
// kernel controls.  The 256 x 512 pair tile moves 25 % fewer operand bytes per FLOP than the
// 256 x 256 tile of gemm_sm100.cuh; the F16-output kernel (gemm_sm100_wide.cuh) showed the
// clock rise that buys.  F32 C needs two more things that kernel does not have:
//
//  * K-chunk promotion (R4): the tensor core's F32 accumulator truncates, so one
//    TMEM chain over K = 8192 sits at ~1e-5 relative error, the bar.  Every `kb_per_chunk`
//    k-blocks the partial sum leaves TMEM and is added into C by a TMA reduce-add (one IEEE
//    round-to-nearest add per element in L2, the same add the register promotion of
//    gemm_sm100.cuh does, in the same fixed order): C = ((C_in + p0) + p1) + ...
//  * no second TMEM buffer (the 128 x 512 F32 accumulator per CTA is all of TMEM), so the
//    drains must hide behind MMAs some other way.  The two accumulator halves h0 = columns
//    [0, 256) and h1 = [256, 512) (one UMMA N=256 each) promote at STAGGERED k-blocks: h0
//    after Cb, 2 Cb, ..., h1 after Cb/2, 3 Cb/2, ... k-blocks (Cb = kb_per_chunk).  While the
//    epilogue drains one half, the MMA issuer runs ahead on the other half through the loaded
//    ring stages and issues the drained half's deferred MMAs once it is free (tcgen05 MMAs
//    execute in issue order, so each stage is released when both halves have used it).  At
//    a tile's end both halves end together; there the last ring_stages - 1 k-blocks issue
//    all their h0 MMAs first (as in gemm_sm100_wide.cuh), so h0 drains under h1's last MMAs.
//
// Determinism: every element's sum is C_in, then its half's chunk partials in K order, each
// a fixed chain of MMAs; a drain's reduce-adds are issued only after the previous drain of
// the same half has completed in memory.  Independent of the grid (bitwise).
//
// Roles (352 threads) as in gemm_sm100.cuh: w0..w7 epilogue, w8 TMA producer, w9 MMA issuer
// (pair leader), w10 TMEM allocator.  Epilogue warp w reads TMEM lanes 32*(w%4).. and, of
// each half, the 128 accumulator columns [256 h + 128 (w/4), +128).
#pragma once
#include "gemm_sm100.cuh"


namespace g16 {

template <int STAGES_, int EPI_SLOTS_>
struct W32Cfg {
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
  static constexpr int CW = 32;              // output chunk: 32 rows x 32 F32 = 32 x 128 B
  static constexpr int NOUT = CPH / CW;      // 4 chunks per warp per drain
  static constexpr int EPI_SLOTS = EPI_SLOTS_;
  static constexpr int EPI_BUF = 32 * 128;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_E = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_E + EPI_WARPS * EPI_SLOTS * EPI_BUF;
  // barriers: full[S], empty[S], acc_full[2 halves], acc_empty[2 halves]; then the TMEM slot
  static constexpr int NBAR = 2 * STAGES + 4;
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static constexpr int THREADS = 352;
  static constexpr int W_PRODUCER = 8, W_MMA = 9, W_ALLOC = 10;
};

// Is the k-block count e (1 <= e < k_blocks) an interior promotion point of half h?
// h0 promotes after Cb, 2 Cb, ... k-blocks, h1 after Cb/2, 3 Cb/2, ...; none in the last
// `guard` k-blocks of a tile (its final chunk then takes them: chains stay <= Cb + guard).
// The host keeps Cb / 2 >= guard, so a half is never asked to promote again before the
// MMA issuer has caught it up.
__device__ __forceinline__ bool w32_bound(const GemmParams& p, int h, int e, int guard) {
  const int cb = p.kb_per_chunk;
  if (cb >= p.k_blocks) return false;
  const int f = h == 0 ? cb : cb / 2;
  return e >= f && (e - f) % cb == 0 && e <= p.k_blocks - guard;
}

// EXT = false: plain C += A.B; EXT = true: beta = 0 (the first drain of each half STORES
// instead of reduce-adding) and/or a bias (added once, in that first drain).
template <class Cfg, bool EXT>
__global__ void __launch_bounds__(352, 1)
gemm_f16_sm100_wide_f32_kernel(const __grid_constant__ CUtensorMap tm_a,
                               const __grid_constant__ CUtensorMap tm_b,
                               const __grid_constant__ CUtensorMap tm_c,
                               const __grid_constant__ GemmParams p,
                               const __grid_constant__ PeerMaps /*unused: no fused gather here*/,
                               const __grid_constant__ CUtensorMap /*unused*/) {
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
  const uint32_t tmem_slot = bar0 + 8 * Cfg::NBAR;
  const int guard = p.ring_stages + 2;            // (w32_bound)

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool trace_me = p.trace != nullptr && blockIdx.x == static_cast<unsigned>(p.trace[8 * 63 + 7]);
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 0] = globaltimer_ns();

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
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 1] = globaltimer_ns();

  const int cluster = static_cast<int>(blockIdx.x) / 2;
  const int nclusters = static_cast<int>(gridDim.x) / 2;

  if (warp == Cfg::W_PRODUCER) {
    // ===================== TMA producer (as gemm_sm100_wide.cuh) =====================
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
      const uint32_t idesc = idesc_f16_f32acc<256, 256>() | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      const int RS = p.ring_stages;
      const int split = RS > 1 ? RS - 1 : 1;   // tile tail: h0 MMAs of the last `split` k-blocks first
      const int KB = p.k_blocks;
      int stage = 0;                 // ring position of the next k-block to consume
      uint32_t phase = 0;
      uint32_t ncommit[2] = {0u, 0u};   // accumulator hand-overs per half so far
      bool blocked[2] = {false, false}; // the half's last chunk is not yet drained: its MMAs wait
      bool post1 = false;               // h1 postponed in a tile's tail (not blocked)
      bool first[2] = {true, true};     // next MMA of the half starts a chain (accumulate = 0)
      int dlo[2] = {0, 0};              // first deferred k-block of a blocked / postponed half
      int dstage[2] = {0, 0};           // ... and its ring stage
      auto mma = [&](int st, int h) {
        const uint32_t a_s = sA + st * Cfg::A_BYTES;
        const uint32_t b_s = sB + st * Cfg::B_BYTES + h * Cfg::B_HALF_BYTES;
#pragma unroll
        for (int k = 0; k < BK / Cfg::UMMA_K; ++k)
          if (leader) umma_f16<2>(tmem_base + static_cast<uint32_t>(h * Cfg::UMMA_N), desc_sw128(a_s + 32 * k, 16, 1024),
                      desc_sw128(b_s + 2048 * k, Cfg::B_ATOM_BYTES, 1024), idesc, (first[h] && k == 0) ? 0u : 1u);
        first[h] = false;
      };
      auto pending = [&](int h, int kb) { return (blocked[h] || (h == 1 && post1)) && kb >= dlo[h]; };
      // issue half h's deferred MMAs for k-blocks [dlo[h], kend); a stage is released once
      // both halves have issued their MMAs on it (the commit tracks every prior MMA)
      auto flush = [&](int h, int kend) {
        int s = dstage[h];
        for (int kb = dlo[h]; kb < kend; ++kb) {
          mma(s, h);
          if (leader && !pending(h ^ 1, kb)) umma_commit_pair(empty_bar + 8 * s, 0x3);
          if (++s == RS) s = 0;
        }
        dlo[h] = kend;
        dstage[h] = s;
      };
      // (test_wait: never suspends the issuer while the other half has work)
      auto try_unblock = [&](int h, int kend) {
        if (!blocked[h]) return;
        const int done = __shfl_sync(0xffffffffu, mbar_test_wait(acce_bar + 8 * h, (ncommit[h] - 1u) & 1u) ? 1 : 0, 0);
        if (!done) return;
        tc_fence_after();
        blocked[h] = false;
        flush(h, kend);
      };
      int it = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters, ++it) {
        const bool tr = trace_me && leader && it < 60;
        uint64_t clk0 = 0;
        if (tr) {
          p.trace[8 * it + 0] = globaltimer_ns();
          clk0 = clock64();
        }
        for (int kb = 0; kb < KB; ++kb) {
          // room in the ring: deferred k-blocks hold their stages
          for (;;) {
            int held = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (blocked[h] || (h == 1 && post1)) held = max(held, kb - dlo[h]);
            if (held < RS) break;
            try_unblock(0, kb);
            try_unblock(1, kb);
          }
          mbar_wait(full_bar + 8 * stage, phase);
          tc_fence_after();
          if (kb == 0 && tr) p.trace[8 * it + 1] = globaltimer_ns();
          if (kb == KB - split && KB > split && !blocked[1] && !post1) {
            post1 = true;   // tail: h1 waits until h0's final MMAs are issued and handed over
            dlo[1] = kb;
            dstage[1] = stage;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            try_unblock(h, kb);
            if (!pending(h, kb)) mma(stage, h);
          }
          if (leader && !pending(0, kb) && !pending(1, kb)) umma_commit_pair(empty_bar + 8 * stage, 0x3);
          if (++stage == RS) { stage = 0; phase ^= 1u; }
          // interior promotion points after this k-block
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (kb + 1 < KB && w32_bound(p, h, kb + 1, guard)) {
              while (blocked[h]) try_unblock(h, kb + 1);   // (host rules keep this a no-op)
              if (leader) umma_commit_pair(accf_bar + 8 * h, 0x3);
              ++ncommit[h];
              blocked[h] = true;
              first[h] = true;
              dlo[h] = kb + 1;
              dstage[h] = stage;
            }
          }
        }
        // tile end: both halves hand over, h0 first
        while (blocked[0]) try_unblock(0, KB);
        if (leader) umma_commit_pair(accf_bar, 0x3);
        if (post1) {
          post1 = false;
          flush(1, KB);
        }
        while (blocked[1]) try_unblock(1, KB);
        if (leader) umma_commit_pair(accf_bar + 8, 0x3);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ++ncommit[h];
          blocked[h] = true;
          first[h] = true;
          dlo[h] = 0;
          dstage[h] = stage;
        }
        if (tr) {
          p.trace[8 * it + 2] = globaltimer_ns();
          p.trace[8 * it + 7] = clock64() - clk0;   // SM cycles of this tile (MMA warp)
        }
      }
    }
  } else if (warp < Cfg::EPI_WARPS) {
    // ===================== epilogue warps =====================
    const uint32_t q = warp & 3;                   // TMEM lane quadrant
    const int grp = static_cast<int>(warp >> 2);   // column group within each half
    const uint32_t ebuf0 = sE + warp * Cfg::EPI_SLOTS * Cfg::EPI_BUF;
    const uint32_t acce_leader = mapa_shared(acce_bar, 0);
    const uint64_t pol_c = p.l2_hints ? policy_evict_first() : policy_evict_normal();
    uint32_t ecount[2] = {0u, 0u};
    int slot = 0;
    int last_h = -1;     // half of the previous drain (-1: none yet / new tile)
    int last_groups = 0; // bulk groups that drain committed
    int it = 0;
    for (int tile = cluster; tile < p.num_tiles; tile += nclusters, ++it) {
      const bool tr = trace_me && warp == 0 && lane == 0 && it < 60;
      if (tr) p.trace[8 * it + 3] = globaltimer_ns();
      int tm, tn;
      tile_coords(tile, p, tm, tn);
      const int row0 = tm * BM * 2 + static_cast<int>(rank) * BM + static_cast<int>(q) * 32;
      bool fresh[2] = {true, true};   // EXT: the first drain of each half in this tile
      last_h = -1;
      // the drains of this tile in hand-over order: interior points, then h0, h1 at the end
      for (int e = 1; e <= p.k_blocks; ++e) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (e < p.k_blocks ? !w32_bound(p, h, e, guard) : false) continue;
          // ---- TMEM -> registers (four 32-column loads in flight), then hand the half back
          mbar_wait(accf_bar + 8 * h, ecount[h] & 1u);
          ++ecount[h];
          tc_fence_after();
          if (tr && e == p.k_blocks && h == 0) p.trace[8 * it + 4] = globaltimer_ns();
          const uint32_t t_row = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(h * Cfg::UMMA_N + grp * Cfg::CPH);
          uint32_t v[Cfg::NOUT][32];
#pragma unroll
          for (int c = 0; c < Cfg::NOUT; ++c) tmem_ld_32x32b_x32(t_row + 32 * c, v[c]);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(acce_leader + 8 * h);
          // ---- registers -> swizzled staging -> TMA reduce-add into C.  The previous drain of
          // this half (same C region) must have completed in memory first: it is the last
          // drain (wait for every group) or the one before (wait for all but its NOUT groups)
          if (lane == 0) {
            const int keep = last_h == h ? 0 : last_groups;   // groups allowed to stay in flight
            if (keep >= 4) bulk_wait_group<4>();
            else if (keep == 3) bulk_wait_group<3>();
            else if (keep == 2) bulk_wait_group<2>();
            else if (keep == 1) bulk_wait_group<1>();
            else bulk_wait_group<0>();
          }
          static_assert(Cfg::NOUT <= 4, "bulk_wait_group immediates above");
          const bool store = EXT && p.beta0 && fresh[h];
          const bool add_bias = EXT && p.bias != nullptr && fresh[h];
          fresh[h] = false;
          last_h = h;
          last_groups = 0;
#pragma unroll
          for (int c = 0; c < Cfg::NOUT; ++c) {
            const int ccol = tn * Cfg::BN + h * Cfg::UMMA_N + grp * Cfg::CPH + c * Cfg::CW;
            if (ccol >= p.N) break;   // warp-uniform
            const uint32_t sbuf = ebuf0 + static_cast<uint32_t>(slot) * Cfg::EPI_BUF;
            if (++slot == Cfg::EPI_SLOTS) slot = 0;
            if (lane == 0) bulk_wait_group_read<Cfg::EPI_SLOTS - 1>();   // the slot's last store has read it
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float o0 = __uint_as_float(v[c][4 * j + 0]), o1 = __uint_as_float(v[c][4 * j + 1]);
              float o2 = __uint_as_float(v[c][4 * j + 2]), o3 = __uint_as_float(v[c][4 * j + 3]);
              if (add_bias) {
                const float4 bb = load_bias4(p.bias, ccol + 4 * j, p.N);
                o0 += bb.x; o1 += bb.y; o2 += bb.z; o3 += bb.w;
              }
              sts128(sbuf + swz<128>(lane, static_cast<uint32_t>(j)), o0, o1, o2, o3);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (store) tma_store_2d_hint(&tm_c, ccol, row0, sbuf, pol_c);
              else tma_reduce_add_2d_hint(&tm_c, ccol, row0, sbuf, pol_c);
              bulk_commit_group();
            }
            ++last_groups;
          }
        }
      }
      if (tr) {
        p.trace[8 * it + 5] = globaltimer_ns();
        p.trace[8 * it + 6] = globaltimer_ns();
      }
    }
    if (lane == 0) bulk_wait_group<0>();
    if (trace_me && warp == 0 && lane == 0) p.trace[8 * 62 + 3] = globaltimer_ns();
  }

  // ===================== teardown =====================
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == Cfg::W_ALLOC) {
    tc_fence_after();
    tmem_dealloc<2>(tmem_base, Cfg::TMEM_COLS);
  }
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 2] = globaltimer_ns();
}

}  // namespace g16
