// gemm_sm100_splitk.cuh -- split-K over a thread-block cluster, for problems whose
// output is too small to fill the GPU with tiles but whose K is long
// (e.g. 1024 x 1024 x 4096, 512 x 512 x 2048):
//     C[M][N] += A[M][K] . B[K][N]        (A, B binary16/bfloat16; C F32 or F16)
// PAPER.md Sec. 4; the paper's per-size "best version" choice
// ("smaller tiles help small sizes through occupancy").
//
// The S CTAs of one cluster (S = 2 or 4) share one 128 x BN output tile: CTA r
// accumulates k-blocks [r kb / S, (r+1) kb / S) in its own TMEM
// (tcgen05.mma.cta_group::1, M=128, N=BN), so S times as many SMs work on the
// problem and each streams 1/S of the operands.  The S partial sums are reduced
// through distributed shared memory, with no workspace and no atomics:
//   1. cluster barrier: every CTA's mainloop is done, so the operand rings are idle;
//   2. CTA r owns columns [r BN / S, (r+1) BN / S) of the tile.  Every CTA reads its
//      partial out of TMEM.  Where everything fits in shared memory (SKCfg::DMA:
//      S4 x 128x128, and S2 x 128x256 with F16 C) it stages the partial slot-major and sends each owner its slot
//      with one bulk DMA copy (cp.async.bulk.shared::cluster, counted on the owner's
//      mbarrier).  Otherwise it pushes each owner's columns into slot r of that
//      owner's receive buffer with plain 16-byte st.shared::cluster stores
//      (fire-and-forget; an st.async per 16 bytes, each updating the owner's
//      mbarrier, measured ~15 us for 128 KB); meanwhile one thread TMA-loads the
//      CTA's own C_in slice;
//   3. cluster barrier (release/acquire: the pushes are visible);
//   4. the owner adds its S slots in the fixed order s = 0..S-1, then C_in (and the
//      optional bias / ReLU), rounds once to the output type and stores its slice
//      with 16-byte global stores.
// The sum order of every element is fixed by (K, S) alone, so results are
// deterministic and independent of the launch.  Shared memory after the mainloop:
// [receive buffer: S slots x 128 rows x BN/S F32][C_in slice 128 x BN/S], both
// inside the idle operand ring.
//
// Roles (192 threads): w0..w3 TMEM drain and reduction (warp w reads TMEM lanes
// 32w..), w4 TMA producer, w5 TMEM allocator + MMA issuer (lane 0).
#pragma once
#include "gemm_sm100.cuh"

namespace g16 {

template <int BN_, int S_, bool OUT_F16_>
struct SKCfg {
  static constexpr int BN = BN_;             // tile columns (UMMA N)
  static constexpr int S = S_;               // CTAs per cluster = K splits
  static constexpr bool OUT_F16 = OUT_F16_;
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int UMMA_K = 16;
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = BM * BK * 2;            // 16 KB
  static constexpr int B_ATOM_BYTES = 64 * BK * 2;       // 64 columns x 64 k = 8 KB
  static constexpr int B_BYTES = BN / 64 * B_ATOM_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int CW = BN / S;                      // columns reduced by each CTA
  static constexpr int U = CW / 4;                       // 16-byte units per slice row
  static_assert(U >= 8 && U % 8 == 0, "the row swizzle needs >= 8 units per row");
  static constexpr int ESIZE = OUT_F16 ? 2 : 4;
  static constexpr int SLOT_BYTES = BM * CW * 4;         // one peer's F32 partial of this slice
  static constexpr int OFF_R = 0;                        // receive buffer (after the mainloop)
  static constexpr int OFF_CIN = S * SLOT_BYTES;         // C_in slice, TMA-loaded
  static constexpr int CIN_BYTES = BM * CW * ESIZE;
  static_assert(OFF_CIN + CIN_BYTES <= RING_BYTES, "receive buffer + C_in must fit in the operand ring");
  // DSMEM exchange by bulk DMA where the own partial (S slots), the S-1 received slots
  // and the C_in slice all fit in the idle ring (S4 x 128x128): one
  // cp.async.bulk.shared::cluster copy per peer instead of 16-byte remote stores
  static constexpr int NBAR = 2 * STAGES + 3;            // full[S], empty[S], acc_full, cin, recv
  // the C_in slice lives past both the ring and the exchange buffers, so its TMA load
  // can be issued at kernel start and land under the mainloop
  static constexpr int OFF_CIN_DMA = RING_BYTES > (2 * S - 1) * SLOT_BYTES ? RING_BYTES : (2 * S - 1) * SLOT_BYTES;
  static constexpr int POST_DMA = OFF_CIN_DMA + CIN_BYTES;
  static constexpr bool DMA = POST_DMA + 1024 + NBAR * 8 + 16 <= 232448;
  static constexpr int OFF_RECV_DMA = S * SLOT_BYTES;
  static constexpr int OFF_BAR = DMA ? POST_DMA : RING_BYTES;
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int THREADS = 192;
  static constexpr int W_PRODUCER = 4, W_MMA = 5;
};

// byte offset of float column `col` of row `row` in one receive slot (rows of CW
// floats; the 16-byte unit index XOR row % 8 spreads the 32 rows a warp pushes at
// once over all banks, and keeps a row's units a permutation for the reads)
template <int CW>
__device__ __forceinline__ uint32_t slot_off(uint32_t row, uint32_t col) {
  return row * (CW * 4) + ((((col >> 2) ^ (row & 7u))) << 4) + ((col & 3u) << 2);
}

template <class Cfg>
__global__ void __launch_bounds__(192, 1)
gemm_f16_sm100_splitk_kernel(const __grid_constant__ CUtensorMap tm_a,
                             const __grid_constant__ CUtensorMap tm_b,
                             const __grid_constant__ CUtensorMap tm_c,   // C, box 32 x 128, 128B swizzle (reduce-add path)
                             const __grid_constant__ GemmParams p,
                             const __grid_constant__ PeerMaps /*unused*/,
                             const __grid_constant__ CUtensorMap tm_cin) {   // C, box CW x 128, no swizzle
  constexpr int BN = Cfg::BN, S = Cfg::S, BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int CW = Cfg::CW, U = Cfg::U;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base + Cfg::OFF_A;
  const uint32_t sB = base + Cfg::OFF_B;
  const uint32_t sR = base + Cfg::OFF_R;
  const uint32_t sC = base + Cfg::OFF_CIN;
  const uint32_t bar0 = base + Cfg::OFF_BAR;
  const uint32_t full_bar = bar0;
  const uint32_t empty_bar = bar0 + 8 * STAGES;
  const uint32_t accf_bar = bar0 + 16 * STAGES;
  const uint32_t cin_bar = accf_bar + 8;
  const uint32_t recv_bar = accf_bar + 16;   // (DMA exchange)
  const uint32_t tmem_slot = bar0 + 8 * Cfg::NBAR;

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t r = cluster_ctarank();
  // DIAGNOSTIC (p.trace): globaltimer stamps of CTA 0, thread 0 -- entry, setup done,
  // accumulator ready, all mainloops done, partial pushed, slots + C_in arrived, exit
  const bool tr = p.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr) p.trace[0] = globaltimer_ns();
  const int tile = static_cast<int>(blockIdx.x) / S;
  const int tm = tile / p.tiles_n, tn = tile % p.tiles_n;
  const int kb0 = static_cast<int>((static_cast<long long>(p.k_blocks) * r) / S);
  const int kb1 = static_cast<int>((static_cast<long long>(p.k_blocks) * (r + 1)) / S);
  const bool load_c = !p.beta0;

  if (warp == Cfg::W_PRODUCER && lane == 0) {
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_cin);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    mbar_init(accf_bar, 1);
    mbar_init(cin_bar, 1);
    mbar_init(recv_bar, 1);
    fence_mbarrier_init();
    // armed before any peer can send (sends start after the second cluster barrier)
    if constexpr (Cfg::DMA) mbar_arrive_expect_tx(recv_bar, (S - 1) * Cfg::SLOT_BYTES);
  }
  if (warp == Cfg::W_MMA) tmem_alloc<1>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");
  tmem_base = __shfl_sync(0xffffffffu, tmem_base, 0);   // (warp-uniform)
  griddep_wait();
  if (tr) p.trace[1] = globaltimer_ns();

  if (warp == Cfg::W_PRODUCER) {
    // ===================== TMA producer: this CTA's share of K =====================
    // (the whole warp runs the loop: warp-uniform TMA operands; the elected lane issues)
    {
      const bool leader = elect_one();
      if (leader) griddep_launch_dependents();
      if constexpr (Cfg::DMA) {
        if (load_c && leader) {   // C_in slice now (its own region), ready long before the reduction
          mbar_arrive_expect_tx(cin_bar, Cfg::CIN_BYTES);
          tma_load_2d_hint(base + Cfg::OFF_CIN_DMA, &tm_cin, tn * BN + static_cast<int>(r) * CW, tm * BM, cin_bar,
                           policy_evict_first());
        }
      }
      const uint64_t pol = policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(empty_bar + 8 * stage, phase ^ 1u);
        const int kc = kb * BK;
        if (leader) {
          mbar_arrive_expect_tx(full_bar + 8 * stage, Cfg::STAGE_BYTES);
          tma_load_2d_hint(sA + stage * Cfg::A_BYTES, &tm_a, kc, tm * BM, full_bar + 8 * stage, pol);
#pragma unroll
          for (int h = 0; h < BN / 64; ++h)
            tma_load_2d_hint(sB + stage * Cfg::B_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, tn * BN + 64 * h, kc,
                             full_bar + 8 * stage, pol);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == Cfg::W_MMA) {
    // ===================== MMA issuer =====================
    // (the whole warp runs the loop: uniform operands; the elected lane issues)
    {
      const bool leader = elect_one();
      const uint32_t idesc = (idesc_f16_f32acc<BM, BN>() & (p.accum_f16 ? ~(3u << 4) : ~0u)) |
                             (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(full_bar + 8 * stage, phase);
        tc_fence_after();
        const uint32_t a_s = sA + stage * Cfg::A_BYTES;
        const uint32_t b_s = sB + stage * Cfg::B_BYTES;
#pragma unroll
        for (int k = 0; k < BK / Cfg::UMMA_K; ++k)
          if (leader)
            umma_f16<1>(tmem_base, desc_sw128(a_s + 32 * k, 16, 1024),
                        desc_sw128(b_s + 2048 * k, Cfg::B_ATOM_BYTES, 1024), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        if (leader) umma_commit(empty_bar + 8 * stage);
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      }
      if (leader) umma_commit(accf_bar);   // with no k-blocks (K split finer than K) it arrives at once
    }
  } else {
    mbar_wait(accf_bar, 0);    // this CTA's accumulator is complete (and its ring idle)
    tc_fence_after();
    if (tr) p.trace[2] = globaltimer_ns();
  }

  // ===================== all mainloops done: the rings become receive buffers =====================
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (tr) p.trace[3] = globaltimer_ns();
  // F32 C, plain C += A.B: no DSMEM exchange at all.  Each CTA stages its whole partial
  // (128B-swizzled 32-column boxes) and the TMA unit adds it into C (reduce-add, one RN
  // add in L2), one column slice per step in a rotation -- in step j CTA r adds slice
  // (r + j) % S -- with a cluster barrier between steps, so every element receives
  // C_in + p_s + p_(s-1) + ... in a fixed order (deterministic).
  const bool red = !Cfg::OUT_F16 && load_c && p.c_reduce && p.bias == nullptr && !p.relu && !p.c_ragged;
  if (red) {
    if (warp < 4) {
      const uint32_t row = warp * 32 + lane;
      const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
      const bool empty_share = kb1 <= kb0;   // -0 is the additive identity for every x
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + 32 * c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = __uint_as_float(v[j]);
          if (p.accum_f16) x = f16x2_to_f32(v[j]).x;
          v[j] = __float_as_uint(empty_share ? -0.f : x);
        }
        const uint32_t box = sR + static_cast<uint32_t>(c) * (BM * 128);   // 128 rows x 128 B
#pragma unroll
        for (int j = 0; j < 8; ++j)
          sts128u(box + swz<128>(row, static_cast<uint32_t>(j)), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
      fence_proxy_async_smem();
    }
    __syncthreads();
    if (tr) p.trace[4] = globaltimer_ns();
#pragma unroll 1
    for (int j = 0; j < S; ++j) {
      if (threadIdx.x == 0) {
        const int sl = (static_cast<int>(r) + j) % S;
#pragma unroll 1
        for (int b = sl * (CW / 32); b < (sl + 1) * (CW / 32); ++b)
          tma_reduce_add_2d_hint(&tm_c, tn * BN + 32 * b, tm * BM, sR + static_cast<uint32_t>(b) * (BM * 128),
                                 policy_evict_first());
        bulk_commit_group();
        bulk_wait_group<0>();   // this step's adds are performed before the barrier
      }
      __syncwarp();
      cluster_sync();
    }
    if (tr) p.trace[5] = globaltimer_ns();
  } else if constexpr (Cfg::DMA) {
    const uint32_t sStage = base;                         // own partial, slot-major by owner
    const uint32_t sRecv = base + Cfg::OFF_RECV_DMA;      // S-1 slots from the peers
    const uint32_t sCin = base + Cfg::OFF_CIN_DMA;        // this CTA's C_in slice
    if (warp < 4) {
      const uint32_t row = warp * 32 + lane;
      const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
      const bool empty_share = kb1 <= kb0;   // this CTA accumulated nothing: its partial is 0
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + 32 * c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = __uint_as_float(v[j]);
          if (p.accum_f16) x = f16x2_to_f32(v[j]).x;
          v[j] = __float_as_uint(empty_share ? 0.f : x);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = 32 * c + 4 * j;          // tile column of this 16-byte unit
          const int sl = col / CW;                 // its owner (a constant after unrolling)
          sts128u(sStage + sl * Cfg::SLOT_BYTES + slot_off<CW>(row, static_cast<uint32_t>(col % CW)), v[4 * j],
                  v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
      fence_proxy_async_smem();   // generic writes before the bulk copies read them
    }
    __syncthreads();
    if (tr) p.trace[4] = globaltimer_ns();
    if (threadIdx.x == 0) {   // one bulk copy per peer: my slot s -> slot (r < s ? r : r - 1) of CTA s
#pragma unroll 1
      for (int sl = 0; sl < S; ++sl) {
        if (sl == static_cast<int>(r)) continue;
        const uint32_t slot = r < static_cast<uint32_t>(sl) ? r : r - 1u;
        bulk_copy_s2dsmem(mapa_shared(sRecv + slot * Cfg::SLOT_BYTES, static_cast<uint32_t>(sl)),
                          sStage + sl * Cfg::SLOT_BYTES, Cfg::SLOT_BYTES,
                          mapa_shared(recv_bar, static_cast<uint32_t>(sl)));
      }
    }
    if (warp < 4) {
      mbar_wait(recv_bar, 0);
      if (load_c) mbar_wait(cin_bar, 0);
      if (tr) p.trace[5] = globaltimer_ns();
#pragma unroll 4
      for (int i = static_cast<int>(threadIdx.x); i < BM * U; i += 128) {
        const int lr = i / U, lc = 4 * (i % U);
        const int grow = tm * BM + lr, gcol = tn * BN + static_cast<int>(r) * CW + lc;
        if (grow >= p.M || gcol >= p.N) continue;
        const uint32_t off = slot_off<CW>(static_cast<uint32_t>(lr), static_cast<uint32_t>(lc));
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int sl = 0; sl < S; ++sl) {   // partials in the fixed order s = 0..S-1
          const uint32_t src = sl == static_cast<int>(r)
                                   ? sStage + sl * Cfg::SLOT_BYTES + off
                                   : sRecv + static_cast<uint32_t>(sl < static_cast<int>(r) ? sl : sl - 1) *
                                                 Cfg::SLOT_BYTES + off;
          const float4 t = lds128(src);
          if (sl == 0) acc = t;
          else { acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w; }
        }
        float o[4] = {acc.x, acc.y, acc.z, acc.w};
        if (load_c) {
          const uint32_t coff = sCin + static_cast<uint32_t>((lr * CW + lc) * Cfg::ESIZE);
          if constexpr (!Cfg::OUT_F16) {
            const float4 ci = lds128(coff);
            o[0] = ci.x + o[0]; o[1] = ci.y + o[1]; o[2] = ci.z + o[2]; o[3] = ci.w + o[3];
          } else {
            uint32_t lo, hi;
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(coff));
            const float2 a = f16x2_to_f32(lo), b = f16x2_to_f32(hi);
            o[0] = a.x + o[0]; o[1] = a.y + o[1]; o[2] = b.x + o[2]; o[3] = b.y + o[3];
          }
        }
        const int nv = min(4, p.N - gcol);           // valid columns of this unit
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (p.bias != nullptr && e < nv) o[e] += __ldg(p.bias + gcol + e);
          if (p.relu) o[e] = relu_keep_nan(o[e]);
        }
        if constexpr (!Cfg::OUT_F16) {
          float* cp = static_cast<float*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc + gcol;
          if (nv == 4) *reinterpret_cast<float4*>(cp) = make_float4(o[0], o[1], o[2], o[3]);
          else for (int e = 0; e < nv; ++e) cp[e] = o[e];
        } else {
          uint16_t* cp = static_cast<uint16_t*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc + gcol;
          const uint32_t lo = cvt_f16x2_rn(o[0], o[1]), hi = cvt_f16x2_rn(o[2], o[3]);
          if (nv == 4) {
            *reinterpret_cast<uint2*>(cp) = make_uint2(lo, hi);
          } else {
            const uint16_t h[4] = {static_cast<uint16_t>(lo), static_cast<uint16_t>(lo >> 16),
                                   static_cast<uint16_t>(hi), static_cast<uint16_t>(hi >> 16)};
            for (int e = 0; e < nv; ++e) cp[e] = h[e];
          }
        }
      }
    }
    if (tr) p.trace[7] = globaltimer_ns();
    // every copy into every CTA has landed (each owner waited) before any CTA exits:
    // the copies read their senders' shared memory
    __syncwarp();
    cluster_sync();
  } else {
  if (warp == Cfg::W_PRODUCER && lane == 0 && load_c) {
    mbar_arrive_expect_tx(cin_bar, Cfg::CIN_BYTES);
    tma_load_2d_hint(sC, &tm_cin, tn * BN + static_cast<int>(r) * CW, tm * BM, cin_bar, policy_evict_first());
  }
  if (warp < 4) {
    // ---- push: TMEM partial -> slot r of each owner's receive buffer
    const uint32_t row = warp * 32 + lane;
    const uint32_t t_row = tmem_base + ((warp * 32u) << 16);
    const bool empty_share = kb1 <= kb0;   // this CTA accumulated nothing: its partial is 0
    uint32_t dst[S];
#pragma unroll
    for (int s = 0; s < S; ++s) dst[s] = mapa_shared(sR + r * Cfg::SLOT_BYTES, static_cast<uint32_t>(s));
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_row + 32 * c, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float x = __uint_as_float(v[j]);
        if (p.accum_f16) x = f16x2_to_f32(v[j]).x;
        v[j] = __float_as_uint(empty_share ? 0.f : x);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = 32 * c + 4 * j;          // tile column of this 16-byte unit
        const int s = col / CW;                  // its owner (a constant after unrolling)
        const uint32_t o = slot_off<CW>(row, static_cast<uint32_t>(col % CW));
        if (static_cast<uint32_t>(s) == r)   // this CTA's own slice: a local store
          sts128u(sR + r * Cfg::SLOT_BYTES + o, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        else
          st_cluster_v4(dst[s] + o, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    if (tr) p.trace[4] = globaltimer_ns();
  }
  __syncwarp();
  cluster_sync();   // every push has landed in its owner's buffer
  if (warp < 4) {
    // ---- reduce this CTA's slice: S slots in order, then C_in; round once; store
    if (load_c) mbar_wait(cin_bar, 0);
    if (tr) p.trace[5] = globaltimer_ns();
#pragma unroll 4
    for (int i = static_cast<int>(threadIdx.x); i < BM * U; i += 128) {
      const int lr = i / U, lc = 4 * (i % U);
      const int grow = tm * BM + lr, gcol = tn * BN + static_cast<int>(r) * CW + lc;
      if (grow >= p.M || gcol >= p.N) continue;
      const uint32_t off = slot_off<CW>(static_cast<uint32_t>(lr), static_cast<uint32_t>(lc));
      float4 acc = lds128(sR + off);
#pragma unroll
      for (int s = 1; s < S; ++s) {
        const float4 t = lds128(sR + s * Cfg::SLOT_BYTES + off);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      float o[4] = {acc.x, acc.y, acc.z, acc.w};
      if (load_c) {
        const uint32_t coff = sC + static_cast<uint32_t>((lr * CW + lc) * Cfg::ESIZE);
        if constexpr (!Cfg::OUT_F16) {
          const float4 ci = lds128(coff);
          o[0] = ci.x + o[0]; o[1] = ci.y + o[1]; o[2] = ci.z + o[2]; o[3] = ci.w + o[3];
        } else {
          uint32_t lo, hi;
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(coff));
          const float2 a = f16x2_to_f32(lo), b = f16x2_to_f32(hi);
          o[0] = a.x + o[0]; o[1] = a.y + o[1]; o[2] = b.x + o[2]; o[3] = b.y + o[3];
        }
      }
      const int nv = min(4, p.N - gcol);           // valid columns of this unit
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (p.bias != nullptr && e < nv) o[e] += __ldg(p.bias + gcol + e);
        if (p.relu) o[e] = relu_keep_nan(o[e]);
      }
      if constexpr (!Cfg::OUT_F16) {
        float* cp = static_cast<float*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc + gcol;
        if (nv == 4) *reinterpret_cast<float4*>(cp) = make_float4(o[0], o[1], o[2], o[3]);
        else for (int e = 0; e < nv; ++e) cp[e] = o[e];
      } else {
        uint16_t* cp = static_cast<uint16_t*>(p.c_ptr) + static_cast<long long>(grow) * p.ldc + gcol;
        const uint32_t lo = cvt_f16x2_rn(o[0], o[1]), hi = cvt_f16x2_rn(o[2], o[3]);
        if (nv == 4) {
          *reinterpret_cast<uint2*>(cp) = make_uint2(lo, hi);
        } else {
          const uint16_t h[4] = {static_cast<uint16_t>(lo), static_cast<uint16_t>(lo >> 16),
                                 static_cast<uint16_t>(hi), static_cast<uint16_t>(hi >> 16)};
          for (int e = 0; e < nv; ++e) cp[e] = h[e];
        }
      }
    }
  }
  }   // DSMEM path
  __syncwarp();
  if (tr) p.trace[6] = globaltimer_ns();
  if (warp == Cfg::W_MMA) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace g16
