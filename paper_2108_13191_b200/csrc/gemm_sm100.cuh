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
//  C in registers, hoisted          accumulator in TMEM for a K chunk, promoted to
//                                               F32 registers of the epilogue warps (see below)
//  1-stage k-loop split (Sec 3.5)    STAGES-deep mbarrier ring (full/empty)
//  __syncthreads around copies (Sec 3.6)        per-stage mbarriers + tcgen05.commit
//  128-bit vector global->smem copies (3.7)     cp.async.bulk.tensor boxes of 8-16 KB
//  one thread block per C tile (Sec 3.9)        persistent clusters, grouped raster schedule
//  C stored once per warp tile      C_in added once in F32; smem -> TMA store,
//                                               overlapped with the next chunk's MMAs
//
// Accumulation (R4): the tensor cores' F32 accumulator truncates on
// every K=16 step, so a single TMEM chain's relative error grows ~1.2e-6 per
// 1024 of K (measured; bitwise the same as cuBLAS) and crosses BASELINE's 1e-5
// bound near K = 8400.  The K loop is therefore cut into chunks of
// `kb_per_chunk` k-blocks: each chunk accumulates in a fresh TMEM buffer
// (double-buffered, so the MMA never waits for the drain), and the epilogue
// warps add the chunk into F32 registers with round-to-nearest adds.  The
// error then scales with the chunk length, not with K.
//
// Warp roles (352 threads): w0..w7 epilogue, w8 TMA producer, w9 MMA issuer
// (pair leader only), w10 TMEM allocator.  The control warps get the highest
// ids because the warp arbiter favours higher warp ids: the single-thread
// producer and MMA loops must not queue behind epilogue bursts on their SMSP.
// Epilogue warp w reads TMEM lanes 32*(w%4).. (hardware quadrant rule) and
// accumulator columns [w/4 * BN/2, +BN/2).
#pragma once
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"

#ifndef G16_DIAG_NO_MMA
#define G16_DIAG_NO_MMA 0   // DIAGNOSTIC builds only (wrong results): 1 = the MMA warp skips the
                            // tcgen05.mma instructions, so the TMA ring runs alone
#endif

namespace g16 {

// Extra destinations of the C tile (fused N-shard all-gather, gemm_f16_gather):
// every finished C chunk is TMA-stored to the local C and to each peer buffer.
constexpr int kMaxPeers = 7;
struct PeerMaps {
  CUtensorMap m[kMaxPeers];
};

struct GemmParams {
  int M, N, K;
  int tiles_m, tiles_n, num_tiles;  // tiles of (128*CG) x BN
  int k_blocks;                     // ceil(K / BK): smem ring stages per tile
  int kb_per_chunk;                 // k-blocks accumulated in TMEM before promotion to registers
  int k_chunks;                     // ceil(k_blocks / kb_per_chunk)
  int k_splits;                     // split-K kernels (gemm_sm100_splitk.cuh): CTAs per cluster,
                                    // each accumulating a contiguous share of the k-blocks
  int group_m;                      // raster group height in tiles
  int snake;                        // 1: odd raster groups walk their columns right to left
  int c_reduce;                     // 1: F32 C += acc by TMA reduce-add (C_in never staged; see epilogue)
  int c_ragged;                     // N * sizeof(C) % 16 != 0: TMA stores would write a
                                    // whole 16-byte granule past column N-1, so the chunk
                                    // holding column N-1 is stored element-wise instead
  void* c_ptr;                      // C base (used only by that ragged-N store path)
  int n_peers;                      // extra destinations of C_out (0 = plain GEMM)
  void* peer_ptr[kMaxPeers];        // their bases, for the ragged-N store path
  long long ldc;                    // C leading dimension in elements
  int ring_stages;                  // smem ring depth in use (1..STAGES; ablation of Sec 3.5)
  int acc_bufs;                     // TMEM accumulator buffers in use (2 = epilogue overlaps MMA)
  unsigned long long* trace;        // DIAGNOSTIC ONLY (null normally): per-tile globaltimer stamps
                                    // of CTA 0 (MMA start/end + SM cycles, epilogue drain/store),
                                    // 8 per tile; row 62 = kernel entry/setup/exit
  // fused epilogue: out = relu?(beta * C_in + A.B + bias[col])
  int in_bf16;                      // 1: A and B are bfloat16 (idesc a/b_format = BF16)
  int beta0;                        // 1: C_in is not read (beta = 0)
  int relu;                         // 1: max(x, 0) with NaN propagated, before the rounding
  const float* bias;                // null, or N floats added per column (16-byte aligned)
  int accum_f16;                    // EXPERIMENT (SURVEY A3 "strict"): idesc c_format = F16, the
                                    // tensor core accumulates in binary16; TMEM cells hold the
                                    // F16 value in their low 16 bits
  int l2_hints;                     // 1: TMA loads/stores carry L2 eviction-priority hints
                                    // (A evict_last: re-read by the next wave of tiles;
                                    //  C evict_first: streamed once)
  // stream-K (kernel built with SK = true; F32 C with the reduce-add epilogue, or F16 C --
  // DESIGN.md R18): tiles [sk_tile0, num_tiles) are shared out as equal runs of (tile,
  // k-block) units, one run per cluster, so the last partial wave is spread over every cluster
  int sk_tile0;
  int sk_snap;                      // run boundaries within this many k-blocks of a tile edge snap to it
  unsigned* sk_flags;               // token counters, one per (cluster boundary, CTA, epilogue warp)
  int tail_ring;                    // 1: the last tile's output chunks are staged all at once in the
                                    // (then idle) operand ring instead of cycling through the slots
};

// The work of one cluster, in the order it is processed: its data-parallel tiles
// cluster, cluster + ncl, ... below sk_tile0, then its run [u0, u1) of the stream-K units
// (unit = tile * k_blocks + k-block over the stream-K tiles), tile by tile from the LAST
// tile of the run down.  A tile split between clusters c and c + 1 is therefore the first
// item of c (k-blocks [0, x)) and the last item of c + 1 (k-blocks [x, k_blocks)): c adds
// its partial into C first and posts a token; c + 1 takes it before adding its own, so the
// two reduce-adds into C happen in a fixed order (deterministic result), and a cluster
// only ever waits on a lower-numbered one that did that work first.  The host gives every
// cluster at least k_blocks units, so a tile is split at most once -- or, below one wave,
// at least k_blocks / 2, so a tile is split at most three ways (a middle part waits for
// cluster - 1 and posts for cluster + 1: chains of waits stay two long).
struct Work {
  int n_dp, n_items, t_hi;
  int u0, u1;   // (the host keeps the stream-K unit count below 2^31)
};
struct Item {
  int tile, kb_lo, kb_hi;
  bool wait, signal;   // wait: k-blocks [0, kb_lo) are cluster-1's; signal: [kb_hi, k_blocks) are cluster+1's
};
// token counter of (cluster boundary b, CTA rank, epilogue warp): the writer warp and
// the waiting warp cover the same 32 x BN/2 region of the shared tile
constexpr int kSkFlagSlots = 1 << 16;   // the device pool; each launch takes a window of it
__device__ __forceinline__ int sk_slot(int b, uint32_t rank, uint32_t ew) {
  return (b * 2 + static_cast<int>(rank)) * 8 + static_cast<int>(ew);
}
// A run boundary that falls within `snap` k-blocks of a tile edge moves onto the edge: no
// sliver of a tile is split off, which would cost a whole extra store phase for a few
// k-blocks of work (the host keeps snap <= k_blocks / 4, so runs stay >= k_blocks / 2)
__device__ __forceinline__ int sk_boundary(long long b, int kb, int snap) {
  const int r = static_cast<int>(b % kb);
  if (r != 0 && r < snap) return static_cast<int>(b - r);
  if (r != 0 && kb - r < snap) return static_cast<int>(b - r + kb);
  return static_cast<int>(b);
}
template <bool SK>
__device__ __forceinline__ Work work_of(const GemmParams& p, int cluster, int ncl) {
  Work w;
  const int dp_end = SK ? p.sk_tile0 : p.num_tiles;
  w.n_dp = cluster < dp_end ? (dp_end - cluster + ncl - 1) / ncl : 0;
  w.n_items = w.n_dp;
  w.t_hi = 0;
  w.u0 = w.u1 = 0;
  if constexpr (SK) {
    const long long units = static_cast<long long>(p.num_tiles - p.sk_tile0) * p.k_blocks;
    w.u0 = sk_boundary(units * cluster / ncl, p.k_blocks, p.sk_snap);
    w.u1 = sk_boundary(units * (cluster + 1) / ncl, p.k_blocks, p.sk_snap);
    if (w.u1 > w.u0) {
      w.t_hi = (w.u1 - 1) / p.k_blocks;
      w.n_items += w.t_hi - w.u0 / p.k_blocks + 1;
    }
  }
  return w;
}
template <bool SK>
__device__ __forceinline__ Item item_of(const GemmParams& p, const Work& w, int cluster, int ncl, int i) {
  Item it;
  if (!SK || i < w.n_dp) {
    it.tile = cluster + i * ncl;
    it.kb_lo = 0;
    it.kb_hi = p.k_blocks;
    it.wait = it.signal = false;
    return it;
  }
  const int t = w.t_hi - (i - w.n_dp);
  const int t0 = t * p.k_blocks;
  it.tile = p.sk_tile0 + t;
  it.kb_lo = max(w.u0, t0) - t0;
  it.kb_hi = min(w.u1, t0 + p.k_blocks) - t0;
  it.wait = it.kb_lo > 0;
  it.signal = it.kb_hi < p.k_blocks;
  return it;
}

template <int CG_, int BN_, int STAGES_, bool OUT_F16_, int EPI_SLOTS_ = 1, int BK_ = 64, bool PEERS_ = false,
          int MC_ = 1, bool SW_ = true>
struct KCfg {
  // SW = false: ABLATION ONLY (option swizzle = -1; the B200 analogue of the paper's
  // unpadded shared memory, Sec. 3.3): operands staged in the no-swizzle
  // "interleaved" UMMA layout (16-byte TMA boxes, core matrices of 8 rows x 16 B) and the
  // epilogue staging in plain rows (32 lanes of a warp hit the same banks)
  static constexpr bool SW = SW_;
  static constexpr int CG = CG_;            // CTAs per MMA (cta_group)
  static constexpr int MC = MC_;            // cta_group::1: CTAs per cluster sharing (multicasting) A along N;
                                            // cta_group::2: CTA pairs per cluster sharing B along M
  static_assert(MC == 1 || (CG == 1 && (MC == 2 || MC == 4)) || (CG == 2 && MC == 2 && !PEERS_ && SW_),
                "multicast: 1-CTA tiles 2 or 4 per cluster (A), or 2 CTA pairs per cluster (B)");
  static constexpr int BN = BN_;            // UMMA N (tile columns)
  static constexpr int STAGES = STAGES_;
  static constexpr bool OUT_F16 = OUT_F16_;
  static constexpr bool PEERS = PEERS_;     // epilogue also stores C to p.n_peers peer buffers
  static constexpr int BM = 128;            // rows per CTA (TMEM lanes)
  static constexpr int BK = BK_;            // K per stage: KH 64-deep (128 B) swizzle spans of F16
  static constexpr int KH = BK / 64;
  static_assert(BK == 64 || BK == 128, "K per stage");
  static constexpr int UMMA_K = 16;
  static constexpr int BN_CTA = BN / CG;    // B columns staged per CTA
  static_assert(BN_CTA % 64 == 0, "B is staged in 64-column (128 B) swizzle atoms");
  static_assert(BN % 64 == 0 && BN <= 256, "UMMA N");
  static constexpr int A_HALF_BYTES = BM * 64 * 2;   // 16 KB: 128 rows x one 64-deep K span
  static constexpr int A_BYTES = KH * A_HALF_BYTES;
  static constexpr int B_ATOM_BYTES = 64 * 64 * 2;    // 64 cols x 64 k = 8 KB
  static constexpr int B_HALF_BYTES = BN_CTA * 64 * 2;
  static constexpr int B_BYTES = KH * B_HALF_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_COLS = BN;                 // one accumulator buffer
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int EPI_WARPS = 8;
  static constexpr int CPW = BN / 2;                  // accumulator columns per epilogue warp
  static constexpr int ESIZE = OUT_F16 ? 2 : 4;
  static constexpr int CW = (128 / ESIZE < CPW) ? 128 / ESIZE : CPW;   // output chunk columns
  static constexpr int RB = CW * ESIZE;               // staging row bytes: 128 or 64
  static_assert(RB == 128 || RB == 64, "staging rows are one 128B or 64B swizzle span");
  static constexpr int NOUT = CPW / CW;               // output chunks per warp per tile
  static constexpr int EPI_SLOTS = EPI_SLOTS_;
  static constexpr int PRE = (EPI_SLOTS < NOUT) ? EPI_SLOTS : NOUT;   // C_in chunks loaded at tile start
  static constexpr int EPI_BUF = 32 * 128;            // 32 rows x up to 128 B
  // the last tile of a CTA can stage every output chunk at once in the idle operand ring
  static constexpr bool TAIL_RING = NOUT > EPI_SLOTS && EPI_WARPS * NOUT * EPI_BUF <= STAGES * (A_BYTES + B_BYTES);
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = STAGES * A_BYTES;
  static constexpr int OFF_E = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_E + EPI_WARPS * EPI_SLOTS * EPI_BUF;
  // barriers: full[S], empty[S], acc_full[2], acc_empty[2], epi[8][slots], tmem slot
  static constexpr int NBAR = 2 * STAGES + 4 + EPI_WARPS * EPI_SLOTS;
  static constexpr int SMEM_BYTES = 1024 + OFF_BAR + NBAR * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static constexpr int THREADS = 352;                 // 11 warps: <= 3 per SMSP x 168 registers
  static constexpr int W_PRODUCER = 8, W_MMA = 9, W_ALLOC = 10;
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

// UMMA shared-memory descriptor, no swizzle ("interleaved" canonical layout, layout type 0):
// core matrices of 8 rows x 16 B stored contiguously.  For both majors LBO is the byte stride
// between core matrices adjacent along K and SBO the stride between those adjacent along M / N
// (cute's make_umma_desc for SWIZZLE_NONE: K-major ((8,m),(T,2)):((1T,SBO),(1,LBO)), MN-major
// ((1,n),(8,k)):((X,SBO),(1,LBO)) in 16-byte units).
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
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
  if (p.snake && (g & 1)) tn = p.tiles_n - 1 - tn;
}

// Byte offset of 16-byte unit j of row r in a TMA-swizzled staging box whose
// rows are RB bytes (128B swizzle: j ^ r%8; 64B swizzle: j ^ (r/2)%4).
template <int RB>
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t j) {
  return r * RB + ((j ^ (((r * RB) >> 7) & (RB / 16 - 1))) << 4);
}

__device__ __forceinline__ float4 load_bias4(const float* bias, int col, int n) {
  if (col + 3 < n) return __ldg(reinterpret_cast<const float4*>(bias + col));
  float4 r;
  r.x = col < n ? __ldg(bias + col) : 0.f;
  r.y = col + 1 < n ? __ldg(bias + col + 1) : 0.f;
  r.z = col + 2 < n ? __ldg(bias + col + 2) : 0.f;
  r.w = 0.f;
  return r;
}
__device__ __forceinline__ float relu_keep_nan(float x) { return (x > 0.f || x != x) ? x : 0.f; }

template <class Cfg, bool SK = false>
__global__ void __launch_bounds__(352, 1)
gemm_f16_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_c,
                      const __grid_constant__ GemmParams p,
                      const __grid_constant__ PeerMaps peers,
                      const __grid_constant__ CUtensorMap /*C_in slice map: split-K kernels only*/) {
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
  // DIAGNOSTIC trace: the CTA to trace is read from trace[8 * 63 + 7] (0 = CTA 0)
  const bool trace_me = p.trace != nullptr && blockIdx.x == static_cast<unsigned>(p.trace[8 * 63 + 7]);
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 0] = globaltimer_ns();
  constexpr int MC = Cfg::MC;
  const uint32_t rank = (CG == 2) ? (cluster_ctarank() & 1u) : 0u;   // rank in the CTA pair
  // A multicast (MC > 1, 1-CTA tiles): the MC CTAs of a cluster own tiles (tm, MC * tg + r),
  // r = rank in the cluster; each loads 128 / MC rows of the shared A box and multicasts them.
  // B multicast (MC = 2, CTA pairs): pair p of the cluster owns tile (2 * tg + p, tn); both pairs
  // need the same B columns, so each loads one of the two 64-column atoms of a CTA's half and
  // multicasts it into the same-rank CTA of the other pair
  // Hybrid launch (GEMM_CFG_PAIR2_256x256_MCH: cluster dim 2, preferred cluster dim 4): the
  // hardware groups blocks 4i..4i+3 into one 4-CTA cluster where it can place one (~132 of 148
  // SMs) and into two 2-CTA clusters elsewhere.  The schedule is the same either way (pair
  // (blockIdx / 2) % 2 of group blockIdx / 4 owns tile (2 tg + p, tn)); only a 4-CTA cluster
  // multicasts B (`mc`), a lone pair loads both of its B atoms itself
  const uint32_t mrank = (MC > 1) ? cluster_ctarank() : 0u;
  const bool mc = (CG == 2 && MC > 1) ? (cluster_nctarank() == 4u) : (MC > 1);
  const uint32_t pidx = (CG == 2 && MC > 1) ? ((blockIdx.x >> 1) & 1u) : 0u;   // pair within the group of 4
  const uint32_t lead = (CG == 2 && MC > 1) ? (mrank & ~1u) : 0u;  // cluster rank of this pair's leader
  // the schedule above assumes a cluster's CTAs are consecutive blocks (ctarank = blockIdx % size),
  // which tools/probe_pref_cluster.cu measured for preferred clusters too; fail loudly otherwise
  if constexpr (CG == 2 && MC > 1)
    if (mrank != (blockIdx.x & (mc ? 3u : 1u))) __trap();

  if (warp == Cfg::W_PRODUCER && lane == 0) {
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
    prefetch_tmap(&tm_c);
    if constexpr (Cfg::PEERS)
      for (int d = 0; d < p.n_peers; ++d) prefetch_tmap(&peers.m[d]);
  }
  if (warp == Cfg::W_MMA && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      // MC > 1: a stage is refilled once every CTA's MMAs used it
      mbar_init(empty_bar + 8 * s, (CG == 2 && MC > 1) ? (mc ? 2 : 1) : MC);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf_bar + 8 * b, 1);
      mbar_init(acce_bar + 8 * b, Cfg::EPI_WARPS * CG);
    }
    for (int i = 0; i < Cfg::EPI_WARPS * Cfg::EPI_SLOTS; ++i) mbar_init(epi_bar + 8 * i, 1);
    fence_mbarrier_init();
  }
  if (warp == Cfg::W_ALLOC) tmem_alloc<CG>(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  if constexpr (CG == 2 || MC > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");
  tmem_base = __shfl_sync(0xffffffffu, tmem_base, 0);   // (warp-uniform)
  // PDL: everything above (barrier init, TMEM allocation, descriptor prefetch)
  // overlapped the previous grid's tail; no global memory is touched before this
  // (bar the diagnostic trace stamps)
  griddep_wait();
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 1] = globaltimer_ns();

  const int cluster = static_cast<int>(blockIdx.x) / (CG * MC);
  const int nclusters = static_cast<int>(gridDim.x) / (CG * MC);
  const Work work = work_of<SK>(p, cluster, nclusters);

  if (warp == Cfg::W_PRODUCER) {
    // ===================== TMA producer =====================
    // The whole warp runs the loop (warp-uniform operands: no per-instruction elect/R2UR
    // waterfall around each TMA); the elected lane issues.
    {
      const bool leader = elect_one();
      const uint32_t full_leader = (CG == 2) ? mapa_shared(full_bar, lead) : full_bar;
      const uint64_t pol_a = p.l2_hints ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_b = policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (; it < work.n_items; ++it) {
        const Item itm = item_of<SK>(p, work, cluster, nclusters, it);
        const int tile = itm.tile;
        int tm, tn;
        tile_coords(tile, p, tm, tn);
        if constexpr (MC > 1 && CG == 1) tn = MC * tn + static_cast<int>(mrank);
        if constexpr (MC > 1 && CG == 2) tm = MC * tm + static_cast<int>(pidx);
        const int a_row = tm * BM * CG + static_cast<int>(rank) * BM;
        const int b_col = tn * BN + static_cast<int>(rank) * Cfg::BN_CTA;
        if (it + 1 == work.n_items && leader) griddep_launch_dependents();   // last tile: let the next grid ramp
        for (int kb = itm.kb_lo; kb < itm.kb_hi; ++kb) {
          mbar_wait(empty_bar + 8 * stage, phase ^ 1u);
          if (leader) {
          if (rank == 0) mbar_arrive_expect_tx(full_bar + 8 * stage, Cfg::STAGE_BYTES * CG);
          const uint32_t fb = full_leader + 8 * stage;
          const uint32_t a_dst = sA + stage * Cfg::A_BYTES;
          const uint32_t b_dst = sB + stage * Cfg::B_BYTES;
#pragma unroll
          for (int kh = 0; kh < Cfg::KH; ++kh) {
            const int kc = kb * BK + 64 * kh;
            if constexpr (CG == 2 && !Cfg::SW) {
              // no swizzle: 16-byte-wide boxes -- A: 8 K-columns x 128 rows (2 KB), B: 8 N-columns
              // x 64 K-rows (1 KB), each one column of core matrices
#pragma unroll
              for (int g = 0; g < 8; ++g)
                tma_load_2d_pair_hint(a_dst + kh * Cfg::A_HALF_BYTES + g * 2048, &tm_a, kc + 8 * g, a_row, fb, pol_a);
#pragma unroll
              for (int g = 0; g < Cfg::BN_CTA / 8; ++g)
                tma_load_2d_pair_hint(b_dst + kh * Cfg::B_HALF_BYTES + g * 1024, &tm_b, b_col + 8 * g, kc, fb, pol_b);
            } else if constexpr (CG == 2 && MC > 1) {
              tma_load_2d_pair_hint(a_dst + kh * Cfg::A_HALF_BYTES, &tm_a, kc, a_row, fb, pol_a);
              static_assert(Cfg::BN_CTA / 64 == MC, "one B atom per pair");
              if (mc) {
                tma_load_2d_pair_mc_hint(b_dst + kh * Cfg::B_HALF_BYTES + pidx * Cfg::B_ATOM_BYTES, &tm_b,
                                         b_col + 64 * static_cast<int>(pidx), kc, fb,
                                         static_cast<uint16_t>((1u << mrank) | (1u << (mrank ^ 2u))), pol_b);
              } else {
#pragma unroll
                for (int h = 0; h < MC; ++h)
                  tma_load_2d_pair_hint(b_dst + kh * Cfg::B_HALF_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h,
                                        kc, fb, pol_b);
              }
            } else if constexpr (CG == 2) {
              tma_load_2d_pair_hint(a_dst + kh * Cfg::A_HALF_BYTES, &tm_a, kc, a_row, fb, pol_a);
#pragma unroll
              for (int h = 0; h < Cfg::BN_CTA / 64; ++h)
                tma_load_2d_pair_hint(b_dst + kh * Cfg::B_HALF_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h,
                                      kc, fb, pol_b);
            } else if constexpr (MC > 1) {
              // this CTA's 128 / MC rows of A, multicast into every CTA of the cluster
              tma_load_2d_mc_hint(a_dst + kh * Cfg::A_HALF_BYTES + mrank * (Cfg::A_HALF_BYTES / MC), &tm_a, kc,
                                  a_row + static_cast<int>(mrank) * (BM / MC), fb, (1u << MC) - 1u, pol_a);
#pragma unroll
              for (int h = 0; h < Cfg::BN_CTA / 64; ++h)
                tma_load_2d_hint(b_dst + kh * Cfg::B_HALF_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h, kc,
                                 fb, pol_b);
            } else {
              tma_load_2d_hint(a_dst + kh * Cfg::A_HALF_BYTES, &tm_a, kc, a_row, fb, pol_a);
#pragma unroll
              for (int h = 0; h < Cfg::BN_CTA / 64; ++h)
                tma_load_2d_hint(b_dst + kh * Cfg::B_HALF_BYTES + h * Cfg::B_ATOM_BYTES, &tm_b, b_col + 64 * h, kc,
                                 fb, pol_b);
            }
          }
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
      const uint32_t idesc = (idesc_f16_f32acc<BM * CG, BN>() & (p.accum_f16 ? ~(3u << 4) : ~0u)) |
                             (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int it = 0;
      for (; it < work.n_items; ++it) {
        const Item itm = item_of<SK>(p, work, cluster, nclusters, it);
        const int n_chunks = SK ? (itm.kb_hi - itm.kb_lo + p.kb_per_chunk - 1) / p.kb_per_chunk : p.k_chunks;
        const bool tr = trace_me && leader && it < 60;
        uint64_t clk0 = 0;
        if (tr) {
          p.trace[8 * it + 0] = globaltimer_ns();
          clk0 = clock64();
        }
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(acce_bar + 8 * acc, acc_phase ^ 1u);
          tc_fence_after();
          if (tr && ch == 0) p.trace[8 * it + 1] = globaltimer_ns();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
          const int kb0 = itm.kb_lo + ch * p.kb_per_chunk;
          const int kb1 = min(kb0 + p.kb_per_chunk, itm.kb_hi);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full_bar + 8 * stage, phase);
            tc_fence_after();
            const uint32_t a_s = sA + stage * Cfg::A_BYTES;
            const uint32_t b_s = sB + stage * Cfg::B_BYTES;
#pragma unroll
            for (int k = 0; k < BK / Cfg::UMMA_K; ++k) {
              // A (K-major): advance 16 elements = 32 B inside the 128B swizzle row.
              uint64_t adesc, bdesc;
              if constexpr (Cfg::SW) {
                adesc = desc_sw128(a_s + (k >> 2) * Cfg::A_HALF_BYTES + 32 * (k & 3), 16, 1024);
                // B (MN-major): advance 16 k-rows = 2 swizzle atoms of 8 rows x 128 B;
                // 64-column groups are B_ATOM_BYTES apart (LBO), 8-row groups 1 KB (SBO).
                bdesc = desc_sw128(b_s + (k >> 2) * Cfg::B_HALF_BYTES + 2048 * (k & 3), Cfg::B_ATOM_BYTES, 1024);
              } else {
                // K-major A: LBO = K-direction core-matrix stride (the 2 KB boxes), SBO = 8-row
                // groups (128 B); a K=16 step spans two boxes.  MN-major B: LBO = K-direction
                // stride (8-k-row groups, 128 B), SBO = N-direction core matrices (the 1 KB
                // boxes); a K=16 step spans two 8-k-row groups.
                adesc = desc_noswz(a_s + (k >> 2) * Cfg::A_HALF_BYTES + 4096 * (k & 3), 2048, 128);
                bdesc = desc_noswz(b_s + (k >> 2) * Cfg::B_HALF_BYTES + 256 * (k & 3), 128, 1024);
              }
#if !G16_DIAG_NO_MMA
              if (leader) umma_f16<CG>(d_tmem, adesc, bdesc, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
#endif
            }
            if (leader) {
              // (B multicast: a stage is refilled into both pairs, so both pairs' MMAs release it)
              if constexpr (CG == 2) umma_commit_pair(empty_bar + 8 * stage, mc ? 0xF : 0x3);
              else if constexpr (MC > 1) umma_commit_mc(empty_bar + 8 * stage, (1u << MC) - 1u);   // every CTA's stage
              else umma_commit(empty_bar + 8 * stage);
            }
            if (++stage == p.ring_stages) { stage = 0; phase ^= 1u; }
          }
          if (leader) {
            if constexpr (CG == 2) umma_commit_pair(accf_bar + 8 * acc, static_cast<uint16_t>(0x3u << (mc ? 2u * pidx : 0u)));
            else umma_commit(accf_bar + 8 * acc);
          }
          if (tr && ch == n_chunks - 1) {
            p.trace[8 * it + 2] = globaltimer_ns();
            p.trace[8 * it + 7] = clock64() - clk0;   // SM cycles of this tile (MMA warp)
          }
          if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1u; }
        }
      }
    }
  } else if (warp < Cfg::EPI_WARPS) {
    // ===================== epilogue warps =====================
    const uint32_t ew = warp;                     // 0..7
    const uint32_t q = warp & 3;                  // TMEM lane quadrant (hardware rule: warp % 4)
    const uint32_t hcol = (ew >> 2) * Cfg::CPW;   // first accumulator column of this warp
    const uint32_t ebuf0 = sE + ew * Cfg::EPI_SLOTS * Cfg::EPI_BUF;
    const uint32_t ebar0 = epi_bar + 8 * Cfg::EPI_SLOTS * ew;
    const uint32_t acce_leader = (CG == 2) ? mapa_shared(acce_bar, lead) : acce_bar;
    const uint64_t pol_c = p.l2_hints ? policy_evict_first() : policy_evict_normal();
    // F32 C, C += A.B (+ bias): the staged accumulator (plus the bias, added in F32 first) is
    // added into C by the TMA unit (cp.reduce.async.bulk .add, one IEEE RN add in L2 --
    // bitwise the same C_in + acc when there is no bias), so C_in is never loaded into shared
    // memory: half the epilogue's shared-memory traffic and no C_in latency chain (findings.md
    // section 14).  ReLU needs the whole sum in registers, so it keeps the staged C_in path
    const bool red = !Cfg::OUT_F16 && !Cfg::PEERS && !p.beta0 && p.c_reduce && !p.relu && !p.c_ragged;
    const bool load_c = !p.beta0 && !red;   // C_in traffic through the staging slots
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t slot_phase = 0;  // bit s = parity to wait for on slot s
    float racc[Cfg::CPW];
    bool sig_pending = false;            // stream-K: a token to post once our reduce-adds complete
    int it = 0;
    for (; it < work.n_items; ++it) {
      const Item itm = item_of<SK>(p, work, cluster, nclusters, it);
      const int tile = itm.tile;
      const int n_chunks = SK ? (itm.kb_hi - itm.kb_lo + p.kb_per_chunk - 1) / p.kb_per_chunk : p.k_chunks;
      const bool tr = trace_me && ew == 0 && lane == 0 && it < 60;
      int tm, tn;
      tile_coords(tile, p, tm, tn);
      if constexpr (MC > 1 && CG == 1) tn = MC * tn + static_cast<int>(mrank);
      if constexpr (MC > 1 && CG == 2) tm = MC * tm + static_cast<int>(pidx);
      const int row0 = tm * BM * CG + static_cast<int>(rank) * BM + static_cast<int>(q) * 32;
      const int col0 = tn * BN + static_cast<int>(hcol);
      // stream-K with F16 C: the second part of a split tile is added into C (which the first
      // part already wrote as C_in + its partial, rounded) by an F16 TMA reduce-add of its own
      // rounded partial -- no C_in load for that item (R18)
      const bool f16_tail = SK && Cfg::OUT_F16 && itm.wait;
      const bool load_it = load_c && !f16_tail;
      const bool red_it = red || f16_tail;
      if (tr) p.trace[8 * it + 3] = globaltimer_ns();
      // C_in for the first PRE output chunks goes straight into the staging slots
      // now, so its latency hides under this tile's MMAs (the slots were freed by
      // the previous tile's stores).
      if (lane == 0) {
        bulk_wait_group_read<0>();
#pragma unroll
        for (int c = 0; c < Cfg::PRE; ++c) {
          const uint32_t sbar = ebar0 + 8 * c;
          if (load_it) {
            mbar_arrive_expect_tx(sbar, 32 * Cfg::RB);
            tma_load_2d_hint(ebuf0 + c * Cfg::EPI_BUF, &tm_c, col0 + c * Cfg::CW, row0, sbar, pol_c);
          } else {
            mbar_arrive(sbar);
          }
        }
      }
      // ---- promote each K chunk's TMEM partial sum into F32 registers (RN adds)
      const uint32_t t_lane = tmem_base + ((q * 32u) << 16) + hcol;
#pragma unroll 1
      for (int ch = 0; ch < n_chunks; ++ch) {
        if (Cfg::PRE < Cfg::NOUT && ch == n_chunks - 1 && lane == 0 && load_it) {
          // the remaining C_in chunks are needed right after this (last) K chunk:
          // pull them into L2 now, one chunk ahead, so they are neither evicted by
          // a whole tile of operand traffic nor fetched from HBM in a burst.
#pragma unroll 1
          for (int c = Cfg::PRE; c < Cfg::NOUT; ++c) tma_prefetch_l2_2d(&tm_c, col0 + c * Cfg::CW, row0);
        }
        mbar_wait(accf_bar + 8 * acc, acc_phase);
        tc_fence_after();
        if (tr && ch == n_chunks - 1) p.trace[8 * it + 4] = globaltimer_ns();
        const uint32_t t_row = t_lane + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
#pragma unroll
        for (int c = 0; c < Cfg::CPW / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + 32 * c, v);
          tmem_wait_ld();
          if (p.accum_f16) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(f16x2_to_f32(v[j]).x);
          }
          if (ch == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) racc[32 * c + j] = __uint_as_float(v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) racc[32 * c + j] = __fadd_rn(racc[32 * c + j], __uint_as_float(v[j]));
          }
        }
        // chunk fully read: hand the TMEM buffer back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(acce_leader + 8 * acc);
          else mbar_arrive(acce_bar + 8 * acc);
        }
        if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1u; }
      }
      if (tr) p.trace[8 * it + 5] = globaltimer_ns();
      // ---- C_out = C_in + acc (F32 add, one rounding to the output type), TMA store.
      const int grow = row0 + static_cast<int>(lane);
      // last tile, nothing to load: every MMA of this CTA pair has completed (the final
      // accumulator barrier), so the operand ring is free -- stage all NOUT chunks there
      // and issue their stores back to back instead of waiting for a slot to be read
      const bool ring = Cfg::TAIL_RING && p.tail_ring && !load_it && it + 1 == work.n_items;
      if (ring) fence_proxy_async_smem();
#pragma unroll
      for (int c = 0; c < Cfg::NOUT; ++c) {
        const uint32_t slot = static_cast<uint32_t>(c % Cfg::EPI_SLOTS);
        const uint32_t sbuf = ring ? sA + (ew * Cfg::NOUT + c) * Cfg::EPI_BUF : ebuf0 + slot * Cfg::EPI_BUF;
        const uint32_t sbar = ebar0 + 8 * slot;
        const int ccol = col0 + c * Cfg::CW;
        const bool manual = p.c_ragged && (ccol + Cfg::CW > p.N);
        if (!ring) {
          mbar_wait(sbar, (slot_phase >> slot) & 1u);
          slot_phase ^= (1u << slot);
        }
#pragma unroll
        for (int j = 0; j < Cfg::RB / 16; ++j) {
          const uint32_t addr = sbuf + (Cfg::SW ? swz<Cfg::RB>(lane, static_cast<uint32_t>(j)) : lane * Cfg::RB + 16u * static_cast<uint32_t>(j));
          const float* a = &racc[c * Cfg::CW + j * (16 / Cfg::ESIZE)];
          constexpr int EPU = 16 / Cfg::ESIZE;      // output elements per 16-byte unit
          float o[EPU];
          if constexpr (!Cfg::OUT_F16) {
            const float z = red ? -0.f : 0.f;   // (reduce-add: stage the accumulator itself, -0 kept)
            float4 ci = make_float4(z, z, z, z);
            if (load_it) ci = lds128(addr);
            o[0] = ci.x + a[0]; o[1] = ci.y + a[1]; o[2] = ci.z + a[2]; o[3] = ci.w + a[3];
          } else {
            uint4 ci = make_uint4(0u, 0u, 0u, 0u);
            if (load_it) ci = lds128u(addr);
            const float2 c0 = f16x2_to_f32(ci.x), c1 = f16x2_to_f32(ci.y);
            const float2 c2 = f16x2_to_f32(ci.z), c3 = f16x2_to_f32(ci.w);
            o[0] = c0.x + a[0]; o[1] = c0.y + a[1]; o[2] = c1.x + a[2]; o[3] = c1.y + a[3];
            o[4] = c2.x + a[4]; o[5] = c2.y + a[5]; o[6] = c3.x + a[6]; o[7] = c3.y + a[7];
          }
          if (p.bias != nullptr) {
#pragma unroll
            for (int h = 0; h < EPU / 4; ++h) {
              const float4 bb = load_bias4(p.bias, ccol + EPU * j + 4 * h, p.N);
              o[4 * h + 0] += bb.x; o[4 * h + 1] += bb.y; o[4 * h + 2] += bb.z; o[4 * h + 3] += bb.w;
            }
          }
          if (p.relu) {
#pragma unroll
            for (int e = 0; e < EPU; ++e) o[e] = relu_keep_nan(o[e]);
          }
          if constexpr (!Cfg::OUT_F16) {
            sts128(addr, o[0], o[1], o[2], o[3]);
          } else {
            sts128u(addr, cvt_f16x2_rn(o[0], o[1]), cvt_f16x2_rn(o[2], o[3]), cvt_f16x2_rn(o[4], o[5]),
                    cvt_f16x2_rn(o[6], o[7]));
          }
        }
        if (!manual) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (SK && c == 0 && sig_pending) {
              // the previous item's partial (a tile cluster + 1 finishes): its reduce-adds
              // were issued a whole drain ago; once they have completed in global memory,
              // post one token for this warp's region.  Posted here, not right after they
              // were issued, so the wait for completion never delays this item's drain.
              bulk_wait_group<0>();
              fence_proxy_async_global();
              red_release_gpu_add(p.sk_flags + sk_slot(cluster, rank, ew), 1u);
              sig_pending = false;
            }
            if (SK && c == 0 && itm.wait) {
              // k-blocks [0, kb_lo) of this tile were added into C by cluster - 1: take
              // its token before adding ours (fixed order of the two RN adds)
              take_token(p.sk_flags + sk_slot(cluster - 1, rank, ew));
              fence_proxy_async_global();
            }
            if (red_it) tma_reduce_add_2d_hint(&tm_c, ccol, row0, sbuf, pol_c);
            else tma_store_2d_hint(&tm_c, ccol, row0, sbuf, pol_c);
            // fused all-gather: the same staged chunk goes to every peer's C
            if constexpr (Cfg::PEERS)
              for (int d = 0; d < p.n_peers; ++d) tma_store_2d_hint(&peers.m[d], ccol, row0, sbuf, pol_c);
            bulk_commit_group();
          }
        } else {
          __syncwarp();
          if (grow < p.M) {
            // ragged N edge: element-wise stores of this thread's row, read back
            // from the staged chunk, clipped at column N, to C and every peer
#pragma unroll 1
            for (int j = 0; j < Cfg::RB / 16; ++j) {
              const uint4 v = lds128u(sbuf + (Cfg::SW ? swz<Cfg::RB>(lane, static_cast<uint32_t>(j)) : lane * Cfg::RB + 16u * static_cast<uint32_t>(j)));
              const uint32_t o[4] = {v.x, v.y, v.z, v.w};
              constexpr int EPU = 16 / Cfg::ESIZE;   // elements per 16-byte unit
              const int cb = ccol + EPU * j;
              const int nd = Cfg::PEERS ? p.n_peers : 0;
#pragma unroll 1
              for (int d = -1; d < nd; ++d) {
                char* base = static_cast<char*>(d < 0 ? p.c_ptr : p.peer_ptr[d]) +
                             (static_cast<long long>(grow) * p.ldc + cb) * Cfg::ESIZE;
#pragma unroll
                for (int e = 0; e < EPU; ++e) {
                  if (cb + e >= p.N) break;
                  if constexpr (Cfg::ESIZE == 4) reinterpret_cast<uint32_t*>(base)[e] = o[e];
                  else reinterpret_cast<uint16_t*>(base)[e] = static_cast<uint16_t>(o[e >> 1] >> (16 * (e & 1)));
                }
              }
            }
          }
        }
        if (!ring && c + Cfg::EPI_SLOTS < Cfg::NOUT && lane == 0) {
          // refill this slot with chunk c + SLOTS once its store has read it
          bulk_wait_group_read<0>();
          if (load_it) {
            mbar_arrive_expect_tx(sbar, 32 * Cfg::RB);
            tma_load_2d_hint(sbuf, &tm_c, ccol + Cfg::EPI_SLOTS * Cfg::CW, row0, sbar, pol_c);
          } else {
            mbar_arrive(sbar);
          }
        }
      }
      if (SK && itm.signal) sig_pending = true;
      if (tr) p.trace[8 * it + 6] = globaltimer_ns();
    }
    if (lane == 0) {
      bulk_wait_group<0>();
      if (SK && sig_pending) {   // (a signalling item that was this CTA's last)
        fence_proxy_async_global();
        red_release_gpu_add(p.sk_flags + sk_slot(cluster, rank, ew), 1u);
      }
    }
    if (trace_me && warp == 0 && lane == 0) p.trace[8 * 62 + 3] = globaltimer_ns();
  }

  // ===================== teardown =====================
  __syncwarp();
  tc_fence_before();
  if constexpr (CG == 2 || MC > 1) cluster_sync(); else __syncthreads();   // (no peer arrives on our barriers any more)
  if (warp == Cfg::W_ALLOC) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
  }
  if (trace_me && threadIdx.x == 0) p.trace[8 * 62 + 2] = globaltimer_ns();
}

}  // namespace g16
