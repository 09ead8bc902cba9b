// gemm_api.cu -- host side of libgemm_f16.so (B2): argument validation,
// per-device capability cache, CUtensorMap encoding, configuration choice and
// cudaLaunchKernelEx with cluster dimensions.  Contract: include/gemm_f16.h.
//
// Replaces the paper's host path (Sec. 3.11: gpu.launch ->
// MLIR CUDA runtime wrappers, JIT via mlir-cpu-runner) with an AOT-compiled
// sm_100a library; the tile-configuration choice plays the role of the
// paper's per-size "best performing version".
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/gemm_f16.h"
#include "../../include/gemm_f16_diag.h"
#include "gemm_sm100.cuh"
#include "gemm_sm100_wide.cuh"
#include "gemm_sm100_wide_f32.cuh"
#include "gemm_sm100_splitk.cuh"
#include "gemm_sm100_nows.cuh"

namespace {

using namespace g16;

constexpr int kDefaultL2Hints = 1;
constexpr int kDefaultPdl = 1;   // profiles/r01/findings.md section 9
constexpr int kDefaultSnake = 0;
constexpr int kDefaultCReduce = 1;   // findings.md section 14: +1-10 %, bitwise identical
// stream-K (auto): taken when the last wave of tiles is at most this full, K >= 4096
// (F32 C; F16 C: 0.4, where the 256 x 512 tile is the alternative) ...
constexpr double kStreamKMaxFill = 0.5;
constexpr double kStreamKMaxFillF16 = 0.4;
// ... or at most this full with K > 2048 (profiles/r01/stream_k.md: the K = 1024-2048 tiles
// are too short to pay for the extra partial-tile store phases)
constexpr double kStreamKMaxFillShortK = 0.3;

// token counters of the stream-K hand-over (gemm_sm100.cuh): every launch leaves them at
// zero (each posted token is taken), so no per-launch reset and no allocation is needed.
// The pool is cut into kSkWindows fixed windows of kSkWindow slots (16 per cluster, for up to
// 128 clusters); successive launches take successive windows round robin, so two stream-K
// GEMMs share counters only if kSkWindows - 1 others were issued between them -- concurrent
// GEMMs on different streams stay isolated up to kSkWindows in flight.
constexpr int kSkWindow = 16 * 128;
constexpr int kSkWindows = kSkFlagSlots / kSkWindow;
static_assert(kSkWindows * kSkWindow == kSkFlagSlots, "whole windows");
__device__ unsigned g_sk_flags[kSkFlagSlots];
uint32_t sk_window_base(uint32_t launch_index) { return (launch_index % kSkWindows) * kSkWindow; }

thread_local int t_last_cuda_error = 0;
thread_local int t_last_launches = 0;
thread_local unsigned long long* t_trace = nullptr;   // gemm_f16_diag_set_trace: armed for the next call

using Cfg1F32 = KCfg<2, 256, 6, false>;
using Cfg1F16 = KCfg<2, 256, 6, true>;
using Cfg2F32 = KCfg<2, 128, 8, false>;
using Cfg2F16 = KCfg<2, 128, 8, true>;
using Cfg3F32 = KCfg<1, 256, 4, false>;
using Cfg3F16 = KCfg<1, 256, 4, true>;
using Cfg4F32 = KCfg<1, 128, 6, false>;
using Cfg4F16 = KCfg<1, 128, 6, true>;
using Cfg5F32 = KCfg<1, 64, 8, false>;
using Cfg5F16 = KCfg<1, 64, 8, true>;
using Cfg6F32 = KCfg<2, 256, 5, false, 2>;
using Cfg6F16 = KCfg<2, 256, 5, true, 2>;
using Cfg7F32 = KCfg<2, 256, 4, false, 3>;
using Cfg7F16 = KCfg<2, 256, 4, true, 3>;
using Cfg8F32 = KCfg<2, 256, 3, false, 1, 128>;
using Cfg8F16 = KCfg<2, 256, 3, true, 1, 128>;
// A multicast across a 4-CTA cluster of 1-CTA tiles along N (small problems)
using Cfg13F32 = KCfg<1, 64, 8, false, 1, 64, false, 4>;
using Cfg13F16 = KCfg<1, 64, 8, true, 1, 64, false, 4>;
using Cfg14F32 = KCfg<1, 128, 6, false, 1, 64, false, 4>;
using Cfg14F16 = KCfg<1, 128, 6, true, 1, 64, false, 4>;
// B multicast across the two CTA pairs of a 4-CTA cluster (the 128-deep pair config otherwise)
using Cfg16F32 = KCfg<2, 256, 3, false, 1, 128, false, 2>;
using Cfg16F16 = KCfg<2, 256, 3, true, 1, 128, false, 2>;
// gemm_f16_gather: the 128-deep pair tile with peer stores compiled in
using CfgGF32 = KCfg<2, 256, 3, false, 1, 128, true>;
using CfgGF16 = KCfg<2, 256, 3, true, 1, 128, true>;

using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const GemmParams, const PeerMaps,
                          const CUtensorMap);

struct ConfigDesc {
  int cta_group, tile_n, stages, threads, bk;
  int smem[2];      // [acc_type]
  int c_box_cols[2];  // epilogue staging box width (elements)
  int c_row_bytes[2]; // 128 -> SWIZZLE_128B, 64 -> SWIZZLE_64B
  KernelFn fn[2];
  int cluster = 0;    // CTAs per cluster (0: = cta_group)
  int k_splits = 0;   // split-K configs: CTAs per cluster sharing one tile's K (non-persistent grid)
  int a_mc = 1;       // A-multicast configs: CTAs per cluster sharing A (tiles (tm, a_mc * tg + r))
  int b_mc = 1;       // B-multicast configs: CTA pairs per cluster sharing B (tiles (b_mc * tg + p, tn))
  KernelFn sk_fn[2] = {nullptr, nullptr};   // [acc_type]: the stream-K build (CTA-pair tiles only)
  bool hybrid = false; // launched with cluster dim cta_group and the preferred cluster dim `cluster`
  int cluster_size() const { return cluster ? cluster : cta_group; }
  int launch_cluster() const { return hybrid ? cta_group : cluster_size(); }
};

template <class C>
constexpr KernelFn sk_fn_of() {
  if constexpr (C::CG == 2 && !C::PEERS && C::MC == 1) return &gemm_f16_sm100_kernel<C, true>;
  else return nullptr;
}

template <class C32, class C16>
constexpr ConfigDesc make_desc() {
  return ConfigDesc{C32::CG, C32::BN, C32::STAGES, C32::THREADS, C32::BK,
                    {C32::SMEM_BYTES, C16::SMEM_BYTES}, {C32::CW, C16::CW}, {C32::RB, C16::RB},
                    {&gemm_f16_sm100_kernel<C32>, &gemm_f16_sm100_kernel<C16>},
                    C32::MC > 1 ? C32::CG * C32::MC : 0, 0, C32::CG == 1 ? C32::MC : 1,
                    C32::CG == 2 ? C32::MC : 1,
                    {sk_fn_of<C32>(), sk_fn_of<C16>()}};
}

template <int BN, int S>
constexpr ConfigDesc make_splitk_desc() {
  using C32 = SKCfg<BN, S, false>;
  using C16 = SKCfg<BN, S, true>;
  return ConfigDesc{1, BN, C32::STAGES, C32::THREADS, C32::BK,
                    {C32::SMEM_BYTES, C16::SMEM_BYTES}, {32, 64}, {128, 128},
                    {&gemm_f16_sm100_splitk_kernel<C32>, &gemm_f16_sm100_splitk_kernel<C16>}, S, S};
}

const ConfigDesc kConfigs[GEMM_CFG_COUNT] = {
    ConfigDesc{0, 0, 0, 0, 0, {0, 0}, {0, 0}, {0, 0}, {nullptr, nullptr}},
    make_desc<Cfg1F32, Cfg1F16>(),
    make_desc<Cfg2F32, Cfg2F16>(),
    make_desc<Cfg3F32, Cfg3F16>(),
    make_desc<Cfg4F32, Cfg4F16>(),
    make_desc<Cfg5F32, Cfg5F16>(),
    make_desc<Cfg6F32, Cfg6F16>(),
    make_desc<Cfg7F32, Cfg7F16>(),
    make_desc<Cfg8F32, Cfg8F16>(),
    ConfigDesc{},   // GEMM_CFG_PAIR_256x512: kWideConfig (defined below)
    make_splitk_desc<256, 2>(),
    make_splitk_desc<256, 4>(),
    make_splitk_desc<128, 4>(),
    make_desc<Cfg13F32, Cfg13F16>(),
    make_desc<Cfg14F32, Cfg14F16>(),
    make_splitk_desc<128, 2>(),
    make_desc<Cfg16F32, Cfg16F16>(),
    [] { ConfigDesc d = make_desc<Cfg16F32, Cfg16F16>(); d.hybrid = true; return d; }(),
};
using CfgW16 = WCfg<4>;
// F32 C (gemm_sm100_wide_f32.cuh): ring depth and epilogue staging slots per warp
#ifndef G16_W32_STAGES
#define G16_W32_STAGES 4
#endif
#ifndef G16_W32_SLOTS
#define G16_W32_SLOTS 1
#endif
using CfgW32 = W32Cfg<G16_W32_STAGES, G16_W32_SLOTS>;
const ConfigDesc kWideConfig{2, CfgW16::BN, CfgW16::STAGES, CfgW16::THREADS, CfgW16::BK,
                             {CfgW32::SMEM_BYTES, CfgW16::SMEM_BYTES}, {CfgW32::CW, CfgW16::CW}, {128, 128},
                             {&gemm_f16_sm100_wide_f32_kernel<CfgW32, false>, &gemm_f16_sm100_wide_kernel<CfgW16, false>}};
// the same tiles with the per-element epilogue options compiled in: F16 C bias, ReLU,
// accum_f16; F32 C beta = 0 and bias (F32 C with ReLU is not built: the reduce-add
// promotion leaves no single point where the final sum is in registers)
const KernelFn kWideExtFn[2] = {&gemm_f16_sm100_wide_f32_kernel<CfgW32, true>,
                                &gemm_f16_sm100_wide_kernel<CfgW16, true>};
const ConfigDesc kGatherConfig = make_desc<CfgGF32, CfgGF16>();
// ABLATION builds (gemm_options_t.swizzle / warp_specialize = -1; never picked by AUTO)
using CfgNsF32 = KCfg<2, 256, 6, false, 1, 64, false, 1, false>;
using CfgNsF16 = KCfg<2, 256, 6, true, 1, 64, false, 1, false>;
const KernelFn kNoSwizzleFn[2] = {&gemm_f16_sm100_kernel<CfgNsF32>, &gemm_f16_sm100_kernel<CfgNsF16>};
const KernelFn kNoWsFn[2] = {&gemm_f16_sm100_nows_kernel<false>, &gemm_f16_sm100_nows_kernel<true>};

const ConfigDesc& config_desc(int c) {
  if (c == GEMM_CFG_COUNT) return kGatherConfig;
  if (c == GEMM_CFG_PAIR_256x512) return kWideConfig;
  return kConfigs[c];
}

// K elements accumulated in TMEM before the partial sum is promoted to F32
// registers (R4): 2048 keeps the truncation error near 2.4e-6.
constexpr int kDefaultPromoteK = 2048;
// the 256 x 512 F32 kernel promotes by TMA reduce-add into C (every drain costs L2 traffic and
// TMEM read time), with chains <= 4096 + a few k-blocks: ~5e-6 relative error, half the bar
constexpr int kDefaultPromoteKWide32 = 4096;

// ---------------------------------------------------------------- device cache
constexpr int kMaxDevices = 64;
struct DeviceInfo {
  gemm_status_t status = GEMM_OK;
  int cuda_error = 0;
  int sm_count = 0;
  int max_clusters[GEMM_CFG_COUNT + 1][2] = {};   // [GEMM_CFG_COUNT] = the gather config
  unsigned* sk_flags = nullptr;                    // this device's g_sk_flags
  std::atomic<uint32_t> sk_next{0};                // next window of the pool
};
std::once_flag g_dev_once[kMaxDevices];
DeviceInfo g_dev[kMaxDevices];

void init_device(int dev) {
  DeviceInfo& d = g_dev[dev];
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
  if (major != 10 || minor != 0) { d.status = GEMM_ERR_UNSUPPORTED_DEVICE; return; }
  for (int c = 1; c <= GEMM_CFG_COUNT; ++c) {
    for (int a = 0; a < 2; ++a) {
      const ConfigDesc& cd = config_desc(c);
      if (cd.fn[a] == nullptr) continue;   // not built for this accumulate mode
      e = cudaFuncSetAttribute(reinterpret_cast<const void*>(cd.fn[a]),
                               cudaFuncAttributeMaxDynamicSharedMemorySize, cd.smem[a]);
      if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
      const int cs = cd.cluster_size();
      if (cs > 1) {
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(cd.fn[a]),
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        // (hybrid: occupancy of the regular 2-CTA clusters; a group of cs CTAs is one 4-CTA
        // cluster or two 2-CTA ones, so all of them fit)
        const int lcs = cd.launch_cluster();
        attr[0].val.clusterDim.x = lcs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(lcs * (d.sm_count / lcs), 1, 1);
        lc.blockDim = dim3(cd.threads, 1, 1);
        lc.dynamicSmemBytes = cd.smem[a];
        lc.attrs = attr;
        lc.numAttrs = 1;
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(cd.fn[a]), &lc);
        if (cd.hybrid) n = n * lcs / cs;
        if (e != cudaSuccess || n <= 0) { d.status = GEMM_ERR_CUDA; d.cuda_error = e ? e : cudaErrorInvalidConfiguration; return; }
        d.max_clusters[c][a] = n;
        if (cd.sk_fn[a] != nullptr) {   // the stream-K build: same smem, same cluster
          e = cudaFuncSetAttribute(reinterpret_cast<const void*>(cd.sk_fn[a]),
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, cd.smem[a]);
          if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
        }
        if (c == GEMM_CFG_PAIR_256x512) {   // the option-carrying twin: same smem, same cluster
          e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kWideExtFn[a]),
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, cd.smem[a]);
          if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
        }
      } else {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cd.fn[a], cd.threads, cd.smem[a]);
        if (e != cudaSuccess || per_sm <= 0) { d.status = GEMM_ERR_CUDA; d.cuda_error = e ? e : cudaErrorInvalidConfiguration; return; }
        d.max_clusters[c][a] = per_sm * d.sm_count;
      }
    }
  }
  for (int a = 0; a < 2; ++a) {   // ablation kernels (same cluster shape as their base configs)
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kNoSwizzleFn[a]), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             a ? CfgNsF16::SMEM_BYTES : CfgNsF32::SMEM_BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kNoWsFn[a]), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               NwsCfg::SMEM_BYTES);
    if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
  }
  void* f = nullptr;
  e = cudaGetSymbolAddress(&f, g_sk_flags);
  if (e != cudaSuccess) { d.status = GEMM_ERR_CUDA; d.cuda_error = e; return; }
  d.sk_flags = static_cast<unsigned*>(f);
}

// Copy streams of the host-buffer path (created once per device, never destroyed).
struct HostStreams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaError_t err = cudaSuccess;
};
std::once_flag g_hs_once[kMaxDevices];
HostStreams g_hs[kMaxDevices];

HostStreams& host_streams(int dev) {
  std::call_once(g_hs_once[dev], [dev]() {
    HostStreams& h = g_hs[dev];
    h.err = cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking);
    if (h.err == cudaSuccess) h.err = cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking);
  });
  return g_hs[dev];
}

// ---------------------------------------------------------------- tensor maps
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = []() -> PFN_encodeTiled {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_encodeTiled>(p);
  }();
  return fn;
}

// Per-thread cache of encoded tensor maps: repeated calls on the same buffers
// (training loops, benchmarks) skip cuTensorMapEncodeTiled.  The key is every
// input of the encoding, so a hit returns exactly what encoding would.
struct TmapKey {
  const void* ptr;
  int64_t rows, cols, ld;
  int dt;
  uint32_t box_cols, box_rows;
  int l2, swz;
  bool operator==(const TmapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && dt == o.dt &&
           box_cols == o.box_cols && box_rows == o.box_rows && l2 == o.l2 && swz == o.swz;
  }
};
constexpr int kTmapCache = 16;
struct TmapCache {
  TmapKey key[kTmapCache];
  CUtensorMap map[kTmapCache];
  bool valid[kTmapCache] = {};
  int next = 0;
};
thread_local TmapCache t_tmap_cache;

// 2-D row-major tensor (rows x cols, ld elements), box = box_cols x box_rows, 128B swizzle.
bool encode_2d_uncached(CUtensorMap* m, CUtensorMapDataType dt, size_t esize, const void* ptr, int64_t rows,
               int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapL2promotion l2,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_2d(CUtensorMap* m, CUtensorMapDataType dt, size_t esize, const void* ptr, int64_t rows,
               int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapL2promotion l2,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  TmapCache& c = t_tmap_cache;
  const TmapKey k{ptr, rows, cols, ld, static_cast<int>(dt), box_cols, box_rows, static_cast<int>(l2),
                  static_cast<int>(swz)};
  for (int i = 0; i < kTmapCache; ++i) {
    if (c.valid[i] && c.key[i] == k) {
      *m = c.map[i];
      return true;
    }
  }
  if (!encode_2d_uncached(m, dt, esize, ptr, rows, cols, ld, box_cols, box_rows, l2, swz)) return false;
  const int slot = c.next;
  c.next = (c.next + 1) % kTmapCache;
  c.key[slot] = k;
  c.map[slot] = *m;
  c.valid[slot] = true;
  return true;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// The stream-K auto rule (profiles/r01/stream_k.md): one to max_waves full waves of pair
// tiles (beyond that the last wave is a small share of the run; measured up to 7), and a last
// wave at most kStreamKMaxFill(F16) full with K >= 4096, or at most kStreamKMaxFillShortK
// full with K > 2048.
// Below one wave (half to 70 % of the clusters have a tile) every tile is shared out; that
// pays only with long K (F16 K >= 4096, F32 K >= 8192: 1792^2 x 8192 -15 % F16, -7 % F32;
// profiles/r01/stream_k.md, one-wave section).
bool stream_k_pays(int64_t tiles, int64_t clusters, int64_t K, int acc_type, int64_t max_waves = 8) {
  if (clusters > 0 && tiles < clusters)
    return 2 * tiles >= clusters && 10 * tiles <= 7 * clusters && K >= (acc_type == GEMM_ACC_F16 ? 4096 : 8192);
  if (clusters <= 0 || tiles % clusters == 0 || tiles / clusters > max_waves) return false;
  const double fill = static_cast<double>(tiles % clusters) / static_cast<double>(clusters);
  const double max_fill = acc_type == GEMM_ACC_F16 ? kStreamKMaxFillF16 : kStreamKMaxFill;
  return (K >= 4096 && fill <= max_fill) || (K > 2048 && fill <= kStreamKMaxFillShortK);
}

// Shape -> configuration (the paper's per-size "best performing version",
// P:903-905, as a fixed table so results stay deterministic).  Measured on B200
// (profiles/r01/cfgsweep.md, epilogue_slots.md, graph_small.md, stage_depth.md):
//  * the 2-CTA 256x256 pair tile wins at every BASELINE shape from 2048^3 up,
//    including the BERT shapes and tails, even below one wave -- smaller tiles
//    lose more to per-FLOP operand traffic than they gain in parallelism;
//  * 128-deep K stages (3 x 64 KB) beat 64-deep ones (6 x 32 KB) by 2-4 %:
//    half the barrier/commit round trips per FLOP and fewer DRAM re-reads;
//  * for F32 C with one K chunk per tile (K <= 2048) the tile is bound by its C
//    traffic: with C_in staged a second epilogue staging slot per warp (5 x 32 KB ring)
//    won; with the reduce-add epilogue the 6-stage ring does;
//  * when the whole problem is under a third of a wave of pair tiles
//    (e.g. 1024^3), fixed per-tile latency dominates and the 1-CTA 128x64 tile
//    (more, shorter tiles) wins (GPU time from CUDA-graph replay);
//  * a short M (<= 128 rows) wastes too much of a 256-row tile;
//  * a small output with a long K (e.g. 512^2 x 2048, 1024^2 x 4096) is split over
//    K across a cluster (gemm_sm100_splitk.cuh), S CTAs per tile;
//  * F16 C: the 256 x 512 pair tile (gemm_sm100_wide.cuh) moves 25 % fewer operand
//    bytes per FLOP and so sustains a higher clock under the power cap; it wins
//    wherever its last wave is about as full as the 256 x 256 tile's
//    (profiles/r01/wide_tile.md: 4096^3 .. 16384^3, 8192^2 x 1024/2048, 4100 x 4096 x 4104,
//    8192 x 1000 x 1000; it loses at 2048^3 and 32768 x 1024 x 4096 on wave quantization).
int pick_config(int64_t M, int64_t N, int64_t K, int acc_type, int sm_count) {
  const int64_t pair_tiles = cdiv(M, 256) * cdiv(N, 256);
  const bool small = M <= 128 || 3 * pair_tiles <= sm_count / 2;   // under 1/3 wave of pair tiles
  const bool half = 2 * pair_tiles <= sm_count / 2;                 // at most half a wave
  if (small || half) {
    // Few output tiles: split K over a cluster when K is long enough to pay for the
    // reduction (profiles/r01/splitk.md; it loses at 1024^3).  Each CTA keeps one
    // truncating TMEM chain over its K / S (no promotion, R4): for F32 C that
    // chain stays <= 4096 long (rel. error <~ 5e-6, bar 1e-5).
    const int64_t kmax_chain = acc_type == GEMM_ACC_F32 ? 4096 : (int64_t(1) << 40);   // (F16: no limit)
    const int64_t t128 = cdiv(M, 128) * cdiv(N, 128), t256 = cdiv(M, 128) * cdiv(N, 256);
    // 4-CTA clusters: only ~132 of 148 SMs can hold them at once (tools/probe_cluster.cu)
    const int64_t sm4 = sm_count - sm_count / 9;
    const bool f32 = acc_type == GEMM_ACC_F32;
    if (K >= 2048 && 4 * t128 <= sm4 && K <= 4 * kmax_chain) return GEMM_CFG_SPLITK_128x128_S4;
    // F32 reduces by TMA reduce-add, F16 through DSMEM (bulk-DMA configs S2 x 128x128 and
    // S2 x 128x256 beat the pushes of S4 x 128x256 until K = 16384, splitk.md v9/v10).
    // The two-way splits pay only from K = 4096 in either mode, the four-way 128x256 split
    // for F32 from K = 8192: below that the 1-CTA tiles win (graph replay, round 2:
    // 1024^2 x 1024 F32 6.4 vs 7.9 us, 1024^2 x 2048 F16 8.8 vs 10.8 us, 768^2 x 4096 F32
    // S2 x 128x128 11.5 vs S4 x 128x256 14.7 us; profiles/r02/graph_small_pick*.jsonl).
    // S2 x 128x256 is not picked: wherever its 2 * t256 CTAs fit one wave the 1-CTA
    // 128 x 128 tiles do too, and win (1024 x 2048 x 4096: 17.7 vs 19.2 us F32, 17.4 vs
    // 21.8 us F16)
    if (f32 && K >= 8192 && 4 * t256 <= sm4 && K <= 4 * kmax_chain) return GEMM_CFG_SPLITK_128x256_S4;
    if (!f32 && K >= 16384 && 4 * t256 <= sm4) return GEMM_CFG_SPLITK_128x256_S4;
    if (K >= 4096 && 2 * t128 <= sm_count && K <= 2 * kmax_chain) return GEMM_CFG_SPLITK_128x128_S2;
    if (small) {
      if (M <= 128) return cdiv(N, 256) >= sm_count ? GEMM_CFG_SOLO_128x256 : GEMM_CFG_SOLO_128x64;
      return GEMM_CFG_SOLO_128x64;
    }
    // at most half a wave of pair tiles: 128 x 128 tiles keep twice as many SMs busy
    // (2048 x 1024 x 1024: 9.2-10.5 us vs 12-13 us for the pair tile; profiles/r01/multicast.md)
    if (t128 <= sm_count) return GEMM_CFG_SOLO_128x128;
  }
  // one wave of pair tiles or less (each cluster runs at most one tile) with K <= 4096:
  // nothing follows a tile's epilogue, so its stores are fully exposed and the 3 staging
  // slots of the 4 x 32 KB ring pipeline them best (2048^3: 18.9 vs 20.1 us F32, 17.9 vs
  // 18.8 us F16; it loses ~4 % at K = 8192, where the deeper ring matters more;
  // profiles/r01/single_wave_cfg.txt)
  if (pair_tiles <= sm_count / 2 && K <= 4096) return GEMM_CFG_PAIR_256x256_S4;
  // F32 C just over one wave (at most 1.25 waves) with 2048 < K <= 4096, where stream-K
  // shares the extra tiles out: the S4 ring's 3 staging slots pipeline the extra partial
  // store phases best (2304^3 31.0 -> 29.6 us, 2304 x 2560 x 2560 33.2 -> 31.4, 2304^2 x 4096
  // 39.1 -> 37.9; not at K = 8192 or beyond 1.25 waves; profiles/r02/f32_one_wave_s4.jsonl)
  if (acc_type == GEMM_ACC_F32 && K > 2048 && K <= 4096 && 4 * pair_tiles <= 5 * (sm_count / 2)) return GEMM_CFG_PAIR_256x256_S4;
  // F32 C with one K chunk: with the reduce-add epilogue (N % 4 == 0) C_in needs no
  // staging slot, and the 6-stage 64-deep ring is best (profiles/r01/f32_short_k_cfg.txt);
  // a ragged N still stages C_in and keeps the second slot of S5
  if (acc_type == GEMM_ACC_F32 && K <= 2048) return N % 4 == 0 ? GEMM_CFG_PAIR_256x256 : GEMM_CFG_PAIR_256x256_S5;
  // a partial last wave that stream-K spreads over every cluster (F16 C: rather than the
  // 256 x 512 tile, whose half as many tiles fill waves no better)
  // (measured against the wide tile up to 4 full waves: 4608^3 -5.5 %, 3840^3 -4 %)
  if (acc_type == GEMM_ACC_F16 && stream_k_pays(pair_tiles, sm_count / 2, K, acc_type, 4))
    return GEMM_CFG_PAIR_256x256_K128;
  if (acc_type == GEMM_ACC_F16) {
    // the 256 x 512 tile runs 5-10 % faster per wave under the power cap
    // (profiles/r01/wide_tile.md) but has half as many tiles: take it unless it
    // fills the last wave of clusters clearly worse than the 256 x 256 tile
    const int64_t clusters = sm_count / 2;
    const int64_t wide_tiles = cdiv(M, 256) * cdiv(N, 512);
    const double eff_pair = double(pair_tiles) / double(cdiv(pair_tiles, clusters) * clusters);
    const double eff_wide = double(wide_tiles) / double(cdiv(wide_tiles, clusters) * clusters);
    if (eff_wide + 0.04 >= eff_pair) return GEMM_CFG_PAIR_256x512;
  }
  return GEMM_CFG_PAIR_256x256_K128;
}

// L2 promotion of an A/B operand map: 256 B when its rows start on 128-byte lines; when
// they do not (ld * 2 % 128 != 0), every 128-byte box row straddles two lines and the
// 128 B promotion is faster (8192x1000x1000 +6-10 %, 4104^3 +11-14 %; profiles/r01/findings.md 18)
CUtensorMapL2promotion operand_promotion(int64_t ld) {
  return (ld * 2) % 128 == 0 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

gemm_status_t cuda_fail(cudaError_t e) {
  t_last_cuda_error = static_cast<int>(e);
  return GEMM_ERR_CUDA;
}

gemm_status_t validate(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                       const void* C, int64_t ldc, int acc_type, bool* no_work) {
  const int64_t kMax = 0x7fffffffLL;
  if (M < 0 || N < 0 || K < 0 || M > kMax || N > kMax || K > kMax) return GEMM_ERR_INVALID_VALUE;
  if (acc_type != GEMM_ACC_F32 && acc_type != GEMM_ACC_F16) return GEMM_ERR_INVALID_VALUE;
  if (lda < std::max<int64_t>(1, K) || ldb < std::max<int64_t>(1, N) || ldc < std::max<int64_t>(1, N))
    return GEMM_ERR_INVALID_VALUE;
  *no_work = (M == 0 || N == 0 || K == 0);
  if (*no_work) return GEMM_OK;
  if (!A || !B || !C) return GEMM_ERR_INVALID_VALUE;
  const int64_t csz = acc_type == GEMM_ACC_F32 ? 4 : 2;
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return GEMM_ERR_MISALIGNED;
  if ((lda * 2) % 16 || (ldb * 2) % 16 || (ldc * csz) % 16) return GEMM_ERR_MISALIGNED;
  if (lda * 2 >= (int64_t(1) << 40) || ldb * 2 >= (int64_t(1) << 40) || ldc * csz >= (int64_t(1) << 40))
    return GEMM_ERR_INVALID_VALUE;
  return GEMM_OK;
}

gemm_status_t device_ready(int* dev_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= kMaxDevices) return GEMM_ERR_UNSUPPORTED_DEVICE;
  std::call_once(g_dev_once[dev], init_device, dev);
  if (g_dev[dev].status == GEMM_ERR_CUDA) {
    t_last_cuda_error = g_dev[dev].cuda_error;
    return GEMM_ERR_CUDA;
  }
  *dev_out = dev;
  return g_dev[dev].status;
}

// ABLATION: the non-warp-specialised kernel (gemm_sm100_nows.cuh), one 128 x 128 tile per CTA
gemm_status_t launch_nows(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                          void* C, int64_t ldc, int acc_type, cudaStream_t stream, const gemm_options_t* opts,
                          const DeviceInfo& di) {
  (void)di;
  if (opts->bias != nullptr || opts->relu || opts->accum_f16 || opts->max_clusters != 0 || opts->stream_k > 0)
    return GEMM_ERR_INVALID_VALUE;
  const int in_type = opts->in_type;
  if (in_type != GEMM_IN_F16 && in_type != GEMM_IN_BF16) return GEMM_ERR_INVALID_VALUE;
  const CUtensorMapDataType in_dt =
      in_type == GEMM_IN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tm_a, tm_b;
  if (!encode_2d(&tm_a, in_dt, 2, A, M, K, lda, 64, 128, operand_promotion(lda)) ||
      !encode_2d(&tm_b, in_dt, 2, B, K, N, ldb, 64, 64, operand_promotion(ldb)))
    return cuda_fail(cudaErrorInvalidValue);
  GemmParams p;
  std::memset(&p, 0, sizeof(p));
  p.M = static_cast<int>(M);
  p.N = static_cast<int>(N);
  p.K = static_cast<int>(K);
  p.tiles_m = static_cast<int>(cdiv(M, 128));
  p.tiles_n = static_cast<int>(cdiv(N, 128));
  const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n;
  if (tiles > 0x7fffffffLL) return GEMM_ERR_INVALID_VALUE;
  p.num_tiles = static_cast<int>(tiles);
  p.k_blocks = static_cast<int>(cdiv(K, 64));
  const int promote = opts->promote_k;
  if (promote < -1 || (promote > 0 && promote % 64 != 0)) return GEMM_ERR_INVALID_VALUE;
  p.kb_per_chunk = promote == -1 ? p.k_blocks : (promote == 0 ? kDefaultPromoteK : promote) / 64;
  const int rs = opts->ring_stages;
  if (rs < 0 || rs > NwsCfg::STAGES) return GEMM_ERR_INVALID_VALUE;
  p.ring_stages = rs == 0 ? NwsCfg::STAGES : rs;
  p.in_bf16 = in_type == GEMM_IN_BF16;
  p.beta0 = opts->beta0 ? 1 : 0;
  p.c_ptr = C;
  p.ldc = ldc;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(tiles), 1, 1);
  lc.blockDim = dim3(NwsCfg::THREADS, 1, 1);
  lc.dynamicSmemBytes = NwsCfg::SMEM_BYTES;
  lc.stream = stream;
  PeerMaps pm;
  std::memset(&pm, 0, sizeof(pm));
  cudaError_t e = cudaLaunchKernelEx(&lc, kNoWsFn[acc_type], tm_a, tm_b, tm_a, p, pm, tm_a);
  if (e != cudaSuccess) return cuda_fail(e);
  t_trace = nullptr;
  t_last_launches = 1;
  return GEMM_OK;
}

gemm_status_t launch(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                     void* C, int64_t ldc, int acc_type, cudaStream_t stream, const gemm_options_t* opts,
                     void* const* peers = nullptr, int n_peers = 0) {
  int dev = 0;
  gemm_status_t st = device_ready(&dev);
  if (st != GEMM_OK) return st;
  const DeviceInfo& di = g_dev[dev];

  int cfg = opts ? opts->config : GEMM_CFG_AUTO;
  if (cfg < 0 || cfg >= GEMM_CFG_COUNT) return GEMM_ERR_INVALID_VALUE;
  const int swz_opt = opts ? opts->swizzle : 0;
  const int ws_opt = opts ? opts->warp_specialize : 0;
  if (swz_opt < -1 || swz_opt > 1 || ws_opt < -1 || ws_opt > 1) return GEMM_ERR_INVALID_VALUE;
  if (ws_opt < 0) {
    if (n_peers > 0 || swz_opt < 0) return GEMM_ERR_INVALID_VALUE;
    return launch_nows(M, N, K, A, lda, B, ldb, C, ldc, acc_type, stream, opts, di);
  }
  const bool no_swizzle = swz_opt < 0;
  if (no_swizzle) {   // ablation build of PAIR_256x256 only
    if ((cfg != GEMM_CFG_AUTO && cfg != GEMM_CFG_PAIR_256x256) || n_peers > 0) return GEMM_ERR_INVALID_VALUE;
    cfg = GEMM_CFG_PAIR_256x256;
  }
  if (cfg == GEMM_CFG_AUTO) {
    cfg = pick_config(M, N, K, acc_type, di.sm_count);
    // an explicit promote_k asks for chunked promotion, which the split-K and 256 x 512
    // kernels do not have (one chain per CTA by design): take the closest kernel that has it
    if (opts && opts->promote_k > 0 &&
        (config_desc(cfg).k_splits || (cfg == GEMM_CFG_PAIR_256x512 && acc_type == GEMM_ACC_F16))) {
      const int64_t pair_tiles = cdiv(M, 256) * cdiv(N, 256);
      cfg = (M <= 128 || 2 * pair_tiles <= di.sm_count / 2) ? GEMM_CFG_SOLO_128x64
            : (opts->promote_k % 128 == 0 ? GEMM_CFG_PAIR_256x256_K128 : GEMM_CFG_PAIR_256x256);
    }
  }
  if (n_peers > 0) cfg = GEMM_CFG_COUNT;   // fused gather: the peer-store build of PAIR_256x256_K128
  const ConfigDesc& cd = config_desc(cfg);
  const int a = acc_type;
  if (cd.fn[a] == nullptr) return GEMM_ERR_INVALID_VALUE;   // e.g. PAIR_256x512 with F32 C

  const int in_type = opts ? opts->in_type : GEMM_IN_F16;
  if (in_type != GEMM_IN_F16 && in_type != GEMM_IN_BF16) return GEMM_ERR_INVALID_VALUE;
  const CUtensorMapDataType in_dt =
      in_type == GEMM_IN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const float* bias = opts ? static_cast<const float*>(opts->bias) : nullptr;
  if (bias && !aligned16(bias)) return GEMM_ERR_MISALIGNED;
  CUtensorMap tm_a, tm_b, tm_c;
  // (no_swizzle ablation: 16-byte-wide boxes, one column of UMMA core matrices each)
  const CUtensorMapSwizzle op_swz = no_swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B;
  const uint32_t op_box = no_swizzle ? 8u : 64u;
  const bool ok =
      encode_2d(&tm_a, in_dt, 2, A, M, K, lda, op_box, static_cast<uint32_t>(128 / cd.a_mc), operand_promotion(lda),
                op_swz) &&
      encode_2d(&tm_b, in_dt, 2, B, K, N, ldb, op_box, 64, operand_promotion(ldb), op_swz) &&
      encode_2d(&tm_c, acc_type == GEMM_ACC_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                acc_type == GEMM_ACC_F32 ? 4 : 2, C, M, N, ldc, static_cast<uint32_t>(cd.c_box_cols[a]),
                cd.k_splits ? 128 : 32,   // split-K: whole 128-row boxes for the reduce-add steps
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                no_swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE
                           : (cd.c_row_bytes[a] == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
  if (!ok) return cuda_fail(cudaErrorInvalidValue);
  // C_in L2-prefetch map: one box = an epilogue warp's whole region (32 rows x tile_n/2
  // columns), unswizzled -- it only drives cp.async.bulk.prefetch, never smem
  // (split-K configs: the C_in slice one CTA reduces, tile_n / k_splits columns x 128 rows, loaded by TMA)
  CUtensorMap tm_cpf;
  if (!encode_2d(&tm_cpf, acc_type == GEMM_ACC_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                 acc_type == GEMM_ACC_F32 ? 4 : 2, C, M, N, ldc,
                 static_cast<uint32_t>(cd.k_splits ? cd.tile_n / cd.k_splits : cd.tile_n / 2), cd.k_splits ? 128 : 32,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cuda_fail(cudaErrorInvalidValue);
  PeerMaps pm;
  std::memset(&pm, 0, sizeof(pm));
  for (int d = 0; d < n_peers; ++d) {
    if (!encode_2d(&pm.m[d], acc_type == GEMM_ACC_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   acc_type == GEMM_ACC_F32 ? 4 : 2, peers[d], M, N, ldc, static_cast<uint32_t>(cd.c_box_cols[a]), 32,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   cd.c_row_bytes[a] == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
      return cuda_fail(cudaErrorInvalidValue);
  }

  GemmParams p;
  std::memset(&p, 0, sizeof(p));
  p.n_peers = n_peers;
  for (int d = 0; d < n_peers; ++d) p.peer_ptr[d] = peers[d];
  p.M = static_cast<int>(M);
  p.N = static_cast<int>(N);
  p.K = static_cast<int>(K);
  const int tile_m = 128 * cd.cta_group;
  const int cl_size = cd.cluster_size();
  p.tiles_m = static_cast<int>(cdiv(cdiv(M, tile_m), cd.b_mc));     // (B multicast: groups of b_mc tiles)
  p.tiles_n = static_cast<int>(cdiv(cdiv(N, cd.tile_n), cd.a_mc));   // (A multicast: groups of a_mc tiles)
  const int64_t tiles = int64_t(p.tiles_m) * p.tiles_n;
  if (tiles * std::max(1, cd.cluster_size()) > 0x7fffffffLL) return GEMM_ERR_INVALID_VALUE;
  p.num_tiles = static_cast<int>(tiles);
  p.k_blocks = static_cast<int>(cdiv(K, cd.bk));
  const int promote = opts ? opts->promote_k : 0;
  if (promote < -1 || (promote > 0 && promote % cd.bk != 0)) return GEMM_ERR_INVALID_VALUE;
  const bool wide32 = cfg == GEMM_CFG_PAIR_256x512 && acc_type == GEMM_ACC_F32;
  p.kb_per_chunk = promote == -1 ? p.k_blocks
                                 : (promote == 0 ? (wide32 ? kDefaultPromoteKWide32 : kDefaultPromoteK) : promote) / cd.bk;
  if ((cfg == GEMM_CFG_PAIR_256x512 && !wide32) || cd.k_splits) {
    if (promote > 0) return GEMM_ERR_INVALID_VALUE;   // one TMEM chain over all of K (its share) by design
    p.kb_per_chunk = std::max(p.k_blocks, 1);
  }
  p.k_splits = cd.k_splits;
  p.k_chunks = static_cast<int>(cdiv(p.k_blocks, p.kb_per_chunk));
  p.group_m = (opts && opts->group_m > 0) ? opts->group_m : 8;
  if (opts && opts->group_m < 0) return GEMM_ERR_INVALID_VALUE;
  const int64_t csize = acc_type == GEMM_ACC_F32 ? 4 : 2;
  p.c_ragged = (N * csize) % 16 != 0;
  p.c_ptr = C;
  p.ldc = ldc;
  const int hints = opts ? opts->l2_hints : 0;
  if (hints < -1 || hints > 1) return GEMM_ERR_INVALID_VALUE;
  p.l2_hints = hints == 0 ? kDefaultL2Hints : (hints > 0 ? 1 : 0);
  p.in_bf16 = in_type == GEMM_IN_BF16;
  p.beta0 = (opts && opts->beta0) ? 1 : 0;
  p.relu = (opts && opts->relu) ? 1 : 0;
  p.accum_f16 = (opts && opts->accum_f16) ? 1 : 0;
  p.bias = bias;
  p.trace = t_trace;
  const int rs = opts ? opts->ring_stages : 0;
  const int stages_max = wide32 ? CfgW32::STAGES : cd.stages;
  if (rs < 0 || rs > stages_max) return GEMM_ERR_INVALID_VALUE;
  p.ring_stages = rs == 0 ? stages_max : rs;
  if (wide32) {
    // reduce-add promotion: no ReLU (no point where the whole sum is in registers), no F16
    // accumulation, N * 4 % 16 == 0 (TMA reduce-adds write whole 16-byte granules); and
    // staggered promotion points at least ring_stages + 2 k-blocks apart (w32_bound)
    if (p.c_ragged || p.relu || p.accum_f16 || n_peers > 0) return GEMM_ERR_INVALID_VALUE;
    if (p.kb_per_chunk < p.k_blocks && p.kb_per_chunk / 2 < p.ring_stages + 2) return GEMM_ERR_INVALID_VALUE;
  }
  const int ab = opts ? opts->acc_bufs : 0;
  if (ab < 0 || ab > 2) return GEMM_ERR_INVALID_VALUE;
  p.acc_bufs = ab == 0 ? 2 : ab;

  // persistent grid: one cluster per resident slot; an explicit max_clusters may
  // also exceed the resident slots (a non-persistent launch, for ablation)
  int clusters = di.max_clusters[cfg][a];
  if (opts && opts->max_clusters > 0) clusters = opts->max_clusters;
  if (opts && opts->max_clusters < 0) return GEMM_ERR_INVALID_VALUE;
  const int grid_cap = clusters;   // (stream-K below one wave uses the whole grid)
  clusters = static_cast<int>(std::min<int64_t>(clusters, tiles));
  if (cd.k_splits) clusters = static_cast<int>(tiles);   // one tile per cluster (non-persistent)

  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(clusters * cl_size), 1, 1);
  lc.blockDim = dim3(static_cast<unsigned>(cd.threads), 1, 1);
  lc.dynamicSmemBytes = cd.smem[a];
  lc.stream = stream;
  cudaLaunchAttribute attr[3];
  if (cl_size > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cd.launch_cluster();
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.numAttrs = 1;
    if (cd.hybrid) {   // (the grid is a whole number of groups of cl_size CTAs)
      attr[1].id = cudaLaunchAttributePreferredClusterDimension;
      attr[1].val.preferredClusterDim.x = cl_size;
      attr[1].val.preferredClusterDim.y = 1;
      attr[1].val.preferredClusterDim.z = 1;
      lc.numAttrs = 2;
    }
  }
  const int raster = opts ? opts->raster : 0;
  if (raster < -1 || raster > 1) return GEMM_ERR_INVALID_VALUE;
  p.snake = raster == 0 ? kDefaultSnake : (raster > 0 ? 1 : 0);
  const int cred = opts ? opts->c_reduce : 0;
  if (cred < -1 || cred > 1) return GEMM_ERR_INVALID_VALUE;
  p.c_reduce = cred == 0 ? kDefaultCReduce : (cred > 0 ? 1 : 0);
  const int pdl_opt = opts ? opts->pdl : 0;
  if (pdl_opt < -1 || pdl_opt > 1) return GEMM_ERR_INVALID_VALUE;
  if (pdl_opt == 0 ? kDefaultPdl : pdl_opt > 0) {
    attr[lc.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[lc.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++lc.numAttrs;
  }
  lc.attrs = lc.numAttrs ? attr : nullptr;
  KernelFn fn = cd.fn[a];
  // stream-K: when the last wave of tiles is partial, the last partial wave plus one full
  // wave are shared out over all clusters as equal runs of k-blocks (gemm_sm100.cuh Work);
  // the partial tiles meet in C through the reduce-add epilogue, in a fixed order
  const int tro = opts ? opts->tail_ring : 0;
  if (tro < -1 || tro > 1) return GEMM_ERR_INVALID_VALUE;
  p.tail_ring = tro >= 0 ? 1 : 0;
  const int skopt = opts ? opts->stream_k : 0;
  void* sk_private = nullptr;   // a captured stream-K launch's own token counters (freed below)
  if (skopt < -1 || skopt > 1) return GEMM_ERR_INVALID_VALUE;
  p.sk_tile0 = p.num_tiles;
  // F32 C: the two partials of a split tile meet by reduce-add (needs the reduce-add epilogue);
  // F16 C: the first part stores C_in + its partial, the second reduce-adds its own (R18)
  const bool sk_ok = cd.sk_fn[a] != nullptr && n_peers == 0 && !no_swizzle && (a == GEMM_ACC_F16 || p.c_reduce) && !p.beta0 &&
                     p.bias == nullptr && !p.relu && !p.accum_f16 && !p.c_ragged &&
                     grid_cap * 16 <= kSkWindow &&
                     (tiles % grid_cap + grid_cap) * static_cast<int64_t>(p.k_blocks) < 0x7fffffffLL;
  const int64_t skc = grid_cap;   // stream-K runs on the whole grid
  const int64_t rem = tiles % skc, waves = tiles / skc;
  const bool sk_want = skopt > 0 || (skopt == 0 && !(opts && opts->max_clusters > 0) &&
                                      stream_k_pays(tiles, skc, K, a));
  // (less than one wave: every tile is shared out, as long as each cluster gets at least
  // half a tile of k-blocks, so a tile is split at most three ways and a chain of waits is
  // at most two long)
  if (sk_ok && sk_want && rem > 0 && (waves >= 1 || 2 * tiles >= skc)) {
    clusters = static_cast<int>(skc);
    lc.gridDim = dim3(static_cast<unsigned>(clusters * cl_size), 1, 1);
    p.sk_tile0 = waves >= 1 ? static_cast<int>(tiles - rem - clusters) : 0;
    // run boundaries within k_blocks / 8 of a tile edge snap to it (at least one full wave;
    // below one wave equal runs matter more: profiles/r01/stream_k.md, snapping)
    p.sk_snap = waves >= 1 ? p.k_blocks / 8 : 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess) cap = cudaStreamCaptureStatusNone;
    if (cap == cudaStreamCaptureStatusActive) {
      // A captured launch replays for the graph's whole lifetime, so a window of the shared
      // pool would be taken again by eager launches on other streams (every kSkWindows
      // launches) while a replay runs.  It gets counters of its own instead: graph memory
      // nodes that every replay allocates, zeroes and frees around the kernel.
      void* buf = nullptr;
      cudaError_t ce = cudaMallocAsync(&buf, kSkWindow * sizeof(unsigned), stream);
      if (ce == cudaSuccess) ce = cudaMemsetAsync(buf, 0, kSkWindow * sizeof(unsigned), stream);
      if (ce != cudaSuccess) return cuda_fail(ce);
      p.sk_flags = static_cast<unsigned*>(buf);
      sk_private = buf;
    } else {
      p.sk_flags = di.sk_flags + sk_window_base(g_dev[dev].sk_next.fetch_add(1u));
    }
    fn = cd.sk_fn[a];
  }
  if (cfg == GEMM_CFG_PAIR_256x512 && a == GEMM_ACC_F16 && (p.bias != nullptr || p.relu || p.accum_f16))
    fn = kWideExtFn[a];
  if (wide32 && (p.bias != nullptr || p.beta0)) fn = kWideExtFn[a];
  if (no_swizzle) fn = kNoSwizzleFn[a];
  cudaError_t e = cudaLaunchKernelEx(&lc, fn, tm_a, tm_b, tm_c, p, pm, tm_cpf);
  if (sk_private) {
    const cudaError_t fe = cudaFreeAsync(sk_private, stream);
    if (e == cudaSuccess) e = fe;
  }
  if (e != cudaSuccess) return cuda_fail(e);
  t_trace = nullptr;   // (a trace is armed for one launch)
  t_last_launches = 1;
  return GEMM_OK;
}

}  // namespace

extern "C" {

gemm_status_t gemm_f16_ex(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                          void* C, int64_t ldc, int acc_type, void* stream, const gemm_options_t* opts) {
  t_last_launches = 0;
  bool no_work = false;
  gemm_status_t st = validate(M, N, K, A, lda, B, ldb, C, ldc, acc_type, &no_work);
  if (st != GEMM_OK || no_work) return st;
  return launch(M, N, K, A, lda, B, ldb, C, ldc, acc_type, static_cast<cudaStream_t>(stream), opts);
}

gemm_status_t gemm_f16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                       void* C, int64_t ldc, int acc_type, void* stream) {
  return gemm_f16_ex(M, N, K, A, lda, B, ldb, C, ldc, acc_type, stream, nullptr);
}

gemm_status_t gemm_f16_gather(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B_r,
                              int64_t ldb, int64_t n0, int64_t nr, void* C, int64_t ldc, void* const* peers,
                              int n_peers, int acc_type, void* stream) {
  t_last_launches = 0;
  if (n0 < 0 || nr < 0 || N < 0 || n0 + nr > N) return GEMM_ERR_INVALID_VALUE;
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && !peers)) return GEMM_ERR_INVALID_VALUE;
  const int64_t csz = acc_type == GEMM_ACC_F32 ? 4 : 2;
  if (acc_type != GEMM_ACC_F32 && acc_type != GEMM_ACC_F16) return GEMM_ERR_INVALID_VALUE;
  if (ldc < std::max<int64_t>(1, N)) return GEMM_ERR_INVALID_VALUE;
  // this rank's slab [n0, n0 + nr) of C, and of every peer buffer (same shape and ld)
  char* C_slab = C ? static_cast<char*>(C) + n0 * csz : nullptr;
  bool no_work = false;
  gemm_status_t st = validate(M, nr, K, A, lda, B_r, ldb, C_slab, ldc, acc_type, &no_work);
  if (st != GEMM_OK || no_work) return st;
  void* peer_slab[kMaxPeers];
  for (int d = 0; d < n_peers; ++d) {
    if (!peers[d]) return GEMM_ERR_INVALID_VALUE;
    peer_slab[d] = static_cast<char*>(peers[d]) + n0 * csz;
    if (!aligned16(peer_slab[d])) return GEMM_ERR_MISALIGNED;
  }
  return launch(M, nr, K, A, lda, B_r, ldb, C_slab, ldc, acc_type, static_cast<cudaStream_t>(stream), nullptr,
                peer_slab, n_peers);
}

gemm_status_t gemm_f16_host(int64_t M, int64_t N, int64_t K, const void* hA, int64_t lda, const void* hB,
                            int64_t ldb, void* hC, int64_t ldc, int acc_type, void* dA, int64_t ldda, void* dB,
                            int64_t lddb, void* dC, int64_t lddc, void* stream) {
  t_last_launches = 0;
  bool no_work = false;
  gemm_status_t st = validate(M, N, K, dA, ldda, dB, lddb, dC, lddc, acc_type, &no_work);
  if (st != GEMM_OK || no_work) return st;
  if (!hC) return GEMM_ERR_INVALID_VALUE;   // hA / hB == NULL: operand already resident in dA / dB
  if ((hA && lda < std::max<int64_t>(1, K)) || (hB && ldb < std::max<int64_t>(1, N)) ||
      ldc < std::max<int64_t>(1, N))
    return GEMM_ERR_INVALID_VALUE;
  int dev = 0;
  st = device_ready(&dev);
  if (st != GEMM_OK) return st;
  HostStreams& hs = host_streams(dev);
  if (hs.err != cudaSuccess) return cuda_fail(hs.err);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t csz = acc_type == GEMM_ACC_F32 ? 4 : 2;

  // Row-block pipeline: B goes first (every block needs it); then block j's A
  // and C_in rows are copied in on the H2D stream, its GEMM runs on the
  // caller's stream, and its C_out rows go back on the D2H stream -- so the
  // two copy directions and the tensor cores overlap.
  const int64_t kMinRows = 1024;
  int64_t nblk = std::min<int64_t>(8, std::max<int64_t>(1, M / kMinRows));
  const int64_t rb = ((cdiv(M, nblk) + 255) / 256) * 256;
  nblk = cdiv(M, rb);
  cudaEvent_t ev_start, ev_done, ev_in[8], ev_gemm[8];
  cudaError_t e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
  for (int j = 0; j < nblk && e == cudaSuccess; ++j) {
    e = cudaEventCreateWithFlags(&ev_in[j], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_gemm[j], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  e = cudaEventRecord(ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hs.h2d, ev_start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hs.d2h, ev_start, 0);
  if (e == cudaSuccess && hB) e = cudaMemcpy2DAsync(dB, lddb * 2, hB, ldb * 2, N * 2, K, cudaMemcpyHostToDevice, hs.h2d);
  int launches = 0;
  for (int64_t j = 0; j < nblk && e == cudaSuccess; ++j) {
    const int64_t r0 = j * rb, mj = std::min(rb, M - r0);
    char* dAj = static_cast<char*>(dA) + r0 * ldda * 2;
    char* hCj = static_cast<char*>(hC) + r0 * ldc * csz;
    char* dCj = static_cast<char*>(dC) + r0 * lddc * csz;
    if (hA) {
      const char* hAj = static_cast<const char*>(hA) + r0 * lda * 2;
      e = cudaMemcpy2DAsync(dAj, ldda * 2, hAj, lda * 2, K * 2, mj, cudaMemcpyHostToDevice, hs.h2d);
    }
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(dCj, lddc * csz, hCj, ldc * csz, N * csz, mj, cudaMemcpyHostToDevice, hs.h2d);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[j], hs.h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_in[j], 0);
    if (e != cudaSuccess) break;
    st = launch(mj, N, K, dAj, ldda, dB, lddb, dCj, lddc, acc_type, s, nullptr);
    if (st != GEMM_OK) break;
    ++launches;
    e = cudaEventRecord(ev_gemm[j], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hs.d2h, ev_gemm[j], 0);
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(hCj, ldc * csz, dCj, lddc * csz, N * csz, mj, cudaMemcpyDeviceToHost, hs.d2h);
  }
  if (e == cudaSuccess && st == GEMM_OK) e = cudaEventRecord(ev_done, hs.d2h);
  if (e == cudaSuccess && st == GEMM_OK) e = cudaStreamWaitEvent(s, ev_done, 0);
  cudaEventDestroy(ev_start);
  cudaEventDestroy(ev_done);
  for (int j = 0; j < nblk; ++j) {
    cudaEventDestroy(ev_in[j]);
    cudaEventDestroy(ev_gemm[j]);
  }
  if (st != GEMM_OK) return st;
  if (e != cudaSuccess) return cuda_fail(e);
  t_last_launches = launches;
  return GEMM_OK;
}

int gemm_f16_pick_config_for(int64_t M, int64_t N, int64_t K, int acc_type, int sm_count) {
  if (acc_type != GEMM_ACC_F32 && acc_type != GEMM_ACC_F16) return -1;
  if (sm_count < 2 || M < 0 || N < 0 || K < 0) return -1;
  return pick_config(M, N, K, acc_type, sm_count);
}

int gemm_f16_pick_config(int64_t M, int64_t N, int64_t K, int acc_type) {
  if (acc_type != GEMM_ACC_F32 && acc_type != GEMM_ACC_F16) return -1;
  int dev = 0;
  if (device_ready(&dev) != GEMM_OK) return -1;
  return pick_config(M, N, K, acc_type, g_dev[dev].sm_count);
}

gemm_status_t gemm_f16_config_info(int config, int acc_type, int* tile_m, int* tile_n, int* cta_group, int* stages,
                                   int* smem_bytes) {
  if (config <= 0 || config >= GEMM_CFG_COUNT) return GEMM_ERR_INVALID_VALUE;
  if (acc_type != GEMM_ACC_F32 && acc_type != GEMM_ACC_F16) return GEMM_ERR_INVALID_VALUE;
  const ConfigDesc& cd = config_desc(config);
  if (cd.fn[acc_type] == nullptr) return GEMM_ERR_INVALID_VALUE;
  if (tile_m) *tile_m = 128 * cd.cta_group;
  if (tile_n) *tile_n = cd.tile_n;
  if (cta_group) *cta_group = cd.cta_group;
  if (stages) *stages = cd.stages;
  if (smem_bytes) *smem_bytes = cd.smem[acc_type];
  return GEMM_OK;
}

int gemm_f16_last_launches(void) { return t_last_launches; }

int gemm_f16_diag_set_trace(void* trace) {
  t_trace = static_cast<unsigned long long*>(trace);
  return 0;
}

uint32_t gemm_f16_diag_sk_window_base(uint32_t launch_index) { return sk_window_base(launch_index); }
uint32_t gemm_f16_diag_sk_window_slots(void) { return kSkWindow; }
uint32_t gemm_f16_diag_sk_pool_slots(void) { return kSkFlagSlots; }

const char* gemm_status_string(gemm_status_t s) {
  switch (s) {
    case GEMM_OK: return "GEMM_OK";
    case GEMM_ERR_INVALID_VALUE: return "GEMM_ERR_INVALID_VALUE";
    case GEMM_ERR_MISALIGNED: return "GEMM_ERR_MISALIGNED";
    case GEMM_ERR_UNSUPPORTED_DEVICE: return "GEMM_ERR_UNSUPPORTED_DEVICE";
    case GEMM_ERR_CUDA: return "GEMM_ERR_CUDA";
  }
  return "GEMM_ERR_UNKNOWN";
}

int gemm_last_cuda_error(void) { return t_last_cuda_error; }

}  // extern "C"
