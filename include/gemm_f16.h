/*
 * gemm_f16.h -- C ABI of the B200 (sm_100a) tensor-core GEMM library
 * (libgemm_f16.so), the one hot path of arXiv 2108.13191:
 *
 *     C[i][j] <- C[i][j] + sum_k A[i][k] * B[k][j]      0 <= i < M, 0 <= j < N
 *
 * PAPER.md Sec. 4: "we consider a matmul of the form C = AB + C (all
 * three matrices are stored in a row-major layout)"; naive loop nest Sec. 3.1
 * P:412-438; F16 inputs with F32 accumulate/output Sec. 4.1; F16
 * inputs with F16 accumulate/output Sec. 4.2 P:976-980.  No alpha / beta.
 *
 * Precision (readings R3/R4): A and B are IEEE binary16.  The tensor
 * cores accumulate in F32 in both modes; GEMM_ACC_F16 reads and writes C as
 * binary16 and rounds once to nearest-even on output (overflow -> +-Inf).
 *
 * Layout: every matrix is row-major with a leading dimension in ELEMENTS
 * (element (r,c) at ptr[r*ld + c]).  Elements of C outside the M x N window
 * (ld padding) are never read or written.
 *
 * Ownership: the caller owns all buffers; the library allocates no device
 * memory.  C must not alias A or B.  Buffers must stay valid until the work
 * enqueued on `stream` has completed.
 *
 * Errors: every argument check happens before anything is enqueued, so an
 * error status means nothing was launched.  Calls are enqueue-only
 * (asynchronous with respect to the host); kernel faults surface at the
 * caller's next synchronisation, as usual in CUDA.  Reentrant and thread-safe.
 * Results are bitwise reproducible for identical inputs, shape, mode and
 * options on the same device model: every element's sum has a fixed order.
 * The F32 epilogue adds the tile into C with a TMA reduce-add, one writer per
 * element.  The split-K configurations combine their partial sums in a fixed
 * order, through distributed shared memory or in reduce-add steps separated
 * by cluster barriers.  No atomics race.
 */
#ifndef GEMM_F16_H_
#define GEMM_F16_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GEMM_ACC_F32 = 0, /* C is float (IEEE binary32); F32 accumulate  */
  GEMM_ACC_F16 = 1  /* C is IEEE binary16; F16 in/out, see R3     */
} gemm_acc_t;

/* Input element type of A and B (gemm_options_t.in_type). */
typedef enum {
  GEMM_IN_F16 = 0,  /* IEEE binary16 (the paper's evaluated inputs) */
  GEMM_IN_BF16 = 1  /* bfloat16 (same tensor-core rate)                      */
} gemm_in_t;

typedef enum {
  GEMM_OK = 0,
  GEMM_ERR_INVALID_VALUE = 1,      /* negative extent, short leading dim, NULL with work, bad mode/option */
  GEMM_ERR_MISALIGNED = 2,         /* pointer not 16-byte aligned or ld*sizeof(elem) not a multiple of 16 */
  GEMM_ERR_UNSUPPORTED_DEVICE = 3, /* current device is not compute capability 10.0 (B200, sm_100a)       */
  GEMM_ERR_CUDA = 4                /* a CUDA runtime/driver call failed; see gemm_last_cuda_error()         */
} gemm_status_t;

/* Kernel configurations (tile = (128 * cta_group) x BN per MMA group). */
typedef enum {
  GEMM_CFG_AUTO = 0,
  GEMM_CFG_PAIR_256x256 = 1, /* cta_group::2, 2-CTA cluster, UMMA 256x256x16 */
  GEMM_CFG_PAIR_256x128 = 2, /* cta_group::2, 2-CTA cluster, UMMA 256x128x16 */
  GEMM_CFG_SOLO_128x256 = 3, /* cta_group::1, UMMA 128x256x16               */
  GEMM_CFG_SOLO_128x128 = 4, /* cta_group::1, UMMA 128x128x16               */
  GEMM_CFG_SOLO_128x64 = 5,  /* cta_group::1, UMMA 128x64x16                */
  GEMM_CFG_PAIR_256x256_S5 = 6, /* as PAIR_256x256, 5 stages, 2 epilogue staging slots per warp */
  GEMM_CFG_PAIR_256x256_S4 = 7, /* as PAIR_256x256, 4 stages, 3 epilogue staging slots per warp */
  GEMM_CFG_PAIR_256x256_K128 = 8, /* as PAIR_256x256 with 128-deep K stages (3 stages)        */
  GEMM_CFG_PAIR_256x512 = 9, /* cta_group::2, 2 UMMAs 256x256x16 per K step (256 x 512 pair
                                tile).  F16 C: one TMEM chain over all of K, C_in held in
                                registers.  F32 C: K-chunk promotion by TMA reduce-add into C
                                at staggered points of the two accumulator halves (default
                                promote_k 4096); N * 4 % 16 == 0 and no ReLU / accum_f16, else
                                GEMM_ERR_INVALID_VALUE.  AUTO picks it for F16 C only */
  GEMM_CFG_SPLITK_128x256_S2 = 10, /* split-K over a 2-CTA cluster: cta_group::1 UMMA 128x256x16, each
                                      CTA one half of K, partials reduced through distributed shared
                                      memory (fixed order, no workspace); one tile per cluster.  Each
                                      CTA keeps one TMEM chain over its K / S (promote_k must be 0 or
                                      -1): with F32 C, K / S > 8192 exceeds the 1e-5 error bar */
  GEMM_CFG_SPLITK_128x256_S4 = 11, /* as SPLITK_128x256_S2 with 4 CTAs (quarters of K) per cluster */
  GEMM_CFG_SPLITK_128x128_S4 = 12, /* as SPLITK_128x256_S4 with UMMA 128x128x16 tiles */
  GEMM_CFG_SOLO_128x64_MC4 = 13,  /* as SOLO_128x64 in 4-CTA clusters along N: each CTA loads a quarter
                                     of the shared A box and TMA-multicasts it to the other three */
  GEMM_CFG_SOLO_128x128_MC4 = 14, /* as SOLO_128x128, with the same A multicast */
  GEMM_CFG_SPLITK_128x128_S2 = 15, /* as SPLITK_128x128_S4 with 2 CTAs (halves of K) per cluster */
  GEMM_CFG_PAIR2_256x256_MCB = 16, /* as PAIR_256x256_K128, two CTA pairs per 4-CTA cluster on
                                      tiles (2t, n) and (2t+1, n): each pair loads half of the
                                      shared B box and TMA-multicasts it into the other pair.  No
                                      stream-K; selectable, not picked (4-CTA clusters fit on only
                                      ~132 of 148 SMs) */
  GEMM_CFG_PAIR2_256x256_MCH = 17, /* the MCB kernel launched with cluster dim 2 and the preferred
                                      cluster dim 4 (cudaLaunchAttributePreferredClusterDimension):
                                      blocks 4i..4i+3 run as one 4-CTA cluster that multicasts B
                                      where the hardware can place one (~132 of 148 SMs) and as two
                                      2-CTA clusters that load B themselves elsewhere, so every SM
                                      holds a CTA.  Same tiles, same order of operations: results
                                      are bitwise those of PAIR_256x256_K128.  No stream-K */
  GEMM_CFG_COUNT = 18
} gemm_config_t;

typedef struct {
  int config;       /* gemm_config_t; GEMM_CFG_AUTO picks from the shape              */
  int max_clusters; /* 0: one persistent cluster per resident slot; >0: exactly this   */
                    /* many clusters (capped at the tile count; more than the resident */
                    /* slots gives a non-persistent launch)                            */
  int group_m;      /* 0: default raster group height (tiles); >0: override            */
  int promote_k;    /* K elements per TMEM accumulation chunk before the partial sum is  */
                    /* added into F32 registers (RN): 0 = default 2048, -1 = never       */
                    /* (one TMEM chain per tile), else a positive multiple of the        */
                    /* config's K stage depth (64, or 128 for PAIR_256x256_K128).  With   */
                    /* config AUTO a positive value steers the choice away from the       */
                    /* split-K and PAIR_256x512 kernels (one chain per CTA by design)     */
  /* Fused epilogue (the paper's fusion motivation):       */
  /*   C <- relu?( beta * C_in + A.B + bias[j] ), one rounding to C's type                */
  int in_type;      /* gemm_in_t: GEMM_IN_F16 (default) or GEMM_IN_BF16 for A and B       */
  int beta0;        /* 0: C += A.B (default); 1: C = A.B (C_in not read)                  */
  int relu;         /* 1: max(x, 0) applied before rounding (NaN propagates)              */
  const void* bias; /* NULL, or device float[N] added to every row (16-byte aligned)      */
  int accum_f16;    /* EXPERIMENT, 0 normally: 1 = the tensor core accumulates in binary16 */
                    /* (instruction c_format F16: the paper's literal F16 accumulation,   */
                    /* P:979-980; DESIGN R3/R16).  Partial sums are still promoted into   */
                    /* F32 registers every promote_k (-1: one binary16 chain per tile)    */
  int stream_k;     /* CTA-pair 256x256 configs, no bias/ReLU/beta=0/ragged N (F32 C:       */
                    /* reduce-add epilogue; F16 C: DESIGN R18).  1 = when the last wave of  */
                    /* tiles is partial, share the last partial wave plus one full wave     */
                    /* (below one wave: every tile) out over all clusters as equal runs of  */
                    /* k-blocks; the parts of a split tile meet in C in a fixed order (F32: */
                    /* reduce-adds; F16: a store, then an F16 reduce-add), so results are   */
                    /* deterministic for a given grid.  0 = default: on when max_clusters   */
                    /* is 0 and stream-K pays (1-8 full waves with the last <= 50 % full,   */
                    /* F16 40 %, for K >= 4096 or <= 30 % for K > 2048; below one wave,     */
                    /* 50-70 % of the clusters busy and K >= 4096 F16 / 8192 F32).  -1 = off */
  /* Ablation knobs (the paper's fig:gradual-opts; profiles/r02/ablation.md).  */
  /* Each 0 = the shipped default; results stay within the parity bars for every value.  */
  int ring_stages;  /* 0: all stages of the config; 1..stages: use a shallower smem ring   */
  int acc_bufs;     /* 0 or 2: double-buffered TMEM accumulator; 1: single (no overlap)   */
  int l2_hints;     /* 0: default; 1: TMA L2 eviction hints on; -1: off                   */
  int pdl;          /* 0: default; 1: programmatic dependent launch (the kernel's prologue */
                    /* overlaps the previous grid's tail in the stream; it waits for that  */
                    /* grid before touching global memory); -1: off                        */
  int raster;       /* 0: default; 1: serpentine raster -- odd groups of group_m tile-rows */
                    /* walk their column strips right to left; -1: plain                   */
  int c_reduce;     /* F32 C, C += A.B (+ bias; no ReLU, N % 4 == 0): 1 = the epilogue adds */
                    /* its tile into C with a TMA reduce-add store instead of loading C_in */
                    /* into shared memory (without a bias bitwise the same single RN add;   */
                    /* with one, C_in + RN(acc + bias)); -1 = off; 0 = default (on)         */
  int tail_ring;    /* 0: default (on); -1: off.  On a CTA's last tile, when no C_in is     */
                    /* staged, all output chunks are staged at once in the idle operand    */
                    /* ring and stored back to back (256x256-class pair, 1-CTA and        */
                    /* PAIR_256x512 configs)                                               */
  int swizzle;      /* 0: default (128B swizzle everywhere); -1: ABLATION -- operands in the */
                    /* no-swizzle UMMA layout (16-byte TMA boxes) and unswizzled epilogue   */
                    /* staging (bank conflicts), the B200 analogue of the paper's unpadded  */
                    /* shared memory (Sec. 3.3).  PAIR_256x256 (or AUTO) only,   */
                    /* else GEMM_ERR_INVALID_VALUE                                         */
  int warp_specialize; /* 0: default; -1: ABLATION -- the non-warp-specialised kernel: one  */
                    /* 128x128 tile per CTA, one thread runs loads and MMAs as a software  */
                    /* pipeline, the epilogue follows the mainloop (no overlap), plain     */
                    /* global stores.  No bias / ReLU / accum_f16 (GEMM_ERR_INVALID_VALUE)  */
} gemm_options_t;

/*
 * gemm_f16: enqueue C += A.B on `stream` (cudaStream_t; NULL = legacy default).
 *   M, N, K    extents, each in [0, 2^31-1].  M == 0 or N == 0 or K == 0:
 *              GEMM_OK with nothing launched (K == 0 leaves C unchanged).
 *   A, lda     device pointer, binary16, M x K row-major, lda >= max(1, K)
 *   B, ldb     device pointer, binary16, K x N row-major, ldb >= max(1, N)
 *   C, ldc     device pointer, float (GEMM_ACC_F32) or binary16 (GEMM_ACC_F16),
 *              M x N row-major, ldc >= max(1, N); read (C_in) and written (C_out)
 *   acc_type   gemm_acc_t
 * Alignment (TMA): A, B, C 16-byte aligned; lda*2, ldb*2 and ldc*sizeof(C elem)
 * multiples of 16 bytes, else GEMM_ERR_MISALIGNED.  There is no slow fallback.
 */
gemm_status_t gemm_f16(int64_t M, int64_t N, int64_t K,
                       const void* A, int64_t lda,
                       const void* B, int64_t ldb,
                       void* C, int64_t ldc,
                       int acc_type, void* stream);

/* gemm_f16 with explicit options (NULL = defaults).  Same contract. */
gemm_status_t gemm_f16_ex(int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda,
                          const void* B, int64_t ldb,
                          void* C, int64_t ldc,
                          int acc_type, void* stream,
                          const gemm_options_t* opts);

/*
 * gemm_f16_gather: one rank's share of an N-sharded C += A.B, fused with the
 * all-gather of C.  Every rank holds a full M x N
 * buffer C; this rank owns the column slab [n0, n0 + nr):
 *     C[:, n0:n0+nr] <- C[:, n0:n0+nr] + A . B_r
 * with C_in read from its own C, and each finished C tile is stored by the
 * epilogue (TMA) into C AND into every peers[d][:, n0:n0+nr], d < n_peers --
 * so the gather overlaps the math tile by tile instead of following it.
 *   A, lda       binary16 M x K (replicated on every rank)
 *   B_r, ldb     binary16 K x nr, this rank's column slab of B, ldb >= nr
 *   C, ldc       this rank's full M x N buffer (float or binary16), read+written
 *   peers        n_peers (<= 7) device addresses of the other ranks' full C
 *                buffers with the same shape, ld and type, mapped into this
 *                process (NVLink peer / symmetric-memory pointers) or plain
 *                buffers on this device; written only in columns [n0, n0+nr)
 * Alignment as gemm_f16, plus n0*sizeof(C elem) a multiple of 16 bytes (slab
 * boundaries at multiples of 8 columns).  Writes to peers are complete when the
 * kernel completes; the caller orders readers after it (e.g. a cross-rank
 * barrier after synchronising `stream`).
 */
gemm_status_t gemm_f16_gather(int64_t M, int64_t N, int64_t K,
                              const void* A, int64_t lda,
                              const void* B_r, int64_t ldb,
                              int64_t n0, int64_t nr,
                              void* C, int64_t ldc,
                              void* const* peers, int n_peers,
                              int acc_type, void* stream);

/*
 * gemm_f16_host: the same operation on HOST buffers (end-to-end path).
 * Copies A, B and C_in into the caller's device scratch (dA/ldda, dB/lddb,
 * dC/lddc: same element types and alignment rules as gemm_f16), runs the GEMM
 * and copies C_out back into hC.  The work is pipelined over row blocks of
 * >= 1024 rows (at most 8): copies in run on a library-owned H2D stream, the
 * GEMMs on `stream`, copies out on a library-owned D2H stream, joined to
 * `stream` by events -- the call is ordered after earlier work on `stream` and
 * later work on `stream` is ordered after it.  Host buffers should be
 * page-locked for the copies to be asynchronous.  The caller synchronises
 * `stream` before reading hC.
 * Resident operands: hA == NULL (resp. hB == NULL) means A (resp. B) is already
 * in dA (dB), written by work ordered before this call on `stream` -- e.g. two
 * GEMMs on the same operands copy A and B once; lda (ldb) is then ignored.
 * hC may not be NULL.
 */
gemm_status_t gemm_f16_host(int64_t M, int64_t N, int64_t K,
                            const void* hA, int64_t lda,
                            const void* hB, int64_t ldb,
                            void* hC, int64_t ldc,
                            int acc_type,
                            void* dA, int64_t ldda,
                            void* dB, int64_t lddb,
                            void* dC, int64_t lddc,
                            void* stream);

/* Configuration gemm_f16 would use for this shape (a gemm_config_t), or -1. */
int gemm_f16_pick_config(int64_t M, int64_t N, int64_t K, int acc_type);

/* The same table for a given SM count, without touching a device (pure host
 * function; -1 for a bad mode or sm_count < 2). */
int gemm_f16_pick_config_for(int64_t M, int64_t N, int64_t K, int acc_type, int sm_count);

/* Static description of a configuration: tile rows/cols, cta_group, pipeline
 * stages, dynamic shared memory bytes.  Returns GEMM_ERR_INVALID_VALUE for an
 * unknown config.  Pure host function (no device needed). */
gemm_status_t gemm_f16_config_info(int config, int acc_type, int* tile_m, int* tile_n,
                                   int* cta_group, int* stages, int* smem_bytes);

/* Number of kernel launches the last successful gemm_f16* call on this host
 * thread enqueued (gemm_f16: 0 or 1; gemm_f16_host: one per row block). */
int gemm_f16_last_launches(void);

const char* gemm_status_string(gemm_status_t s);

/* Thread-local cudaError_t behind the last GEMM_ERR_CUDA on this thread. */
int gemm_last_cuda_error(void);

#ifdef __cplusplus
}
#endif

#endif /* GEMM_F16_H_ */
