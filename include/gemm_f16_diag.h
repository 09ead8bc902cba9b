/*
 * gemm_f16_diag.h -- DIAGNOSTIC entry points of libgemm_f16.so.  Not part of the
 * product contract (include/gemm_f16.h): they never change a result, and no
 * product path calls them.  Used by bench.py (the SM clock the kernel ran at)
 * and tools/trace_tiles.py (per-tile timelines behind profiles/*.md).
 */
#ifndef GEMM_F16_DIAG_H_
#define GEMM_F16_DIAG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Arm a per-tile trace for the NEXT gemm_f16 / gemm_f16_ex call on this host
 * thread (the call consumes it; gemm_f16_diag_set_trace(NULL) disarms).
 *   trace   device buffer of 512 uint64 (8 per tile for 60 tiles, rows 62-63 for
 *           kernel entry/setup/exit).  The traced CTA index is read from element
 *           511 (0 = CTA 0), which the caller sets before the call.  The kernel
 *           writes globaltimer stamps (ns) and SM cycle counts (clock64) of that
 *           CTA's MMA and epilogue warps per tile.
 * Returns 0.  The buffer must stay valid until the traced kernel completes.
 */
int gemm_f16_diag_set_trace(void* trace);

/*
 * First token-counter slot of the stream-K window that the launch with this
 * index (the library's per-device launch counter) takes: windows are whole,
 * fixed and taken round robin, so two windows handed out fewer than
 * (pool / window) launches apart never overlap.  Pure host function, exported
 * so the CPU tests can pin the allocator (no overlap at the wrap).
 */
uint32_t gemm_f16_diag_sk_window_base(uint32_t launch_index);

/* Size of one stream-K window and of the whole pool, in token-counter slots. */
uint32_t gemm_f16_diag_sk_window_slots(void);
uint32_t gemm_f16_diag_sk_pool_slots(void);

#ifdef __cplusplus
}
#endif

#endif /* GEMM_F16_DIAG_H_ */
