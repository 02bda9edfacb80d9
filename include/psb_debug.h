/* psb_debug.h -- diagnostics exported by libpsb.so (NOT part of the drop-in
 * boundary in psb.h; used by tools/probe_*.py to measure the design).
 *
 * Step milestones: with PSB_STEP_MARKS=1 in the environment at ctx creation,
 * every psb_sync_step records CUDA events between its phases; this returns
 * the milliseconds between consecutive events recorded since the last call
 * (synchronizes the device). */
#ifndef PSB_DEBUG_H_
#define PSB_DEBUG_H_

#include "psb.h"

#ifdef __cplusplus
extern "C" {
#endif

PSB_API int psb_debug_marks(psb_ctx* ctx, float* out_ms, int max);

/* NVLink probes (one process, several GPUs): enable peer access, and a
 * 16-byte SM copy / an update-list scatter theta[idx] = val between any two
 * pointers of the process's address space. */
PSB_API int psb_debug_enable_peer(int dev, int peer);
PSB_API int psb_debug_copy16(void* dst, const void* src, size_t bytes, int ctas, void* stream);
PSB_API int psb_debug_scatter(float* theta, const uint32_t* idx, const float* val, size_t cnt, int ctas,
                              void* stream);

/* `iters` bare payload exchanges of bytes_per_rank between the ranks of a
 * multi-rank ctx (every rank calls it together). */
PSB_API psb_status psb_debug_exchange(psb_ctx* ctx, size_t bytes_per_rank, int iters, psb_stream_t stream);

/* Only in a build with EXTRA_NVFLAGS=-DPSB_APPLY_TRACE: per-phase CTA time
 * sums of the sparse apply. */
PSB_API void psb_debug_apply_trace(unsigned long long* out8, int reset);

/* Only in a build with EXTRA_NVFLAGS=-DPSB_SCAN_TRACE: globaltimer (ns) at
 * entry and exit of every CTA of the last K1 streaming pass, as pairs; returns
 * the number of CTAs copied (0 in a normal build). */
PSB_API int psb_debug_scan_trace(unsigned long long* out, int max_ctas);
/* Same build: per CTA of the last candidate phase, 16 words -- globaltimer at
 * its phase boundaries (unused slots 0) and, in word 15, (tiles << 32 |
 * entries) of its slice. */
PSB_API int psb_debug_cand_trace(unsigned long long* out, int max_ctas);

/* Device timestamps (globaltimer, ns) recorded by a 1-thread kernel at points
 * the caller chooses (graph-capturable: the slot advances on the device);
 * psb_debug_stamps copies up to max of them and resets the count. */
PSB_API psb_status psb_debug_stamp(psb_ctx* ctx, psb_stream_t stream);
PSB_API int psb_debug_stamps(unsigned long long* out, int max);

#ifdef __cplusplus
}
#endif

#endif /* PSB_DEBUG_H_ */
