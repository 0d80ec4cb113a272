/*
 * dv_baselines.h -- prior-art copy methods kept ONLY as measured baselines (SURVEY §2.6 B14,
 * BASELINE.md §4). They implement the paper's own mechanisms with CUDA runtime copies:
 *   dvb_per_run_copy   -- Fig. 11 "Baseline": "transferring all contiguous memory regions one by
 *                         one", one cudaMemcpyAsync per contiguous run.
 *   dvb_buffered_copy  -- Opt (1) "buffered copies" as runtime copies: 2-D DMA of
 *                         every (layer, kv, request) block into a device staging buffer, then one
 *                         contiguous copy to the destination.
 * Both produce the canonical wire chunk of dv.h at `dst`.
 */
#ifndef DV_BASELINES_H_
#define DV_BASELINES_H_
#include "dv.h"
#ifdef __cplusplus
extern "C" {
#endif
/* Returns the number of runtime copy calls issued in *n_calls (may be NULL). */
DV_API dv_status dvb_per_run_copy(const dv_cache* src, const dv_region* region, void* dst,
                                  void* stream, uint64_t* n_calls);
/* `staging` must be local device memory of at least the region's bytes. */
DV_API dv_status dvb_buffered_copy(const dv_cache* src, const dv_region* region, void* staging,
                                   void* dst, void* stream, uint64_t* n_calls);
#ifdef __cplusplus
}
#endif
#endif
