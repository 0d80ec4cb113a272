/*
 * dv_trace.h -- introspection hooks of libdvstream.so (SURVEY §5 "tracing"): latency tracing of
 * the fused publish and the release-scope decision. Part of the product library (they read or set
 * context state); no kernels of their own.
 */
#ifndef DV_TRACE_H_
#define DV_TRACE_H_
#include "dv.h"
#ifdef __cplusplus
extern "C" {
#endif

/* Latency tracing: while `ts` (device memory, 4 x uint64) is set, every fused copy of `ctx` that
 * publishes a flag records %globaltimer (ns): ts[0] = right after the release store of the flag,
 * ts[1] = min over CTAs of "resident" (before the programmatic-dependency wait; initialise to
 * UINT64_MAX), ts[2] = min over CTAs of "past the wait" (initialise to UINT64_MAX), ts[3] = max
 * over CTAs of "stores issued". NULL disables. */
DV_API dv_status dvt_trace(dv_ctx* ctx, uint64_t* ts);

/* Release scope the fused publish of `ctx` would use for a flag at `flag` after stores to
 * `payload`: *gpu_scope = 1 when both are this context's GPU's own device memory (not mapped from
 * another process), 0 otherwise (system scope). Host-only query; DESIGN.md §6 protocols 2/3. */
DV_API dv_status dvt_release_scope(dv_ctx* ctx, const void* flag, const void* payload,
                                   int32_t* gpu_scope);

/* Engine tracing: while `stamps` (device memory, 5 * n uint64) is set, the engine writes, for step
 * k of plan p, five %globaltimer stamps into stamps[5 * ((k * n_plans + p) % n) + 0..4]: the flag
 * release, the doorbell found by the poll, past the posting cluster barrier, the copy's stores
 * issued (rank 0), past the collecting cluster barrier (n_plans = plans registered). Set it while
 * the engine is parked or idle. */
DV_API dv_status dvt_engine_trace(dv_engine* e, uint64_t* stamps, uint64_t n);

/* Launches so far (all contexts of this process) of one kernel form: "tma_transpose" = the FT6D
 * key transpose whose packet-major side is moved by TMA tensor copies (DESIGN.md §6 "FT6D keys");
 * "all" = every library kernel (as dv_stats). DV_EINVAL for an unknown name. */
DV_API dv_status dvt_launch_count(const char* form, uint64_t* n);

/* Change one experiment knob of the copy kernels at run time (names as the environment variables
 * read at load: "DV_TRS" packet-transpose form -- 0 automatic, 1 shared-memory tiles, 2 / 3
 * registers with PK 1 / <= 2, 4 registers even over a link; "DV_PK", "DV_PP", "DV_RDBULK",
 * "DV_BULK", "DV_CLUSTER"; "DV_TMA" 1 / 0 = FT6D key transposes by TMA rows on / off, "DV_TMA_TS"
 * positions per TMA tile). Not thread-safe against concurrent data calls; DV_EINVAL for an unknown
 * name. For measurements that compare forms in one process. */
DV_API dv_status dvt_tune(const char* name, int64_t value);

#ifdef __cplusplus
}
#endif
#endif
