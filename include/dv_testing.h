/*
 * dv_testing.h -- test-only utilities of dvstream, exported by the SEPARATE
 * library libdvstream_testing.so (which links libdvstream.so); NOT part of the streaming path and
 * not in the product library: a synthetic KV "writer" that fills caches with the seeded generator
 * of kvgen/__init__.py (same counter-based splitmix64 coordinate hash, implemented independently
 * on the device), an on-device verifier, flag watchers / consumers and a spin kernel for latency
 * and overlap measurements. Errors are reported through libdvstream's dv_last_error().
 */
#ifndef DV_TESTING_H_
#define DV_TESTING_H_
#include "dv.h"
#ifdef __cplusplus
extern "C" {
#endif

enum { DVT_FILL_HASH = 0, DVT_FILL_UID = 1, DVT_FILL_CONST = 2 };

/* Write the generator's word at every (kv, l, r, h, s, d) of `region` of cache `c` (global layer
 * and request ids; NULL region = the whole cache). Positions outside [valid_begin, valid_end) get
 * the POISON word 0xFFFE. kind:
 *   DVT_FILL_HASH  word = bits 48..63 of splitmix64(key XOR seed*0xD1B54A32D192ED03), key =
 *                  kv<<62 | l<<52 | r<<40 | h<<30 | s<<10 | d  (elem_bytes must be 2);
 *   DVT_FILL_UID   word = ((((kv*L + l)*R + r)*H + h)*S + s)*D + d with box = {L,R,H,S,D};
 *   DVT_FILL_CONST word = (uint16_t)seed.
 * If t_end is non-NULL (device memory), the kernel atomically maxes %globaltimer (ns) into it after
 * its stores -- "the new K/V is written" time for latency measurements. The kernel triggers
 * programmatic dependent launch at its start, like a PDL-aware attention kernel would.
 * Stream-ordered; no synchronisation. */
DV_API dv_status dvt_fill(const dv_cache* c, int32_t kind, uint64_t seed, const int32_t* box,
                   int32_t valid_begin, int32_t valid_end, const dv_region* region,
                   uint64_t* t_end, void* stream);

/* dvt_fill (hash kind, whole positions of `region`) whose LAST CTA then rings a dv_engine doorbell
 * with `step` (dv_device.cuh dv_engine_ring) once every CTA's stores are ordered before it -- a
 * producer that starts the engine's copy itself. `ticket` is a device uint32 counter, zero before
 * the call (the last CTA resets it). */
DV_API dv_status dvt_fill_ring(const dv_cache* c, uint64_t seed, const dv_region* region, uint64_t* t_end,
                               uint64_t* doorbell, uint64_t step, uint32_t* ticket, void* stream);

/* A vectorised synthetic PRODUCER (dvt_fill's words of `kind` / `seed` / `box` -- HASH is ALU-heavy,
 * UID a few integer ops per word, i.e. a memory-bound producer -- for `region` of cache `c`, KV5D or
 * FT6D key, 16-byte stores,
 * one thread per 16-byte chunk in a grid-stride loop of at most 4 x SMs CTAs of 256 threads -- the
 * shape of a producer's grid, so few CTAs join the plans' release). With `n_plans` plans (include/dv.h
 * dv_dplan_*; <= DV_DPLAN_SET_MAX, disjoint regions, e.g. a dv_dplan_set) it also stores every
 * packet inside a plan's region at step `step` to that plan's destination and releases every
 * plan's flag from its last CTA -- the stream-out fused into the producer (include/dv_device.cuh
 * dv_dplan_set_packet / dv_dplan_set_release). t_start / t_end (optional,
 * device uint64, preset by the caller): min over CTAs of %globaltimer at kernel start / max after
 * the CTA's stores. Triggers programmatic dependent launch at its start. */
DV_API dv_status dvt_fill_rows(const dv_cache* c, int32_t kind, uint64_t seed, const int32_t* box,
                               const dv_region* region, const dv_dplan* plans, int32_t n_plans, int32_t step,
                               uint64_t* t_start, uint64_t* t_end, void* stream);

/* Verifier (the second, on-device parity check of SURVEY §8(c) C-5 at full sizes): adds to
 * *mismatches (device memory, uint64) the number of words of `region` that differ from the
 * generator word dvt_fill would write there (same kind / seed / box / valid range). wire == NULL:
 * the words are read from cache `c` (either layout). wire != NULL: they are read from the dense
 * canonical wire [l][kv][r][h][s][d] of `region` at `wire` (device or mapped pinned host memory;
 * `c` then only supplies head_dim, head range and the global-id frame). Stream-ordered. */
DV_API dv_status dvt_verify(const dv_cache* c, const void* wire, int32_t kind, uint64_t seed,
                     const int32_t* box, int32_t valid_begin, int32_t valid_end,
                     const dv_region* region, uint64_t* mismatches, void* stream);

/* Flag watcher: one GPU thread polls `flag` (device memory, or pinned host memory through its
 * device-mapped address) with system-scope acquire loads and writes %globaltimer to ts[i] (device
 * memory) the first time it reads >= seq0 + i, i = 0..n-1; gives up after timeout_ns. Launch it on
 * its own stream, concurrent with the producer. Latency measurement: "flag visible to an
 * independent observer". */
DV_API dv_status dvt_watch(const uint64_t* flag, uint64_t seq0, int32_t n, uint64_t* ts,
                           uint64_t timeout_ns, void* stream);

/* In-kernel consumer (include/dv_device.cuh): 4 CTAs; thread 0 of each waits with dv_flag_wait
 * until *flag >= seq, then the CTAs copy `bytes` (multiple of 16) from src to dst (device
 * memory). *ok (device int32, preset to 1 by the caller) becomes 0 if the wait timed out. */
DV_API dv_status dvt_consume(const uint64_t* flag, uint64_t seq, const void* src, void* dst,
                             uint64_t bytes, uint64_t timeout_ns, int32_t* ok, void* stream);

/* Busy-wait kernel: `ctas` CTAs of 128 threads spin for `ns` nanoseconds (globaltimer). */
DV_API dv_status dvt_spin(uint64_t ns, int32_t ctas, void* stream);

#ifdef __cplusplus
}
#endif
#endif
