/* dv_device.cuh -- device-side helpers of dvstream (header only, CUDA): consumers acquiring a
 * sequence flag (below), PRODUCERS storing the K/V rows they compute straight to a stream-out
 * destination through a device plan and releasing its flag (dv_dplan_*, end of file; include/dv.h),
 * and producers ringing a persistent-engine doorbell.
 *
 * SURVEY §8(a) A5 / PAPER.md:123-135: a chunk is complete once its 64-bit monotone sequence flag
 * reaches the chunk's seq. Host code waits with dv_wait (a stream-ordered cuStreamWaitValue64);
 * a consumer KERNEL (e.g. a decode kernel reading streamed-in KV) can instead acquire the flag
 * itself with these helpers. The flag may live in this GPU's HBM, in a peer GPU's memory mapped
 * with dv_ipc_open, or in pinned host memory (device-mapped address); the loads are system-scope
 * acquires, so every payload byte released before the flag (dvstream's st.release) is visible to
 * the calling thread afterwards -- other threads of the CTA must synchronise with it (e.g.
 * __syncthreads()) before reading the payload.
 *
 * Note: create the dv_ctx (dv_create loads every library kernel) before launching a kernel that
 * spins on a dvstream flag; see include/dv.h dv_create.
 */
#ifndef DV_DEVICE_CUH
#define DV_DEVICE_CUH
#include <stdint.h>

#include "dv.h"

/* One system-scope acquire load of the flag. */
static __device__ __forceinline__ uint64_t dv_flag_load(const uint64_t* flag) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
  return v;
}

/* Spin until *flag >= seq (acquire). Returns 1, or 0 if timeout_ns (by %globaltimer) passed first;
 * timeout_ns = 0 waits forever. Backs off with nanosleep between polls of a remote/host flag. */
static __device__ __forceinline__ int dv_flag_wait(const uint64_t* flag, uint64_t seq,
                                                   uint64_t timeout_ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  for (;;) {
    if (dv_flag_load(flag) >= seq) return 1;
    if (timeout_ns) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) return 0;
    }
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

/* Ring a dv_engine doorbell (dv_engine_doorbell) from a producer kernel: ask for every step of the
 * plan up to `step`. Call it from ONE thread once every store of the producer that the plan reads
 * is ordered before it (e.g. after a __syncthreads() in the last CTA of a ticket chain, or in a
 * single-CTA producer): a gpu-scope release max, so the engine's acquire sees the data. */
static __device__ __forceinline__ void dv_engine_ring(uint64_t* doorbell, uint64_t step) {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("red.release.gpu.global.max.u64 [%0], %1;" ::"l"(doorbell), "l"(step + 1) : "memory");
}

/* ---- device plans (include/dv.h dv_dplan_*): the stream-out inside the producer kernel ------
 * Destination of the 16-byte packet u of the row (kv, l, r, h, s) -- global ids -- at step k, or
 * NULL when the row is outside the plan's region at that step. The producer stores each packet it
 * computes there in addition to its own cache store (16-byte aligned). */
static __device__ __forceinline__ uint8_t* dv_dplan_packet(const dv_dplan* p, int32_t k, int kv, int32_t l,
                                                           int32_t r, int32_t h, int32_t s, int32_t u) {
  const int32_t sk = s - k;   /* the position at step 0 */
  if (l < p->l0 || l >= p->l1 || r < p->r0 || r >= p->r1 || h < p->h0 || h >= p->h1 || sk < p->s0 ||
      sk >= p->s1)
    return (uint8_t*)0;
  const int32_t os = p->o_s + (p->pos_shift ? k : 0);
  return p->dst[kv] + (int64_t)k * p->step_bytes + (int64_t)(l - p->o_l) * p->st_l +
         (int64_t)(r - p->o_r) * p->st_r + (int64_t)(h - p->o_h) * p->st_h + (int64_t)(s - os) * p->st_s[kv] +
         (int64_t)u * p->st_u[kv];
}
/* Whether rows of kv are contiguous at the destination (every wire; KV5D caches; the V half of an
 * FT6D cache): then dv_dplan_row gives the row's start and the producer may store it with wider
 * vectors. */
static __device__ __forceinline__ int dv_dplan_row_contiguous(const dv_dplan* p, int kv) {
  return p->st_u[kv] == 16;
}
static __device__ __forceinline__ uint8_t* dv_dplan_row(const dv_dplan* p, int32_t k, int kv, int32_t l,
                                                        int32_t r, int32_t h, int32_t s) {
  return dv_dplan_packet(p, k, kv, l, r, h, s, 0);
}

/* Release of step k, called by EVERY thread of EVERY CTA of the producer grid once the CTA's row
 * stores are issued (n_ctas = the grid's CTA count): each CTA orders its stores at gpu scope and
 * takes a ticket; the last CTA releases flag = seq + k with ONE release at the plan's scope
 * (st.release.sys for host / peer memory: causality order is cumulative, so every CTA's rows are
 * visible to any observer of the flag). Contains a __syncthreads(). */
static __device__ __forceinline__ void dv_dplan_release_cta(const dv_dplan* p, int32_t k, uint32_t n_ctas) {
  /* the part after the CTA's barrier: one thread of the CTA */
  if (!p->flag) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const uint32_t prev = atomicAdd(p->ticket, 1u);
  if (prev == n_ctas - 1) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    *(volatile uint32_t*)p->ticket = 0u;
    const uint64_t v = p->seq + (uint64_t)k;
    if (p->sys_scope)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p->flag), "l"(v) : "memory");
    else
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p->flag), "l"(v) : "memory");
    if (p->trace) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      *p->trace = t;
    }
  }
}
static __device__ __forceinline__ void dv_dplan_release(const dv_dplan* p, int32_t k, uint32_t n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) dv_dplan_release_cta(p, k, n_ctas);
}

/* Plan sets (dv_dplan_stream_out_direct): the destination of a packet is the one plan whose piece
 * holds it (NULL if none); the release runs every plan's ticket chain after ONE barrier. */
static __device__ __forceinline__ uint8_t* dv_dplan_set_packet(const dv_dplan_set* s, int32_t k, int kv,
                                                               int32_t l, int32_t r, int32_t h, int32_t pos,
                                                               int32_t u) {
  for (int i = 0; i < s->n; ++i) {
    uint8_t* d = dv_dplan_packet(&s->plan[i], k, kv, l, r, h, pos, u);
    if (d) return d;
  }
  return (uint8_t*)0;
}
static __device__ __forceinline__ void dv_dplan_set_release(const dv_dplan_set* s, int32_t k, uint32_t n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0)
    for (int i = 0; i < s->n; ++i) dv_dplan_release_cta(&s->plan[i], k, n_ctas);
}

#endif
