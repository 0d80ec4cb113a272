/* dv_device.cuh -- device-side consumer helpers for dvstream sequence flags (header only, CUDA).
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

#endif
