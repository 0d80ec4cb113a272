// The data-movement kernel of dvstream for sm_100a: a batched strided "run copy".
//
// Every hot-path step that moves KV bytes is one instance of it:
//   pack   (paper: scatter + Opt (1) buffered copies): cache runs -> wire
//   unpack (paper: gather):                                 wire -> cache runs
//   remap  (pack+unpack fused):                                            cache -> cache
// with the destination (or source) in local HBM, in pinned host memory over PCIe ("zero-copy"),
// or in a peer GPU's HBM over NVLink (CUDA-IPC mapped). A run is n*D*e contiguous bytes
// (positions [s0,s1) of one (layer, kv, request, head)); runs are enumerated row-major over up to
// 4 dims, so consecutive threads move consecutive 16/32-byte vectors of the wire order and both
// the strided side (whole 32 B sectors, >= 256 B per run) and the contiguous side coalesce.
//
// Design notes (B200):
//   * one flat vector index per thread, decoded with multiply-shift division (no 64-bit div);
//   * U independent 16/32-byte loads in flight per thread before the stores (latency hiding:
//     HBM ~1 us, NVLink ~1-2 us, PCIe ~2 us round trip);
//   * loads use ld.global.nc.L1::no_allocate (streaming, read once), 32-byte vectors become
//     LDG.E.NA.ENL2.256 / STG.E.ENL2.256 on sm_100a;
//   * words are moved as raw bits in integer registers: fp16/bf16 NaN payloads are preserved;
//   * optional fused publish: after its stores each CTA fences at system scope and bumps a
//     ticket; the last CTA stores the 64-bit sequence flag with st.release.sys (peer / host
//     observers then see the payload before the flag).
#include <cuda.h>
#include <stdlib.h>

#include <mutex>

#include <algorithm>

#include "dv_internal.h"

namespace dv {

std::atomic<uint64_t> g_kernel_launches{0};
std::atomic<uint64_t> g_dma_calls{0};
std::atomic<uint64_t> g_tma_launches{0};

struct DevDiv {
  uint32_t d, mul, shr;
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = (d == 1) ? n : (__umulhi(n, mul) >> shr);
    r = n - q * d;
  }
};

struct KParams {
  const uint8_t* src;
  uint8_t* dst;
  int64_t ss[kDims];
  int64_t ds[kDims];
  DevDiv fv;          // vectors per run
  DevDiv fd[kDims];   // n[k] (fd[0] unused: the outermost index is what remains)
  uint32_t q_begin;  // first run of this launch
  uint32_t n_vec;    // vectors in this launch (< 2^31)
  int32_t pub;  // publish protocol (see publish())
  unsigned long long* flag;
  unsigned long long seq;
  unsigned int* ticket;
  unsigned long long* ts;  // optional: %globaltimer right after the flag store (latency tracing)
  const int32_t* dyn;      // optional device step counter (see CopyPlan::dyn)
  int64_t dyn_ss, dyn_ds;
  int32_t dyn_max;
};

template <int VEC>
struct alignas(VEC) Vec {
  uint32_t w[VEC / 4];
};

// DV_LD_PREFETCH=N (build-time experiment, N = 64/128/256): .L2::NB prefetch-size hint on the loads.
#ifndef DV_LD_PREFETCH
#define DV_LD_PREFETCH 0
#endif
#if DV_LD_PREFETCH == 256
#define DV_LDQ ".L2::256B"
#elif DV_LD_PREFETCH == 128
#define DV_LDQ ".L2::128B"
#elif DV_LD_PREFETCH == 64
#define DV_LDQ ".L2::64B"
#else
#define DV_LDQ ""
#endif
__device__ __forceinline__ void ld_vec(Vec<16>& v, const uint8_t* p) {
  asm volatile("ld.global.nc.L1::no_allocate" DV_LDQ ".v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3])
               : "l"(p));
}
// Store cache-operator variants (PTX st.{wb,cs,wt}); selected per launch for sysmem experiments.
template <int STM>
__device__ __forceinline__ void st_vec_m(uint8_t* p, const Vec<32>& v) {
  if (STM == 1)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
                 "r"(v.w[7])
                 : "memory");
  else if (STM == 2)
    asm volatile("st.global.wt.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
                 "r"(v.w[7])
                 : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
                 "r"(v.w[7])
                 : "memory");
}
template <int STM>
__device__ __forceinline__ void st_vec_m(uint8_t* p, const Vec<16>& v) {
  if (STM == 1)
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
  else if (STM == 2)
    asm volatile("st.global.wt.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
  else
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
}

__device__ __forceinline__ void st_vec(uint8_t* p, const Vec<16>& v) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
               "r"(v.w[2]), "r"(v.w[3])
               : "memory");
}
__device__ __forceinline__ void ld_vec(Vec<32>& v, const uint8_t* p) {
  asm volatile("ld.global.nc.L1::no_allocate" DV_LDQ ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]),
                 "=r"(v.w[5]), "=r"(v.w[6]), "=r"(v.w[7])
               : "l"(p));
}
__device__ __forceinline__ void st_vec(uint8_t* p, const Vec<32>& v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
               "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
               "r"(v.w[7])
               : "memory");
}

// Programmatic dependent launch, both roles. As a dependent: wait (griddepcontrol.wait) until the
// grid that wrote our input has completed and its memory is visible. As a primary: let the NEXT
// PDL kernel on the stream be scheduled right away (griddepcontrol.launch_dependents) -- it only
// becomes resident and then blocks in its own wait until this grid completes. Measured OFF by
// default: back-to-back C2 token-step packs take 4.65 us with the early trigger vs 4.03 us with the
// implicit trigger at grid exit (tools/probe_token_pack.py); build with -DDV_TRIGGER=1 to try it.
#ifndef DV_TRIGGER
#define DV_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_enter() {
#if DV_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <int VEC>
__device__ __forceinline__ void locate(const KParams& p, const uint8_t* src, uint8_t* dst,
                                       uint32_t g, const uint8_t*& s, uint8_t*& d) {
  uint32_t q, w;
  p.fv.divmod(g, q, w);
  q += p.q_begin;
  const int64_t wo = (int64_t)w * VEC;
  int64_t so = wo, dof = wo;
#pragma unroll
  for (int k = kDims - 1; k >= 1; --k) {
    uint32_t i;
    p.fd[k].divmod(q, q, i);
    so += (int64_t)i * p.ss[k];
    dof += (int64_t)i * p.ds[k];
  }
  s = src + so + (int64_t)q * p.ss[0];
  d = dst + dof + (int64_t)q * p.ds[0];
}

// Publish protocol: every CTA orders its stores before a GPU-scope release
// (bar.sync, then thread 0's fence.acq_rel.gpu + ticket atomic); the CTA that takes the last
// ticket has, by the acquire on that atomic, every CTA's stores ordered before it, and makes them
// visible to the system with the ONE system-scope release of the flag, st.release.sys (PTX memory
// model: causality order is transitive, fences are cumulative). Protocols (`pub`, DV_PUBLISH;
// measured per-layer latency in DESIGN.md §6):
//   0  system fence in every CTA before the ticket (the most conservative form);
//   1  gpu-scope ticket chain, then fence.sc.sys + st.release.sys in the last CTA;
//   2  gpu-scope ticket chain, then st.release.sys alone (its own fence is the cumulative one);
//   3  gpu-scope ticket chain, then st.release.gpu: only when payload and flag both live in this
//      GPU's HBM, whose every reader (SMs, copy engines, stream memory ops, peers over NVLink) is
//      served by this GPU's L2, where the gpu-scope release has already made the stores visible.
__device__ __forceinline__ void publish(const KParams& p, int pub, unsigned long long seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pub == 0) {
      __threadfence_system();
    } else {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    unsigned int prev = atomicAdd(p.ticket, 1u);
    if (prev == gridDim.x - 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire side of the ticket chain
      if (pub <= 1) __threadfence_system();            // fence.sc.sys: everything -> system scope
      *p.ticket = 0u;  // ready for the next stream-ordered user of this ticket
      if (pub == 3)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.flag), "l"(seq) : "memory");
      else
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.flag), "l"(seq) : "memory");
      if (p.ts) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.ts[0] = t;  // flag published
      }
    }
  }
}

// The grid-stride body of the run copy: CTA `bid` of `nb` moves chunks of THREADS*U vectors.
template <int VEC, int U, int THREADS, int STM = 0>
__device__ __forceinline__ void run_chunks(const KParams& p, const uint8_t* src, uint8_t* dst,
                                           uint32_t bid, uint32_t nb) {
  const uint32_t chunk = THREADS * U;
  for (uint32_t base = bid * chunk; base < p.n_vec; base += nb * chunk) {
    Vec<VEC> v[U];
    uint8_t* d[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) {
        const uint8_t* s;
        locate<VEC>(p, src, dst, g, s, d[i]);
        ld_vec(v[i], s);
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) st_vec_m<STM>(d[i], v[i]);
    }
  }
}

#ifndef DV_MIN_BLOCKS
#define DV_MIN_BLOCKS 1
#endif
template <int VEC, int U, int THREADS, int STM = 0>
__global__ void __launch_bounds__(THREADS, (THREADS == 256 ? DV_MIN_BLOCKS : 1)) k_run_copy(const KParams p) {
  // Programmatic dependent launch: this grid may become resident while the kernel that wrote the
  // K/V (e.g. attention) is still draining; wait here until that grid's memory is visible.
  if (p.ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(p.ts + 1, t);  // first CTA resident
  }
  pdl_enter();
  if (p.ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(p.ts + 2, t);  // first CTA past the dependency wait
  }
  int32_t k = 0;
  if (p.dyn) {
    k = *p.dyn;
    if (k < 0 || k > p.dyn_max) return;  // uniform across the grid: nothing moves, nothing published
  }
  run_chunks<VEC, U, THREADS, STM>(p, p.src + (int64_t)k * p.dyn_ss, p.dst + (int64_t)k * p.dyn_ds,
                                   blockIdx.x, gridDim.x);
  if (p.ts) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(p.ts + 3, t);  // last CTA done with its stores (issued)
    }
  }
  if (p.flag) publish(p, p.pub, p.seq + (unsigned long long)k);
}

// Small released copies as ONE thread-block cluster (kClusterCtas CTAs): the CTAs meet at a
// cluster barrier instead of a global ticket, so the publish needs no L2 atomic round trip.
// Every thread orders its own stores at gpu scope (fence.acq_rel.gpu: its stores are performed
// in L2), arrives at the cluster barrier with release and waits with acquire; cluster rank 0's
// thread 0 then holds every CTA's stores in its causality past and releases the flag at the
// scope the destination needs (st.release.gpu for this GPU's HBM, st.release.sys otherwise).
constexpr int kClusterCtas = 8;   // the portable cluster size (see cluster_ctas())
template <int VEC, int U>
__global__ void __launch_bounds__(1024) k_copy_cluster(const KParams p) {
  if (p.ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(p.ts + 1, t);
  }
  pdl_enter();
  if (p.ts && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(p.ts + 2, t);
  }
  int32_t k = 0;
  if (p.dyn) {
    k = *p.dyn;
    if (k < 0 || k > p.dyn_max) return;  // uniform across the cluster
  }
  const uint8_t* src = p.src + (int64_t)k * p.dyn_ss;
  uint8_t* dst = p.dst + (int64_t)k * p.dyn_ds;
  const uint32_t T = blockDim.x * gridDim.x;
  const uint32_t g0 = blockIdx.x * blockDim.x + threadIdx.x;
  Vec<VEC> v[U];
  uint8_t* d[U];
#pragma unroll
  for (int i = 0; i < U; ++i) {
    const uint32_t g = g0 + i * T;
    d[i] = nullptr;
    if (g < p.n_vec) {
      const uint8_t* sp;
      locate<VEC>(p, src, dst, g, sp, d[i]);
      ld_vec(v[i], sp);
    }
  }
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (d[i]) st_vec(d[i], v[i]);
  if (p.ts) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(p.ts + 3, t);
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (p.flag && rank == 0 && threadIdx.x == 0) {
    const unsigned long long seq = p.seq + (unsigned long long)k;
    if (p.pub == 3)
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.flag), "l"(seq) : "memory");
    else
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.flag), "l"(seq) : "memory");
    if (p.ts) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.ts[0] = t;
    }
  }
}

// Two plans in one launch (K and V with different structures, e.g. an FT6D key + a KV5D value
// at a token step): vector g < a.n_vec belongs to plan a, the rest to plan b. Release fields
// travel in `a`. One launch instead of two halves the fixed cost of small two-plan copies.
template <int VEC, int U, int THREADS>
__global__ void __launch_bounds__(THREADS) k_run_copy2(const KParams a, const KParams b) {
  pdl_enter();
  int32_t k = 0;
  if (a.dyn) {
    k = *a.dyn;
    if (k < 0 || k > a.dyn_max) return;
  }
  const uint8_t* sa = a.src + (int64_t)k * a.dyn_ss;
  uint8_t* da = a.dst + (int64_t)k * a.dyn_ds;
  const uint8_t* sb = b.src + (int64_t)k * b.dyn_ss;
  uint8_t* db = b.dst + (int64_t)k * b.dyn_ds;
  const uint32_t total = a.n_vec + b.n_vec;
  const uint32_t chunk = THREADS * U;
  for (uint32_t base = blockIdx.x * chunk; base < total; base += gridDim.x * chunk) {
    Vec<VEC> v[U];
    uint8_t* d[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < total) {
        const uint8_t* s;
        if (g < a.n_vec)
          locate<VEC>(a, sa, da, g, s, d[i]);
        else
          locate<VEC>(b, sb, db, g - a.n_vec, s, d[i]);
        ld_vec(v[i], s);
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < total) st_vec(d[i], v[i]);
    }
  }
  if (a.flag) publish(a, a.pub, a.seq + (unsigned long long)k);
}

// Dense-destination variant: the destination of vectors [q_begin*vpr, ...) is one contiguous
// range (packing into a wire chunk). Each CTA gathers THREADS*U vectors into shared memory and one
// thread moves the whole chunk with a bulk async copy (cp.async.bulk, the TMA engine: UBLKCP),
// double-buffered. Large, well-formed writes matter most over PCIe and NVLink.
template <int VEC, int U, int THREADS>
__global__ void __launch_bounds__(THREADS) k_pack_bulk(const KParams p, uint8_t* dst0) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_enter();
  constexpr uint32_t chunk = THREADS * U;
  int stage = 0;
  for (uint32_t base = blockIdx.x * chunk; base < p.n_vec; base += gridDim.x * chunk) {
    uint8_t* buf = smem + stage * (chunk * VEC);
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    Vec<VEC> v[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) {
        const uint8_t* s;
        uint8_t* d;
        locate<VEC>(p, p.src, p.dst, g, s, d);
        ld_vec(v[i], s);
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) *reinterpret_cast<Vec<VEC>*>(buf + (i * THREADS + threadIdx.x) * VEC) = v[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t n = min(chunk, p.n_vec - base) * VEC;
      uint8_t* d = dst0 + (uint64_t)base * VEC;
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sa),
                   "r"(n)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    stage ^= 1;
  }
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  if (p.flag) publish(p, p.pub, p.seq);
}

// Dense-SOURCE variant for reads over a link (unpacking a wire chunk that sits in pinned host
// memory, or in a peer GPU's memory): the wire is read with bulk asynchronous copies (the TMA
// engine, cp.async.bulk global -> shared, SASS UBLKCP.S.G) of `ch` contiguous bytes, completion on
// an mbarrier per stage, `st` stages in flight per CTA; all threads then scatter the staged bytes
// into the destination runs with 16/32-byte stores. The per-thread 32-byte zero-copy loads of
// k_run_copy reach pinned host memory as many small PCIe read requests (ncu: pcie__read_bytes =
// 2.18 x payload, profiles/r01g_ncu_hbm_kernels.md); a bulk copy lets the copy engine of the SM's
// TMA unit issue large ones.
constexpr int kRdStagesMax = 8;
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(b);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_load(uint8_t* smem_dst, const uint8_t* src, uint32_t bytes,
                                          unsigned long long* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(smem_dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

template <int VEC>
__global__ void __launch_bounds__(256) k_unpack_bulk(const KParams p, const uint8_t* src0, uint32_t ch,
                                                     uint32_t st) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) unsigned long long bar[kRdStagesMax];
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < st; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  const uint64_t total = (uint64_t)p.n_vec * VEC;
  const uint32_t nchunks = (uint32_t)((total + ch - 1) / ch);
  if (threadIdx.x == 0)
    for (uint32_t i = 0; i < st; ++i) {
      const uint32_t c = blockIdx.x + i * gridDim.x;
      if (c < nchunks)
        bulk_load(smem + i * ch, src0 + (uint64_t)c * ch, (uint32_t)(uint32_t)(total - (uint64_t)c * ch < ch ? total - (uint64_t)c * ch : ch),
                  &bar[i]);
    }
  uint32_t it = 0;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const uint32_t s = it % st;
    mbar_wait(&bar[s], (it / st) & 1);
    const uint32_t nbytes = (uint32_t)(uint32_t)(total - (uint64_t)c * ch < ch ? total - (uint64_t)c * ch : ch);
    const uint32_t g0 = (uint32_t)((uint64_t)c * ch / VEC);
    const uint8_t* buf = smem + s * ch;
    for (uint32_t v = threadIdx.x; v < nbytes / VEC; v += blockDim.x) {
      const Vec<VEC> x = *reinterpret_cast<const Vec<VEC>*>(buf + v * VEC);
      const uint8_t* sp;
      uint8_t* d;
      locate<VEC>(p, p.src, p.dst, g0 + v, sp, d);
      st_vec(d, x);
    }
    __syncthreads();  // every thread is done reading stage s
    if (threadIdx.x == 0) {
      const uint32_t c2 = c + st * gridDim.x;
      if (c2 < nchunks)
        bulk_load(smem + s * ch, src0 + (uint64_t)c2 * ch,
                  (uint32_t)(total - (uint64_t)c2 * ch < ch ? total - (uint64_t)c2 * ch : ch), &bar[s]);
    }
  }
  if (p.flag) publish(p, p.pub, p.seq);
}

// 16-byte packet transpose through shared memory (NEXT-1, FasterTransformer's 6-D key layout):
// inside each slab the packet-major side holds [u][s] (a column of positions per packet, each
// column contiguous), the position-major side [s][u] (the wire, KV5D). A CTA moves a tile of all
// U packets x kTS positions: loads coalesced along the source's contiguous axis, stores coalesced
// along the destination's, the transposition happens in shared memory (rows padded by one
// packet so neither phase has bank conflicts).
constexpr int kTS = 64;

struct TParams {
  const uint8_t* src;
  uint8_t* dst;
  int64_t ss[4], ds[4];
  DevDiv fd[4];
  uint32_t n_tiles, tiles_per_slab;
  DevDiv fU, fT;
  uint32_t U, N;
  int64_t su, sps;  // packet stride of the packet-major side, position stride of the position-major side
  unsigned long long* flag;
  unsigned long long seq;
  unsigned int* ticket;
  unsigned long long* ts;
  int32_t pub;
  const int32_t* dyn;
  int64_t dyn_ss, dyn_ds;
  int32_t dyn_max;
  // register form (transpose_regs): items = slabs x (U / PK) packet groups x N positions
  uint32_t n_items;
  DevDiv fN, fG;
  int32_t pk;    // packets per thread item (1, 2, 4, 8, 16); 0 = shared-memory tiles
  // TMA-row form (transpose_tma): the packet-major side through a 5-D tensor map (16-byte words
  // of a packet row, packet, up to 3 slab dims); slab dim d contributes i_d * tm_mul[d] to map
  // coordinate tm_dim[d] (2..4; -1 = unit dim)
  int32_t tm_nst;          // stages in flight per CTA (0 = not this form)
  int32_t tm_dim[4];
  uint32_t tm_mul[4];
  uint32_t tm_tps;         // tiles per slab
  DevDiv fTm;              // division by tm_tps
};

// Register form of the packet transpose: no shared memory, no barrier. A thread item is PK
// adjacent packets of ONE position: on the packet-major side the PK 16-byte loads (or stores) of a
// warp's 32 consecutive positions are PK fully coalesced 512-byte segments; on the position-major
// side each item is one contiguous PK*16-byte piece moved as 32-byte vectors (PK = 16: a whole
// 256-byte row, i.e. two full 128-byte lines per thread). IT items per thread are in flight before
// the first store (PK*IT*16 = 128 bytes for PK <= 4 and 8, 256 for PK = 16).
template <int PK>
struct TrIt {
  static constexpr int value = PK >= 8 ? 1 : PK == 4 ? 2 : 4;
};
template <int DIR, int PK>
__device__ __forceinline__ void transpose_regs(const TParams& p, const uint8_t* src0, uint8_t* dst0,
                                               uint32_t bid, uint32_t nb) {
  constexpr int IT = TrIt<PK>::value;
  for (uint32_t b0 = bid * IT * 256; b0 < p.n_items; b0 += nb * IT * 256) {
    Vec<16 * PK> v[IT];
    uint8_t* d[IT];
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const uint32_t i = b0 + j * 256 + threadIdx.x;
      d[j] = nullptr;
      if (i < p.n_items) {
        uint32_t rest, s, slab, g;
        p.fN.divmod(i, rest, s);
        p.fG.divmod(rest, slab, g);
        int64_t so = 0, dof = 0;
        uint32_t q = slab;
#pragma unroll
        for (int k = 3; k >= 1; --k) {
          uint32_t x;
          p.fd[k].divmod(q, q, x);
          so += (int64_t)x * p.ss[k];
          dof += (int64_t)x * p.ds[k];
        }
        so += (int64_t)q * p.ss[0];
        dof += (int64_t)q * p.ds[0];
        const uint32_t u0 = g * PK;
        if (DIR == 0) {  // packet-major source, position-major destination
          const uint8_t* a = src0 + so + (int64_t)u0 * p.su + (int64_t)s * 16;
#pragma unroll
          for (int k = 0; k < PK; ++k) {
            Vec<16> w;
            ld_vec(w, a + (int64_t)k * p.su);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[j].w[4 * k + c] = w.w[c];
          }
          d[j] = dst0 + dof + (int64_t)s * p.sps + (int64_t)u0 * 16;
        } else {         // position-major source, packet-major destination
          const uint8_t* a = src0 + so + (int64_t)s * p.sps + (int64_t)u0 * 16;
          if constexpr (PK == 1) {
            ld_vec(v[j], a);
          } else {
#pragma unroll
            for (int k = 0; k < PK / 2; ++k) {
              Vec<32> x;
              ld_vec(x, a + 32 * k);
#pragma unroll
              for (int c = 0; c < 8; ++c) v[j].w[8 * k + c] = x.w[c];
            }
          }
          d[j] = dst0 + dof + (int64_t)u0 * p.su + (int64_t)s * 16;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      if (!d[j]) continue;
      if (DIR == 0) {
        if constexpr (PK == 1) {
          st_vec(d[j], v[j]);
        } else {
#pragma unroll
          for (int k = 0; k < PK / 2; ++k) {
            Vec<32> x;
#pragma unroll
            for (int c = 0; c < 8; ++c) x.w[c] = v[j].w[8 * k + c];
            st_vec(d[j] + 32 * k, x);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < PK; ++k) {
          Vec<16> w;
#pragma unroll
          for (int c = 0; c < 4; ++c) w.w[c] = v[j].w[4 * k + c];
          st_vec(d[j] + (int64_t)k * p.su, w);
        }
      }
    }
  }
}

template <int DIR>
__device__ __forceinline__ void transpose_tiles(const TParams& p, uint4* tile, const uint8_t* src0,
                                                uint8_t* dst0, uint32_t bid, uint32_t nb) {
  const uint32_t row = p.U + 1;
  const uint32_t elems = p.U * kTS;
  for (uint32_t t = bid; t < p.n_tiles; t += nb) {
    uint32_t slab, ti;
    p.fT.divmod(t, slab, ti);
    const uint32_t s0 = ti * kTS;
    const uint32_t ns = min((uint32_t)kTS, p.N - s0);
    int64_t so = 0, dof = 0;
    uint32_t q = slab;
#pragma unroll
    for (int d = 3; d >= 1; --d) {
      uint32_t i;
      p.fd[d].divmod(q, q, i);
      so += (int64_t)i * p.ss[d];
      dof += (int64_t)i * p.ds[d];
    }
    so += (int64_t)q * p.ss[0];
    dof += (int64_t)q * p.ds[0];
    const uint8_t* sb = src0 + so;
    uint8_t* db = dst0 + dof;
    // 4 independent 16-byte loads in flight per thread before their shared-memory stores
    for (uint32_t i0 = threadIdx.x; i0 < elems; i0 += 4 * 256) {
      uint4 v[4];
      uint32_t slot[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t i = i0 + j * 256;
        uint32_t u = 0, s = kTS;
        if (i < elems) {
          if (DIR == 0) {  // packet-major source: consecutive threads walk positions of one packet
            u = i / kTS;
            s = i % kTS;
          } else {         // position-major source: consecutive threads walk packets of one position
            p.fU.divmod(i, s, u);
          }
        }
        slot[j] = s < ns ? s * row + u : 0xFFFFFFFFu;
        if (s < ns) {
          const uint8_t* a = DIR == 0 ? sb + (int64_t)u * p.su + (int64_t)(s0 + s) * 16
                                      : sb + (int64_t)(s0 + s) * p.sps + (int64_t)u * 16;
          asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                       : "l"(a));
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (slot[j] != 0xFFFFFFFFu) tile[slot[j]] = v[j];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < elems; i += 256) {
      uint32_t u, s;
      if (DIR == 0) {  // position-major destination: consecutive threads write packets of a position
        p.fU.divmod(i, s, u);
      } else {
        u = i / kTS;
        s = i % kTS;
      }
      if (s < ns) {
        const uint4 v = tile[s * row + u];
        uint8_t* a = DIR == 0 ? db + (int64_t)(s0 + s) * p.sps + (int64_t)u * 16
                              : db + (int64_t)u * p.su + (int64_t)(s0 + s) * 16;
        asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w)
                     : "memory");
      }
    }
    __syncthreads();
  }
}

// Two-position register form (PK packets x 2 adjacent positions per item, DV_PP=2): the
// packet-major side moves 32-byte vectors (positions s, s+1 of one packet are adjacent there), the
// position-major side two PK*16-byte row pieces. Items = slabs x (U / PK) x (N / 2); N even.
template <int DIR, int PK>
__device__ __forceinline__ void transpose_regs2(const TParams& p, const uint8_t* src0, uint8_t* dst0,
                                                uint32_t bid, uint32_t nb) {
  for (uint32_t i = bid * 256 + threadIdx.x; i < p.n_items; i += nb * 256) {
    uint32_t rest, s2, slab, g;
    p.fN.divmod(i, rest, s2);   // fN = N / 2
    p.fG.divmod(rest, slab, g);
    int64_t so = 0, dof = 0;
    uint32_t q = slab;
#pragma unroll
    for (int k = 3; k >= 1; --k) {
      uint32_t x;
      p.fd[k].divmod(q, q, x);
      so += (int64_t)x * p.ss[k];
      dof += (int64_t)x * p.ds[k];
    }
    so += (int64_t)q * p.ss[0];
    dof += (int64_t)q * p.ds[0];
    const uint32_t u0 = g * PK, s = 2 * s2;
    Vec<32> v[PK];   // v[k]: packet u0 + k at positions s (words 0..3) and s + 1 (words 4..7)
    if (DIR == 0) {  // packet-major source
      const uint8_t* a = src0 + so + (int64_t)u0 * p.su + (int64_t)s * 16;
#pragma unroll
      for (int k = 0; k < PK; ++k) ld_vec(v[k], a + (int64_t)k * p.su);
      uint8_t* d = dst0 + dof + (int64_t)s * p.sps + (int64_t)u0 * 16;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < PK; k += 2) {
          Vec<32> x;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            x.w[c] = v[k].w[4 * r + c];
            x.w[4 + c] = v[k + 1].w[4 * r + c];
          }
          st_vec(d + (int64_t)r * p.sps + 16 * k, x);
        }
    } else {         // position-major source
      const uint8_t* a = src0 + so + (int64_t)s * p.sps + (int64_t)u0 * 16;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < PK; k += 2) {
          Vec<32> x;
          ld_vec(x, a + (int64_t)r * p.sps + 16 * k);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            v[k].w[4 * r + c] = x.w[c];
            v[k + 1].w[4 * r + c] = x.w[4 + c];
          }
        }
      uint8_t* d = dst0 + dof + (int64_t)u0 * p.su + (int64_t)s * 16;
#pragma unroll
      for (int k = 0; k < PK; ++k) st_vec(d + (int64_t)k * p.su, v[k]);
    }
  }
}

// PK is a template parameter of the kernels (not a runtime branch): the register budget of each
// instantiation is that of its own form (59-64 registers at PK <= 4, 1024 threads per SM).
// PK > 32 selects the two-position form with PK - 32 packets per item.
template <int DIR, int PK>
__device__ __forceinline__ void transpose_any(const TParams& p, uint4* tile, const uint8_t* src0,
                                              uint8_t* dst0, uint32_t bid, uint32_t nb) {
  if constexpr (PK == 0)
    transpose_tiles<DIR>(p, tile, src0, dst0, bid, nb);
  else if constexpr (PK > 32)
    transpose_regs2<DIR, PK - 32>(p, src0, dst0, bid, nb);
  else
    transpose_regs<DIR, PK>(p, src0, dst0, bid, nb);
}

template <int DIR, int PK>
__global__ void __launch_bounds__(256) k_packet_transpose(const TParams p) {
  extern __shared__ uint4 tile[];  // kTS rows x (U + 1) packets
  pdl_enter();
  int32_t k = 0;
  if (p.dyn) {
    k = *p.dyn;
    if (k < 0 || k > p.dyn_max) return;
  }
  const uint8_t* src0 = p.src + (int64_t)k * p.dyn_ss;
  uint8_t* dst0 = p.dst + (int64_t)k * p.dyn_ds;
  transpose_any<DIR, PK>(p, tile, src0, dst0, blockIdx.x, gridDim.x);
  if (p.flag) {
    KParams kp{};
    kp.flag = p.flag;
    kp.ticket = p.ticket;
    kp.ts = p.ts;
    publish(kp, p.pub, p.seq + (unsigned long long)k);
  }
}

// An FT6D key transpose and the value's run copy in ONE launch: CTAs [0, t_blocks) transpose, the
// rest run-copy; both halves share the dependency wait, the step counter and the release.
template <int DIR, int VEC, int PK>
__global__ void __launch_bounds__(256) k_transpose_run(const TParams t, const KParams r,
                                                       uint32_t t_blocks) {
  extern __shared__ uint4 tile[];
  pdl_enter();
  int32_t k = 0;
  if (t.dyn) {
    k = *t.dyn;
    if (k < 0 || k > t.dyn_max) return;
  }
  if (t_blocks == 0) {  // every CTA takes its share of both halves
    transpose_any<DIR, PK>(t, tile, t.src + (int64_t)k * t.dyn_ss, t.dst + (int64_t)k * t.dyn_ds,
                       blockIdx.x, gridDim.x);
    run_chunks<VEC, 4, 256>(r, r.src + (int64_t)k * r.dyn_ss, r.dst + (int64_t)k * r.dyn_ds,
                            blockIdx.x, gridDim.x);
  } else if (blockIdx.x < t_blocks)
    transpose_any<DIR, PK>(t, tile, t.src + (int64_t)k * t.dyn_ss, t.dst + (int64_t)k * t.dyn_ds,
                       blockIdx.x, t_blocks);
  else
    run_chunks<VEC, 4, 256>(r, r.src + (int64_t)k * r.dyn_ss, r.dst + (int64_t)k * r.dyn_ds,
                            blockIdx.x - t_blocks, gridDim.x - t_blocks);
  if (t.flag) {
    KParams kp{};
    kp.flag = t.flag;
    kp.ticket = t.ticket;
    kp.ts = t.ts;
    publish(kp, t.pub, t.seq + (unsigned long long)k);
  }
}

// TMA-row form of the packet transpose (NEXT-1; DESIGN.md §6 "FT6D keys"). The packet-major
// side (the FT6D key cache, in this GPU's HBM) is moved by the TMA engine, one 2-D box per packet
// row of TS positions (TS*16 contiguous bytes), through a tensor map whose position extent ends at
// the region's end (stores past it are clipped by the hardware: bytes outside the region are never
// written); shared memory holds a tile as [u][s][16 B]. The position-major side is moved by the
// CTA's threads as 32-byte vectors (two packets of one position; a warp's lanes walk 32 positions
// of one packet pair: conflict-free 16-byte shared-memory accesses, whole 32-byte sectors in HBM).
//   DIR 0 (pack / FT6D -> KV5D): thread 0 keeps tm_nst tile loads in flight (mbarrier
//     complete_tx per stage); all threads store the staged tile.
//   DIR 1 (unpack / KV5D -> FT6D): all threads load a tile into shared memory, a proxy fence and a
//     barrier hand it to thread 0, which stores the U packet rows by TMA (bulk async-group); a
//     stage is refilled only after its stores have read it (cp.async.bulk.wait_group.read).
// Measured against the register form (PK = 16) on the C2 prompt layer: DESIGN.md §6.
__device__ __forceinline__ void tma_row_load(const CUtensorMap* m, uint8_t* sdst, unsigned long long* bar,
                                             const int32_t c[5]) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(sdst)),
      "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
      "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_row_store(const CUtensorMap* m, const uint8_t* ssrc, const int32_t c[5]) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(m),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read(int n) {   // at most n bulk groups still reading shared memory
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
  }
}
constexpr int kTmaStagesMax = 4;

// tile t -> map coordinates of its first packet row (c[1] = packet 0) and the position-major
// side's byte offset of its first position
__device__ __forceinline__ void tma_tile(const TParams& p, uint32_t t, int TS, int32_t c[5], int64_t& pos_off,
                                         uint32_t& ns, int DIR) {
  uint32_t slab, ti;
  p.fTm.divmod(t, slab, ti);
  const uint32_t s0 = ti * TS;
  ns = min((uint32_t)TS, p.N - s0);
  c[0] = (int32_t)(s0 * 4);
  c[1] = 0;
  c[2] = c[3] = c[4] = 0;
  int64_t off = 0;
  uint32_t q = slab;
#pragma unroll
  for (int d = 3; d >= 0; --d) {
    uint32_t i;
    if (d > 0)
      p.fd[d].divmod(q, q, i);
    else
      i = q;
    off += (int64_t)i * (DIR == 0 ? p.ds[d] : p.ss[d]);
    const int32_t v = (int32_t)(i * p.tm_mul[d]);   // (register-resident: no dynamic index into c)
    c[2] += p.tm_dim[d] == 2 ? v : 0;
    c[3] += p.tm_dim[d] == 3 ? v : 0;
    c[4] += p.tm_dim[d] == 4 ? v : 0;
  }
  pos_off = off + (int64_t)s0 * p.sps;
}

template <int DIR, int TS>
__device__ __forceinline__ void transpose_tma(const TParams& p, const CUtensorMap* map, uint8_t* sm,
                                              unsigned long long* bar, uint32_t bid, uint32_t nb) {
  const int nst = p.tm_nst;
  const uint32_t U = p.U;
  const uint32_t stage = U * TS * 16;
  const uint32_t mine = bid < p.n_tiles ? (p.n_tiles - bid + nb - 1) / nb : 0;
  const uint32_t items = TS * (U / 2);   // (position, packet pair) items of a tile
  if (DIR == 0) {
    auto issue = [&](uint32_t j) {
      int32_t c[5];
      int64_t po;
      uint32_t ns;
      tma_tile(p, bid + j * nb, TS, c, po, ns, 0);
      uint8_t* buf = sm + (j % nst) * stage;
      unsigned long long* b = &bar[j % nst];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(b)),
                   "r"(stage)
                   : "memory");
      for (uint32_t u = 0; u < U; ++u) {
        c[1] = (int32_t)u;
        tma_row_load(map, buf + u * TS * 16, b, c);
      }
    };
    if (threadIdx.x == 0)
      for (uint32_t j = 0; j < (uint32_t)nst && j < mine; ++j) issue(j);
    for (uint32_t j = 0; j < mine; ++j) {
      int32_t c[5];
      int64_t po;
      uint32_t ns;
      tma_tile(p, bid + j * nb, TS, c, po, ns, 0);
      mbar_wait(&bar[j % nst], (j / nst) & 1);
      const uint8_t* buf = sm + (j % nst) * stage;
      uint8_t* out = p.dst + po;
      for (uint32_t i = threadIdx.x; i < items; i += 256) {
        const uint32_t s = i % TS, pr = i / TS;
        if (s < ns) {
          Vec<32> x;
          *reinterpret_cast<uint4*>(&x.w[0]) = *reinterpret_cast<const uint4*>(buf + (2 * pr) * TS * 16 + s * 16);
          *reinterpret_cast<uint4*>(&x.w[4]) = *reinterpret_cast<const uint4*>(buf + (2 * pr + 1) * TS * 16 + s * 16);
          st_vec(out + (int64_t)s * p.sps + pr * 32, x);
        }
      }
      __syncthreads();   // every thread is done reading this stage
      if (threadIdx.x == 0 && j + nst < mine) issue(j + nst);
    }
  } else {
    for (uint32_t j = 0; j < mine; ++j) {
      int32_t c[5];
      int64_t po;
      uint32_t ns;
      tma_tile(p, bid + j * nb, TS, c, po, ns, 1);
      uint8_t* buf = sm + (j % nst) * stage;
      if (j >= (uint32_t)nst) {   // the stores issued from this stage nst tiles ago have read it
        if (threadIdx.x == 0) bulk_wait_read(nst - 1);
        __syncthreads();
      }
      const uint8_t* in = p.src + po;
      for (uint32_t i0 = threadIdx.x; i0 < items; i0 += 512) {   // two items in flight per thread
        Vec<32> x[2];
        bool ok[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint32_t i = i0 + k * 256, s = i % TS, pr = i / TS;
          ok[k] = i < items && s < ns;
          if (ok[k]) ld_vec(x[k], in + (int64_t)s * p.sps + pr * 32);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint32_t i = i0 + k * 256, s = i % TS, pr = i / TS;
          if (ok[k]) {
            *reinterpret_cast<uint4*>(buf + (2 * pr) * TS * 16 + s * 16) = *reinterpret_cast<const uint4*>(&x[k].w[0]);
            *reinterpret_cast<uint4*>(buf + (2 * pr + 1) * TS * 16 + s * 16) =
                *reinterpret_cast<const uint4*>(&x[k].w[4]);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy
      __syncthreads();
      if (threadIdx.x == 0) {
        for (uint32_t u = 0; u < U; ++u) {
          c[1] = (int32_t)u;
          tma_row_store(map, buf + u * TS * 16, c);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // stores complete (before any release)
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
}

// The TMA-row transpose and the value's run copy in ONE launch (CTAs [0, t_blocks) transpose; with
// t_blocks == gridDim.x it is the transpose alone). The tensor map is a __grid_constant__ parameter.
template <int DIR, int VEC, int TS>
__global__ void __launch_bounds__(256) k_transpose_tma_run(const TParams t, const KParams r, uint32_t t_blocks,
                                                           const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ __align__(8) unsigned long long bar[kTmaStagesMax];
  if (blockIdx.x < t_blocks && threadIdx.x == 0) {
    for (int i = 0; i < t.tm_nst; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  if (blockIdx.x < t_blocks)
    transpose_tma<DIR, TS>(t, &map, tsm, bar, blockIdx.x, t_blocks);
  else
    run_chunks<VEC, 4, 256>(r, r.src, r.dst, blockIdx.x - t_blocks, gridDim.x - t_blocks);
  if (t.flag) {
    KParams kp{};
    kp.flag = t.flag;
    kp.ticket = t.ticket;
    kp.ts = t.ts;
    publish(kp, t.pub, t.seq);
  }
}

// Credit wait on peer memory (api.cu credit_wait): thread 0 polls with system-scope acquire loads
// and backs off; the copy kernel behind it passes its griddepcontrol.wait only once this grid
// has completed.
__global__ void k_wait_geq(const unsigned long long* p, unsigned long long v) {
  if (threadIdx.x != 0) return;
  unsigned ns = 32;
  for (;;) {
    unsigned long long x;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    if (x >= v) break;
    __nanosleep(ns);
    if (ns < 1024) ns *= 2;
  }
}

// Stream-ordered release of a word in peer memory (api.cu stream_signal): every earlier grid of the
// stream has completed; one thread fences at system scope and releases the value.
__global__ void k_store_release(unsigned long long* p, unsigned long long v) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

dv_status launch_store_release(uint64_t* p, uint64_t v, cudaStream_t stream) {
  (void)cudaGetLastError();
  k_store_release<<<1, 32, 0, stream>>>((unsigned long long*)p, (unsigned long long)v);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "release kernel launch");
  return DV_OK;
}

dv_status launch_wait_geq(const uint64_t* p, uint64_t v, cudaStream_t stream) {
  (void)cudaGetLastError();
  k_wait_geq<<<1, 32, 0, stream>>>((const unsigned long long*)p, (unsigned long long)v);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "credit wait kernel launch");
  return DV_OK;
}

static DevDiv to_dev(const FastDiv& f) { return DevDiv{f.d, f.mul, f.shr}; }

// Per-device "attribute already set" bits (function attributes are per device context).
static bool first_use_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  return !(mask.fetch_or(bit) & bit);
}
template <int VEC>
static std::atomic<uint64_t>& bulk_mask() {
  static std::atomic<uint64_t> m{0};
  return m;
}

static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int VEC, int U, int THREADS, int STM = 0>
static cudaError_t go(const KParams& kp, int blocks, cudaStream_t st) {
  (void)cudaGetLastError();  // clear stale non-sticky errors of unrelated earlier calls
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_run_copy<VEC, U, THREADS, STM>, kp);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Launch-shape tunables (environment, read once; for experiments -- DESIGN.md "Kernel tuning").
struct Tune {
  int u = 0;          // DV_U: vectors in flight per thread (1,2,4,8); 0 = automatic
  int vec = 0;        // DV_VEC: force 16-byte vectors when 16
  int bulk = 0;       // DV_BULK: 1 = dense-destination copies use k_pack_bulk
  int pub = 2;  // DV_PUBLISH: publish protocol (see publish()); 3 only where the scope allows
  uint64_t max_vec_per_launch = (1ull << 31) - 1;  // DV_MAX_VEC (tests of the launch split)
  int stm = 0;  // DV_STM: store cache operator for U=4 copies (0 default .wb, 1 .cs, 2 .wt)
  uint64_t small = 148ull * 128 * 4;  // DV_SMALL: copies up to this many vectors use U=1, 128 thr
  int trs = 0;  // DV_TRS: packet transpose form (0 registers PK<=pk; 1 shared-memory tiles; 2 PK=1; 3 PK<=2)
  int pk = 16;  // DV_PK: largest packets per register-transpose item (1, 2, 4, 8, 16)
  int pp = 1;       // DV_PP: positions per register-transpose item (1, or 2 = the two-position form)
  int cluster = 1;  // DV_CLUSTER: small released copies as one cluster (0 off; 1 gpu-scope releases of
                    // <= 8192 vectors; 2 whenever it fits -- see launch_copy)
  int rdbulk = 0;     // DV_RDBULK: dense-source copies reading over a link use k_unpack_bulk (2: any source)
  uint32_t rdch = 8192;  // DV_RDCH: bytes per bulk read
  uint32_t rdst = 4;     // DV_RDST: bulk reads in flight per CTA (<= kRdStagesMax)
  int tma = 0;           // DV_TMA: FT6D key transposes with the packet-major side moved by TMA rows
  int tma_ts = 0;        // DV_TMA_TS: positions per TMA tile (32 / 64; 0 = per direction)
  double tma_split = 1.0;  // DV_TMA_TSPLIT: transpose CTAs' share weight (x their byte share)
};
static Tune& tune_mut() {
  static Tune t = [] {
    Tune x;
    if (const char* e = getenv("DV_U")) x.u = atoi(e);
    if (const char* e = getenv("DV_VEC")) x.vec = atoi(e);
    if (const char* e = getenv("DV_BULK")) x.bulk = atoi(e);
    if (const char* e = getenv("DV_PUBLISH")) x.pub = atoi(e);
    if (const char* e = getenv("DV_STM")) x.stm = atoi(e);
    if (const char* e = getenv("DV_MAX_VEC")) {
      const uint64_t v = strtoull(e, nullptr, 10);
      if (v > 0 && v < x.max_vec_per_launch) x.max_vec_per_launch = v;
    }
    if (const char* e = getenv("DV_SMALL")) x.small = strtoull(e, nullptr, 10);
    if (const char* e = getenv("DV_TRS")) x.trs = atoi(e);
    if (const char* e = getenv("DV_PK")) x.pk = atoi(e);
    if (const char* e = getenv("DV_CLUSTER")) x.cluster = atoi(e);
    if (const char* e = getenv("DV_PP")) x.pp = atoi(e);
    if (const char* e = getenv("DV_RDBULK")) x.rdbulk = atoi(e);
    if (const char* e = getenv("DV_RDCH")) x.rdch = (uint32_t)std::max(16, atoi(e) / 16 * 16);
    if (const char* e = getenv("DV_RDST")) x.rdst = (uint32_t)std::min(kRdStagesMax, std::max(1, atoi(e)));
    if (const char* e = getenv("DV_TMA")) x.tma = atoi(e);
    if (const char* e = getenv("DV_TMA_TS")) x.tma_ts = atoi(e);
    if (const char* e = getenv("DV_TMA_TSPLIT")) x.tma_split = atof(e);
    return x;
  }();
  return t;
}
static const Tune& tune() { return tune_mut(); }

// dvt_tune (dv_trace.h): change one experiment knob at run time (same names as the environment).
dv_status set_tune(const char* name, int64_t value) {
  Tune& t = tune_mut();
  const std::string n = name ? name : "";
  if (n == "DV_TRS") t.trs = (int)value;
  else if (n == "DV_PK") t.pk = (int)value;
  else if (n == "DV_PP") t.pp = (int)value;
  else if (n == "DV_RDBULK") t.rdbulk = (int)value;
  else if (n == "DV_BULK") t.bulk = (int)value;
  else if (n == "DV_CLUSTER") t.cluster = (int)value;
  else if (n == "DV_TMA") t.tma = (int)value;
  else if (n == "DV_TMA_TS") t.tma_ts = (int)value;
  else return fail(DV_EINVAL, "unknown tunable '%s'", n.c_str());
  return DV_OK;
}

// Publish protocol of a release: the environment's (default 2, system scope), narrowed to gpu
// scope (3) when payload and flag are all in this GPU's HBM; DV_PUBLISH=0/1 keep their forms.
static int pub_of(const Release& rel) {
  const int t = tune().pub;
  if (t < 2) return t;
  return rel.gpu_scope ? 3 : 2;
}

template <int VEC>
static cudaError_t launch_vec(const KParams& kp, int u, int max_ctas, cudaStream_t st) {
  const int threads = u == 1 ? 128 : 256;
  const uint64_t need = (kp.n_vec + (uint64_t)threads * u - 1) / ((uint64_t)threads * u);
  const int blocks = (int)std::min<uint64_t>(need, (uint64_t)(u == 1 ? (1u << 30) : max_ctas));
  switch (u) {
    case 1: return go<VEC, 1, 128>(kp, blocks, st);
    case 2: return go<VEC, 2, 256>(kp, blocks, st);
    case 8: return go<VEC, 8, 256>(kp, blocks, st);
    default:
      if (tune().stm == 1) return go<VEC, 4, 256, 1>(kp, blocks, st);
      if (tune().stm == 2) return go<VEC, 4, 256, 2>(kp, blocks, st);
      return go<VEC, 4, 256>(kp, blocks, st);
  }
}

// Cluster form of a small released copy (DV_CLUSTER=1): one cluster of kClusterCtas CTAs, up to
// 1024 threads each, U <= 4 vectors per thread. Returns cudaErrorNotSupported when it does not fit.
// Cluster size of the small-copy publish: 16 CTAs (non-portable, allowed per kernel) when the
// device accepts it, else the portable 8. Measured (tools/probe_latency.py, C2 layer into HBM):
// 8 CTAs 3.23 us, 16 CTAs 2.78 us writer end -> flag. DV_CLUSTER_CTAS=8 forces the portable size.
static int cluster_ctas() {
  static const int n = [] {
    const char* e = getenv("DV_CLUSTER_CTAS");
    if (e && atoi(e) == 8) return 8;
    bool ok = true;
    ok &= cudaFuncSetAttribute(k_copy_cluster<16, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    ok &= cudaFuncSetAttribute(k_copy_cluster<16, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    ok &= cudaFuncSetAttribute(k_copy_cluster<16, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    ok &= cudaFuncSetAttribute(k_copy_cluster<32, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    ok &= cudaFuncSetAttribute(k_copy_cluster<32, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    ok &= cudaFuncSetAttribute(k_copy_cluster<32, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    (void)cudaGetLastError();
    return ok ? 16 : kClusterCtas;
  }();
  return n;
}
template <int VEC, int U>
static cudaError_t go_cluster(const KParams& kp, int threads, cudaStream_t st) {
  (void)cudaGetLastError();
  const int nc = cluster_ctas();
  if (nc > 8) {   // the attribute is per device: set it on every device this process uses
    static std::atomic<uint64_t> mask{0};
    if (first_use_on_device(mask)) {
      cudaFuncSetAttribute(k_copy_cluster<16, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_copy_cluster<16, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_copy_cluster<16, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_copy_cluster<32, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_copy_cluster<32, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_copy_cluster<32, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc);
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_copy_cluster<VEC, U>, kp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}
// The last stream on which a cluster launch was refused (a small green-context partition).
static std::atomic<uintptr_t> g_no_cluster_stream{UINTPTR_MAX};   // none yet
static bool cluster_fits(uint64_t n_vec) { return n_vec <= (uint64_t)cluster_ctas() * 1024 * 4; }
// Measured (tools/probe_latency.py, C2 layer 160 KiB = 5,120 vectors): into HBM (gpu-scope
// release) writer end -> flag 3.55 (ticket) -> 3.20 (8-CTA cluster) -> 2.78 us (16-CTA cluster); to
// pinned host (system scope) 5.89 (ticket) / 6.05 (8) / 5.89 us (16) -- no gain, the PCIe flush
// dominates; a 576 KiB peer put with 8 CTAs got slower (ping-pong RTT 11.3 -> 12.5 us). So by
// default only gpu-scope releases of <= 8,192 vectors use it.
static bool use_cluster(const KParams& kp) {
  const int c = tune().cluster;
  if (c == 2) return cluster_fits(kp.n_vec);
  return c == 1 && kp.pub == 3 && kp.n_vec <= (uint64_t)kClusterCtas * 1024;
}
static cudaError_t launch_cluster(const KParams& kp, int vec, cudaStream_t st) {
  const uint64_t per_cta = (kp.n_vec + cluster_ctas() - 1) / cluster_ctas();
  const int u = per_cta <= 1024 ? 1 : per_cta <= 2048 ? 2 : 4;
  const int threads = (int)std::min<uint64_t>(1024, ((per_cta + u - 1) / u + 31) / 32 * 32);
  if (vec == 32)
    return u == 1 ? go_cluster<32, 1>(kp, threads, st) : u == 2 ? go_cluster<32, 2>(kp, threads, st)
                                                         : go_cluster<32, 4>(kp, threads, st);
  return u == 1 ? go_cluster<16, 1>(kp, threads, st) : u == 2 ? go_cluster<16, 2>(kp, threads, st)
                                                       : go_cluster<16, 4>(kp, threads, st);
}

// Small copies (per-token updates): one vector per thread, 128-thread CTAs, as many CTAs as
// needed -> lowest latency. Large copies: U vectors in flight per thread, grid capped at max_ctas.
static cudaError_t launch_cfg(const KParams& kp, int vec, int max_ctas, cudaStream_t st) {
  const Tune& t = tune();
  int u = t.u ? t.u : (kp.n_vec <= t.small ? 1 : 4);
  return vec == 32 ? launch_vec<32>(kp, u, max_ctas, st) : launch_vec<16>(kp, u, max_ctas, st);
}

// Is the destination of run q at dst + q*run_bytes (row-major dense over the loop dims)?
static bool dense_dst(const CopyPlan& p) {
  int64_t expect = (int64_t)p.run_bytes;
  for (int k = kDims - 1; k >= 0; --k) {
    if (p.n[k] == 1) continue;
    if (p.ds[k] != expect) return false;
    expect *= p.n[k];
  }
  return true;
}

// Is the source of run q at src + q*run_bytes (a dense wire chunk)?
static bool dense_src(const CopyPlan& p) {
  int64_t expect = (int64_t)p.run_bytes;
  for (int k = kDims - 1; k >= 0; --k) {
    if (p.n[k] == 1) continue;
    if (p.ss[k] != expect) return false;
    expect *= p.n[k];
  }
  return true;
}

template <int VEC>
static cudaError_t launch_unpack_bulk_vec(const KParams& kp, const uint8_t* src0, int max_ctas,
                                          cudaStream_t st) {
  const uint32_t ch = std::min<uint32_t>(tune().rdch, 64u << 10);
  const uint32_t nst = std::max<uint32_t>(1, std::min<uint32_t>(tune().rdst, (200u << 10) / ch));
  const int smem = (int)(ch * nst);
  static std::atomic<uint64_t> mask{0};
  if (first_use_on_device(mask))
    cudaFuncSetAttribute(k_unpack_bulk<VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const uint64_t chunks = ((uint64_t)kp.n_vec * VEC + ch - 1) / ch;
  const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>(chunks, (uint64_t)max_ctas));
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_unpack_bulk<VEC>, kp, src0, ch, nst);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int VEC>
static cudaError_t launch_bulk_vec(const KParams& kp, uint8_t* dst0, int max_ctas, cudaStream_t st) {
  constexpr int T = 256, U = 4;
  const int smem = 2 * T * U * VEC;
  if (first_use_on_device(bulk_mask<VEC>()))
    cudaFuncSetAttribute(k_pack_bulk<VEC, U, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const uint64_t need = (kp.n_vec + T * U - 1) / (T * U);
  const int blocks = (int)std::min<uint64_t>(need, (uint64_t)max_ctas);
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_pack_bulk<VEC, U, T>, kp, dst0);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

static cudaError_t launch_bulk(const KParams& kp, int vec, uint8_t* dst0, int max_ctas,
                               cudaStream_t st) {
  return vec == 32 ? launch_bulk_vec<32>(kp, dst0, max_ctas, st)
                   : launch_bulk_vec<16>(kp, dst0, max_ctas, st);
}

// Is `p` reached over a link (pinned host memory over PCIe, or another GPU's memory over NVLink)
// rather than this GPU's own HBM?
static bool over_link(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered) return true;
  int dev = 0;
  cudaGetDevice(&dev);
  return at.type == cudaMemoryTypeDevice && at.device != dev;
}

static dv_status fill_tparams(const CopyPlan& p, const Release& rel, TParams* out) {
  TParams tp{};
  tp.src = p.src;
  tp.dst = p.dst;
  // slab dims: the last four loop dims of the plan (the builder leaves the others at 1)
  uint64_t slabs = 1;
  for (int d = 0; d < 4; ++d) {
    const int k = kDims - 4 + d;
    tp.ss[d] = p.ss[k];
    tp.ds[d] = p.ds[k];
    tp.fd[d] = to_dev(make_fastdiv(p.n[k]));
    slabs *= p.n[k];
  }
  for (int k = 0; k < kDims - 4; ++k)
    if (p.n[k] != 1) return fail(DV_ENOTSUP, "transpose plan with more than 4 slab dims");
  const uint64_t tiles = (p.tN + kTS - 1) / kTS;
  if (slabs * tiles >= (1ull << 31) || p.tU > 256) return fail(DV_ENOTSUP, "transpose too large");
  if (kTS * (p.tU + 1) * 16 > 64 * 1024) return fail(DV_ENOTSUP, "head_dim too large for the packet transpose");
  tp.n_tiles = (uint32_t)(slabs * tiles);
  tp.tiles_per_slab = (uint32_t)tiles;
  tp.fT = to_dev(make_fastdiv((uint32_t)tiles));
  tp.fU = to_dev(make_fastdiv(p.tU));
  tp.U = p.tU;
  tp.N = p.tN;
  tp.su = p.t_su;
  tp.sps = p.t_ss;
  tp.flag = rel.flag;
  tp.seq = rel.seq;
  tp.ticket = rel.ticket;
  tp.ts = rel.ts;
  tp.pub = pub_of(rel);
  tp.dyn = p.dyn;
  tp.dyn_ss = p.dyn_ss;
  tp.dyn_ds = p.dyn_ds;
  tp.dyn_max = p.dyn_max;
  // register form: PK = 2 when the packet count is even and the position-major side's 32-byte
  // vectors are aligned (base, position stride, slab strides, step stride)
  const uint64_t items1 = slabs * p.tN * p.tU;
  uint64_t pm = p.t_ss | (uint64_t)(p.tdir == 0 ? p.dyn_ds : p.dyn_ss) |
                (uint64_t)(uintptr_t)(p.tdir == 0 ? p.dst : p.src);
  for (int d = 0; d < 4; ++d) pm |= (uint64_t)(p.tdir == 0 ? tp.ds[d] : tp.ss[d]);
  const int want = tune().trs == 3 ? 2 : tune().trs == 2 ? 1 : tune().pk;
  // Pinned host memory on either side: the shared-memory tile form, whose warps store (load)
  // consecutive 16-byte packets of a position row -- whole 128-byte lines per warp instruction,
  // which PCIe carries in full TLPs. The register form's per-thread 256-byte rows leave partial
  // lines per instruction: C2 FT6D prompt layer to pinned host 35 GB/s (registers) vs 48-49 GB/s
  // (tiles), tools/probe_ft6d_host_ctas.py. In HBM the register form is the faster one. A peer
  // GPU's memory is treated like the host's (NVLink is packetised like PCIe; not measurable on
  // one GPU -- memory IPC-mapped from another process on the SAME GPU stays on the register form).
  // (DV_TRS=4: the register form even over a link -- the peer-memory experiment of bench_peer)
  const bool host_side = tune().trs == 0 && (over_link(p.src) || over_link(p.dst));
  tp.pk = 0;
  if (tune().trs != 1 && !host_side && items1 < (1ull << 31)) {
    tp.pk = 1;
    for (int k = 16; k >= 2; k /= 2)
      if (want >= k && p.tU % k == 0 && pm % 32 == 0) {
        tp.pk = k;
        break;
      }
  }
  // DV_PP=2: the two-position form, when N is even and the packet-major side's 32-byte vectors
  // are aligned too (base, packet stride, slab strides, step stride)
  uint64_t km = p.t_su | (uint64_t)(p.tdir == 0 ? p.dyn_ss : p.dyn_ds) |
                (uint64_t)(uintptr_t)(p.tdir == 0 ? p.src : p.dst);
  for (int d = 0; d < 4; ++d) km |= (uint64_t)(p.tdir == 0 ? tp.ss[d] : tp.ds[d]);
  if (tune().pp == 2 && (tp.pk == 16 || tp.pk == 8 || tp.pk == 4) && p.tN % 2 == 0 && km % 32 == 0) {
    const int pk2 = tp.pk == 4 ? 4 : 8;
    tp.n_items = (uint32_t)(items1 / pk2 / 2);
    tp.fN = to_dev(make_fastdiv(p.tN / 2));
    tp.fG = to_dev(make_fastdiv(p.tU / pk2));
    tp.pk = 32 + pk2;
  } else if (tp.pk) {
    tp.n_items = (uint32_t)(items1 / tp.pk);
    tp.fN = to_dev(make_fastdiv(p.tN));
    tp.fG = to_dev(make_fastdiv(p.tU / tp.pk));
  }
  *out = tp;
  return DV_OK;
}

// CTAs a transpose plan can use, and its dynamic shared memory.
static uint64_t transpose_ctas(const TParams& tp) {
  if (!tp.pk) return tp.n_tiles;
  const uint64_t per = tp.pk >= 8 ? 256 : tp.pk == 4 ? 512 : 1024;  // IT * 256 items per CTA pass
  return (tp.n_items + per - 1) / per;
}
static int transpose_smem(const TParams& tp) { return tp.pk ? 0 : kTS * (tp.U + 1) * 16; }

static void set_transpose_smem() {
  static std::atomic<uint64_t> mask{0};
  if (first_use_on_device(mask)) {
    cudaFuncSetAttribute(k_packet_transpose<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_packet_transpose<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_transpose_run<0, 16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_transpose_run<1, 16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_transpose_run<0, 32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_transpose_run<1, 32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  }
}

// Kernel instantiation for a (direction, vector width, PK) triple.
using PtFn = void (*)(TParams);
using TrFn = void (*)(TParams, KParams, uint32_t);
template <int DIR>
static PtFn pt_fn(int pk) {
  switch (pk) {
    case 40: return k_packet_transpose<DIR, 40>;
    case 36: return k_packet_transpose<DIR, 36>;
    case 16: return k_packet_transpose<DIR, 16>;
    case 8: return k_packet_transpose<DIR, 8>;
    case 4: return k_packet_transpose<DIR, 4>;
    case 2: return k_packet_transpose<DIR, 2>;
    case 1: return k_packet_transpose<DIR, 1>;
    default: return k_packet_transpose<DIR, 0>;
  }
}
template <int DIR, int VEC>
static TrFn tr_fn(int pk) {
  switch (pk) {
    case 40: return k_transpose_run<DIR, VEC, 40>;
    case 36: return k_transpose_run<DIR, VEC, 36>;
    case 16: return k_transpose_run<DIR, VEC, 16>;
    case 8: return k_transpose_run<DIR, VEC, 8>;
    case 4: return k_transpose_run<DIR, VEC, 4>;
    case 2: return k_transpose_run<DIR, VEC, 2>;
    case 1: return k_transpose_run<DIR, VEC, 1>;
    default: return k_transpose_run<DIR, VEC, 0>;
  }
}

static void fill_kparams(const CopyPlan& p, int VEC, KParams* kp);
static uint64_t align_bits(const CopyPlan& p);

// ---- TMA-row transpose: the tensor map of the packet-major side ------------------------------
typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode() {
  static const TmapEncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      f = nullptr;
    }
    return (TmapEncodeFn)f;
  }();
  return fn;
}
static bool own_hbm(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  return at.type == cudaMemoryTypeDevice && at.device == dev;
}
static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    (void)cudaGetLastError();
    n = 148;
  }
  return n;
}
constexpr int kTmaSmem = 64 * 1024;   // dynamic shared memory budget of a TMA-row transpose CTA

// The TMA-row form applies when DV_TMA is on, the packet-major side is this GPU's HBM (not a step-
// shifted graph plan), the position-major side is in HBM too and 32-byte aligned, U is even, and
// the slab dims fit the map's three remaining dims (unit dims dropped, nested ones merged).
// Fills tp's tm_* fields, *map and *ts_out; false = use the other forms.
static bool tma_rows_setup(const CopyPlan& p, TParams& tp, CUtensorMap* map, int* ts_out) {
  if (!tune().tma || p.dyn || p.tU % 2 || p.tU > 128 || !tmap_encode()) return false;
  const uint8_t* pm = p.tdir == 0 ? p.src : p.dst;   // packet-major side
  const uint8_t* ps = p.tdir == 0 ? p.dst : p.src;   // position-major side
  if ((uintptr_t)pm % 16 || p.t_su % 16 || p.t_su <= 0) return false;
  uint64_t al = (uint64_t)p.t_ss | (uint64_t)(uintptr_t)ps;
  for (int d = 0; d < 4; ++d) al |= (uint64_t)(p.tdir == 0 ? tp.ds[d] : tp.ss[d]);
  if (al % 32) return false;
  if (!own_hbm(pm) || !own_hbm(ps)) return false;
  int TS = tune().tma_ts ? tune().tma_ts : (p.tdir == 0 ? 32 : 64);
  while (TS > 8 && (uint64_t)p.tU * TS * 16 * 2 > (uint64_t)kTmaSmem) TS /= 2;
  if (TS != 8 && TS != 16 && TS != 32 && TS != 64) return false;
  const uint32_t stage = p.tU * TS * 16;
  const int nst = std::min(kTmaStagesMax, (int)(kTmaSmem / stage));
  if (nst < 2) return false;
  // slab dims (inner -> outer) -> map dims 2..4
  uint64_t gn[3] = {1, 1, 1};
  int64_t gs[3] = {16, 16, 16};
  int ng = 0;
  uint64_t slabs = 1;
  for (int d = 3; d >= 0; --d) {
    const int k = kDims - 4 + d;
    const uint64_t n = p.n[k];
    const int64_t st = p.tdir == 0 ? p.ss[k] : p.ds[k];
    slabs *= n;
    if (n == 1) {
      tp.tm_dim[d] = -1;
      tp.tm_mul[d] = 0;
      continue;
    }
    if (st <= 0 || st % 16 || st >= (1ll << 40)) return false;
    if (ng > 0 && st == gs[ng - 1] * (int64_t)gn[ng - 1] && gn[ng - 1] * n < (1ull << 31)) {
      tp.tm_dim[d] = 2 + ng - 1;   // nests outside the current map dim
      tp.tm_mul[d] = (uint32_t)gn[ng - 1];
      gn[ng - 1] *= n;
      continue;
    }
    if (ng == 3) return false;
    tp.tm_dim[d] = 2 + ng;
    tp.tm_mul[d] = 1;
    gn[ng] = n;
    gs[ng] = st;
    ++ng;
  }
  const uint64_t tps = (p.tN + TS - 1) / TS;
  if (slabs * tps >= (1ull << 31)) return false;
  const cuuint64_t dims[5] = {(cuuint64_t)p.tN * 4, p.tU, gn[0], gn[1], gn[2]};
  const cuuint64_t strides[4] = {(cuuint64_t)p.t_su, (cuuint64_t)gs[0], (cuuint64_t)gs[1], (cuuint64_t)gs[2]};
  const cuuint32_t box[5] = {(cuuint32_t)TS * 4, 1, 1, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  if (tmap_encode()(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, (void*)pm, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tp.tm_nst = nst;
  tp.tm_tps = (uint32_t)tps;
  tp.fTm = to_dev(make_fastdiv((uint32_t)tps));
  tp.n_tiles = (uint32_t)(slabs * tps);
  *ts_out = TS;
  return true;
}

using TmFn = void (*)(TParams, KParams, uint32_t, CUtensorMap);
template <int DIR, int VEC>
static TmFn tm_fn(int ts) {
  switch (ts) {
    case 8: return k_transpose_tma_run<DIR, VEC, 8>;
    case 16: return k_transpose_tma_run<DIR, VEC, 16>;
    case 32: return k_transpose_tma_run<DIR, VEC, 32>;
    default: return k_transpose_tma_run<DIR, VEC, 64>;
  }
}
static void set_tma_smem() {
  static std::atomic<uint64_t> mask{0};
  if (first_use_on_device(mask))
    for (int ts : {8, 16, 32, 64}) {
      cudaFuncSetAttribute(tm_fn<0, 16>(ts), cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
      cudaFuncSetAttribute(tm_fn<1, 16>(ts), cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
      cudaFuncSetAttribute(tm_fn<0, 32>(ts), cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
      cudaFuncSetAttribute(tm_fn<1, 32>(ts), cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
    }
}

// One launch: the TMA-row transpose of `t` (+ the run copy `r` when given). Every CTA is resident
// at once (grid = SMs x CTAs per SM that the shared memory allows, <= max_ctas); the transpose
// CTAs get DV_TMA_TSPLIT x their byte share.
static dv_status launch_tma_run(const CopyPlan& t, const TParams& tp, const CUtensorMap& map, int TS,
                                const CopyPlan* r, int max_ctas, cudaStream_t stream) {
  const int smem = tp.tm_nst * (int)tp.U * TS * 16;
  KParams kr{};
  int VEC = 32;
  uint64_t grid, t_blocks;
  if (r) {
    const uint64_t orall = align_bits(*r);
    if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
    VEC = (orall % 32 == 0 && tune().vec != 16) ? 32 : 16;
    fill_kparams(*r, VEC, &kr);
  }
  const TmFn fn = t.tdir == 0 ? (VEC == 32 ? tm_fn<0, 32>(TS) : tm_fn<0, 16>(TS))
                              : (VEC == 32 ? tm_fn<1, 32>(TS) : tm_fn<1, 16>(TS));
  set_tma_smem();
  int per_sm = 1;   // resident CTAs per SM (registers, threads and shared memory together)
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess || per_sm < 1) {
    (void)cudaGetLastError();
    per_sm = 1;
  }
  if (r) {
    grid = std::max<uint64_t>(2, std::min<uint64_t>((uint64_t)max_ctas, (uint64_t)sm_count() * per_sm));
    const double tb = (double)t.runs() * t.tN * t.tU * 16, rb = (double)r->runs() * r->run_bytes, w = tune().tma_split;
    t_blocks = (uint64_t)(grid * w * tb / (w * tb + rb) + 0.5);
    t_blocks = std::min(std::max<uint64_t>(1, t_blocks), grid - 1);
  } else {
    grid = std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)max_ctas, (uint64_t)sm_count() * per_sm,
                                                     (uint64_t)tp.n_tiles}));
    t_blocks = grid;
  }
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, tp, kr, (uint32_t)t_blocks, map);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  g_tma_launches.fetch_add(1, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "TMA transpose kernel launch");
  return DV_OK;
}

static dv_status launch_transpose(const CopyPlan& p, const Release& rel, int max_ctas,
                                  cudaStream_t stream) {
  TParams tp;
  DV_TRY(fill_tparams(p, rel, &tp));
  {
    CUtensorMap map;
    int TS = 0;
    if (tma_rows_setup(p, tp, &map, &TS)) return launch_tma_run(p, tp, map, TS, nullptr, max_ctas, stream);
  }
  const int smem = transpose_smem(tp);
  set_transpose_smem();
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(transpose_ctas(tp), (uint64_t)max_ctas)));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, p.tdir == 0 ? pt_fn<0>(tp.pk) : pt_fn<1>(tp.pk), tp);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "transpose kernel launch");
  return DV_OK;
}

// Kernel parameters of a whole run plan at vector width VEC (no split; caller checked sizes).
static void fill_kparams(const CopyPlan& p, int VEC, KParams* kp) {
  *kp = KParams{};
  kp->src = p.src;
  kp->dst = p.dst;
  for (int k = 0; k < kDims; ++k) {
    kp->ss[k] = p.ss[k];
    kp->ds[k] = p.ds[k];
    kp->fd[k] = to_dev(make_fastdiv(p.n[k]));
  }
  const uint64_t vpr = p.run_bytes / VEC;
  kp->fv = to_dev(make_fastdiv((uint32_t)vpr));
  kp->q_begin = 0;
  kp->n_vec = (uint32_t)(p.runs() * vpr);
  kp->dyn = p.dyn;
  kp->dyn_ss = p.dyn_ss;
  kp->dyn_ds = p.dyn_ds;
  kp->dyn_max = p.dyn_max;
}

static uint64_t align_bits(const CopyPlan& p) {
  uint64_t orall = (uint64_t)(uintptr_t)p.src | (uint64_t)(uintptr_t)p.dst | p.run_bytes;
  for (int k = 0; k < kDims; ++k) orall |= (uint64_t)p.ss[k] | (uint64_t)p.ds[k];
  return orall | (uint64_t)p.dyn_ss | (uint64_t)p.dyn_ds;
}

template <int VEC, int U, int THREADS>
static cudaError_t go2(const KParams& a, const KParams& b, int blocks, cudaStream_t st) {
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_run_copy2<VEC, U, THREADS>, a, b);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// FT6D key transpose + value run copy in one launch; CTAs split in proportion to the bytes.
static dv_status launch_transpose_run(const CopyPlan& t, const CopyPlan& r, const Release& rel,
                                      int max_ctas, cudaStream_t stream) {
  TParams tp;
  DV_TRY(fill_tparams(t, rel, &tp));
  {
    CUtensorMap map;
    int TS = 0;
    if (tma_rows_setup(t, tp, &map, &TS)) return launch_tma_run(t, tp, map, TS, &r, max_ctas, stream);
  }
  const uint64_t orall = align_bits(r);
  if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
  const int VEC = (orall % 32 == 0 && tune().vec != 16) ? 32 : 16;
  KParams kr;
  fill_kparams(r, VEC, &kr);
  const double tb = (double)tp.n_tiles * kTS * t.tU * 16, rb = (double)r.runs() * r.run_bytes;
  const uint64_t t_need = transpose_ctas(tp), r_need = (kr.n_vec + 1023) / 1024;
  const uint64_t grid = std::max<uint64_t>(2, std::min<uint64_t>((uint64_t)max_ctas, t_need + r_need));
  // transpose CTAs get 0.6 of their byte share (C2 FT6D prompt layer, PK = 16, both directions,
  // tools/ft6d_cmp.sh + tools/probe_ft6d_dirs.py: pack / unpack / KV5D->FT6D remap 0.954 / 0.942 /
  // 0.935 of HBM peak at 0.6, 0.950 / 0.934 / 0.925 at 0.7, 0.939 / 0.933 / 0.924 at 1.0;
  // DV_TSPLIT=0 = every CTA does both halves)
  static const double tscale = getenv("DV_TSPLIT") ? atof(getenv("DV_TSPLIT")) : 0.6;
  uint64_t t_blocks = (uint64_t)(grid * tscale * tb / (tscale * tb + rb) + 0.5);
  t_blocks = std::min(std::max<uint64_t>(1, t_blocks), grid - 1);
  if (tscale == 0) t_blocks = 0;
  set_transpose_smem();
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = transpose_smem(tp);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const uint32_t tbk = (uint32_t)t_blocks;
  cudaError_t e;
  const TrFn fn = t.tdir == 0 ? (VEC == 32 ? tr_fn<0, 32>(tp.pk) : tr_fn<0, 16>(tp.pk))
                               : (VEC == 32 ? tr_fn<1, 32>(tp.pk) : tr_fn<1, 16>(tp.pk));
  e = cudaLaunchKernelEx(&cfg, fn, tp, kr, tbk);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "transpose+run kernel launch");
  return DV_OK;
}

// ---- persistent stream engine (dv_engine_*, DESIGN.md §6 "Persistent engine") -----------------
// ONE thread-block cluster of W <= 16 CTAs stays resident on its own highest-priority stream.
// Registered plans (a run copy whose source and destination move by k positions / k*step bytes at
// step k, and the flag it releases with seq + k) are triggered by doorbells: want[plan] = k + 1 (a
// stream memory write after the producer, or a release by the producer kernel itself). Warp 0 of
// cluster rank 0 polls the doorbells (one L2 round trip per scan: every lane's loads in flight at
// once) and posts the next (plan, step) in its shared memory; a cluster barrier hands it to every
// CTA (read through distributed shared memory), each CTA copies its static share (1,024-vector
// units rank, rank + W, ...), a second cluster barrier (release / acquire) collects every CTA's
// stores, and rank 0 releases the flag at the scope the memory needs. Jobs run in lockstep, so
// every flag is released in step order. No launch, no SM-slot wait, no dependency wait and no
// global-memory ticket sit between the producer's doorbell and the copy. The plans' parameters
// live in every CTA's shared memory.
constexpr int kEngineMaxCtas = 16;   // the non-portable cluster size (8 where refused)
struct EPlan {
  KParams kp;        // whole plan at step 0 (q_begin 0); dyn_ss / dyn_ds: bytes per step
  int32_t vec;       // 16 or 32
  int32_t max_step;
};
struct EState {
  unsigned long long want[kEngineMaxPlans];    // doorbells (steps requested + 1)
  unsigned long long done[kEngineMaxPlans];    // steps completed (flag released)
  unsigned long long issued[kEngineMaxPlans];  // rank 0's progress, kept across park / relaunch
  unsigned int stop;
  int32_t n_plans;                             // registered plans (polled: [0, n_plans))
  unsigned long long* stamps;                  // optional: %globaltimer after (plan, step)'s release
  unsigned long long n_stamps;                 // stamps[(step * n_plans + plan) % n_stamps]
};

__device__ __forceinline__ unsigned long long ld_rlx_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Warp 0 of rank 0: the next pending plan (lowest index), or -1 (stop requested, nothing pending);
// *np_out = the registered plans seen by the scan.
__device__ __forceinline__ int engine_poll(EState* s, const EPlan* plans, const unsigned long long* issued,
                                           int* np_out) {
  const int lane = threadIdx.x;
  bool stopping = false;
  for (;;) {
    const int np = *(volatile int32_t*)&s->n_plans;   // plans registered while the engine runs
    *np_out = np;
    // one round trip per scan: every lane's doorbell loads and the stop word in flight together
    const unsigned st = *(volatile unsigned int*)&s->stop;
    unsigned long long w[kEngineMaxPlans / 32];
#pragma unroll
    for (int i = 0; i < kEngineMaxPlans / 32; ++i) {
      const int p = lane + 32 * i;
      w[i] = p < np ? ld_rlx_gpu(&s->want[p]) : 0ull;
    }
#pragma unroll
    for (int i = 0; i < kEngineMaxPlans / 32; ++i) {
      const int p = lane + 32 * i;
      // a step beyond the plan's validated max_step (a producer ringing too far) is never run
      const bool pend = p < np && w[i] > issued[p] && issued[p] <= (unsigned long long)plans[p].max_step;
      const unsigned m = __ballot_sync(0xffffffffu, pend);
      if (m) return 32 * i + __ffs(m) - 1;
    }
    if (stopping) return -1;   // stop seen, and a full scan after it found nothing pending
    if (st) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");   // every doorbell released before the stop
      stopping = true;
    }
  }
}

__global__ void __launch_bounds__(256) k_engine(EState* s, const EPlan* plans) {
  extern __shared__ __align__(16) uint8_t esm[];
  KParams* sp = reinterpret_cast<KParams*>(esm);                                   // [kEngineMaxPlans]
  int32_t* svec = reinterpret_cast<int32_t*>(sp + kEngineMaxPlans);
  __shared__ unsigned long long issued[kEngineMaxPlans];   // rank 0 only
  __shared__ __align__(16) int32_t job[4];                   // rank 0's copy is the broadcast
  uint32_t rank, W;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(W));
  uint32_t job_addr;   // rank 0's `job` in the cluster's shared window
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(job_addr) : "r"((uint32_t)__cvta_generic_to_shared(job)));
  if (rank == 0)
    for (int p = threadIdx.x; p < kEngineMaxPlans; p += blockDim.x) issued[p] = s->issued[p];
  __syncthreads();
  int loaded = 0;
  __shared__ unsigned long long t_found;
  for (;;) {
    if (rank == 0 && threadIdx.x < 32) {
      int np = 0;
      const int plan = engine_poll(s, plans, issued, &np);
      if (threadIdx.x == 0) {
        if (plan >= 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");   // the producer's data
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_found));
        job[0] = plan;
        job[1] = plan >= 0 ? (int32_t)issued[plan] : 0;
        job[2] = np;
        // taken: the next poll (after the barriers below) must not see this step as pending
        if (plan >= 0) issued[plan] += 1;
      }
    }
    cluster_sync_all();   // B1: the job is posted
    unsigned long long t_b1 = 0, t_copied = 0, t_b2 = 0;
    if (rank == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_b1));
    int32_t plan, k, np, pad_;
    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(plan), "=r"(k), "=r"(np), "=r"(pad_) : "r"(job_addr) : "memory");
    if (plan < 0) {       // park: rank 0 keeps its progress for the relaunch
      if (rank == 0)
        for (int p = threadIdx.x; p < kEngineMaxPlans; p += blockDim.x) s->issued[p] = issued[p];
      cluster_sync_all();   // nobody leaves while a peer may still read rank 0's shared memory
      return;
    }
    if (np > loaded) {    // newly registered plans' parameters into shared memory
      for (int p = loaded; p < np; ++p) {
        const int* from = reinterpret_cast<const int*>(&plans[p].kp);
        int* to = reinterpret_cast<int*>(&sp[p]);
        for (int i = threadIdx.x; i < (int)(sizeof(KParams) / sizeof(int)); i += blockDim.x) to[i] = from[i];
        if (threadIdx.x == 0) svec[p] = plans[p].vec;
      }
      loaded = np;
      __syncthreads();
    }
    const KParams& kp = sp[plan];
    if (svec[plan] == 32)
      run_chunks<32, 4, 256>(kp, kp.src + (int64_t)k * kp.dyn_ss, kp.dst + (int64_t)k * kp.dyn_ds, rank, W);
    else
      run_chunks<16, 4, 256>(kp, kp.src + (int64_t)k * kp.dyn_ss, kp.dst + (int64_t)k * kp.dyn_ds, rank, W);
    if (rank == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_copied));
    asm volatile("fence.acq_rel.gpu;" ::: "memory");   // this thread's stores, performed at gpu scope
    cluster_sync_all();   // B2: every CTA's stores are in rank 0's causality past
    if (rank == 0 && threadIdx.x == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_b2));
      if (kp.flag) {
        const unsigned long long seq = kp.seq + (unsigned long long)k;
        if (kp.pub == 3)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(kp.flag), "l"(seq) : "memory");
        else
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(kp.flag), "l"(seq) : "memory");
      }
      unsigned long long* stamps = s->stamps;
      const unsigned long long n_stamps = s->n_stamps;
      if (stamps && n_stamps) {   // [flag released, job found, past B1, copy issued, past B2]
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        unsigned long long* r = stamps + 5 * (((unsigned long long)k * (unsigned long long)np + plan) % n_stamps);
        r[0] = t;
        r[1] = t_found;
        r[2] = t_b1;
        r[3] = t_copied;
        r[4] = t_b2;
      }
      st_rel_gpu(&s->done[plan], (unsigned long long)k + 1);
    }
  }
}

int engine_smem() { return (int)(kEngineMaxPlans * (sizeof(KParams) + sizeof(int32_t))); }

// Cluster size of the engine: n_ctas when the device accepts it (> 8 needs the non-portable
// attribute), else an error.
static dv_status engine_cfg(int n_ctas) {
  static std::atomic<uint64_t> mask{0};
  if (first_use_on_device(mask)) {
    cudaFuncSetAttribute(k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, engine_smem());
    cudaFuncSetAttribute(k_engine, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    (void)cudaGetLastError();
  }
  if (n_ctas < 1 || n_ctas > kEngineMaxCtas) return fail(DV_EINVAL, "engine CTAs %d outside [1, %d]", n_ctas, kEngineMaxCtas);
  return DV_OK;
}

dv_status engine_alloc(void** state, void** plans) {
  DV_CUDA(cudaMalloc(state, sizeof(EState)));
  DV_CUDA(cudaMalloc(plans, sizeof(EPlan) * kEngineMaxPlans));
  DV_CUDA(cudaMemset(*state, 0, sizeof(EState)));
  DV_CUDA(cudaMemset(*plans, 0, sizeof(EPlan) * kEngineMaxPlans));
  return DV_OK;
}

dv_status engine_launch(void* state, const void* plans, int n_ctas, cudaStream_t st) {
  DV_TRY(engine_cfg(n_ctas));
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = engine_smem();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;   // the whole grid is ONE cluster
  at[0].val.clusterDim.x = n_ctas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_engine, (EState*)state, (const EPlan*)plans);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "engine kernel launch");
  return DV_OK;
}

unsigned long long* engine_word(void* state, int which, int plan) {
  EState* s = (EState*)state;
  switch (which) {
    case 0: return &s->want[plan];
    case 1: return &s->done[plan];
    case 2: return nullptr;
    default: return nullptr;
  }
}
size_t engine_field_offset(int which) {
  switch (which) {
    case 0: return offsetof(EState, stop);
    case 1: return offsetof(EState, n_plans);
    case 2: return offsetof(EState, stamps);
    default: return offsetof(EState, n_stamps);
  }
}

// Plan `id` := the whole run plan p (one launch's worth; at most 2^31 vectors), released into
// `flag` with seq + k at step k.
dv_status engine_set_plan(void* plans, int id, const CopyPlan& p, const Release& rel, int32_t max_step,
                          cudaStream_t st) {
  if (p.kind != kRun) return fail(DV_ENOTSUP, "engine plans are run copies (no packet transpose)");
  uint64_t orall = (uint64_t)(uintptr_t)p.src | (uint64_t)(uintptr_t)p.dst | p.run_bytes;
  for (int k = 0; k < kDims; ++k) orall |= (uint64_t)p.ss[k] | (uint64_t)p.ds[k];
  orall |= (uint64_t)p.dyn_ss | (uint64_t)p.dyn_ds;
  if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
  const int VEC = (orall % 32 == 0) ? 32 : 16;
  if (p.runs() * (p.run_bytes / VEC) >= (1ull << 31)) return fail(DV_ENOTSUP, "engine plan too large");
  EPlan e{};
  fill_kparams(p, VEC, &e.kp);
  e.kp.dyn = nullptr;
  e.kp.flag = rel.flag;
  e.kp.seq = rel.seq;
  e.kp.pub = pub_of(rel) >= 2 ? pub_of(rel) : 2;
  e.vec = VEC;
  e.max_step = max_step;
  DV_CUDA(cudaMemcpyAsync((EPlan*)plans + id, &e, sizeof e, cudaMemcpyHostToDevice, st));
  DV_CUDA(cudaStreamSynchronize(st));
  return DV_OK;
}

// Load every kernel of the library on the current device now (cudaFuncGetAttributes needs the
// loaded function). Under CUDA lazy loading a kernel is otherwise loaded at its first launch, and
// that load waits for the device: a consumer kernel already spinning on one of our flags would
// then block the very stream-out it waits for (observed with the dvt_watch latency observer).
template <typename F>
static void load_fn(F f) {
  cudaFuncAttributes a;
  (void)cudaFuncGetAttributes(&a, f);
}
template <int VEC>
static void load_vec() {
  load_fn(k_run_copy<VEC, 1, 128>);
  load_fn(k_run_copy<VEC, 2, 256>);
  load_fn(k_run_copy<VEC, 4, 256>);
  load_fn(k_run_copy<VEC, 8, 256>);
  load_fn(k_run_copy<VEC, 4, 256, 1>);
  load_fn(k_run_copy<VEC, 4, 256, 2>);
  load_fn(k_run_copy2<VEC, 1, 128>);
  load_fn(k_run_copy2<VEC, 4, 256>);
  load_fn(k_pack_bulk<VEC, 4, 256>);
  load_fn(k_unpack_bulk<VEC>);
  load_fn(k_copy_cluster<VEC, 1>);
  load_fn(k_copy_cluster<VEC, 2>);
  load_fn(k_copy_cluster<VEC, 4>);
  for (int pk : {0, 1, 2, 4, 8, 16, 36, 40}) {
    load_fn(tr_fn<0, VEC>(pk));
    load_fn(tr_fn<1, VEC>(pk));
  }
}
void preload_kernels() {
  (void)cluster_ctas();   // decide the cluster size (and set the attribute) outside any capture
  load_fn(k_run_copy<16, 1, 32>);
  load_fn(k_wait_geq);
  load_fn(k_store_release);
  load_fn(k_engine);
  load_vec<16>();
  load_vec<32>();
  for (int pk : {0, 1, 2, 4, 8, 16, 36, 40}) {
    load_fn(pt_fn<0>(pk));
    load_fn(pt_fn<1>(pk));
  }
  for (int ts : {8, 16, 32, 64}) {
    load_fn(tm_fn<0, 16>(ts));
    load_fn(tm_fn<1, 16>(ts));
    load_fn(tm_fn<0, 32>(ts));
    load_fn(tm_fn<1, 32>(ts));
  }
  (void)cudaGetLastError();
}

dv_status launch_copy2(const CopyPlan& a, const CopyPlan& b, const Release& rel, int max_ctas,
                       cudaStream_t stream) {
  if ((a.kind == kTranspose) != (b.kind == kTranspose) && a.dyn == b.dyn) {
    const CopyPlan& t = a.kind == kTranspose ? a : b;
    const CopyPlan& r = a.kind == kTranspose ? b : a;
    if (r.runs() && r.run_bytes && r.runs() * r.run_bytes / 16 < (1ull << 31))
      return launch_transpose_run(t, r, rel, max_ctas, stream);
  }
  // Fall back to two launches when the pair does not fit the single-launch form.
  const bool fits = a.kind == kRun && b.kind == kRun && a.run_bytes && b.run_bytes &&
                    a.runs() && b.runs() && a.dyn == b.dyn &&
                    (a.runs() + b.runs()) * std::max(a.run_bytes, b.run_bytes) / 16 < (1ull << 31);
  if (!fits) {
    DV_TRY(launch_copy(a, 0, a.runs(), Release{nullptr, 0, nullptr}, max_ctas, stream));
    return launch_copy(b, 0, b.runs(), rel, max_ctas, stream);
  }
  const uint64_t orall = align_bits(a) | align_bits(b);
  if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
  const int VEC = (orall % 32 == 0 && tune().vec != 16) ? 32 : 16;
  KParams ka, kb;
  fill_kparams(a, VEC, &ka);
  fill_kparams(b, VEC, &kb);
  ka.flag = rel.flag;
  ka.seq = rel.seq;
  ka.ticket = rel.ticket;
  ka.ts = rel.ts;
  ka.pub = pub_of(rel);
  const uint64_t total = (uint64_t)ka.n_vec + kb.n_vec;
  cudaError_t e;
  if (total <= tune().small) {
    const int blocks = (int)((total + 127) / 128);
    e = VEC == 32 ? go2<32, 1, 128>(ka, kb, blocks, stream) : go2<16, 1, 128>(ka, kb, blocks, stream);
  } else {
    const int blocks = (int)std::min<uint64_t>((total + 1023) / 1024, (uint64_t)max_ctas);
    e = VEC == 32 ? go2<32, 4, 256>(ka, kb, blocks, stream) : go2<16, 4, 256>(ka, kb, blocks, stream);
  }
  if (e != cudaSuccess) return cuda_fail(e, "copy kernel launch");
  return DV_OK;
}

dv_status launch_copy(const CopyPlan& p, uint64_t q_first, uint64_t q_last, const Release& rel,
                      int max_ctas, cudaStream_t stream) {
  if (p.kind == kTranspose) {
    if (q_first != 0 || q_last < p.runs()) return fail(DV_ENOTSUP, "partial transpose plan");
    return launch_transpose(p, rel, max_ctas, stream);
  }
  if (q_last > p.runs()) q_last = p.runs();
  if (q_first > q_last) q_first = q_last;
  if (q_last == q_first || p.run_bytes == 0) {
    if (rel.flag) {  // nothing to move: still publish in stream order
      KParams kp{};
      kp.fv = DevDiv{1, 0, 0};
      for (int k = 0; k < kDims; ++k) kp.fd[k] = DevDiv{1, 0, 0};
      kp.flag = rel.flag;
      kp.seq = rel.seq;
      kp.ticket = rel.ticket;
      kp.ts = rel.ts;
      kp.pub = pub_of(rel);
      kp.dyn = p.dyn;
      kp.dyn_max = p.dyn_max;
      cudaError_t e = go<16, 1, 32>(kp, 1, stream);
      if (e != cudaSuccess) return cuda_fail(e, "publish kernel launch");
    }
    return DV_OK;
  }
  // 32-byte vectors when every address and stride allows it.
  uint64_t orall = (uint64_t)(uintptr_t)p.src | (uint64_t)(uintptr_t)p.dst | p.run_bytes;
  for (int k = 0; k < kDims; ++k) orall |= (uint64_t)p.ss[k] | (uint64_t)p.ds[k];
  orall |= (uint64_t)p.dyn_ss | (uint64_t)p.dyn_ds;
  if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
  const int VEC = (orall % 32 == 0 && tune().vec != 16) ? 32 : 16;
  const uint64_t vpr = p.run_bytes / VEC;
  if (vpr >= (1ull << 31)) return fail(DV_ENOTSUP, "run of %llu bytes too long", (unsigned long long)p.run_bytes);
  for (int k = 1; k < kDims; ++k)
    if (p.n[k] >= (1u << 31)) return fail(DV_ENOTSUP, "copy extent too large");
  if (p.runs() >= (1ull << 31)) return fail(DV_ENOTSUP, "too many runs");

  KParams kp{};
  kp.src = p.src;
  kp.dst = p.dst;
  for (int k = 0; k < kDims; ++k) {
    kp.ss[k] = p.ss[k];
    kp.ds[k] = p.ds[k];
    kp.fd[k] = to_dev(make_fastdiv(p.n[k]));
  }
  kp.fv = to_dev(make_fastdiv((uint32_t)vpr));
  kp.dyn = p.dyn;
  kp.dyn_ss = p.dyn_ss;
  kp.dyn_ds = p.dyn_ds;
  kp.dyn_max = p.dyn_max;

  // Split into launches of < 2^31 vectors at run boundaries.
  const uint64_t runs_per_launch = std::max<uint64_t>(1, tune().max_vec_per_launch / vpr);
  for (uint64_t q0 = q_first; q0 < q_last; q0 += runs_per_launch) {
    const uint64_t nq = std::min(runs_per_launch, q_last - q0);
    const bool last = q0 + nq == q_last;
    kp.q_begin = (uint32_t)q0;
    kp.n_vec = (uint32_t)(nq * vpr);
    kp.flag = last ? rel.flag : nullptr;
    kp.seq = rel.seq;
    kp.ticket = rel.ticket;
    kp.ts = last ? rel.ts : nullptr;
    kp.pub = pub_of(rel);
    const bool rd_bulk = tune().rdbulk && !p.dyn && dense_src(p) &&
                         (tune().rdbulk == 2 || over_link(p.src));
    cudaError_t e = rd_bulk ? (VEC == 32 ? launch_unpack_bulk_vec<32>(kp, p.src + q0 * p.run_bytes, max_ctas, stream)
                                         : launch_unpack_bulk_vec<16>(kp, p.src + q0 * p.run_bytes, max_ctas, stream))
                    : (tune().bulk && dense_dst(p) && !p.dyn)
                        ? launch_bulk(kp, VEC, p.dst + q0 * p.run_bytes, max_ctas, stream)
                    : (kp.flag && q0 == 0 && last && use_cluster(kp) &&
                       (uintptr_t)stream != g_no_cluster_stream.load())
                        ? launch_cluster(kp, VEC, stream)
                        : launch_cfg(kp, VEC, max_ctas, stream);
    if (e == cudaErrorInvalidClusterSize) {
      // a stream of a green context with fewer SMs than the cluster (e.g. an 8-SM streaming
      // partition, DESIGN.md §6 "SM partitions"): nothing was launched; the ticket form instead,
      // and for this stream from now on (one remembered stream: no failed launch per call)
      (void)cudaGetLastError();
      g_no_cluster_stream.store((uintptr_t)stream);
      e = launch_cfg(kp, VEC, max_ctas, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "copy kernel launch");
  }
  return DV_OK;
}

}  // namespace dv
