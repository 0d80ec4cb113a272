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
#include <stdlib.h>

#include <algorithm>

#include "dv_internal.h"

namespace dv {

std::atomic<uint64_t> g_kernel_launches{0};
std::atomic<uint64_t> g_dma_calls{0};

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
  int64_t ss0, ss1, ss2, ss3;
  int64_t ds0, ds1, ds2, ds3;
  DevDiv fv;   // vectors per run
  DevDiv f3;   // n[3]
  DevDiv f2;   // n[2]
  DevDiv f1;   // n[1]
  uint32_t q_begin;  // first run of this launch
  uint32_t n_vec;    // vectors in this launch (< 2^31)
  unsigned long long* flag;
  unsigned long long seq;
  unsigned int* ticket;
  unsigned long long* ts;  // optional: %globaltimer right after the flag store (latency tracing)
};

template <int VEC>
struct alignas(VEC) Vec {
  uint32_t w[VEC / 4];
};

__device__ __forceinline__ void ld_vec(Vec<16>& v, const uint8_t* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3])
               : "l"(p));
}
__device__ __forceinline__ void st_vec(uint8_t* p, const Vec<16>& v) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
               "r"(v.w[2]), "r"(v.w[3])
               : "memory");
}
__device__ __forceinline__ void ld_vec(Vec<32>& v, const uint8_t* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
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

template <int VEC>
__device__ __forceinline__ void locate(const KParams& p, uint32_t g, const uint8_t*& s,
                                       uint8_t*& d) {
  uint32_t q, w, i3, i2, i1;
  p.fv.divmod(g, q, w);
  q += p.q_begin;
  p.f3.divmod(q, q, i3);
  p.f2.divmod(q, q, i2);
  p.f1.divmod(q, q, i1);  // q is now i0
  const int64_t wo = (int64_t)w * VEC;
  s = p.src + (int64_t)q * p.ss0 + (int64_t)i1 * p.ss1 + (int64_t)i2 * p.ss2 +
      (int64_t)i3 * p.ss3 + wo;
  d = p.dst + (int64_t)q * p.ds0 + (int64_t)i1 * p.ds1 + (int64_t)i2 * p.ds2 +
      (int64_t)i3 * p.ds3 + wo;
}

__device__ __forceinline__ void publish(const KParams& p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's payload (ordered before by the barrier) -> system scope
    unsigned int prev = atomicAdd(p.ticket, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      *p.ticket = 0u;  // ready for the next stream-ordered user of this ticket
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.flag), "l"(p.seq) : "memory");
      if (p.ts) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        *p.ts = t;
      }
    }
  }
}

template <int VEC, int U, int THREADS>
__global__ void __launch_bounds__(THREADS) k_run_copy(const KParams p) {
  // Programmatic dependent launch: this grid may become resident while the kernel that wrote the
  // K/V (e.g. attention) is still draining; wait here until that grid's memory is visible.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t chunk = THREADS * U;
  for (uint32_t base = blockIdx.x * chunk; base < p.n_vec; base += gridDim.x * chunk) {
    Vec<VEC> v[U];
    uint8_t* d[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) {
        const uint8_t* s;
        locate<VEC>(p, g, s, d[i]);
        ld_vec(v[i], s);
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t g = base + i * THREADS + threadIdx.x;
      if (g < p.n_vec) st_vec(d[i], v[i]);
    }
  }
  if (p.flag) publish(p);
}

static DevDiv to_dev(const FastDiv& f) { return DevDiv{f.d, f.mul, f.shr}; }

static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int VEC, int U, int THREADS>
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_run_copy<VEC, U, THREADS>, kp);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Launch-shape tunables (environment, read once; for experiments -- DESIGN.md "Kernel tuning").
struct Tune {
  int u = 0;          // DV_U: vectors in flight per thread (1,2,4,8); 0 = automatic
  int vec = 0;        // DV_VEC: force 16-byte vectors when 16
  uint64_t small = 148ull * 128 * 4;  // DV_SMALL: copies up to this many vectors use U=1, 128 thr
};
static const Tune& tune() {
  static Tune t = [] {
    Tune x;
    if (const char* e = getenv("DV_U")) x.u = atoi(e);
    if (const char* e = getenv("DV_VEC")) x.vec = atoi(e);
    if (const char* e = getenv("DV_SMALL")) x.small = strtoull(e, nullptr, 10);
    return x;
  }();
  return t;
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
    default: return go<VEC, 4, 256>(kp, blocks, st);
  }
}

// Small copies (per-token updates): one vector per thread, 128-thread CTAs, as many CTAs as
// needed -> lowest latency. Large copies: U vectors in flight per thread, grid capped at max_ctas.
static cudaError_t launch_cfg(const KParams& kp, int vec, int max_ctas, cudaStream_t st) {
  const Tune& t = tune();
  int u = t.u ? t.u : (kp.n_vec <= t.small ? 1 : 4);
  return vec == 32 ? launch_vec<32>(kp, u, max_ctas, st) : launch_vec<16>(kp, u, max_ctas, st);
}

dv_status launch_copy(const CopyPlan& p, uint64_t q_first, uint64_t q_last, const Release& rel,
                      int max_ctas, cudaStream_t stream) {
  if (q_last > p.runs()) q_last = p.runs();
  if (q_first > q_last) q_first = q_last;
  if (q_last == q_first || p.run_bytes == 0) {
    if (rel.flag) {  // nothing to move: still publish in stream order
      KParams kp{};
      kp.fv = kp.f1 = kp.f2 = kp.f3 = DevDiv{1, 0, 0};
      kp.flag = rel.flag;
      kp.seq = rel.seq;
      kp.ticket = rel.ticket;
      kp.ts = rel.ts;
      cudaError_t e = go<16, 1, 32>(kp, 1, stream);
      if (e != cudaSuccess) return cuda_fail(e, "publish kernel launch");
    }
    return DV_OK;
  }
  // 32-byte vectors when every address and stride allows it.
  uint64_t orall = (uint64_t)(uintptr_t)p.src | (uint64_t)(uintptr_t)p.dst | p.run_bytes;
  for (int k = 0; k < 4; ++k) orall |= (uint64_t)p.ss[k] | (uint64_t)p.ds[k];
  if (orall % 16) return fail(DV_EALIGN, "copy plan not 16-byte aligned");
  const int VEC = (orall % 32 == 0 && tune().vec != 16) ? 32 : 16;
  const uint64_t vpr = p.run_bytes / VEC;
  if (vpr >= (1ull << 31)) return fail(DV_ENOTSUP, "run of %llu bytes too long", (unsigned long long)p.run_bytes);
  for (int k = 1; k < 4; ++k)
    if (p.n[k] >= (1u << 31)) return fail(DV_ENOTSUP, "copy extent too large");
  if (p.runs() >= (1ull << 31)) return fail(DV_ENOTSUP, "too many runs");

  KParams kp{};
  kp.src = p.src;
  kp.dst = p.dst;
  kp.ss0 = p.ss[0]; kp.ss1 = p.ss[1]; kp.ss2 = p.ss[2]; kp.ss3 = p.ss[3];
  kp.ds0 = p.ds[0]; kp.ds1 = p.ds[1]; kp.ds2 = p.ds[2]; kp.ds3 = p.ds[3];
  kp.fv = to_dev(make_fastdiv((uint32_t)vpr));
  kp.f3 = to_dev(make_fastdiv(p.n[3]));
  kp.f2 = to_dev(make_fastdiv(p.n[2]));
  kp.f1 = to_dev(make_fastdiv(p.n[1]));

  // Split into launches of < 2^31 vectors at run boundaries.
  const uint64_t runs_per_launch = std::max<uint64_t>(1, ((1ull << 31) - 1) / vpr);
  for (uint64_t q0 = q_first; q0 < q_last; q0 += runs_per_launch) {
    const uint64_t nq = std::min(runs_per_launch, q_last - q0);
    const bool last = q0 + nq == q_last;
    kp.q_begin = (uint32_t)q0;
    kp.n_vec = (uint32_t)(nq * vpr);
    kp.flag = last ? rel.flag : nullptr;
    kp.seq = rel.seq;
    kp.ticket = rel.ticket;
    kp.ts = last ? rel.ts : nullptr;
    cudaError_t e = launch_cfg(kp, VEC, max_ctas, stream);
    if (e != cudaSuccess) return cuda_fail(e, "copy kernel launch");
  }
  return DV_OK;
}

}  // namespace dv
