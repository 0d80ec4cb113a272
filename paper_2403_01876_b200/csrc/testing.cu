// Test-only kernels (include/dv_testing.h): synthetic KV writer with the kvgen generator, spin.
#include "../../include/dv_device.cuh"
#include "../../include/dv_testing.h"
#include "dv_internal.h"

#include <algorithm>

namespace dv {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct FillParams {
  uint16_t* k;
  uint16_t* v;
  int64_t s_l, s_r, s_h;  // element strides of the cache
  int32_t lb, rb, hb;     // cache layer_begin / req_begin / head_begin
  int32_t l0, r0, s0, h0; // region origin (global ids)
  int32_t nR, H, n, D;    // region extents (H = heads in the region)
  int32_t S;              // cache max_seq
  int32_t ft6d;           // K in FasterTransformer 6-D layout [..][D/x][S][x]
  int32_t kind;
  uint64_t seedmix;
  int32_t box[5];
  int32_t vlo, vhi;
  unsigned long long* t_end;  // optional: max over CTAs of %globaltimer after their stores
  uint64_t* ring;             // optional: a dv_engine doorbell the last CTA rings (dvt_fill_ring)
  uint64_t ring_step;
  unsigned int* ticket;       // CTA counter for the last-CTA ring (zero between uses)
};

// The generator's word at global coordinate (kv, l, r, h, s, d) (kvgen.hash_words / uid / const).
__device__ __forceinline__ uint16_t gen_word(const FillParams& p, int kv, int l, int r, int h, int s,
                                             int d) {
  if (s < p.vlo || s >= p.vhi) return 0xFFFE;
  if (p.kind == DVT_FILL_HASH) {
    const uint64_t key = ((uint64_t)kv << 62) | ((uint64_t)l << 52) | ((uint64_t)r << 40) |
                         ((uint64_t)h << 30) | ((uint64_t)s << 10) | (uint64_t)d;
    return (uint16_t)(splitmix64(key ^ p.seedmix) >> 48);
  }
  if (p.kind == DVT_FILL_UID)
    return (uint16_t)((((((int64_t)kv * p.box[0] + l) * p.box[1] + r) * p.box[2] + h) * p.box[3] +
                       s) * p.box[4] + d);
  return (uint16_t)p.seedmix;
}

__global__ void k_fill(const FillParams p) {
  // Behave like a PDL-aware producer (an attention kernel would do the same): let the dependent
  // streaming kernel be scheduled now; it still waits (griddepcontrol.wait) for our memory.
  asm volatile("griddepcontrol.launch_dependents;");
  // blockIdx.x = slab (l, r, h) of the region, blockIdx.y = kv
  uint32_t slab = blockIdx.x;
  const int h = p.h0 + (int)(slab % p.H);  // global head id
  slab /= p.H;
  const int r = p.r0 + (int)(slab % p.nR);
  const int l = p.l0 + (int)(slab / p.nR);
  const int kv = blockIdx.y;
  uint16_t* base = (kv ? p.v : p.k) + (int64_t)(l - p.lb) * p.s_l + (int64_t)(r - p.rb) * p.s_r +
                   (int64_t)(h - p.hb) * p.s_h;
  const bool ft = p.ft6d && kv == 0;
  const int64_t words = (int64_t)p.n * p.D;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) {
    const int s = p.s0 + (int)(i / p.D);
    const int d = (int)(i % p.D);
    const uint16_t w = gen_word(p, kv, l, r, h, s, d);
    if (ft)  // x = 8 16-bit words per 16-byte packet
      base[((int64_t)(d >> 3) * p.S + s) * 8 + (d & 7)] = w;
    else
      base[(int64_t)s * p.D + d] = w;
  }
  if (p.t_end) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(p.t_end, t);
    }
  }
  if (p.ring) {   // a producer ringing the engine itself: the last CTA, after every CTA's stores
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      const unsigned prev = atomicAdd(p.ticket, 1u);
      if (prev == gridDim.x * gridDim.y - 1) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        *p.ticket = 0u;
        dv_engine_ring(p.ring, p.ring_step);
      }
    }
  }
}

// Vectorised producer (dvt_fill_rows): the generator's words of the region with 16-byte stores,
// one CTA per (slab, kv); with a device plan it also stores every row of the plan's region to the
// plan's destination and releases the plan's flag from its last CTA (the stream-out fused into
// the producer, include/dv_device.cuh).
struct RowsParams {
  FillParams f;
  dv_dplan_set plans;   // n == 0: no plan
  int32_t step;
  int64_t slabs;        // (layer, request, head) slabs of the region
  unsigned long long* t_start;
};
__global__ void k_fill_rows(const RowsParams rp) {
  asm volatile("griddepcontrol.launch_dependents;");
  const FillParams& p = rp.f;
  if (rp.t_start && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(rp.t_start, t);
  }
  // grid-stride over every 16-byte chunk of the region: (kv, slab, position, chunk), chunk fastest
  const int cpr = p.D / 8;   // 16-byte chunks per row
  const int64_t per_slab = (int64_t)p.n * cpr;
  const int64_t total = 2 * rp.slabs * per_slab;
  // (32-bit index math: the host keeps total < 2^32)
  const uint32_t ps32 = (uint32_t)per_slab, slabs32 = (uint32_t)rp.slabs;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (uint32_t)total; i += gridDim.x * blockDim.x) {
    const uint32_t ks = i / ps32;                 // kv * slabs + slab
    const uint32_t in_slab = i - ks * ps32;
    const int kv = (int)(ks / slabs32);
    uint32_t slab = ks - (uint32_t)kv * slabs32;
    const int h = p.h0 + (int)(slab % (uint32_t)p.H);
    slab /= (uint32_t)p.H;
    const int r = p.r0 + (int)(slab % (uint32_t)p.nR);
    const int l = p.l0 + (int)(slab / (uint32_t)p.nR);
    const int s = p.s0 + (int)(in_slab / (uint32_t)cpr);
    const int d0 = (int)(in_slab % (uint32_t)cpr) * 8;
    uint16_t* base = (kv ? p.v : p.k) + (int64_t)(l - p.lb) * p.s_l + (int64_t)(r - p.rb) * p.s_r +
                     (int64_t)(h - p.hb) * p.s_h;
    uint32_t w[4];
    if (p.kind == DVT_FILL_UID && s >= p.vlo && s < p.vhi) {   // the uid of d0, then + 1 per word
      const uint32_t u0 = (uint32_t)gen_word(p, kv, l, r, h, s, d0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = ((u0 + 2 * j) & 0xFFFFu) | (((u0 + 2 * j + 1) & 0xFFFFu) << 16);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = (uint32_t)gen_word(p, kv, l, r, h, s, d0 + 2 * j) |
               ((uint32_t)gen_word(p, kv, l, r, h, s, d0 + 2 * j + 1) << 16);
    }
    const uint4 v = make_uint4(w[0], w[1], w[2], w[3]);
    if (p.ft6d && kv == 0)   // the producer's own FT6D key: packet d0/8 of position s, S*16 bytes apart
      *reinterpret_cast<uint4*>(base + ((int64_t)(d0 >> 3) * p.S + s) * 8) = v;
    else
      *reinterpret_cast<uint4*>(base + (int64_t)s * p.D + d0) = v;
    if (rp.plans.n) {   // packet d0/8 of the row (FT6D-key destinations: packets S*16 bytes apart)
      uint8_t* dst = dv_dplan_set_packet(&rp.plans, rp.step, kv, l, r, h, s, d0 / 8);
      if (dst) *reinterpret_cast<uint4*>(dst) = v;
    }
  }
  if (p.t_end) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(p.t_end, t);
    }
  }
  if (rp.plans.n) dv_dplan_set_release(&rp.plans, rp.step, gridDim.x);
}

// Verifier: counts the words of a region that differ from the generator. Cache form (wire == NULL):
// the same slab walk and addressing as k_fill. Wire form: the canonical wire [l][kv][r][h][s][d]
// of the region, dense, at `wire` (device or mapped pinned host memory).
__global__ void k_verify(const FillParams p, const uint16_t* wire, unsigned long long* bad) {
  uint32_t slab = blockIdx.x;
  const int hi = (int)(slab % p.H);
  slab /= p.H;
  const int ri = (int)(slab % p.nR);
  const int li = (int)(slab / p.nR);
  const int h = p.h0 + hi, r = p.r0 + ri, l = p.l0 + li;
  const int kv = blockIdx.y;
  const int64_t words = (int64_t)p.n * p.D;
  const uint16_t* base;
  if (wire)
    base = wire + ((((int64_t)li * 2 + kv) * p.nR + ri) * p.H + hi) * words;
  else
    base = (kv ? p.v : p.k) + (int64_t)(l - p.lb) * p.s_l + (int64_t)(r - p.rb) * p.s_r +
           (int64_t)(h - p.hb) * p.s_h;
  const bool ft = !wire && p.ft6d && kv == 0;
  unsigned long long n_bad = 0;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) {
    const int si = (int)(i / p.D);
    const int s = p.s0 + si;
    const int d = (int)(i % p.D);
    const uint16_t got = wire ? base[i]
                         : ft ? base[((int64_t)(d >> 3) * p.S + s) * 8 + (d & 7)]
                              : base[(int64_t)s * p.D + d];
    n_bad += got != gen_word(p, kv, l, r, h, s, d);
  }
  if (n_bad) atomicAdd(bad, n_bad);
}

__global__ void k_spin(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// One thread watches a 64-bit seq flag (device or mapped pinned host memory) with system-scope
// acquire loads and stamps %globaltimer the first time it reads >= seq0 + i, for i = 0..n-1:
// "the flag became visible to an independent observer" (for a host flag every poll is a PCIe
// read, so a stamp includes up to one read round trip). Gives up after timeout_ns.
__global__ void k_watch(const unsigned long long* flag, unsigned long long seq0, int32_t n,
                        unsigned long long* ts, unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int32_t i = 0; i < n; ++i) {
    for (;;) {
      const unsigned long long v = dv_flag_load((const uint64_t*)flag);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (v >= seq0 + (unsigned long long)i) break;
      if (t - t0 > timeout_ns) return;
    }
    ts[i] = t;
  }
}

// An in-kernel consumer (A5's second form, include/dv_device.cuh): thread 0 acquires the flag
// (dv_flag_wait), the CTA synchronises, then every thread copies the released payload. *ok = 0
// if the wait timed out.
__global__ void k_consume(const uint64_t* flag, uint64_t seq, const uint4* src, uint4* dst,
                          uint64_t n16, uint64_t timeout_ns, int32_t* ok) {
  __shared__ int got;
  if (threadIdx.x == 0) got = dv_flag_wait(flag, seq, timeout_ns);
  __syncthreads();
  if (!got) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *ok = 0;
    return;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    dst[i] = v;
  }
}

}  // namespace dv

using namespace dv;

// FillParams of `region` (NULL = whole cache) of cache `c`; *slabs = (l, r, h) slabs in it.
static dv_status fill_params(const dv_cache* c, int32_t kind, uint64_t seed, const int32_t* box,
                             int32_t valid_begin, int32_t valid_end, const dv_region* region,
                             FillParams* out, uint64_t* slabs) {
  DV_TRY(check_cache(c, "cache"));
  if (c->elem_bytes != 2) return fail(DV_ENOTSUP, "dvt_fill supports 16-bit words only");
  dv_region whole{c->layer_begin, c->layer_begin + c->n_layers, c->req_begin,
                  c->req_begin + c->n_reqs, 0, c->max_seq, 0, 0};
  const dv_region rr = resolve_heads(region ? region : &whole, c);
  const dv_region* r = &rr;
  DV_TRY(check_region_shape(r));
  DV_TRY(check_cache_holds(c, r, "cache"));
  if (kind == DVT_FILL_UID && !box) return fail(DV_EINVAL, "uid fill needs a box");
  FillParams p{};
  p.k = (uint16_t*)c->k;
  p.v = (uint16_t*)c->v;
  p.s_h = (int64_t)c->max_seq * c->head_dim;
  p.s_r = p.s_h * c->n_heads;
  p.s_l = p.s_r * c->n_reqs;
  p.lb = c->layer_begin;
  p.rb = c->req_begin;
  p.hb = c->head_begin;
  p.l0 = r->layer_begin;
  p.r0 = r->req_begin;
  p.h0 = r->head_begin;
  p.s0 = r->pos_begin;
  p.nR = r->req_end - r->req_begin;
  p.H = r->head_end - r->head_begin;
  p.S = c->max_seq;
  p.ft6d = c->layout == DV_LAYOUT_FT6D;
  p.n = r->pos_end - r->pos_begin;
  p.D = c->head_dim;
  p.kind = kind;
  p.seedmix = kind == DVT_FILL_CONST ? seed : seed * 0xD1B54A32D192ED03ull;
  if (box)
    for (int i = 0; i < 5; ++i) p.box[i] = box[i];
  p.vlo = valid_begin;
  p.vhi = valid_end;
  *slabs = p.n ? (uint64_t)(r->layer_end - r->layer_begin) * p.nR * p.H : 0;
  if (*slabs >= (1ull << 31)) return fail(DV_ENOTSUP, "region too large for dvt_fill / dvt_verify");
  *out = p;
  return DV_OK;
}

extern "C" dv_status dvt_fill(const dv_cache* c, int32_t kind, uint64_t seed, const int32_t* box,
                              int32_t valid_begin, int32_t valid_end, const dv_region* region,
                              uint64_t* t_end, void* stream) {
  FillParams p;
  uint64_t slabs;
  DV_TRY(fill_params(c, kind, seed, box, valid_begin, valid_end, region, &p, &slabs));
  p.t_end = (unsigned long long*)t_end;
  if (!slabs) return DV_OK;
  const int threads = p.n * p.D >= 256 ? 256 : 128;
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)slabs, 2);
  cfg.blockDim = dim3(threads);
  cfg.stream = (cudaStream_t)stream;
  DV_CUDA(cudaLaunchKernelEx(&cfg, k_fill, p));
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_fill_ring(const dv_cache* c, uint64_t seed, const dv_region* region,
                                   uint64_t* t_end, uint64_t* doorbell, uint64_t step,
                                   uint32_t* ticket, void* stream) {
  if (!doorbell || !ticket) return fail(DV_EINVAL, "NULL doorbell or ticket");
  FillParams p;
  uint64_t slabs;
  DV_TRY(fill_params(c, DVT_FILL_HASH, seed, nullptr, 0, 1 << 30, region, &p, &slabs));
  p.t_end = (unsigned long long*)t_end;
  p.ring = doorbell;
  p.ring_step = step;
  p.ticket = ticket;
  if (!slabs) return fail(DV_EINVAL, "empty region");
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)slabs, 2);
  cfg.blockDim = dim3(p.n * p.D >= 256 ? 256 : 128);
  cfg.stream = (cudaStream_t)stream;
  DV_CUDA(cudaLaunchKernelEx(&cfg, k_fill, p));
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_fill_rows(const dv_cache* c, int32_t kind, uint64_t seed, const int32_t* box,
                                   const dv_region* region, const dv_dplan* plans, int32_t n_plans, int32_t step,
                                   uint64_t* t_start, uint64_t* t_end, void* stream) {
  RowsParams rp{};
  uint64_t slabs;
  DV_TRY(fill_params(c, kind, seed, box, 0, 1 << 30, region, &rp.f, &slabs));
  if (c->head_dim % 8) return fail(DV_EALIGN, "dvt_fill_rows needs head_dim %% 8 == 0");
  if (!slabs) return fail(DV_EINVAL, "empty region");
  rp.f.t_end = (unsigned long long*)t_end;
  rp.t_start = (unsigned long long*)t_start;
  if (n_plans < 0 || n_plans > DV_DPLAN_SET_MAX || (n_plans && !plans))
    return fail(DV_EINVAL, "dvt_fill_rows: %d plans (0 .. %d)", n_plans, DV_DPLAN_SET_MAX);
  for (int i = 0; i < n_plans; ++i) {
    if (plans[i].row_bytes != c->head_dim * 2) return fail(DV_EMAP, "plan row size differs from the cache's");
    rp.plans.plan[i] = plans[i];
  }
  rp.plans.n = n_plans;
  rp.step = step;
  rp.slabs = (int64_t)slabs;
  if (2 * (int64_t)slabs * rp.f.n * (c->head_dim / 8) >= (1ll << 32))
    return fail(DV_ENOTSUP, "dvt_fill_rows: region too large for one launch (2^32 chunks)");
  // one thread per 16-byte chunk, 256-thread CTAs, at most 4 CTAs per SM (a producer's grid):
  // few CTAs take part in the plans' release ticket chains
  const int64_t chunks = 2 * (int64_t)slabs * rp.f.n * (c->head_dim / 8);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((chunks + 255) / 256, 4 * (int64_t)nsm));
  (void)cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  DV_CUDA(cudaLaunchKernelEx(&cfg, k_fill_rows, rp));
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_verify(const dv_cache* c, const void* wire, int32_t kind, uint64_t seed,
                                const int32_t* box, int32_t valid_begin, int32_t valid_end,
                                const dv_region* region, uint64_t* mismatches, void* stream) {
  if (!mismatches) return fail(DV_EINVAL, "NULL mismatch counter");
  FillParams p;
  uint64_t slabs;
  DV_TRY(fill_params(c, kind, seed, box, valid_begin, valid_end, region, &p, &slabs));
  if (!slabs) return DV_OK;
  (void)cudaGetLastError();
  k_verify<<<dim3((unsigned)slabs, 2), p.n * p.D >= 256 ? 256 : 128, 0, (cudaStream_t)stream>>>(
      p, (const uint16_t*)wire, (unsigned long long*)mismatches);
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_watch(const uint64_t* flag, uint64_t seq0, int32_t n, uint64_t* ts,
                               uint64_t timeout_ns, void* stream) {
  if (!flag || !ts || n < 0) return fail(DV_EINVAL, "bad dvt_watch arguments");
  (void)cudaGetLastError();
  k_watch<<<1, 1, 0, (cudaStream_t)stream>>>((const unsigned long long*)flag, seq0, n,
                                             (unsigned long long*)ts, timeout_ns);
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_consume(const uint64_t* flag, uint64_t seq, const void* src, void* dst,
                                 uint64_t bytes, uint64_t timeout_ns, int32_t* ok, void* stream) {
  if (!flag || !src || !dst || !ok || bytes % 16) return fail(DV_EINVAL, "bad dvt_consume arguments");
  (void)cudaGetLastError();
  k_consume<<<4, 256, 0, (cudaStream_t)stream>>>(flag, seq, (const uint4*)src, (uint4*)dst,
                                                 bytes / 16, timeout_ns, ok);
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}

extern "C" dv_status dvt_spin(uint64_t ns, int32_t ctas, void* stream) {
  if (ctas < 1) return fail(DV_EINVAL, "ctas must be >= 1");
  (void)cudaGetLastError();
  k_spin<<<ctas, 128, 0, (cudaStream_t)stream>>>(ns);
  DV_CUDA(cudaGetLastError());
  return DV_OK;
}
