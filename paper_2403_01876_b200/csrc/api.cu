// dvstream C ABI: context, memory, peers, and the three primitive levels of DejaVuLib
// (Table 1) on top of the run-copy kernel (copy_kernels.cu) and the route
// planner (route.cpp).
#include <cuda.h>
#include <limits.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "dv_internal.h"

namespace dv {

// ---------------------------------------------------------------------------------------------
// driver entry points (stream memory operations, address ranges) via the runtime
// ---------------------------------------------------------------------------------------------
static Driver g_drv;
static std::once_flag g_drv_once;
static dv_status g_drv_status = DV_OK;
static std::string g_drv_err;

dv_status driver(const Driver** out) {
  std::call_once(g_drv_once, [] {
    struct E {
      const char* name;
      void** slot;
    } es[] = {
        {"cuStreamWaitValue64", (void**)&g_drv.streamWaitValue64},
        {"cuStreamWriteValue64", (void**)&g_drv.streamWriteValue64},
        {"cuMemGetAddressRange", (void**)&g_drv.memGetAddressRange},
        {"cuGetErrorString", (void**)&g_drv.getErrorString},
    };
    for (auto& e : es) {
      cudaDriverEntryPointQueryResult q;
      cudaError_t r = cudaGetDriverEntryPointByVersion(e.name, e.slot, 12000, cudaEnableDefault, &q);
      if (r != cudaSuccess || q != cudaDriverEntryPointSuccess || !*e.slot) {
        g_drv_status = DV_ECUDA;
        g_drv_err = std::string("cannot resolve driver entry point ") + e.name + ": " +
                    cudaGetErrorString(r);
        return;
      }
    }
  });
  if (g_drv_status != DV_OK) return fail(g_drv_status, "%s", g_drv_err.c_str());
  *out = &g_drv;
  return DV_OK;
}

static dv_status drv_fail(int r, const char* what) {
  const char* s = "?";
  if (g_drv.getErrorString) g_drv.getErrorString(r, &s);
  return fail(DV_ECUDA, "%s: CUresult %d (%s)", what, r, s);
}

// Keeps the calling thread's current device unchanged across a call on ctx->device.
struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) {
      err = cudaSetDevice(dev);
      switched = err == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};
#define DV_ON_DEVICE(dev)                                              \
  DeviceGuard _guard(dev);                                             \
  if (_guard.err != cudaSuccess) return cuda_fail(_guard.err, "select device")

// ---------------------------------------------------------------------------------------------
// staging pool
// ---------------------------------------------------------------------------------------------
dv_status Staging::init(int device, uint64_t bytes) {
  (void)device;
  cap_ = (bytes + 255) & ~255ull;
  head_ = 0;
  DV_CUDA(cudaMalloc(&base_, cap_));
  return DV_OK;
}

void Staging::destroy() {
  for (auto& r : recs_) cudaEventDestroy(r.ev);
  for (auto e : free_ev_) cudaEventDestroy(e);
  recs_.clear();
  free_ev_.clear();
  if (base_) cudaFree(base_);
  base_ = nullptr;
}

dv_status Staging::acquire(uint64_t n, cudaStream_t stream, uint8_t** out, uint64_t* off) {
  std::lock_guard<std::mutex> lk(mu_);
  n = (n + 255) & ~255ull;
  if (n > cap_) return fail(DV_ENOMEM, "staging request %llu > pool %llu", (unsigned long long)n,
                            (unsigned long long)cap_);
  if (head_ + n > cap_) head_ = 0;
  const uint64_t a = head_, b = head_ + n;
  // records are in allocation order; wait for (and retire) every one overlapping [a, b)
  for (auto it = recs_.begin(); it != recs_.end();) {
    if (it->off < b && a < it->off + it->len) {
      cudaError_t e = cudaStreamWaitEvent(stream, it->ev, 0);
      if (e != cudaSuccess) return cuda_fail(e, "staging wait");
      free_ev_.push_back(it->ev);
      it = recs_.erase(it);
    } else {
      ++it;
    }
  }
  head_ = b;
  *out = base_ + a;
  *off = a;
  return DV_OK;
}

dv_status Staging::release(uint64_t off, uint64_t n, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(mu_);
  n = (n + 255) & ~255ull;
  cudaEvent_t ev;
  if (!free_ev_.empty()) {
    ev = free_ev_.back();
    free_ev_.pop_back();
  } else {
    DV_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  DV_CUDA(cudaEventRecord(ev, stream));
  recs_.push_back(Rec{off, n, ev});
  return DV_OK;
}

// ---------------------------------------------------------------------------------------------
// descriptors -> copy plans
// ---------------------------------------------------------------------------------------------
// One side of a copy: address of word (l0, r0, h=0, s0, d=0) of K, and byte strides.
struct Side {
  const uint8_t* base;
  int64_t s_kv, s_l, s_r, s_h;
};

static Side cache_side(const dv_cache* c, const dv_region* r) {
  const int64_t row = (int64_t)c->head_dim * c->elem_bytes;
  const int64_t sh = (int64_t)c->max_seq * row;
  const int64_t sr = (int64_t)c->n_heads * sh;
  const int64_t sl = (int64_t)c->n_reqs * sr;
  const int64_t off = (int64_t)(r->layer_begin - c->layer_begin) * sl +
                      (int64_t)(r->req_begin - c->req_begin) * sr + (int64_t)r->pos_begin * row;
  Side s;
  s.base = (const uint8_t*)c->k + off;
  s.s_kv = (int64_t)((const uint8_t*)c->v - (const uint8_t*)c->k);
  s.s_l = sl;
  s.s_r = sr;
  s.s_h = sh;
  return s;
}

// Canonical wire chunk [l][kv][r][h][s][d] of a region (reading Q3).
static Side wire_side(const uint8_t* w, const dv_region* r, int32_t H, int64_t run) {
  const int64_t nR = r->req_end - r->req_begin;
  Side s;
  s.base = w;
  s.s_h = run;
  s.s_r = (int64_t)H * run;
  s.s_kv = nR * s.s_r;
  s.s_l = 2 * s.s_kv;
  return s;
}

enum Order { ORDER_WIRE /* [l][kv][r][h] */, ORDER_KV_OUTER /* [kv][l][r][h] */ };

static CopyPlan make_plan(const Side& s, const Side& d, const dv_region* r, int32_t H, int64_t run,
                          Order order) {
  CopyPlan p{};
  p.src = s.base;
  p.dst = (uint8_t*)d.base;
  const uint32_t nL = r->layer_end - r->layer_begin, nR = r->req_end - r->req_begin;
  p.n[0] = 1;
  if (order == ORDER_WIRE) {
    p.n[1] = nL; p.ss[1] = s.s_l;  p.ds[1] = d.s_l;
    p.n[2] = 2;  p.ss[2] = s.s_kv; p.ds[2] = d.s_kv;
  } else {
    p.n[1] = 2;  p.ss[1] = s.s_kv; p.ds[1] = d.s_kv;
    p.n[2] = nL; p.ss[2] = s.s_l;  p.ds[2] = d.s_l;
  }
  p.n[3] = nR; p.ss[3] = s.s_r; p.ds[3] = d.s_r;
  p.n[4] = H;  p.ss[4] = s.s_h; p.ds[4] = d.s_h;
  p.run_bytes = (uint64_t)run;
  collapse(p);
  return p;
}

static uint64_t region_bytes(const dv_region* r, const dv_cache* c) {
  return 2ull * (uint64_t)(r->layer_end - r->layer_begin) * (uint64_t)(r->req_end - r->req_begin) *
         (uint64_t)(r->pos_end - r->pos_begin) * (uint64_t)c->n_heads * (uint64_t)c->head_dim *
         (uint64_t)c->elem_bytes;
}

static int64_t run_bytes(const dv_region* r, const dv_cache* c) {
  return (int64_t)(r->pos_end - r->pos_begin) * c->head_dim * c->elem_bytes;
}

static dv_status check_ep(const dv_endpoint* ep, uint64_t off, uint64_t bytes, int32_t slot,
                          bool use_flag, const char* name) {
  if (!ep) return fail(DV_EINVAL, "%s: NULL endpoint", name);
  if (ep->kind != DV_EP_DEVICE && ep->kind != DV_EP_HOST && ep->kind != DV_EP_PEER)
    return fail(DV_EINVAL, "%s: bad endpoint kind %d", name, ep->kind);
  if (!ep->base && bytes) return fail(DV_EINVAL, "%s: NULL endpoint base", name);
  if (((uintptr_t)ep->base | off) % 16)
    return fail(DV_EALIGN, "%s: endpoint base/offset not 16-byte aligned", name);
  if (off > ep->bytes || bytes > ep->bytes - off)
    return fail(DV_EINVAL, "%s: [%llu, +%llu) exceeds endpoint capacity %llu", name,
                (unsigned long long)off, (unsigned long long)bytes, (unsigned long long)ep->bytes);
  if (use_flag && slot >= 0) {
    if (!ep->flags || slot >= ep->n_flags)
      return fail(DV_EINVAL, "%s: flag slot %d but endpoint has %d flags", name, slot, ep->n_flags);
    if ((uintptr_t)ep->flags % 8) return fail(DV_EALIGN, "%s: flags not 8-byte aligned", name);
  }
  return DV_OK;
}

static dv_status check_ctx(dv_ctx* ctx) {
  if (!ctx) return fail(DV_EINVAL, "NULL context");
  return DV_OK;
}

static Release ticket_release(dv_ctx* ctx, const dv_endpoint* ep, int32_t slot, uint64_t seq,
                              bool use_flag) {
  Release r{nullptr, 0, nullptr};
  if (use_flag && slot >= 0 && ep && ep->flags) {
    r.flag = (unsigned long long*)&ep->flags[slot];
    r.seq = seq;
    r.ticket = ctx->tickets + (ctx->next_ticket.fetch_add(1) % dv_ctx::kTickets);
    r.ts = ctx->trace_ts;
  }
  return r;
}

static dv_status stream_signal(const dv_endpoint* ep, int32_t slot, uint64_t seq,
                               cudaStream_t stream) {
  const Driver* d;
  DV_TRY(driver(&d));
  int r = d->streamWriteValue64(stream, (unsigned long long)(uintptr_t)&ep->flags[slot], seq,
                                CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r) return drv_fail(r, "cuStreamWriteValue64");
  return DV_OK;
}

static dv_status stream_wait(const dv_endpoint* ep, int32_t slot, uint64_t seq,
                             cudaStream_t stream) {
  const Driver* d;
  DV_TRY(driver(&d));
  int r = d->streamWaitValue64(stream, (unsigned long long)(uintptr_t)&ep->flags[slot], seq,
                               CU_STREAM_WAIT_VALUE_GEQ);
  if (r) return drv_fail(r, "cuStreamWaitValue64");
  return DV_OK;
}

// One fused kernel, then the flag: by the kernel itself (fenced st.release.sys from the last CTA)
// or, with DV_PUBLISH_STREAMOP, by a stream memory operation after it.
static dv_status launch_publish(dv_ctx* ctx, const CopyPlan& p, const dv_endpoint* ep, int32_t slot,
                                uint64_t seq, bool use_flag, uint32_t xfer, cudaStream_t st) {
  const bool streamop = (xfer & DV_PUBLISH_STREAMOP) != 0;
  const Release none{nullptr, 0, nullptr};
  DV_TRY(launch_copy(p, 0, p.runs(), streamop ? none : ticket_release(ctx, ep, slot, seq, use_flag),
                     ctx->max_ctas, st));
  if (streamop && use_flag) DV_TRY(stream_signal(ep, slot, seq, st));
  return DV_OK;
}

// Chooses FUSED or STAGED for a data call (measured in
// profiles/r01_tune_host*.jsonl): writes to pinned host go through the kernel's own PCIe stores
// (same throughput as pack+DMA, lower latency, no staging); reads from pinned host go through the
// copy engine (SM zero-copy reads do not overlap with concurrent D2H traffic).
static uint32_t pick_xfer(uint32_t xfer, const dv_endpoint* ep, uint64_t bytes, bool reading) {
  uint32_t m = xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  if (m == DV_XFER_FUSED || m == DV_XFER_STAGED) {
    if (m == DV_XFER_STAGED && ep->kind == DV_EP_DEVICE) return DV_XFER_FUSED;  // already local
    return m;
  }
  if (ep->kind == DV_EP_HOST && reading) return DV_XFER_STAGED;
  (void)bytes;
  return DV_XFER_FUSED;
}

// ---- scatter / gather / remap bodies (validated inputs) -------------------------------------
struct ScatterOp {
  const dv_cache* src;
  dv_region reg;
  const dv_endpoint* dst;
  uint64_t dst_off;
  int32_t slot;
  uint64_t seq;
  uint32_t xfer;
};

static dv_status scatter_check(dv_ctx* ctx, const ScatterOp& op) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_cache(op.src, "source"));
  DV_TRY(check_region_shape(&op.reg));
  DV_TRY(check_cache_holds(op.src, &op.reg, "source"));
  const bool use_flag = !(op.xfer & DV_NO_FLAG);
  return check_ep(op.dst, op.dst_off, region_bytes(&op.reg, op.src), op.slot, use_flag,
                  "destination");
}

static dv_status scatter_run(dv_ctx* ctx, const ScatterOp& op, cudaStream_t st) {
  const dv_cache* c = op.src;
  const uint64_t bytes = region_bytes(&op.reg, c);
  const int64_t run = run_bytes(&op.reg, c);
  const bool use_flag = !(op.xfer & DV_NO_FLAG) && op.slot >= 0;
  const uint32_t mode = pick_xfer(op.xfer, op.dst, bytes, false);
  uint8_t* wire = (uint8_t*)op.dst->base + op.dst_off;
  if (mode == DV_XFER_FUSED) {
    CopyPlan p = make_plan(cache_side(c, &op.reg), wire_side(wire, &op.reg, c->n_heads, run),
                           &op.reg, c->n_heads, run, ORDER_WIRE);
    return launch_publish(ctx, p, op.dst, op.slot, op.seq, use_flag, op.xfer, st);
  }
  // STAGED: pack chunks of runs into staging, copy engine moves each chunk.
  if (bytes) {
    CopyPlan p = make_plan(cache_side(c, &op.reg), wire_side(wire, &op.reg, c->n_heads, run),
                           &op.reg, c->n_heads, run, ORDER_WIRE);
    const uint64_t rb = p.run_bytes, runs = p.runs();
    const uint64_t chunk = std::max<uint64_t>(1, (ctx->staging.capacity() / 2) / rb);
    if (rb > ctx->staging.capacity() / 2)
      return fail(DV_ENOMEM, "run of %llu bytes exceeds half the staging pool",
                  (unsigned long long)rb);
    for (uint64_t q0 = 0; q0 < runs; q0 += chunk) {
      const uint64_t q1 = std::min(runs, q0 + chunk), nb = (q1 - q0) * rb;
      uint8_t* stg;
      uint64_t off;
      DV_TRY(ctx->staging.acquire(nb, st, &stg, &off));
      CopyPlan pc = p;
      pc.dst = stg - q0 * rb;  // run q lands at stg + (q - q0) * rb (wire side is dense)
      DV_TRY(launch_copy(pc, q0, q1, Release{nullptr, 0, nullptr}, ctx->max_ctas, st));
      DV_DMA(cudaMemcpyAsync(wire + q0 * rb, stg, nb, cudaMemcpyDefault, st));
      DV_TRY(ctx->staging.release(off, nb, st));
    }
  }
  if (use_flag) DV_TRY(stream_signal(op.dst, op.slot, op.seq, st));
  return DV_OK;
}

struct GatherOp {
  const dv_endpoint* src;
  uint64_t src_off;
  int32_t slot;
  uint64_t wait_seq;
  const dv_cache* dst;
  dv_region reg;
  uint32_t xfer;
};

static dv_status gather_check(dv_ctx* ctx, const GatherOp& op) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_cache(op.dst, "destination"));
  DV_TRY(check_region_shape(&op.reg));
  DV_TRY(check_cache_holds(op.dst, &op.reg, "destination"));
  const bool use_flag = !(op.xfer & DV_NO_FLAG);
  return check_ep(op.src, op.src_off, region_bytes(&op.reg, op.dst), op.slot, use_flag, "source");
}

// Runs an unpack plan whose source side is a dense wire chunk at `wire` (run q at wire + q*run):
// FUSED = one kernel reading the endpoint memory directly; STAGED = the copy engine brings chunks
// of runs into HBM staging, the kernel unpacks each chunk.
static dv_status unpack_plan(dv_ctx* ctx, const CopyPlan& p, const uint8_t* wire, uint32_t mode,
                             cudaStream_t st) {
  const Release none{nullptr, 0, nullptr};
  if (mode == DV_XFER_FUSED) return launch_copy(p, 0, p.runs(), none, ctx->max_ctas, st);
  const uint64_t rb = p.run_bytes, runs = p.runs();
  if (rb > ctx->staging.capacity() / 2)
    return fail(DV_ENOMEM, "run of %llu bytes exceeds half the staging pool",
                (unsigned long long)rb);
  const uint64_t chunk = std::max<uint64_t>(1, (ctx->staging.capacity() / 2) / rb);
  for (uint64_t q0 = 0; q0 < runs; q0 += chunk) {
    const uint64_t q1 = std::min(runs, q0 + chunk), nb = (q1 - q0) * rb;
    uint8_t* stg;
    uint64_t off;
    DV_TRY(ctx->staging.acquire(nb, st, &stg, &off));
    DV_DMA(cudaMemcpyAsync(stg, wire + q0 * rb, nb, cudaMemcpyDefault, st));
    CopyPlan pc = p;
    pc.src = stg - q0 * rb;
    DV_TRY(launch_copy(pc, q0, q1, none, ctx->max_ctas, st));
    DV_TRY(ctx->staging.release(off, nb, st));
  }
  return DV_OK;
}

static dv_status gather_run(dv_ctx* ctx, const GatherOp& op, cudaStream_t st) {
  const dv_cache* c = op.dst;
  const uint64_t bytes = region_bytes(&op.reg, c);
  const int64_t run = run_bytes(&op.reg, c);
  if (!(op.xfer & DV_NO_FLAG) && op.slot >= 0 && op.wait_seq)
    DV_TRY(stream_wait(op.src, op.slot, op.wait_seq, st));
  if (!bytes) return DV_OK;
  const uint32_t mode = pick_xfer(op.xfer, op.src, bytes, true);
  const uint8_t* wire = (const uint8_t*)op.src->base + op.src_off;
  CopyPlan p = make_plan(wire_side(wire, &op.reg, c->n_heads, run), cache_side(c, &op.reg),
                         &op.reg, c->n_heads, run, ORDER_WIRE);
  return unpack_plan(ctx, p, wire, mode, st);
}

struct RemapOp {
  const dv_cache* src;
  const dv_cache* dst;
  dv_region reg;
  const dv_endpoint* signal;
  int32_t slot;
  uint64_t seq;
  uint32_t xfer;
};

static dv_status remap_check(dv_ctx* ctx, const RemapOp& op) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_cache(op.src, "source"));
  DV_TRY(check_cache(op.dst, "destination"));
  DV_TRY(check_region_shape(&op.reg));
  DV_TRY(check_cache_holds(op.src, &op.reg, "source"));
  DV_TRY(check_cache_holds(op.dst, &op.reg, "destination"));
  if (op.src->n_heads != op.dst->n_heads || op.src->head_dim != op.dst->head_dim ||
      op.src->elem_bytes != op.dst->elem_bytes)
    return fail(DV_EMAP, "source and destination caches differ in heads/head_dim/elem_bytes");
  if (op.signal && !(op.xfer & DV_NO_FLAG) && op.slot >= 0)
    DV_TRY(check_ep(op.signal, 0, 0, op.slot, true, "signal"));
  return DV_OK;
}

static dv_status remap_run(dv_ctx* ctx, const RemapOp& op, cudaStream_t st) {
  const dv_cache* c = op.src;
  const int64_t run = run_bytes(&op.reg, c);
  const bool use_flag = op.signal && !(op.xfer & DV_NO_FLAG) && op.slot >= 0;
  CopyPlan p = make_plan(cache_side(op.src, &op.reg), cache_side(op.dst, &op.reg), &op.reg,
                         c->n_heads, run, ORDER_KV_OUTER);
  uint32_t m = op.xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  if (m != DV_XFER_FUSED && m != DV_XFER_STAGED)  // AUTO (profiles/r01_configs*.jsonl, C4):
    m = (op.src->device < 0 && op.dst->device >= 0) ? DV_XFER_STAGED : DV_XFER_FUSED;
  if (m == DV_XFER_STAGED && p.runs() && p.run_bytes) {
    // Copy-engine form (paper-style DMA, used for pinned-host mirror arenas): one
    // 2-D copy per (kv, layer, request) over the heads, or one 1-D copy when the heads are
    // contiguous on both sides.
    const Side s = cache_side(op.src, &op.reg), d = cache_side(op.dst, &op.reg);
    const int nL = op.reg.layer_end - op.reg.layer_begin, nR = op.reg.req_end - op.reg.req_begin;
    const int H = c->n_heads;
    const bool flat = s.s_h == run && d.s_h == run;
    for (int kv = 0; kv < 2; ++kv)
      for (int l = 0; l < nL; ++l)
        for (int r = 0; r < nR; ++r) {
          const uint8_t* sp = s.base + kv * s.s_kv + l * s.s_l + r * s.s_r;
          uint8_t* dp = (uint8_t*)d.base + kv * d.s_kv + l * d.s_l + r * d.s_r;
          if (flat || H == 1) {
            DV_DMA(cudaMemcpyAsync(dp, sp, (size_t)run * (flat ? H : 1), cudaMemcpyDefault, st));
          } else {
            DV_DMA(cudaMemcpy2DAsync(dp, (size_t)d.s_h, sp, (size_t)s.s_h, (size_t)run, H,
                                      cudaMemcpyDefault, st));
          }
        }
    if (use_flag) DV_TRY(stream_signal(op.signal, op.slot, op.seq, st));
    return DV_OK;
  }
  return launch_publish(ctx, p, op.signal, op.slot, op.seq, use_flag, op.xfer, st);
}

// ---------------------------------------------------------------------------------------------
// IPC registry
// ---------------------------------------------------------------------------------------------
struct Blob {
  uint32_t magic;
  uint32_t version;
  int32_t pid;
  int32_t device;
  cudaIpcMemHandle_t handle;  // 64 bytes
  uint64_t offset;            // ptr - allocation base
  uint64_t ptr;               // exporter's address (same-process fast path)
};
static_assert(sizeof(Blob) <= sizeof(dv_ipc_blob), "blob too large");
static const uint32_t kBlobMagic = 0x44564950;  // "DVIP"
static std::mutex g_ipc_mu;
static std::map<uintptr_t, std::pair<void*, int>> g_ipc_open;  // mapped -> (base, refcount)

}  // namespace dv

using namespace dv;

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

dv_status dv_create(int32_t device, const dv_config* cfg, dv_ctx** out) {
  if (!out) return fail(DV_EINVAL, "NULL out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(DV_ECUDA, "no CUDA device available (dvstream has no CPU fallback): %s",
                cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(DV_EINVAL, "device %d out of range [0,%d)", device, n);
  const Driver* d;
  DV_TRY(driver(&d));
  DV_ON_DEVICE(device);
  dv_ctx* c = new dv_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  c->max_ctas = (cfg && cfg->max_ctas > 0) ? cfg->max_ctas : c->sm_count * 8;
  uint64_t stg = (cfg && cfg->staging_bytes) ? cfg->staging_bytes : (256ull << 20);
  dv_status s = c->staging.init(device, stg);
  if (s != DV_OK) {
    delete c;
    return s;
  }
  e = cudaMalloc(&c->tickets, sizeof(unsigned int) * dv_ctx::kTickets);
  if (e == cudaSuccess) e = cudaMemset(c->tickets, 0, sizeof(unsigned int) * dv_ctx::kTickets);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    c->staging.destroy();
    delete c;
    return cuda_fail(e, "dv_create");
  }
  *out = c;
  return DV_OK;
}

dv_status dv_destroy(dv_ctx* ctx) {
  if (!ctx) return DV_OK;
  {
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    ctx->staging.destroy();
    cudaFree(ctx->tickets);
    cudaStreamDestroy(ctx->aux);
  }
  delete ctx;
  return DV_OK;
}

dv_status dv_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(DV_EINVAL, "NULL out");
  DV_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
  return DV_OK;
}

dv_status dv_host_free(void* p) {
  if (p) DV_CUDA(cudaFreeHost(p));
  return DV_OK;
}

dv_status dv_device_alloc(int32_t device, uint64_t bytes, void** out) {
  if (!out) return fail(DV_EINVAL, "NULL out");
  DV_ON_DEVICE(device);
  DV_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  return DV_OK;
}

dv_status dv_device_free(void* p) {
  if (p) DV_CUDA(cudaFree(p));
  return DV_OK;
}

dv_status dv_ipc_export(const void* ptr, dv_ipc_blob* out) {
  if (!ptr || !out) return fail(DV_EINVAL, "NULL argument");
  const Driver* d;
  DV_TRY(driver(&d));
  cudaPointerAttributes at;
  DV_CUDA(cudaPointerGetAttributes(&at, ptr));
  if (at.type != cudaMemoryTypeDevice) return fail(DV_EPEER, "ipc export: not device memory");
  unsigned long long base = 0;
  size_t size = 0;
  int r = d->memGetAddressRange(&base, &size, (unsigned long long)(uintptr_t)ptr);
  if (r) return drv_fail(r, "cuMemGetAddressRange");
  Blob b{};
  b.magic = kBlobMagic;
  b.version = DV_ABI_VERSION;
  b.pid = (int32_t)getpid();
  b.device = at.device;
  b.offset = (uint64_t)(uintptr_t)ptr - base;
  b.ptr = (uint64_t)(uintptr_t)ptr;
  {
    DeviceGuard g(at.device);
    cudaError_t e = cudaIpcGetMemHandle(&b.handle, (void*)(uintptr_t)base);
    if (e != cudaSuccess) return fail(DV_EPEER, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  memset(out, 0, sizeof *out);
  memcpy(out->bytes, &b, sizeof b);
  return DV_OK;
}

dv_status dv_ipc_open(const dv_ipc_blob* blob, void** out) {
  if (!blob || !out) return fail(DV_EINVAL, "NULL argument");
  Blob b;
  memcpy(&b, blob->bytes, sizeof b);
  if (b.magic != kBlobMagic || b.version != DV_ABI_VERSION)
    return fail(DV_EPEER, "malformed IPC blob");
  if (b.pid == (int32_t)getpid()) {  // same process (loopback peer): the address is valid here
    *out = (void*)(uintptr_t)b.ptr;
    return DV_OK;
  }
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(DV_EPEER, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  void* mapped = (uint8_t*)base + b.offset;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto& ent = g_ipc_open[(uintptr_t)mapped];
  ent.first = base;
  ent.second += 1;
  *out = mapped;
  return DV_OK;
}

dv_status dv_ipc_close(void* mapped) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_open.find((uintptr_t)mapped);
  if (it == g_ipc_open.end()) return DV_OK;  // same-process mapping or already closed
  if (--it->second.second == 0) {
    cudaError_t e = cudaIpcCloseMemHandle(it->second.first);
    g_ipc_open.erase(it);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  }
  return DV_OK;
}

dv_status dv_stats(uint64_t* kernel_launches, uint64_t* dma_calls) {
  if (kernel_launches) *kernel_launches = g_kernel_launches.load();
  if (dma_calls) *dma_calls = g_dma_calls.load();
  return DV_OK;
}

// ---- level 3 --------------------------------------------------------------------------------
dv_status dv_flush(dv_ctx* ctx, const void* src, uint64_t bytes, const dv_endpoint* dst,
                   uint64_t dst_off, int32_t flag_slot, uint64_t seq, uint32_t xfer,
                   void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!src && bytes) return fail(DV_EINVAL, "NULL source");
  const bool use_flag = !(xfer & DV_NO_FLAG) && flag_slot >= 0;
  DV_TRY(check_ep(dst, dst_off, bytes, flag_slot, !(xfer & DV_NO_FLAG), "destination"));
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* d = (uint8_t*)dst->base + dst_off;
  const uint32_t m = xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  if (m == DV_XFER_FUSED && bytes % 16 == 0 && (uintptr_t)src % 16 == 0) {
    CopyPlan p{};
    p.src = (const uint8_t*)src;
    p.dst = d;
    for (int k = 0; k < kDims; ++k) p.n[k] = 1;
    p.run_bytes = bytes;
    // split one long run into 1 MiB runs so the kernel's 32-bit vector index suffices
    if (bytes > (1u << 20) && bytes % (1u << 20) == 0) {
      p.n[kDims - 1] = (uint32_t)(bytes >> 20);
      p.ss[kDims - 1] = p.ds[kDims - 1] = 1 << 20;
      p.run_bytes = 1u << 20;
    }
    return launch_publish(ctx, p, dst, flag_slot, seq, use_flag, xfer, st);
  }
  if (bytes) DV_DMA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyDefault, st));
  if (use_flag) DV_TRY(stream_signal(dst, flag_slot, seq, st));
  return DV_OK;
}

dv_status dv_fetch(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                   uint64_t wait_seq, void* dst, uint64_t bytes, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!dst && bytes) return fail(DV_EINVAL, "NULL destination");
  DV_TRY(check_ep(src, src_off, bytes, flag_slot, !(xfer & DV_NO_FLAG), "source"));
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!(xfer & DV_NO_FLAG) && flag_slot >= 0 && wait_seq)
    DV_TRY(stream_wait(src, flag_slot, wait_seq, st));
  const uint8_t* s = (const uint8_t*)src->base + src_off;
  const uint32_t m = xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  if (m == DV_XFER_FUSED && bytes % 16 == 0 && (uintptr_t)dst % 16 == 0 && bytes) {
    CopyPlan p{};
    p.src = s;
    p.dst = (uint8_t*)dst;
    for (int k = 0; k < kDims; ++k) p.n[k] = 1;
    p.run_bytes = bytes;
    if (bytes > (1u << 20) && bytes % (1u << 20) == 0) {
      p.n[kDims - 1] = (uint32_t)(bytes >> 20);
      p.ss[kDims - 1] = p.ds[kDims - 1] = 1 << 20;
      p.run_bytes = 1u << 20;
    }
    return launch_copy(p, 0, p.runs(), Release{nullptr, 0, nullptr}, ctx->max_ctas, st);
  }
  if (bytes) DV_DMA(cudaMemcpyAsync(dst, s, bytes, cudaMemcpyDefault, st));
  return DV_OK;
}

// ---- level 2 --------------------------------------------------------------------------------
dv_status dv_scatter(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                     const dv_endpoint* dst, uint64_t dst_off, int32_t flag_slot, uint64_t seq,
                     uint32_t xfer, void* stream) {
  if (!region) return fail(DV_EINVAL, "NULL region");
  ScatterOp op{src, *region, dst, dst_off, flag_slot, seq, xfer};
  DV_TRY(scatter_check(ctx, op));
  DV_ON_DEVICE(ctx->device);
  return scatter_run(ctx, op, (cudaStream_t)stream);
}

dv_status dv_gather(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                    uint64_t wait_seq, const dv_cache* dst, const dv_region* region,
                    uint32_t xfer, void* stream) {
  if (!region) return fail(DV_EINVAL, "NULL region");
  GatherOp op{src, src_off, flag_slot, wait_seq, dst, *region, xfer};
  DV_TRY(gather_check(ctx, op));
  DV_ON_DEVICE(ctx->device);
  return gather_run(ctx, op, (cudaStream_t)stream);
}

dv_status dv_gather_chunks(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                           uint64_t wait_seq, const dv_cache* dst, const dv_region* first,
                           int32_t n_chunks, int32_t pos_step, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!first) return fail(DV_EINVAL, "NULL region");
  if (n_chunks < 0) return fail(DV_EINVAL, "negative n_chunks");
  DV_TRY(check_cache(dst, "destination"));
  DV_TRY(check_region_shape(first));
  const int32_t n = first->pos_end - first->pos_begin;
  if (n_chunks > 1 && pos_step < n)
    return fail(DV_EINVAL, "pos_step %d smaller than the chunk's %d positions", pos_step, n);
  dv_region last = *first;
  if (n_chunks > 0) {
    const int64_t shift = (int64_t)(n_chunks - 1) * pos_step;
    if (first->pos_end + shift > INT32_MAX) return fail(DV_ERANGE, "chunk positions overflow");
    last.pos_begin += (int32_t)shift;
    last.pos_end += (int32_t)shift;
  }
  DV_TRY(check_cache_holds(dst, first, "destination"));
  DV_TRY(check_cache_holds(dst, &last, "destination"));
  const uint64_t chunk_bytes = region_bytes(first, dst);
  const uint64_t total = chunk_bytes * (uint64_t)n_chunks;
  DV_TRY(check_ep(src, src_off, total, flag_slot, !(xfer & DV_NO_FLAG), "source"));
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!(xfer & DV_NO_FLAG) && flag_slot >= 0 && wait_seq)
    DV_TRY(stream_wait(src, flag_slot, wait_seq, st));
  if (!total) return DV_OK;
  const int64_t run = run_bytes(first, dst);
  const uint8_t* wire = (const uint8_t*)src->base + src_off;
  // dims [chunk][l][kv][r][h]: the log side is dense in this order
  const Side ws = wire_side(wire, first, dst->n_heads, run);
  const Side cs = cache_side(dst, first);
  CopyPlan p{};
  p.src = ws.base;
  p.dst = (uint8_t*)cs.base;
  p.n[0] = (uint32_t)n_chunks; p.ss[0] = (int64_t)chunk_bytes;
  p.ds[0] = (int64_t)pos_step * dst->head_dim * dst->elem_bytes;
  p.n[1] = first->layer_end - first->layer_begin; p.ss[1] = ws.s_l; p.ds[1] = cs.s_l;
  p.n[2] = 2; p.ss[2] = ws.s_kv; p.ds[2] = cs.s_kv;
  p.n[3] = first->req_end - first->req_begin; p.ss[3] = ws.s_r; p.ds[3] = cs.s_r;
  p.n[4] = dst->n_heads; p.ss[4] = ws.s_h; p.ds[4] = cs.s_h;
  p.run_bytes = (uint64_t)run;
  collapse(p);
  return unpack_plan(ctx, p, wire, pick_xfer(xfer, src, total, true), st);
}

dv_status dv_remap(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst, const dv_region* region,
                   const dv_endpoint* signal, int32_t flag_slot, uint64_t seq, uint32_t xfer,
                   void* stream) {
  if (!region) return fail(DV_EINVAL, "NULL region");
  RemapOp op{src, dst, *region, signal, flag_slot, seq, xfer};
  DV_TRY(remap_check(ctx, op));
  DV_ON_DEVICE(ctx->device);
  return remap_run(ctx, op, (cudaStream_t)stream);
}

// ---- level 1 --------------------------------------------------------------------------------
static dv_status my_pieces(const dv_setup* src_setup, const dv_setup* dst_setup,
                           const dv_region* region, const dv_cache* c, int32_t stage,
                           int32_t micro, bool sender, std::vector<dv_piece>* out) {
  DV_TRY(check_cache(c, sender ? "source" : "destination"));
  std::vector<dv_piece> all;
  DV_TRY(route(src_setup, dst_setup, region, c->n_heads, c->head_dim, c->elem_bytes, &all));
  const dv_setup* mine = sender ? src_setup : dst_setup;
  if (stage < 0 || stage >= mine->n_stages || micro < 0 || micro >= mine->n_micro)
    return fail(DV_EINVAL, "block (%d,%d) not in the %s setup", stage, micro,
                sender ? "source" : "destination");
  out->clear();
  for (auto& p : all)
    if (sender ? (p.src_stage == stage && p.src_micro == micro)
               : (p.dst_stage == stage && p.dst_micro == micro))
      out->push_back(p);
  return DV_OK;
}

dv_status dv_stream_out(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                        const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                        const dv_setup* dst_setup, const dv_endpoint* inboxes, int32_t n_inboxes,
                        uint64_t seq, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, true, &ps));
  if (!inboxes && !ps.empty()) return fail(DV_EINVAL, "NULL inboxes");
  const int32_t slot = my_stage * src_setup->n_micro + my_micro;
  std::vector<ScatterOp> ops;
  for (auto& p : ps) {
    const int32_t k = p.dst_stage * dst_setup->n_micro + p.dst_micro;
    if (k >= n_inboxes) return fail(DV_EINVAL, "inbox %d missing (n_inboxes %d)", k, n_inboxes);
    dv_region r{p.layer_begin, p.layer_end, p.req_begin, p.req_end, p.pos_begin, p.pos_end};
    ScatterOp op{src, r, &inboxes[k], p.dst_wire_off, slot, seq, xfer};
    DV_TRY(scatter_check(ctx, op));  // validate every piece before enqueueing any
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(scatter_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

dv_status dv_stream_in(dv_ctx* ctx, const dv_cache* dst, const dv_region* region,
                       const dv_setup* src_setup, const dv_setup* dst_setup, int32_t my_stage,
                       int32_t my_micro, const dv_endpoint* inbox, uint64_t wait_seq,
                       uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, dst, my_stage, my_micro, false, &ps));
  std::vector<GatherOp> ops;
  for (auto& p : ps) {
    dv_region r{p.layer_begin, p.layer_end, p.req_begin, p.req_end, p.pos_begin, p.pos_end};
    const int32_t slot = p.src_stage * src_setup->n_micro + p.src_micro;
    GatherOp op{inbox, p.dst_wire_off, slot, wait_seq, dst, r, xfer};
    DV_TRY(gather_check(ctx, op));
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(gather_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

dv_status dv_stream_out_direct(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                               const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                               const dv_setup* dst_setup, const dv_cache* dst_caches,
                               const dv_endpoint* signals, int32_t n_dst, uint64_t seq,
                               uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, true, &ps));
  if (!dst_caches && !ps.empty()) return fail(DV_EINVAL, "NULL dst_caches");
  const int32_t slot = my_stage * src_setup->n_micro + my_micro;
  std::vector<RemapOp> ops;
  for (auto& p : ps) {
    const int32_t k = p.dst_stage * dst_setup->n_micro + p.dst_micro;
    if (k >= n_dst) return fail(DV_EINVAL, "destination %d missing (n_dst %d)", k, n_dst);
    dv_region r{p.layer_begin, p.layer_end, p.req_begin, p.req_end, p.pos_begin, p.pos_end};
    RemapOp op{src, &dst_caches[k], r, signals ? &signals[k] : nullptr, slot, seq, xfer};
    DV_TRY(remap_check(ctx, op));
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(remap_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

// ---- completion -----------------------------------------------------------------------------
dv_status dv_wait(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq,
                  void* stream) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_ep(ep, 0, 0, flag_slot, true, "endpoint"));
  if (flag_slot < 0) return fail(DV_EINVAL, "negative flag slot");
  DV_ON_DEVICE(ctx->device);
  return stream_wait(ep, flag_slot, seq, (cudaStream_t)stream);
}

dv_status dv_signal(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq,
                    void* stream) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_ep(ep, 0, 0, flag_slot, true, "endpoint"));
  if (flag_slot < 0) return fail(DV_EINVAL, "negative flag slot");
  DV_ON_DEVICE(ctx->device);
  return stream_signal(ep, flag_slot, seq, (cudaStream_t)stream);
}

dv_status dv_query(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq,
                   int32_t* done) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_ep(ep, 0, 0, flag_slot, true, "endpoint"));
  if (flag_slot < 0 || !done) return fail(DV_EINVAL, "bad flag slot or NULL done");
  cudaPointerAttributes at;
  DV_CUDA(cudaPointerGetAttributes(&at, &ep->flags[flag_slot]));
  uint64_t v;
  if (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered) {
    v = __atomic_load_n(&ep->flags[flag_slot], __ATOMIC_ACQUIRE);
  } else {
    DV_ON_DEVICE(ctx->device);
    DV_CUDA(cudaMemcpyAsync(&v, &ep->flags[flag_slot], 8, cudaMemcpyDefault, ctx->aux));
    DV_CUDA(cudaStreamSynchronize(ctx->aux));
  }
  *done = v >= seq;
  return DV_OK;
}

}  // extern "C"
