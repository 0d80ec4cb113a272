// dvstream C ABI: context, memory, peers, and the three primitive levels of DejaVuLib
// (Table 1) on top of the run-copy kernel (copy_kernels.cu) and the route
// planner (route.cpp).
#include <cuda.h>
#include <limits.h>
#include <string.h>
#include <time.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "dv_internal.h"
#include "../../include/dv_trace.h"

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
  // Wait for every record overlapping [a, b). Retire only the records [a, b) covers entirely: the
  // record this acquisition's release() adds is ordered after them and stands in for them. A
  // partly covered record stays: another stream may later acquire its uncovered rest, and must
  // still wait for the work that reads or writes it.
  for (auto it = recs_.begin(); it != recs_.end();) {
    if (it->off < b && a < it->off + it->len) {
      cudaError_t e = cudaStreamWaitEvent(stream, it->ev, 0);
      if (e != cudaSuccess) return cuda_fail(e, "staging wait");
      if (a <= it->off && it->off + it->len <= b) {
        free_ev_.push_back(it->ev);
        it = recs_.erase(it);
        continue;
      }
    }
    ++it;
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
// One tensor (K or V) of one side of a copy: the address of word (l0, r0, h0, s0, d=0) and the
// byte strides of the dims (layer, request, head, position, 16-byte packet of d). The packet
// granularity expresses both cache layouts and the wire:
//   KV5D (and V of FT6D): position stride D*e, packet stride 16       (d contiguous)
//   FT6D K:               position stride 16,  packet stride S*16     (x = 16/e words per packet)
//   wire [l][kv][r][h][s][d]: position stride D*e, packet stride 16
enum { DL = 0, DR, DH, DS, DU, NDIM };
struct TView {
  const uint8_t* base;
  int64_t st[NDIM];
};

// `r` must have its heads resolved (explicit head range).
static TView cache_view(const dv_cache* c, int kv, const dv_region* r) {
  const int64_t row = (int64_t)c->head_dim * c->elem_bytes;
  const int64_t sh = (int64_t)c->max_seq * row;  // a head's [S][D] (or [D/x][S][x]) block
  const int64_t sr = (int64_t)c->n_heads * sh;
  const int64_t sl = (int64_t)c->n_reqs * sr;
  const bool ft = c->layout == DV_LAYOUT_FT6D && kv == 0;
  TView t;
  t.st[DL] = sl;
  t.st[DR] = sr;
  t.st[DH] = sh;
  t.st[DS] = ft ? 16 : row;
  t.st[DU] = ft ? (int64_t)c->max_seq * 16 : 16;
  const int64_t off = (int64_t)(r->layer_begin - c->layer_begin) * sl +
                      (int64_t)(r->req_begin - c->req_begin) * sr +
                      (int64_t)(r->head_begin - c->head_begin) * sh +
                      (int64_t)r->pos_begin * t.st[DS];
  t.base = (const uint8_t*)(kv ? c->v : c->k) + off;
  return t;
}

// Canonical wire chunk [l][kv][r][h][s][d] of a region (reading Q3), heads resolved.
static TView wire_view(const uint8_t* w, int kv, const dv_region* r, int64_t row) {
  const int64_t run = (int64_t)(r->pos_end - r->pos_begin) * row;
  const int64_t nH = r->head_end - r->head_begin, nR = r->req_end - r->req_begin;
  TView t;
  t.st[DH] = run;
  t.st[DR] = nH * run;
  const int64_t kvs = nR * nH * run;
  t.st[DL] = 2 * kvs;
  t.st[DS] = row;
  t.st[DU] = 16;
  t.base = w + kv * kvs;
  return t;
}

static bool same_strides(const TView& a, const TView& b) {
  for (int k = 0; k < NDIM; ++k)
    if (a.st[k] != b.st[k]) return false;
  return true;
}

enum Order { ORDER_WIRE /* [l][kv][r][h] */, ORDER_KV_OUTER /* [kv][l][r][h] */ };

// An optional outer dim in front of everything (the chunk index of a log).
struct Outer {
  uint32_t n = 1;
  int64_t ss = 0, ds = 0;
};

// Copy plans moving K and V of a (heads-resolved) region from views `sv` to views `dv_`: one plan
// with kv as a loop dim when K and V have the same strides on both sides, else one per tensor.
// The (position, packet) dims are pre-merged into the run when contiguous on both sides.
// only = 0 / 1: a single plan for that tensor alone.
static int build_plans(const TView sv[2], const TView dv_[2], const dv_region* r, int64_t row,
                       Order order, const Outer& outer, CopyPlan out[2], int only = -1) {
  const uint32_t ext[NDIM] = {(uint32_t)(r->layer_end - r->layer_begin),
                              (uint32_t)(r->req_end - r->req_begin),
                              (uint32_t)(r->head_end - r->head_begin),
                              (uint32_t)(r->pos_end - r->pos_begin), (uint32_t)(row / 16)};
  const bool one = only < 0 && same_strides(sv[0], sv[1]) && same_strides(dv_[0], dv_[1]);
  const int nplans = (one || only >= 0) ? 1 : 2;
  for (int q = 0; q < nplans; ++q) {
    const TView& a = sv[only >= 0 ? only : q];
    const TView& b = dv_[only >= 0 ? only : q];
    // exactly one side packet-major (FT6D key): a 16-byte packet transpose through shared memory
    const bool a_um = a.st[DS] == 16 && a.st[DU] != 16, b_um = b.st[DS] == 16 && b.st[DU] != 16;
    // (only for >= 32 positions: a token step's single position is better served by the run copy)
    if (a_um != b_um && !one && ext[DS] >= 32) {
      CopyPlan t{};
      t.kind = kTranspose;
      t.src = a.base;
      t.dst = (uint8_t*)b.base;
      t.tdir = a_um ? 0 : 1;
      t.tU = ext[DU];
      t.tN = ext[DS];
      t.t_su = (a_um ? a : b).st[DU];
      t.t_ss = (a_um ? b : a).st[DS];
      t.run_bytes = 16;
      const uint32_t sn[4] = {outer.n, ext[DL], ext[DR], ext[DH]};
      const int64_t s1[4] = {outer.ss, a.st[DL], a.st[DR], a.st[DH]};
      const int64_t d1[4] = {outer.ds, b.st[DL], b.st[DR], b.st[DH]};
      for (int k = 0; k < kDims; ++k) {
        const int j = k - (kDims - 4);
        t.n[k] = j < 0 ? 1 : sn[j];
        t.ss[k] = j < 0 ? 0 : s1[j];
        t.ds[k] = j < 0 ? 0 : d1[j];
      }
      out[q] = t;
      continue;
    }
    // dims outer -> inner, before collapsing
    uint32_t n[8];
    int64_t ss[8], ds[8];
    int m = 0;
    auto push = [&](uint32_t e, int64_t x, int64_t y) {
      n[m] = e;
      ss[m] = x;
      ds[m] = y;
      ++m;
    };
    push(outer.n, outer.ss, outer.ds);
    if (one && order == ORDER_KV_OUTER) push(2, sv[1].base - sv[0].base, dv_[1].base - dv_[0].base);
    push(ext[DL], a.st[DL], b.st[DL]);
    if (one && order == ORDER_WIRE) push(2, sv[1].base - sv[0].base, dv_[1].base - dv_[0].base);
    push(ext[DR], a.st[DR], b.st[DR]);
    push(ext[DH], a.st[DH], b.st[DH]);
    uint64_t run = 16;
    if (a.st[DU] == 16 && b.st[DU] == 16 && a.st[DS] == row && b.st[DS] == row) {
      run = (uint64_t)ext[DS] * row;  // positions x packets are one contiguous run on both sides
    } else {
      push(ext[DS], a.st[DS], b.st[DS]);
      push(ext[DU], a.st[DU], b.st[DU]);
    }
    // drop unit dims; keep at most kDims (merging happens in collapse())
    CopyPlan p{};
    p.src = a.base;
    p.dst = (uint8_t*)b.base;
    p.run_bytes = run;
    int w = 0;
    uint32_t nn[8];
    int64_t s2[8], d2[8];
    for (int k = 0; k < m; ++k)
      if (n[k] != 1) {
        nn[w] = n[k];
        s2[w] = ss[k];
        d2[w] = ds[k];
        ++w;
      }
    if (w > kDims) return -1;  // not expressible (cannot happen for the layouts above)
    for (int k = 0; k < kDims; ++k) {
      const int j = k - (kDims - w);
      p.n[k] = j < 0 ? 1 : nn[j];
      p.ss[k] = j < 0 ? 0 : s2[j];
      p.ds[k] = j < 0 ? 0 : d2[j];
    }
    collapse(p);
    out[q] = p;
  }
  return nplans;
}

static uint64_t region_bytes(const dv_region* r, const dv_cache* c) {
  const dv_region x = resolve_heads(r, c);
  return region_bytes_h(&x, c->n_heads, c->head_dim, c->elem_bytes);
}

static int64_t row_bytes(const dv_cache* c) { return (int64_t)c->head_dim * c->elem_bytes; }

static dv_status check_mapped(const void* p, uint64_t extent, const char* name);
static dv_status check_cache_mapped(const dv_cache* c, const char* name);

// Endpoint structure and the capacity for `bytes` at `off` (inside one ring slot for a ring).
static dv_status check_ep(const dv_endpoint* ep, uint64_t off, uint64_t bytes, int32_t slot,
                          bool use_flag, const char* name) {
  if (!ep) return fail(DV_EINVAL, "%s: NULL endpoint", name);
  if (ep->kind != DV_EP_DEVICE && ep->kind != DV_EP_HOST && ep->kind != DV_EP_PEER)
    return fail(DV_EINVAL, "%s: bad endpoint kind %d", name, ep->kind);
  if (!ep->base && bytes) return fail(DV_EINVAL, "%s: NULL endpoint base", name);
  if (((uintptr_t)ep->base | off) % 16)
    return fail(DV_EALIGN, "%s: endpoint base/offset not 16-byte aligned", name);
  if (ep->n_slots < 0) return fail(DV_EINVAL, "%s: negative n_slots", name);
  if (ep->n_slots > 0) {
    if (!ep->slot_bytes || ep->slot_bytes % 16)
      return fail(DV_EALIGN, "%s: ring slot_bytes %llu not a positive multiple of 16", name,
                  (unsigned long long)ep->slot_bytes);
    if ((uint64_t)ep->n_slots > ep->bytes / ep->slot_bytes)
      return fail(DV_EINVAL, "%s: ring of %d x %llu B exceeds endpoint capacity %llu", name,
                  ep->n_slots, (unsigned long long)ep->slot_bytes, (unsigned long long)ep->bytes);
    if (off > ep->slot_bytes || bytes > ep->slot_bytes - off)
      return fail(DV_EINVAL, "%s: [%llu, +%llu) exceeds the ring slot of %llu B", name,
                  (unsigned long long)off, (unsigned long long)bytes,
                  (unsigned long long)ep->slot_bytes);
    if ((uintptr_t)ep->credits % 8) return fail(DV_EALIGN, "%s: credits not 8-byte aligned", name);
    if (ep->credits && !ep->flags)
      return fail(DV_EINVAL, "%s: credits need flags (one credit word per flag slot)", name);
  } else if (off > ep->bytes || bytes > ep->bytes - off) {
    return fail(DV_EINVAL, "%s: [%llu, +%llu) exceeds endpoint capacity %llu", name,
                (unsigned long long)off, (unsigned long long)bytes, (unsigned long long)ep->bytes);
  }
  if (use_flag && slot >= 0) {
    if (!ep->flags || slot >= ep->n_flags)
      return fail(DV_EINVAL, "%s: flag slot %d but endpoint has %d flags", name, slot, ep->n_flags);
    if ((uintptr_t)ep->flags % 8) return fail(DV_EALIGN, "%s: flags not 8-byte aligned", name);
  }
  if (ep->base) DV_TRY(check_mapped(ep->base, ep->bytes, name));
  if (ep->flags) DV_TRY(check_mapped(ep->flags, 8ull * (uint64_t)std::max(ep->n_flags, 0), name));
  if (ep->credits) DV_TRY(check_mapped(ep->credits, 8ull * (uint64_t)std::max(ep->n_flags, 0), name));
  return DV_OK;
}

// ---- inbox rings and credits (dv.h, dv_endpoint) ----------------------------------------------
static bool has_ring(const dv_endpoint* ep) { return ep && ep->n_slots > 0; }
static uint64_t ring_off(const dv_endpoint* ep, uint64_t seq) {
  return has_ring(ep) ? (seq % (uint64_t)ep->n_slots) * ep->slot_bytes : 0;
}
// A data call into / out of a ring needs a flag slot and a sequence number >= 1.
static dv_status check_ring_use(const dv_endpoint* ep, int32_t slot, uint64_t seq, bool use_flag,
                                const char* name) {
  if (!has_ring(ep)) return DV_OK;
  if (!use_flag || slot < 0 || seq < 1)
    return fail(DV_EINVAL, "%s: a ring endpoint needs a flag slot and a sequence number >= 1", name);
  return DV_OK;
}
static bool local_vidmem(const dv_ctx* ctx, const void* p);
// The value of a 64-bit word in host, device or mapped peer memory, read now from the host (a
// small synchronous copy for device memory).
static dv_status read_word(dv_ctx* ctx, const uint64_t* p, uint64_t* out) {
  cudaPointerAttributes at;
  DV_CUDA(cudaPointerGetAttributes(&at, p));
  if (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered) {
    *out = __atomic_load_n(p, __ATOMIC_ACQUIRE);
    return DV_OK;
  }
  DV_ON_DEVICE(ctx->device);   // validation may run before the caller switched to ctx's device
  DV_CUDA(cudaMemcpyAsync(out, p, 8, cudaMemcpyDefault, ctx->aux));
  DV_CUDA(cudaStreamSynchronize(ctx->aux));
  return DV_OK;
}
// Sender side, validation time: with DV_NOWAIT a seq whose ring slot has no credit yet -> DV_EBUSY
// (nothing has been enqueued; the caller retries).
static dv_status credit_check_nowait(dv_ctx* ctx, const dv_endpoint* ep, int32_t slot, uint64_t seq,
                                     uint32_t xfer) {
  if (!has_ring(ep) || !ep->credits || !(xfer & DV_NOWAIT) || seq <= (uint64_t)ep->n_slots)
    return DV_OK;
  uint64_t c = 0;
  DV_TRY(read_word(ctx, &ep->credits[slot], &c));
  if (c + (uint64_t)ep->n_slots < seq)
    return fail(DV_EBUSY, "inbox ring slot %llu busy: source %d's credit is %llu, seq %llu needs %llu",
                (unsigned long long)(seq % (uint64_t)ep->n_slots), slot, (unsigned long long)c,
                (unsigned long long)seq, (unsigned long long)(seq - (uint64_t)ep->n_slots));
  return DV_OK;
}
// Sender side, enqueue time: order the writes of seq s after credits[slot] >= s - n_slots. A
// stream memory-op wait where the word is pinned host memory or this GPU's own HBM; a one-thread
// acquire-spin kernel for peer memory (mapped over NVLink).
static dv_status stream_wait_word(const uint64_t* p, uint64_t v, cudaStream_t st);
static dv_status credit_wait(dv_ctx* ctx, const dv_endpoint* ep, int32_t slot, uint64_t seq,
                             uint32_t xfer, cudaStream_t st) {
  if (!has_ring(ep) || !ep->credits || seq <= (uint64_t)ep->n_slots || (xfer & DV_NOWAIT))
    return DV_OK;   // NOWAIT: the credit was already there at validation (credits only grow)
  (void)ctx;
  return stream_wait_word(&ep->credits[slot], seq - (uint64_t)ep->n_slots, st);
}

static dv_status check_ctx(dv_ctx* ctx) {
  if (!ctx) return fail(DV_EINVAL, "NULL context");
  return DV_OK;
}

static bool in_ipc_mapping(const void* p);

// Is `p` memory of this context's GPU (its own HBM)? Then every reader of it -- SMs, copy
// engines, stream memory operations, peers over NVLink -- is served by this GPU's L2. Memory
// mapped from another process (dv_ipc_open) never counts as local, whatever GPU it lives on.
static bool local_vidmem(const dv_ctx* ctx, const void* p) {
  if (in_ipc_mapping(p)) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device == ctx->device;
}

// The release of a fused copy: the endpoint's flag, a ticket, and the scope. Payload (the plans'
// destinations) and flag all in this GPU's HBM -> a gpu-scope release suffices (publish() protocol
// 3); anything in pinned host or peer memory -> system scope.
static dv_status word_release(dv_ctx* ctx, uint64_t* word, uint64_t seq, const CopyPlan* p, int np,
                              cudaStream_t st, Release* out);
static dv_status ticket_release(dv_ctx* ctx, const dv_endpoint* ep, int32_t slot, uint64_t seq,
                                bool use_flag, const CopyPlan* p, int np, cudaStream_t st,
                                Release* out) {
  *out = Release{nullptr, 0, nullptr};
  if (use_flag && slot >= 0 && ep && ep->flags) return word_release(ctx, &ep->flags[slot], seq, p, np, st, out);
  return DV_OK;
}
// The receiver's credit (dv.h, rings): released by the unpack kernel once it has read the chunk.
// Its loads completed before its stores, which the release orders; the scope is the credit word's
// (gpu scope for this GPU's HBM -- peers polling it over NVLink are served by this GPU's L2).
static dv_status credit_release(dv_ctx* ctx, const dv_endpoint* src, int32_t slot, uint64_t seq,
                                cudaStream_t st, Release* out) {
  *out = Release{nullptr, 0, nullptr};
  if (!has_ring(src) || !src->credits) return DV_OK;
  return word_release(ctx, &src->credits[slot], seq, nullptr, 0, st, out);
}
// A release of `seq` into `word` after a copy kernel's plans `p` (their destinations decide the
// scope together with the word's memory).
static dv_status word_release(dv_ctx* ctx, uint64_t* word, uint64_t seq, const CopyPlan* p, int np,
                              cudaStream_t st, Release* out) {
  Release r{nullptr, 0, nullptr};
  {
    r.flag = (unsigned long long*)word;
    r.seq = seq;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    DV_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) {  // a graph keeps this ticket: never hand it out again
      const uint32_t g = ctx->next_graph_ticket.fetch_add(1);
      if (g >= dv_ctx::kGraphTickets)
        return fail(DV_ENOMEM, "more than %u publishing launches captured into CUDA graphs by this "
                    "context", dv_ctx::kGraphTickets);
      r.ticket = ctx->tickets + dv_ctx::kTickets + g;
    } else {
      r.ticket = ctx->tickets + (ctx->next_ticket.fetch_add(1) % dv_ctx::kTickets);
    }
    r.ts = ctx->trace_ts;
    bool local = local_vidmem(ctx, r.flag);
    for (int q = 0; q < np && local; ++q)
      if (p[q].dst && p[q].runs() && p[q].run_bytes) local = local_vidmem(ctx, p[q].dst);
    r.gpu_scope = local;
  }
  *out = r;
  return DV_OK;
}

// Stream memory operations serve words in pinned host memory and in the calling GPU's own HBM;
// a word in peer memory (another GPU's, or mapped from another process) is written / waited on by
// a one-thread kernel instead (system-scope release / acquire over the link).
static bool memop_ok(const void* p) {
  if (in_ipc_mapping(p)) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeHost) return true;
  int dev = -1;
  cudaGetDevice(&dev);
  return at.type == cudaMemoryTypeDevice && at.device == dev;
}

static dv_status stream_signal(const dv_endpoint* ep, int32_t slot, uint64_t seq,
                               cudaStream_t stream) {
  uint64_t* p = &ep->flags[slot];
  if (!memop_ok(p)) return launch_store_release(p, seq, stream);
  const Driver* d;
  DV_TRY(driver(&d));
  int r = d->streamWriteValue64(stream, (unsigned long long)(uintptr_t)p, seq,
                                CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r) return drv_fail(r, "cuStreamWriteValue64");
  return DV_OK;
}

static dv_status stream_wait_word(const uint64_t* p, uint64_t v, cudaStream_t stream) {
  if (!memop_ok(p)) return launch_wait_geq(p, v, stream);
  const Driver* d;
  DV_TRY(driver(&d));
  int r = d->streamWaitValue64(stream, (unsigned long long)(uintptr_t)p, v, CU_STREAM_WAIT_VALUE_GEQ);
  if (r) return drv_fail(r, "cuStreamWaitValue64");
  return DV_OK;
}
static dv_status stream_wait(const dv_endpoint* ep, int32_t slot, uint64_t seq,
                             cudaStream_t stream) {
  return stream_wait_word(&ep->flags[slot], seq, stream);
}

static dv_status hand_off(dv_ctx* ctx, cudaStream_t from, cudaStream_t to);
// Once this context has published a decoupled flag (on ctx->flag_st, after its DMA), a publish to
// a pinned-host flag from another stream is ordered after flag_st: a slot used in both modes then
// never sees seq t+1 before step t's decoupled flag (and never drops back).
// Costs nothing when every decoupled flag has already landed (the event has completed), so the
// per-layer latency path keeps its programmatic dependent launch behind the writer. Not applied
// to launches captured into a CUDA graph (a graph cannot wait on work outside it; event queries
// are illegal during capture): the caller orders a replay after earlier decoupled transfers of
// the same slot (dv.h, DV_XFER_DECOUPLED).
static dv_status after_decoupled_flags(dv_ctx* ctx, cudaStream_t st) {
  if (!ctx->decoupled_used.load(std::memory_order_relaxed)) return DV_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DV_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) return DV_OK;
  std::lock_guard<std::mutex> lk(ctx->pipe_mu);
  const cudaError_t q = cudaEventQuery(ctx->flag_ev);
  if (q == cudaSuccess) return DV_OK;
  if (q != cudaErrorNotReady) return cuda_fail(q, "decoupled flag event");
  (void)cudaGetLastError();
  DV_CUDA(cudaStreamWaitEvent(st, ctx->flag_ev, 0));
  return DV_OK;
}
// A decoupled flag store was just enqueued on ctx->flag_st (pipe_mu held).
static dv_status note_decoupled_flag(dv_ctx* ctx) {
  DV_CUDA(cudaEventRecord(ctx->flag_ev, ctx->flag_st));
  ctx->decoupled_used.store(true, std::memory_order_relaxed);
  return DV_OK;
}

// The fused kernels of 1-2 plans, then the flag: by the last kernel itself (fenced st.release.sys
// from its last CTA) or, with DV_PUBLISH_STREAMOP, by a stream memory operation after it.
static dv_status launch_publish(dv_ctx* ctx, const CopyPlan* p, int np, const dv_endpoint* ep,
                                int32_t slot, uint64_t seq, bool use_flag, uint32_t xfer,
                                cudaStream_t st, int ctas) {
  const bool streamop = (xfer & DV_PUBLISH_STREAMOP) != 0;
  const Release none{nullptr, 0, nullptr};
  Release rel = none;
  if (!streamop) DV_TRY(ticket_release(ctx, ep, slot, seq, use_flag, p, np, st, &rel));
  if (use_flag && ep->kind == DV_EP_HOST) DV_TRY(after_decoupled_flags(ctx, st));
  if (np == 2) {
    DV_TRY(launch_copy2(p[0], p[1], rel, ctas, st));
    if (streamop && use_flag) DV_TRY(stream_signal(ep, slot, seq, st));
    return DV_OK;
  }
  for (int q = 0; q < np; ++q) {
    const bool last = q == np - 1;
    DV_TRY(launch_copy(p[q], 0, p[q].runs(), last ? rel : none, ctas, st));
  }
  if (streamop && use_flag) DV_TRY(stream_signal(ep, slot, seq, st));
  return DV_OK;
}

// Chooses FUSED or STAGED for a data call (measured in
// profiles/r01_tune_host*.jsonl): writes to pinned host go through the kernel's own PCIe stores up
// to 32 MB (same throughput as pack+DMA for a 6.55 MB token step, lower latency, no staging) and
// through pipelined pack + copy-engine DMA above (54.8 vs 52.6 GB/s for a 163.8 MB prompt layer,
// and no SMs held during the transfer); reads from pinned host below 4 MiB are SM zero-copy loads,
// larger ones go through the copy engine (see below).
static uint32_t pick_xfer(uint32_t xfer, const dv_endpoint* ep, uint64_t bytes, bool reading) {
  uint32_t m = xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  // decoupled host writes: pack + DMA on the context's DMA stream overlaps consecutive steps
  if (!reading && (xfer & DV_XFER_DECOUPLED) && ep->kind == DV_EP_HOST && m != DV_XFER_FUSED)
    return DV_XFER_STAGED;
  if (m == DV_XFER_FUSED || m == DV_XFER_STAGED) {
    if (m == DV_XFER_STAGED && ep->kind == DV_EP_DEVICE) return DV_XFER_FUSED;  // already local
    return m;
  }
  // reads: SM zero-copy loads win alone at every size (160 KiB 6.8 vs 12.3 us, 1.3 MB 28.6 vs
  // 39.3 us, 6.55 MB 130.6 vs 132.7 us -- tools/probe_small_reads.py) but do not overlap with a
  // concurrent D2H stream (e2e 25 vs 39.8 GB/s at 6.55 MB), so the copy engine takes reads from
  // 4 MiB up, where a read is a bulk transfer rather than a latency-bound one
  if (ep->kind == DV_EP_HOST && reading) return bytes < (4ull << 20) ? DV_XFER_FUSED : DV_XFER_STAGED;
  if (ep->kind == DV_EP_HOST && bytes >= (32ull << 20)) return DV_XFER_STAGED;
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

static dv_status staged_capacity_check(dv_ctx* ctx, uint32_t xfer, const dv_endpoint* ep,
                                       const dv_cache* c, const dv_region& reg0, uint64_t off,
                                       bool pack);

static dv_status scatter_check(dv_ctx* ctx, const ScatterOp& op) {
  DV_TRY(check_ctx(ctx));
  DV_TRY(check_cache(op.src, "source"));
  DV_TRY(check_cache_mapped(op.src, "source"));
  DV_TRY(check_region_shape(&op.reg));
  DV_TRY(check_cache_holds(op.src, &op.reg, "source"));
  const bool use_flag = !(op.xfer & DV_NO_FLAG);
  if ((op.xfer & DV_XFER_DECOUPLED) && op.dst && op.dst->kind == DV_EP_HOST &&
      (!use_flag || op.slot < 0))
    return fail(DV_EINVAL, "DV_XFER_DECOUPLED needs a flag: the flag is its only completion signal");
  DV_TRY(check_ep(op.dst, op.dst_off, region_bytes(&op.reg, op.src), op.slot, use_flag,
                  "destination"));
  DV_TRY(check_ring_use(op.dst, op.slot, op.seq, use_flag, "destination"));
  DV_TRY(staged_capacity_check(ctx, op.xfer, op.dst, op.src, op.reg,
                               op.dst_off + ring_off(op.dst, op.seq), true));
  return credit_check_nowait(ctx, op.dst, op.slot, op.seq, op.xfer);   // last: DV_EBUSY
}

// Layer slabs of a region's wire: [l][...] -- slab l starts at (l - l0) * slab bytes.
static uint64_t layer_slab_bytes(const dv_region* r, int64_t row) {
  return 2ull * (uint64_t)(r->req_end - r->req_begin) * (uint64_t)(r->head_end - r->head_begin) *
         (uint64_t)(r->pos_end - r->pos_begin) * (uint64_t)row;
}

// Pipelined staging: kernels run on the caller's stream, copy-engine DMAs on ctx->dma; each
// hand-off is an event (record on one stream, wait on the other), so chunk k's DMA overlaps
// chunk k+1's kernel and the transfer time approaches the DMA time alone.
static cudaEvent_t next_event(dv_ctx* ctx) {
  return ctx->pipe_ev[ctx->next_ev.fetch_add(1) % ctx->pipe_ev.size()];
}
static dv_status hand_off(dv_ctx* ctx, cudaStream_t from, cudaStream_t to) {
  if (from == to) return DV_OK;
  cudaEvent_t ev = next_event(ctx);
  DV_CUDA(cudaEventRecord(ev, from));
  DV_CUDA(cudaStreamWaitEvent(to, ev, 0));
  return DV_OK;
}
// Transfers below this size are not worth the cross-stream hand-offs (measured: a 6.55 MB token
// step took 151 us pipelined in 1 MiB chunks vs 137 us as one chunk on one stream).
static const uint64_t kPipeMin = 32ull << 20;
// Chunk size of a staged transfer: one chunk below kPipeMin; else ~8 chunks >= 4 MiB; <= half pool.
static uint64_t pipe_chunk(uint64_t total, uint64_t half) {
  if (total < kPipeMin) return half;
  return std::min<uint64_t>(half, std::max<uint64_t>(4ull << 20, total / 8));
}

// Can the staged path move `reg` of cache `c` with this context's staging pool? A single run plan
// is chunked by runs (one run must fit half the pool); two plans (K and V of different structure)
// are staged per layer slab, or per (layer, K or V) half-slab when a slab does not fit half the
// pool (one half-slab must).
static bool staged_fits(dv_ctx* ctx, const dv_cache* c, const dv_region& reg, const uint8_t* wire,
                        bool pack) {
  const int64_t row = row_bytes(c);
  const uint64_t half = ctx->staging.capacity() / 2;
  TView cv[2] = {cache_view(c, 0, &reg), cache_view(c, 1, &reg)};
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  CopyPlan p[2];
  const int np = pack ? build_plans(cv, wv, &reg, row, ORDER_WIRE, Outer{}, p)
                      : build_plans(wv, cv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np < 0) return true;   // let the staged path report it
  if (np == 1 && p[0].run_bytes <= half) return true;
  return layer_slab_bytes(&reg, row) / 2 <= half;   // per (layer, K or V) when a slab is too big
}

// Validation-time capacity check (so a multi-piece call fails before enqueueing anything): an
// EXPLICIT staged / decoupled host transfer whose staging unit does not fit the pool -> DV_ENOMEM.
// (AUTO falls back to the kernel's own copies instead, in scatter_run / gather_run.)
static dv_status staged_capacity_check(dv_ctx* ctx, uint32_t xfer, const dv_endpoint* ep,
                                       const dv_cache* c, const dv_region& reg0, uint64_t off,
                                       bool pack) {
  if (!(xfer & (DV_XFER_STAGED | DV_XFER_DECOUPLED)) || (xfer & DV_XFER_FUSED)) return DV_OK;
  const dv_region reg = resolve_heads(&reg0, c);
  const uint64_t bytes = region_bytes(&reg, c);
  if (!bytes || pick_xfer(xfer, ep, bytes, !pack) != DV_XFER_STAGED) return DV_OK;
  const uint8_t* wire = (const uint8_t*)ep->base + off;
  if (staged_fits(ctx, c, reg, wire, pack)) return DV_OK;
  return fail(DV_ENOMEM, "one layer slab (%llu B) exceeds the staging pool; use a larger "
              "dv_config.staging_bytes or DV_XFER_FUSED",
              (unsigned long long)layer_slab_bytes(&reg, row_bytes(c)));
}

// Pack `reg` (heads resolved) of cache `c` into a wire chunk at `wire` through HBM staging:
// the kernel packs a group of layer slabs (or, with one plan, a range of runs) into staging, the
// copy engine moves that contiguous piece to its place in the wire.
// decoupled: the DMAs (and the caller's flag after them) stay on ctx->dma, the caller's stream only
// waits for the packs; *flag_stream is the stream the flag must be published on.
static dv_status staged_pack(dv_ctx* ctx, const dv_cache* c, const dv_region& reg, uint8_t* wire,
                             cudaStream_t st, bool decoupled, cudaStream_t* flag_stream) {
  *flag_stream = st;
  const int64_t row = row_bytes(c);
  const uint64_t half = ctx->staging.capacity() / 2;
  const Release none{nullptr, 0, nullptr};
  TView sv[2] = {cache_view(c, 0, &reg), cache_view(c, 1, &reg)};
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  CopyPlan p[2];
  const int np = build_plans(sv, wv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  std::lock_guard<std::mutex> lk(ctx->pipe_mu);
  const uint64_t total = region_bytes_h(&reg, c->n_heads, c->head_dim, c->elem_bytes);
  cudaStream_t ds = (total >= kPipeMin || decoupled) ? ctx->dma : st;  // copy-engine stream
  // the caller's stream rejoins after the DMAs, or (decoupled) after the last pack
  auto finish = [&]() -> dv_status {
    if (!decoupled) return hand_off(ctx, ds, st);
    *flag_stream = ds;
    return DV_OK;
  };
  if (np == 1 && p[0].run_bytes <= half) {  // dense wire in run order: chunk by runs
    const uint64_t rb = p[0].run_bytes, runs = p[0].runs();
    const uint64_t chunk = std::max<uint64_t>(1, pipe_chunk(runs * rb, half) / rb);
    DV_TRY(hand_off(ctx, st, ds));  // the DMA stream must not run ahead of the caller's work
    for (uint64_t q0 = 0; q0 < runs; q0 += chunk) {
      const uint64_t q1 = std::min(runs, q0 + chunk), nb = (q1 - q0) * rb;
      uint8_t* stg;
      uint64_t off;
      DV_TRY(ctx->staging.acquire(nb, st, &stg, &off));
      CopyPlan pc = p[0];
      pc.dst = stg - q0 * rb;  // run q lands at stg + (q - q0) * rb (wire side is dense)
      DV_TRY(launch_copy(pc, q0, q1, none, ctx->max_ctas, st));
      DV_TRY(hand_off(ctx, st, ds));
      DV_DMA(cudaMemcpyAsync(wire + q0 * rb, stg, nb, cudaMemcpyDefault, ds));
      DV_TRY(ctx->staging.release(off, nb, ds));
    }
    return finish();
  }
  const uint64_t slab = layer_slab_bytes(&reg, row);
  if (slab / 2 > half)
    return fail(DV_ENOMEM, "one layer slab (%llu B) exceeds the staging pool; use a larger "
                "dv_config.staging_bytes or DV_XFER_FUSED", (unsigned long long)slab);
  if (slab > half) {
    // one layer slab does not fit half the pool: stage per (layer, K or V) -- each half of a
    // layer slab is contiguous in the wire ([l][kv][...]); one plan per tensor (the K plan may be
    // a packet transpose, which moves a whole layer's key in one launch)
    const uint64_t hs = slab / 2;
    DV_TRY(hand_off(ctx, st, ds));
    for (int32_t la = reg.layer_begin; la < reg.layer_end; ++la) {
      dv_region sub = reg;
      sub.layer_begin = la;
      sub.layer_end = la + 1;
      for (int kv = 0; kv < 2; ++kv) {
        uint8_t* stg;
        uint64_t off;
        DV_TRY(ctx->staging.acquire(hs, st, &stg, &off));
        // the wire view of tensor kv starts kv*hs into the layer: shift it back onto the staging
        TView s2[2] = {cache_view(c, 0, &sub), cache_view(c, 1, &sub)};
        TView w2[2] = {wire_view(stg - kv * hs, 0, &sub, row), wire_view(stg - kv * hs, 1, &sub, row)};
        CopyPlan ps[2];
        if (build_plans(s2, w2, &sub, row, ORDER_WIRE, Outer{}, ps, kv) != 1)
          return fail(DV_ENOTSUP, "copy not expressible");
        DV_TRY(launch_copy(ps[0], 0, ps[0].runs(), none, ctx->max_ctas, st));
        DV_TRY(hand_off(ctx, st, ds));
        DV_DMA(cudaMemcpyAsync(wire + (uint64_t)(la - reg.layer_begin) * slab + kv * hs, stg, hs,
                               cudaMemcpyDefault, ds));
        DV_TRY(ctx->staging.release(off, hs, ds));
      }
    }
    return finish();
  }
  const int32_t per = (int32_t)std::max<uint64_t>(
      1, pipe_chunk((uint64_t)(reg.layer_end - reg.layer_begin) * slab, half) / slab);
  DV_TRY(hand_off(ctx, st, ds));
  for (int32_t la = reg.layer_begin; la < reg.layer_end; la += per) {
    dv_region sub = reg;
    sub.layer_begin = la;
    sub.layer_end = std::min(reg.layer_end, la + per);
    const uint64_t nb = (uint64_t)(sub.layer_end - la) * slab;
    uint8_t* stg;
    uint64_t off;
    DV_TRY(ctx->staging.acquire(nb, st, &stg, &off));
    TView s2[2] = {cache_view(c, 0, &sub), cache_view(c, 1, &sub)};
    TView w2[2] = {wire_view(stg, 0, &sub, row), wire_view(stg, 1, &sub, row)};
    CopyPlan ps[2];
    const int n2 = build_plans(s2, w2, &sub, row, ORDER_WIRE, Outer{}, ps);
    if (n2 == 2)
      DV_TRY(launch_copy2(ps[0], ps[1], none, ctx->max_ctas, st));
    else
      DV_TRY(launch_copy(ps[0], 0, ps[0].runs(), none, ctx->max_ctas, st));
    DV_TRY(hand_off(ctx, st, ds));
    DV_DMA(cudaMemcpyAsync(wire + (uint64_t)(la - reg.layer_begin) * slab, stg, nb,
                           cudaMemcpyDefault, ds));
    DV_TRY(ctx->staging.release(off, nb, ds));
  }
  return finish();
}

// Unpack a wire chunk at `wire` (any memory) into `reg` of cache `c` through HBM staging.
static dv_status staged_unpack(dv_ctx* ctx, const uint8_t* wire, const dv_cache* c,
                               const dv_region& reg, cudaStream_t st) {
  const int64_t row = row_bytes(c);
  const uint64_t half = ctx->staging.capacity() / 2;
  const Release none{nullptr, 0, nullptr};
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  TView cv[2] = {cache_view(c, 0, &reg), cache_view(c, 1, &reg)};
  CopyPlan p[2];
  const int np = build_plans(wv, cv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  std::lock_guard<std::mutex> lk(ctx->pipe_mu);
  const uint64_t total = region_bytes_h(&reg, c->n_heads, c->head_dim, c->elem_bytes);
  cudaStream_t ds = total >= kPipeMin ? ctx->dma : st;
  DV_TRY(hand_off(ctx, st, ds));  // DMAs start after the caller's prior work (flag waits)
  if (np == 1 && p[0].run_bytes <= half) {
    const uint64_t rb = p[0].run_bytes, runs = p[0].runs();
    const uint64_t chunk = std::max<uint64_t>(1, pipe_chunk(runs * rb, half) / rb);
    for (uint64_t q0 = 0; q0 < runs; q0 += chunk) {
      const uint64_t q1 = std::min(runs, q0 + chunk), nb = (q1 - q0) * rb;
      uint8_t* stg;
      uint64_t off;
      DV_TRY(ctx->staging.acquire(nb, ds, &stg, &off));
      DV_DMA(cudaMemcpyAsync(stg, wire + q0 * rb, nb, cudaMemcpyDefault, ds));
      DV_TRY(hand_off(ctx, ds, st));
      CopyPlan pc = p[0];
      pc.src = stg - q0 * rb;
      DV_TRY(launch_copy(pc, q0, q1, none, ctx->max_ctas, st));
      DV_TRY(ctx->staging.release(off, nb, st));
    }
    return DV_OK;
  }
  const uint64_t slab = layer_slab_bytes(&reg, row);
  if (slab / 2 > half)
    return fail(DV_ENOMEM, "one layer slab (%llu B) exceeds the staging pool; use a larger "
                "dv_config.staging_bytes or DV_XFER_FUSED", (unsigned long long)slab);
  if (slab > half) {   // per (layer, K or V), as in staged_pack
    const uint64_t hs = slab / 2;
    for (int32_t la = reg.layer_begin; la < reg.layer_end; ++la) {
      dv_region sub = reg;
      sub.layer_begin = la;
      sub.layer_end = la + 1;
      for (int kv = 0; kv < 2; ++kv) {
        uint8_t* stg;
        uint64_t off;
        DV_TRY(ctx->staging.acquire(hs, ds, &stg, &off));
        DV_DMA(cudaMemcpyAsync(stg, wire + (uint64_t)(la - reg.layer_begin) * slab + kv * hs, hs,
                               cudaMemcpyDefault, ds));
        DV_TRY(hand_off(ctx, ds, st));
        TView w2[2] = {wire_view(stg - kv * hs, 0, &sub, row), wire_view(stg - kv * hs, 1, &sub, row)};
        TView c2[2] = {cache_view(c, 0, &sub), cache_view(c, 1, &sub)};
        CopyPlan ps[2];
        if (build_plans(w2, c2, &sub, row, ORDER_WIRE, Outer{}, ps, kv) != 1)
          return fail(DV_ENOTSUP, "copy not expressible");
        DV_TRY(launch_copy(ps[0], 0, ps[0].runs(), none, ctx->max_ctas, st));
        DV_TRY(ctx->staging.release(off, hs, st));
      }
    }
    return DV_OK;
  }
  const int32_t per = (int32_t)std::max<uint64_t>(
      1, pipe_chunk((uint64_t)(reg.layer_end - reg.layer_begin) * slab, half) / slab);
  for (int32_t la = reg.layer_begin; la < reg.layer_end; la += per) {
    dv_region sub = reg;
    sub.layer_begin = la;
    sub.layer_end = std::min(reg.layer_end, la + per);
    const uint64_t nb = (uint64_t)(sub.layer_end - la) * slab;
    uint8_t* stg;
    uint64_t off;
    DV_TRY(ctx->staging.acquire(nb, ds, &stg, &off));
    DV_DMA(cudaMemcpyAsync(stg, wire + (uint64_t)(la - reg.layer_begin) * slab, nb,
                           cudaMemcpyDefault, ds));
    DV_TRY(hand_off(ctx, ds, st));
    TView w2[2] = {wire_view(stg, 0, &sub, row), wire_view(stg, 1, &sub, row)};
    TView c2[2] = {cache_view(c, 0, &sub), cache_view(c, 1, &sub)};
    CopyPlan ps[2];
    const int n2 = build_plans(w2, c2, &sub, row, ORDER_WIRE, Outer{}, ps);
    if (n2 == 2)
      DV_TRY(launch_copy2(ps[0], ps[1], none, ctx->max_ctas, st));
    else
      DV_TRY(launch_copy(ps[0], 0, ps[0].runs(), none, ctx->max_ctas, st));
    DV_TRY(ctx->staging.release(off, nb, st));
  }
  return DV_OK;
}

static dv_status scatter_run(dv_ctx* ctx, const ScatterOp& op, cudaStream_t st) {
  const dv_cache* c = op.src;
  const dv_region reg = resolve_heads(&op.reg, c);
  const uint64_t bytes = region_bytes(&reg, c);
  const bool use_flag = !(op.xfer & DV_NO_FLAG) && op.slot >= 0;
  uint32_t mode = pick_xfer(op.xfer, op.dst, bytes, false);
  uint8_t* wire = (uint8_t*)op.dst->base + op.dst_off + ring_off(op.dst, op.seq);
  const int64_t row = row_bytes(c);
  // a credited ring slot is overwritten only after the receiver consumed its previous chunk
  DV_TRY(credit_wait(ctx, op.dst, op.slot, op.seq, op.xfer, st));
  // AUTO picked staging but the pool cannot hold one layer slab of this region: the kernel's own
  // stores move it instead (an explicit STAGED / DECOUPLED request still reports DV_ENOMEM)
  if (mode == DV_XFER_STAGED && !(op.xfer & (DV_XFER_FUSED | DV_XFER_STAGED | DV_XFER_DECOUPLED)) &&
      !region_empty(&reg) && !staged_fits(ctx, c, reg, wire, true))
    mode = DV_XFER_FUSED;
  const bool decoupled = (op.xfer & DV_XFER_DECOUPLED) && op.dst->kind == DV_EP_HOST;
  if (decoupled && use_flag && region_empty(&reg)) {
    // nothing to move: the flag still goes out on the flag stream, behind the caller's prior work
    // and behind every earlier decoupled flag (FIFO), so the slot's seq never runs ahead of a
    // DMA still in flight
    std::lock_guard<std::mutex> lk(ctx->pipe_mu);
    DV_TRY(hand_off(ctx, st, ctx->flag_st));
    DV_TRY(stream_signal(op.dst, op.slot, op.seq, ctx->flag_st));
    return note_decoupled_flag(ctx);
  }
  if (mode == DV_XFER_FUSED || region_empty(&reg)) {
    CopyPlan p[2];
    int np = 0;
    if (!region_empty(&reg)) {
      TView sv[2] = {cache_view(c, 0, &reg), cache_view(c, 1, &reg)};
      TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
      np = build_plans(sv, wv, &reg, row, ORDER_WIRE, Outer{}, p);
      if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
    } else {
      p[0] = CopyPlan{};
      np = 1;  // empty plan: still publishes the flag in stream order
    }
    return launch_publish(ctx, p, np, op.dst, op.slot, op.seq, use_flag, op.xfer, st,
                          (op.dst->kind == DV_EP_HOST || c->device < 0) ? ctx->host_ctas
                                                                         : ctx->max_ctas);
  }
  cudaStream_t fs;
  DV_TRY(staged_pack(ctx, c, reg, wire, st, decoupled, &fs));
  if (use_flag && fs != st) {
    // A stream memory op serialises its stream for ~5.7 us (tools/probe_dma_gaps.py): the flag
    // store goes to its own stream, ordered after this DMA by an event, so the next step's DMA
    // starts at once. One flag stream per context keeps flags monotonic.
    std::lock_guard<std::mutex> lk(ctx->pipe_mu);
    DV_TRY(hand_off(ctx, fs, ctx->flag_st));
    DV_TRY(stream_signal(op.dst, op.slot, op.seq, ctx->flag_st));
    return note_decoupled_flag(ctx);
  }
  if (use_flag) {
    if (op.dst->kind == DV_EP_HOST) DV_TRY(after_decoupled_flags(ctx, fs));
    DV_TRY(stream_signal(op.dst, op.slot, op.seq, fs));
  }
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
  DV_TRY(check_cache_mapped(op.dst, "destination"));
  DV_TRY(check_region_shape(&op.reg));
  DV_TRY(check_cache_holds(op.dst, &op.reg, "destination"));
  const bool use_flag = !(op.xfer & DV_NO_FLAG);
  DV_TRY(check_ep(op.src, op.src_off, region_bytes(&op.reg, op.dst), op.slot, use_flag, "source"));
  DV_TRY(check_ring_use(op.src, op.slot, op.wait_seq, use_flag, "source"));
  return staged_capacity_check(ctx, op.xfer, op.src, op.dst, op.reg,
                               op.src_off + ring_off(op.src, op.wait_seq), false);
}

static dv_status gather_run(dv_ctx* ctx, const GatherOp& op, cudaStream_t st) {
  const dv_cache* c = op.dst;
  const dv_region reg = resolve_heads(&op.reg, c);
  const uint64_t bytes = region_bytes(&reg, c);
  uint32_t mode = bytes ? pick_xfer(op.xfer, op.src, bytes, true) : DV_XFER_FUSED;
  const uint8_t* wire = (const uint8_t*)op.src->base + op.src_off + ring_off(op.src, op.wait_seq);
  // decided before anything is enqueued (no partial effect): AUTO falls back to the kernel's own
  // loads when one layer slab does not fit half the staging pool; explicit STAGED reports it
  if (mode == DV_XFER_STAGED && !staged_fits(ctx, c, reg, wire, false)) {
    if (op.xfer & DV_XFER_STAGED)
      return fail(DV_ENOMEM, "one layer slab (%llu B) exceeds the staging pool; use a larger "
                  "dv_config.staging_bytes or DV_XFER_FUSED",
                  (unsigned long long)layer_slab_bytes(&reg, row_bytes(c)));
    mode = DV_XFER_FUSED;
  }
  const bool use_flag = !(op.xfer & DV_NO_FLAG) && op.slot >= 0;
  if (use_flag && op.wait_seq) DV_TRY(stream_wait(op.src, op.slot, op.wait_seq, st));
  // the receiver's credit for this chunk (ring inboxes): released once the chunk has been read
  Release credit{nullptr, 0, nullptr};
  if (use_flag) DV_TRY(credit_release(ctx, op.src, op.slot, op.wait_seq, st, &credit));
  const int ctas = (op.src->kind == DV_EP_HOST || c->device < 0) ? ctx->host_ctas : ctx->max_ctas;
  if (!bytes || mode == DV_XFER_STAGED) {
    if (bytes) DV_TRY(staged_unpack(ctx, wire, c, reg, st));
    if (!credit.flag) return DV_OK;
    return launch_copy(CopyPlan{}, 0, 0, credit, ctas, st);   // publish only
  }
  const int64_t row = row_bytes(c);
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  TView cv[2] = {cache_view(c, 0, &reg), cache_view(c, 1, &reg)};
  CopyPlan p[2];
  const int np = build_plans(wv, cv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  if (np == 2) return launch_copy2(p[0], p[1], credit, ctas, st);
  return launch_copy(p[0], 0, p[0].runs(), credit, ctas, st);
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
  DV_TRY(check_cache_mapped(op.src, "source"));
  DV_TRY(check_cache_mapped(op.dst, "destination"));
  DV_TRY(check_region_shape(&op.reg));
  const dv_region reg = resolve_heads(&op.reg, op.src);
  DV_TRY(check_cache_holds(op.src, &reg, "source"));
  DV_TRY(check_cache_holds(op.dst, &reg, "destination"));
  if (op.src->head_dim != op.dst->head_dim || op.src->elem_bytes != op.dst->elem_bytes)
    return fail(DV_EMAP, "source and destination caches differ in head_dim/elem_bytes");
  if (op.signal && !(op.xfer & DV_NO_FLAG) && op.slot >= 0)
    DV_TRY(check_ep(op.signal, 0, 0, op.slot, true, "signal"));
  return DV_OK;
}

static dv_status remap_run(dv_ctx* ctx, const RemapOp& op, cudaStream_t st) {
  const dv_region reg = resolve_heads(&op.reg, op.src);
  const int64_t row = row_bytes(op.src);
  const bool use_flag = op.signal && !(op.xfer & DV_NO_FLAG) && op.slot >= 0;
  uint32_t m = op.xfer & (DV_XFER_FUSED | DV_XFER_STAGED);
  if (m != DV_XFER_FUSED && m != DV_XFER_STAGED)  // AUTO (profiles/r01_configs*.jsonl, C4):
    m = (op.src->device < 0 && op.dst->device >= 0) ? DV_XFER_STAGED : DV_XFER_FUSED;
  const bool both5 = op.src->layout == DV_LAYOUT_KV5D && op.dst->layout == DV_LAYOUT_KV5D;
  if (m == DV_XFER_STAGED && both5 && !region_empty(&reg)) {
    // Copy-engine form (paper-style DMA, used for pinned-host mirror arenas): one
    // 2-D copy per (kv, layer, request) over the heads, or one 1-D copy when the heads are
    // contiguous on both sides.
    const int64_t run = (int64_t)(reg.pos_end - reg.pos_begin) * row;
    const int nL = reg.layer_end - reg.layer_begin, nR = reg.req_end - reg.req_begin;
    const int H = reg.head_end - reg.head_begin;
    for (int kv = 0; kv < 2; ++kv) {
      const TView s = cache_view(op.src, kv, &reg), d = cache_view(op.dst, kv, &reg);
      const bool flat = s.st[DH] == run && d.st[DH] == run;
      for (int l = 0; l < nL; ++l)
        for (int r = 0; r < nR; ++r) {
          const uint8_t* sp = s.base + l * s.st[DL] + r * s.st[DR];
          uint8_t* dp = (uint8_t*)d.base + l * d.st[DL] + r * d.st[DR];
          if (flat || H == 1) {
            DV_DMA(cudaMemcpyAsync(dp, sp, (size_t)run * (flat ? H : 1), cudaMemcpyDefault, st));
          } else {
            DV_DMA(cudaMemcpy2DAsync(dp, (size_t)d.st[DH], sp, (size_t)s.st[DH], (size_t)run, H,
                                     cudaMemcpyDefault, st));
          }
        }
    }
    if (use_flag) {
      if (op.signal->kind == DV_EP_HOST) DV_TRY(after_decoupled_flags(ctx, st));
      DV_TRY(stream_signal(op.signal, op.slot, op.seq, st));
    }
    return DV_OK;
  }
  CopyPlan p[2];
  int np = 1;
  p[0] = CopyPlan{};
  if (!region_empty(&reg)) {
    TView sv[2] = {cache_view(op.src, 0, &reg), cache_view(op.src, 1, &reg)};
    TView dv_[2] = {cache_view(op.dst, 0, &reg), cache_view(op.dst, 1, &reg)};
    np = build_plans(sv, dv_, &reg, row, ORDER_KV_OUTER, Outer{}, p);
    if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  }
  return launch_publish(ctx, p, np, op.signal, op.slot, op.seq, use_flag, op.xfer, st,
                        (op.src->device < 0 || op.dst->device < 0) ? ctx->host_ctas
                                                                   : ctx->max_ctas);
}

// ---------------------------------------------------------------------------------------------
// IPC registry
// ---------------------------------------------------------------------------------------------
struct Blob {
  uint32_t magic;
  uint32_t version;
  uint64_t token;             // random per exporting process (same-process fast path; not the pid,
                              // which two PID namespaces on one host can share)
  int32_t device;
  int32_t pad;
  cudaIpcMemHandle_t handle;  // 64 bytes
  uint64_t offset;            // ptr - allocation base
  uint64_t ptr;               // exporter's address (same-process fast path)
  uint64_t extent;            // bytes from ptr to the end of its allocation
};
static_assert(sizeof(Blob) <= sizeof(dv_ipc_blob), "blob too large");
static const uint32_t kBlobMagic = 0x44564950;  // "DVIP"
static std::mutex g_ipc_mu;
static std::map<uintptr_t, std::pair<void*, int>> g_ipc_open;  // mapped -> (base, refcount)
static std::map<uintptr_t, std::pair<uint64_t, int>> g_ipc_ranges;  // base -> (end, refcount)

// This process's blob token: 64 random bits drawn once (getrandom), mixed with the pid and a
// clock as a fallback.
static uint64_t process_token() {
  static const uint64_t tok = [] {
    uint64_t t = 0;
    if (syscall(SYS_getrandom, &t, sizeof t, 0) != (long)sizeof t) t = 0;
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    t ^= ((uint64_t)getpid() << 32) ^ (uint64_t)ts.tv_nsec ^ ((uint64_t)ts.tv_sec << 20);
    return t ? t : 1;
  }();
  return tok;
}

static bool in_ipc_mapping(const void* p) {
  const uintptr_t a = (uintptr_t)p;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  if (g_ipc_ranges.empty()) return false;
  auto it = g_ipc_ranges.upper_bound(a);
  if (it == g_ipc_ranges.begin()) return false;
  --it;
  return a < it->second.first;
}

// A descriptor that starts inside an IPC mapping must end inside it too: caches and endpoints
// built from raw mapped pointers are checked against the mapped allocation's extent.
static dv_status check_mapped(const void* p, uint64_t extent, const char* name) {
  const uintptr_t a = (uintptr_t)p;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  if (g_ipc_ranges.empty()) return DV_OK;
  auto it = g_ipc_ranges.upper_bound(a);
  if (it == g_ipc_ranges.begin()) return DV_OK;
  --it;
  if (a >= it->second.first) return DV_OK;   // not IPC-mapped memory
  if (extent > it->second.first - a)
    return fail(DV_EPEER, "%s: %llu bytes at an IPC-mapped address exceed the mapped allocation "
                "(%llu bytes left): descriptor geometry does not match what the peer exported", name,
                (unsigned long long)extent, (unsigned long long)(it->second.first - a));
  return DV_OK;
}

static uint64_t cache_extent(const dv_cache* c) {
  return (uint64_t)c->n_layers * c->n_reqs * c->n_heads * c->max_seq * c->head_dim * c->elem_bytes;
}
static dv_status check_cache_mapped(const dv_cache* c, const char* name) {
  DV_TRY(check_mapped(c->k, cache_extent(c), name));
  return check_mapped(c->v, cache_extent(c), name);
}

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
  {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0)   // the kernels are built for sm_100a only (B200)
      return fail(DV_ENOTSUP, "device %d is sm_%d%d; libdvstream is built for sm_100a (B200) only",
                  device, major, minor);
  }
  const Driver* d;
  DV_TRY(driver(&d));
  DV_ON_DEVICE(device);
  dv_ctx* c = new dv_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  c->max_ctas = (cfg && cfg->max_ctas > 0) ? cfg->max_ctas : c->sm_count * 8;
  c->host_ctas = std::min(c->max_ctas, (cfg && cfg->host_ctas > 0) ? cfg->host_ctas : 16);
  if (!getenv("DV_NO_PRELOAD")) preload_kernels();  // before a spinning consumer can wait on a flag
  uint64_t stg = (cfg && cfg->staging_bytes) ? cfg->staging_bytes : (256ull << 20);
  dv_status s = c->staging.init(device, stg);
  if (s != DV_OK) {
    delete c;
    return s;
  }
  e = cudaMalloc(&c->tickets, sizeof(unsigned int) * (dv_ctx::kTickets + dv_ctx::kGraphTickets));
  if (e == cudaSuccess) e = cudaMemset(c->tickets, 0, sizeof(unsigned int) * (dv_ctx::kTickets + dv_ctx::kGraphTickets));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->dma, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->flag_st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->flag_ev, cudaEventDisableTiming);
  for (int i = 0; e == cudaSuccess && i < 64; ++i) {
    cudaEvent_t ev;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) c->pipe_ev.push_back(ev);
  }
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
    std::vector<dv_engine*> es;
    {
      std::lock_guard<std::mutex> lk(ctx->engine_mu);
      es = ctx->engines;
    }
    for (auto* e : es) dv_engine_destroy(e);   // a resident engine would block the device sync
  }
  {
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    ctx->staging.destroy();
    cudaFree(ctx->tickets);
    cudaStreamDestroy(ctx->aux);
    cudaStreamDestroy(ctx->dma);
    cudaStreamDestroy(ctx->flag_st);
    cudaEventDestroy(ctx->flag_ev);
    for (auto ev : ctx->pipe_ev) cudaEventDestroy(ev);
  }
  delete ctx;
  return DV_OK;
}

dv_status dv_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(DV_EINVAL, "NULL out");
  DV_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
  return DV_OK;
}

// NUMA-bound arenas from dv_host_alloc_near: registered mmap regions (ptr -> bytes).
static std::mutex g_near_mu;
static std::map<void*, uint64_t> g_near;

dv_status dv_host_alloc_near(int32_t device, uint64_t bytes, void** out, int32_t* node_out) {
  if (!out) return fail(DV_EINVAL, "NULL out");
  int node = -1;
  if (cudaDeviceGetAttribute(&node, cudaDevAttrHostNumaId, device) != cudaSuccess) node = -1;
  (void)cudaGetLastError();
  if (node_out) *node_out = node;
  if (node < 0 || node >= 1024) return dv_host_alloc(bytes, out);
  const uint64_t page = (uint64_t)sysconf(_SC_PAGESIZE);
  const uint64_t len = ((bytes ? bytes : 1) + page - 1) / page * page;
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return fail(DV_ENOMEM, "mmap of %llu bytes failed", (unsigned long long)len);
  unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
  mask[node / (8 * sizeof(unsigned long))] = 1ul << (node % (8 * sizeof(unsigned long)));
  const long MPOL_BIND_ = 2;
  if (syscall(SYS_mbind, p, len, MPOL_BIND_, mask, 1024ul, 0u) != 0 && node_out)
    *node_out = -1;  // binding refused (e.g. a container without the capability): first touch
  memset(p, 0, len);  // populate on the bound node
  cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    munmap(p, len);
    return cuda_fail(e, "cudaHostRegister");
  }
  {
    std::lock_guard<std::mutex> lk(g_near_mu);
    g_near[p] = len;
  }
  *out = p;
  return DV_OK;
}

dv_status dv_host_free(void* p) {
  if (!p) return DV_OK;
  uint64_t len = 0;
  {
    std::lock_guard<std::mutex> lk(g_near_mu);
    auto it = g_near.find(p);
    if (it != g_near.end()) {
      len = it->second;
      g_near.erase(it);
    }
  }
  if (len) {
    DV_CUDA(cudaHostUnregister(p));
    munmap(p, len);
    return DV_OK;
  }
  DV_CUDA(cudaFreeHost(p));
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

dv_status dv_peer_enable(int32_t device, int32_t peer) {
  int n = 0;
  DV_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n || peer < 0 || peer >= n)
    return fail(DV_EINVAL, "device pair (%d,%d) out of range [0,%d)", device, peer, n);
  if (device == peer) return DV_OK;  // a device always reaches its own memory
  int can = 0;
  DV_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail(DV_EPEER, "device %d cannot access device %d", device, peer);
  DV_ON_DEVICE(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();
    return DV_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
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
  b.token = process_token();
  b.device = at.device;
  b.offset = (uint64_t)(uintptr_t)ptr - base;
  b.ptr = (uint64_t)(uintptr_t)ptr;
  b.extent = base + size - (uint64_t)(uintptr_t)ptr;
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
  if (b.token == process_token()) {  // same process (loopback peer): the address is valid here
    *out = (void*)(uintptr_t)b.ptr;
    return DV_OK;
  }
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(DV_EPEER, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  void* mapped = (uint8_t*)base + b.offset;
  unsigned long long rb = 0;
  size_t rsize = 0;
  const Driver* d;
  DV_TRY(driver(&d));
  if (d->memGetAddressRange(&rb, &rsize, (unsigned long long)(uintptr_t)base))
    rsize = ~0ull - (uintptr_t)base;  // unknown extent: treat everything above as mapped
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto& rg = g_ipc_ranges[(uintptr_t)base];
  rg.first = std::max<uint64_t>(rg.first, (uint64_t)(uintptr_t)base + rsize);
  rg.second += 1;
  auto& ent = g_ipc_open[(uintptr_t)mapped];
  ent.first = base;
  ent.second += 1;
  *out = mapped;
  return DV_OK;
}

dv_status dv_ipc_blob_bytes(const dv_ipc_blob* blob, uint64_t* out) {
  if (!blob || !out) return fail(DV_EINVAL, "NULL argument");
  Blob b;
  memcpy(&b, blob->bytes, sizeof b);
  if (b.magic != kBlobMagic || b.version != DV_ABI_VERSION) return fail(DV_EPEER, "malformed IPC blob");
  *out = b.extent;
  return DV_OK;
}

dv_status dv_ipc_close(void* mapped) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_open.find((uintptr_t)mapped);
  if (it == g_ipc_open.end()) return DV_OK;  // same-process mapping or already closed
  auto rg = g_ipc_ranges.find((uintptr_t)it->second.first);
  if (rg != g_ipc_ranges.end() && --rg->second.second == 0) g_ipc_ranges.erase(rg);
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
  DV_TRY(check_ring_use(dst, flag_slot, seq, use_flag, "destination"));
  DV_TRY(credit_check_nowait(ctx, dst, flag_slot, seq, xfer));
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* d = (uint8_t*)dst->base + dst_off + ring_off(dst, seq);
  DV_TRY(credit_wait(ctx, dst, flag_slot, seq, xfer, st));
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
    return launch_publish(ctx, &p, 1, dst, flag_slot, seq, use_flag, xfer, st,
                          dst->kind == DV_EP_HOST ? ctx->host_ctas : ctx->max_ctas);
  }
  if (bytes) DV_DMA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyDefault, st));
  if (use_flag) {
    if (dst->kind == DV_EP_HOST) DV_TRY(after_decoupled_flags(ctx, st));
    DV_TRY(stream_signal(dst, flag_slot, seq, st));
  }
  return DV_OK;
}

dv_status dv_fetch(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                   uint64_t wait_seq, void* dst, uint64_t bytes, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!dst && bytes) return fail(DV_EINVAL, "NULL destination");
  DV_TRY(check_ep(src, src_off, bytes, flag_slot, !(xfer & DV_NO_FLAG), "source"));
  const bool use_flag = !(xfer & DV_NO_FLAG) && flag_slot >= 0;
  DV_TRY(check_ring_use(src, flag_slot, wait_seq, use_flag, "source"));
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (use_flag && wait_seq) DV_TRY(stream_wait(src, flag_slot, wait_seq, st));
  const uint8_t* s = (const uint8_t*)src->base + src_off + ring_off(src, wait_seq);
  Release credit{nullptr, 0, nullptr};
  if (use_flag) DV_TRY(credit_release(ctx, src, flag_slot, wait_seq, st, &credit));
  const int ctas = src->kind == DV_EP_HOST ? ctx->host_ctas : ctx->max_ctas;
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
    return launch_copy(p, 0, p.runs(), credit, ctas, st);
  }
  if (bytes) DV_DMA(cudaMemcpyAsync(dst, s, bytes, cudaMemcpyDefault, st));
  if (credit.flag) return launch_copy(CopyPlan{}, 0, 0, credit, ctas, st);   // publish only
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
                           uint64_t wait_seq, const dv_cache* dst, const dv_region* first0,
                           int32_t n_chunks, int32_t pos_step, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!first0) return fail(DV_EINVAL, "NULL region");
  if (n_chunks < 0) return fail(DV_EINVAL, "negative n_chunks");
  DV_TRY(check_cache(dst, "destination"));
  DV_TRY(check_region_shape(first0));
  const dv_region first = resolve_heads(first0, dst);
  const int32_t n = first.pos_end - first.pos_begin;
  if (n_chunks > 1 && pos_step < n)
    return fail(DV_EINVAL, "pos_step %d smaller than the chunk's %d positions", pos_step, n);
  dv_region last = first;
  if (n_chunks > 0) {
    const int64_t shift = (int64_t)(n_chunks - 1) * pos_step;
    if (first.pos_end + shift > INT32_MAX) return fail(DV_ERANGE, "chunk positions overflow");
    last.pos_begin += (int32_t)shift;
    last.pos_end += (int32_t)shift;
  }
  DV_TRY(check_cache_holds(dst, &first, "destination"));
  DV_TRY(check_cache_holds(dst, &last, "destination"));
  const uint64_t chunk_bytes = region_bytes(&first, dst);
  const uint64_t total = chunk_bytes * (uint64_t)n_chunks;
  DV_TRY(check_ep(src, src_off, total, flag_slot, !(xfer & DV_NO_FLAG), "source"));
  if (has_ring(src)) return fail(DV_EINVAL, "dv_gather_chunks reads a log, not a ring inbox");
  DV_ON_DEVICE(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t row = row_bytes(dst);
  const uint8_t* wire = (const uint8_t*)src->base + src_off;
  uint32_t mode = total ? pick_xfer(xfer, src, total, true) : DV_XFER_FUSED;
  // decided before anything is enqueued (no partial effect), as in gather_run: when one chunk's
  // staging unit does not fit the pool, AUTO unpacks with the kernel's own loads and an explicit
  // STAGED request reports DV_ENOMEM
  if (mode == DV_XFER_STAGED && chunk_bytes > ctx->staging.capacity() / 2 &&
      !staged_fits(ctx, dst, first, wire, false)) {
    if (xfer & DV_XFER_STAGED)
      return fail(DV_ENOMEM, "one layer slab (%llu B) of a chunk exceeds the staging pool; use a "
                  "larger dv_config.staging_bytes or DV_XFER_FUSED",
                  (unsigned long long)layer_slab_bytes(&first, row));
    mode = DV_XFER_FUSED;
  }
  if (!(xfer & DV_NO_FLAG) && flag_slot >= 0 && wait_seq)
    DV_TRY(stream_wait(src, flag_slot, wait_seq, st));
  if (!total) return DV_OK;
  const Release none{nullptr, 0, nullptr};
  // groups of chunks [k0, k1): the log side is dense over [chunk][l][kv][r][h][s][d]
  auto unpack_group = [&](const uint8_t* base, int32_t k0, int32_t k1) -> dv_status {
    dv_region f = first;
    f.pos_begin += k0 * pos_step;
    f.pos_end += k0 * pos_step;
    TView wv[2] = {wire_view(base, 0, &f, row), wire_view(base, 1, &f, row)};
    TView cv[2] = {cache_view(dst, 0, &f), cache_view(dst, 1, &f)};
    // chunk dim: log stride = chunk bytes; cache stride = pos_step positions (per tensor; equal
    // for K and V unless K is FT6D, whose position stride is 16 B -- then two plans anyway)
    CopyPlan p[2];
    const bool one = same_strides(wv[0], wv[1]) && same_strides(cv[0], cv[1]);
    int np = 0;
    for (int q = 0; q < (one ? 1 : 2); ++q) {
      Outer o;
      o.n = (uint32_t)(k1 - k0);
      o.ss = (int64_t)chunk_bytes;
      o.ds = (int64_t)pos_step * cv[q].st[DS];
      const int r = build_plans(wv, cv, &f, row, ORDER_WIRE, o, &p[np], one ? -1 : q);
      if (r < 0) return fail(DV_ENOTSUP, "copy not expressible");
      np += 1;
    }
    const int ctas = (base == wire && src->kind == DV_EP_HOST) ? ctx->host_ctas : ctx->max_ctas;
    if (np == 2) return launch_copy2(p[0], p[1], none, ctas, st);
    return launch_copy(p[0], 0, p[0].runs(), none, ctas, st);
  };
  if (mode == DV_XFER_FUSED) return unpack_group(wire, 0, n_chunks);
  const uint64_t half = ctx->staging.capacity() / 2;
  if (chunk_bytes > half) {  // big chunks: one staged gather per chunk
    for (int32_t k = 0; k < n_chunks; ++k) {
      dv_region f = first;
      f.pos_begin += k * pos_step;
      f.pos_end += k * pos_step;
      DV_TRY(staged_unpack(ctx, wire + (uint64_t)k * chunk_bytes, dst, f, st));
    }
    return DV_OK;
  }
  const int32_t per = (int32_t)std::max<uint64_t>(1, pipe_chunk(total, half) / chunk_bytes);
  std::lock_guard<std::mutex> lk(ctx->pipe_mu);
  cudaStream_t ds = total >= kPipeMin ? ctx->dma : st;
  DV_TRY(hand_off(ctx, st, ds));  // DMAs start after the caller's prior work (flag waits)
  for (int32_t k0 = 0; k0 < n_chunks; k0 += per) {
    const int32_t k1 = std::min(n_chunks, k0 + per);
    const uint64_t nb = (uint64_t)(k1 - k0) * chunk_bytes;
    uint8_t* stg;
    uint64_t off;
    DV_TRY(ctx->staging.acquire(nb, ds, &stg, &off));
    DV_DMA(cudaMemcpyAsync(stg, wire + (uint64_t)k0 * chunk_bytes, nb, cudaMemcpyDefault, ds));
    DV_TRY(hand_off(ctx, ds, st));
    DV_TRY(unpack_group(stg, k0, k1));
    DV_TRY(ctx->staging.release(off, nb, st));
  }
  return DV_OK;
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

// ---- CUDA-graph forms --------------------------------------------------------------------------
// dst_step < 0: the destination is a cache and moves by k positions; else by k*dst_step bytes.
static void set_dyn(CopyPlan* p, int np, const TView* sv, const TView* dv_, int64_t dst_step,
                    const int32_t* d, int32_t max_step) {
  for (int q = 0; q < np; ++q) {
    p[q].dyn = d;
    p[q].dyn_max = max_step;
    p[q].dyn_ss = sv[np == 1 ? 0 : q].st[DS];
    p[q].dyn_ds = dst_step >= 0 ? dst_step : dv_[np == 1 ? 0 : q].st[DS];
  }
}

static dv_region shift_pos(const dv_region& r, int32_t k) {
  dv_region x = r;
  x.pos_begin += k;
  x.pos_end += k;
  return x;
}

dv_status dv_scatter_dyn(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                         const dv_endpoint* dst, uint64_t dst_off, uint64_t dst_step_bytes,
                         int32_t flag_slot, uint64_t seq, const int32_t* d_step, int32_t max_step,
                         void* stream) {
  DV_TRY(check_ctx(ctx));
  if (!region || !d_step) return fail(DV_EINVAL, "NULL region or d_step");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  if (dst_step_bytes % 16) return fail(DV_EALIGN, "dst_step_bytes not a multiple of 16");
  DV_TRY(check_cache(src, "source"));
  DV_TRY(check_region_shape(region));
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  DV_TRY(check_cache_holds(src, &reg, "source"));
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  const uint64_t bytes = region_bytes(&reg, src);
  if (has_ring(dst)) return fail(DV_EINVAL, "dv_scatter_dyn writes a log, not a ring inbox");
  DV_TRY(check_ep(dst, dst_off, bytes + (uint64_t)max_step * dst_step_bytes, flag_slot, true,
                  "destination"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  DV_ON_DEVICE(ctx->device);
  const int64_t row = row_bytes(src);
  uint8_t* wire = (uint8_t*)dst->base + dst_off;
  TView sv[2] = {cache_view(src, 0, &reg), cache_view(src, 1, &reg)};
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  CopyPlan p[2];
  const int np = build_plans(sv, wv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  set_dyn(p, np, sv, wv, (int64_t)dst_step_bytes, d_step, max_step);
  return launch_publish(ctx, p, np, dst, flag_slot, seq, flag_slot >= 0, DV_XFER_FUSED,
                        (cudaStream_t)stream,
                        (dst->kind == DV_EP_HOST || src->device < 0) ? ctx->host_ctas : ctx->max_ctas);
}

// ---- device plans (dv.h dv_dplan_*): the stream-out fused into the producer -------------------
}  // extern "C"
namespace dv {
// The plan's own ticket: taken from the never-recycled range (like a graph-captured launch).
static dv_status dplan_ticket(dv_ctx* ctx, uint32_t** out) {
  {
    std::lock_guard<std::mutex> lk(ctx->dplan_mu);
    if (!ctx->dplan_free.empty()) {
      *out = ctx->dplan_free.back();
      ctx->dplan_free.pop_back();
      return DV_OK;
    }
  }
  const uint32_t g = ctx->next_graph_ticket.fetch_add(1);
  if (g >= dv_ctx::kGraphTickets)
    return fail(DV_ENOMEM, "more than %u device plans / captured publishing launches in this context",
                dv_ctx::kGraphTickets);
  *out = ctx->tickets + dv_ctx::kTickets + g;
  return DV_OK;
}
static void dplan_region(dv_dplan* p, const dv_region& reg, const dv_cache* src) {
  p->l0 = reg.layer_begin;
  p->l1 = reg.layer_end;
  p->r0 = reg.req_begin;
  p->r1 = reg.req_end;
  p->h0 = reg.head_begin;
  p->h1 = reg.head_end;
  p->s0 = reg.pos_begin;
  p->s1 = reg.pos_end;
  p->row_bytes = (int32_t)row_bytes(src);
}
}  // namespace dv
extern "C" {

dv_status dv_dplan_free(dv_ctx* ctx, dv_dplan* plan) {
  DV_TRY(check_ctx(ctx));
  if (!plan) return fail(DV_EINVAL, "NULL plan");
  if (plan->ticket) {
    const uint32_t* lo = ctx->tickets + dv_ctx::kTickets;
    if (plan->ticket < lo || plan->ticket >= lo + dv_ctx::kGraphTickets)
      return fail(DV_EINVAL, "the plan's ticket is not one of this context's plan tickets");
    std::lock_guard<std::mutex> lk(ctx->dplan_mu);
    ctx->dplan_free.push_back(plan->ticket);
  }
  plan->ticket = nullptr;
  plan->flag = nullptr;   // a freed plan releases nothing
  return DV_OK;
}

dv_status dv_dplan_set_free(dv_ctx* ctx, dv_dplan_set* set) {
  DV_TRY(check_ctx(ctx));
  if (!set) return fail(DV_EINVAL, "NULL plan set");
  for (int i = 0; i < set->n && i < DV_DPLAN_SET_MAX; ++i) DV_TRY(dv_dplan_free(ctx, &set->plan[i]));
  set->n = 0;
  return DV_OK;
}

dv_status dv_dplan_scatter(dv_ctx* ctx, const dv_cache* src, const dv_region* region, const dv_endpoint* dst,
                           uint64_t dst_off, uint64_t dst_step_bytes, int32_t flag_slot, uint64_t seq,
                           int32_t max_step, dv_dplan* out) {
  DV_TRY(check_ctx(ctx));
  if (!region || !out) return fail(DV_EINVAL, "NULL region or plan");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  if (dst_step_bytes % 16) return fail(DV_EALIGN, "dst_step_bytes not a multiple of 16");
  DV_TRY(check_cache(src, "source"));
  DV_TRY(check_region_shape(region));
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  DV_TRY(check_cache_holds(src, &reg, "source"));
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  const uint64_t bytes = region_bytes(&reg, src);
  if (has_ring(dst)) return fail(DV_EINVAL, "a device plan writes a log, not a ring inbox");
  DV_TRY(check_ep(dst, dst_off, bytes + (uint64_t)max_step * dst_step_bytes, flag_slot, true, "destination"));
  DV_ON_DEVICE(ctx->device);
  dv_dplan p;
  memset(&p, 0, sizeof p);
  const int64_t row = row_bytes(src);
  uint8_t* wire = (uint8_t*)dst->base + dst_off;
  const TView w0 = wire_view(wire, 0, &reg, row), w1 = wire_view(wire, 1, &reg, row);
  p.dst[0] = (uint8_t*)w0.base;
  p.dst[1] = (uint8_t*)w1.base;
  p.st_l = w0.st[DL];
  p.st_r = w0.st[DR];
  p.st_h = w0.st[DH];
  p.st_s[0] = p.st_s[1] = w0.st[DS];
  p.st_u[0] = p.st_u[1] = 16;
  p.step_bytes = (int64_t)dst_step_bytes;
  p.o_l = reg.layer_begin;
  p.o_r = reg.req_begin;
  p.o_h = reg.head_begin;
  p.o_s = reg.pos_begin;
  p.pos_shift = 1;
  dplan_region(&p, reg, src);
  if (flag_slot >= 0 && dst->flags) {
    p.flag = &dst->flags[flag_slot];
    p.seq = seq;
    DV_TRY(dplan_ticket(ctx, &p.ticket));
    p.sys_scope = !(local_vidmem(ctx, p.flag) && local_vidmem(ctx, wire));
  }
  *out = p;
  return DV_OK;
}

dv_status dv_dplan_remap(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst, const dv_region* region,
                         const dv_endpoint* signal, int32_t flag_slot, uint64_t seq, int32_t max_step,
                         dv_dplan* out) {
  if (!region || !out) return fail(DV_EINVAL, "NULL region or plan");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  RemapOp op{src, dst, *region, signal, flag_slot, seq, DV_XFER_FUSED};
  DV_TRY(remap_check(ctx, op));
  if (dst->device < 0 && !dst->k) return fail(DV_EINVAL, "NULL destination cache");
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  DV_TRY(check_cache_holds(dst, &last, "destination"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  DV_ON_DEVICE(ctx->device);
  dv_dplan p;
  memset(&p, 0, sizeof p);
  // the destination cache's origin: (layer_begin, req_begin, head_begin, position 0)
  dv_region o = reg;
  o.layer_begin = dst->layer_begin;
  o.req_begin = dst->req_begin;
  o.head_begin = dst->head_begin;
  o.pos_begin = 0;
  const TView c0 = cache_view(dst, 0, &o), c1 = cache_view(dst, 1, &o);
  p.dst[0] = (uint8_t*)c0.base;
  p.dst[1] = (uint8_t*)c1.base;
  p.st_l = c0.st[DL];
  p.st_r = c0.st[DR];
  p.st_h = c0.st[DH];
  p.st_s[0] = c0.st[DS];
  p.st_s[1] = c1.st[DS];
  p.st_u[0] = c0.st[DU];
  p.st_u[1] = c1.st[DU];
  p.o_l = dst->layer_begin;
  p.o_r = dst->req_begin;
  p.o_h = dst->head_begin;
  p.o_s = 0;
  p.pos_shift = 0;
  dplan_region(&p, reg, src);
  if (signal && flag_slot >= 0) {
    p.flag = &signal->flags[flag_slot];
    p.seq = seq;
    DV_TRY(dplan_ticket(ctx, &p.ticket));
    p.sys_scope = !(local_vidmem(ctx, p.flag) && local_vidmem(ctx, dst->k) && local_vidmem(ctx, dst->v));
  }
  *out = p;
  return DV_OK;
}

dv_status dv_remap_dyn(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst,
                       const dv_region* region, const dv_endpoint* signal, int32_t flag_slot,
                       uint64_t seq, const int32_t* d_step, int32_t max_step, void* stream) {
  if (!region || !d_step) return fail(DV_EINVAL, "NULL region or d_step");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  RemapOp op{src, dst, *region, signal, flag_slot, seq, DV_XFER_FUSED};
  DV_TRY(remap_check(ctx, op));
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  DV_TRY(check_cache_holds(dst, &last, "destination"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  DV_ON_DEVICE(ctx->device);
  const int64_t row = row_bytes(src);
  TView sv[2] = {cache_view(src, 0, &reg), cache_view(src, 1, &reg)};
  TView dv_[2] = {cache_view(dst, 0, &reg), cache_view(dst, 1, &reg)};
  CopyPlan p[2];
  const int np = build_plans(sv, dv_, &reg, row, ORDER_KV_OUTER, Outer{}, p);
  if (np < 0) return fail(DV_ENOTSUP, "copy not expressible");
  set_dyn(p, np, sv, dv_, -1, d_step, max_step);
  const bool use_flag = signal && flag_slot >= 0;
  return launch_publish(ctx, p, np, signal, flag_slot, seq, use_flag, DV_XFER_FUSED,
                        (cudaStream_t)stream,
                        (src->device < 0 || dst->device < 0) ? ctx->host_ctas : ctx->max_ctas);
}

// ---- level 1 --------------------------------------------------------------------------------
static int32_t flat_block(const dv_setup* s, int32_t stage, int32_t micro, int32_t tp) {
  return (stage * s->n_micro + micro) * std::max(s->n_tp, 1) + tp;
}

static dv_status my_pieces(const dv_setup* src_setup, const dv_setup* dst_setup,
                           const dv_region* region, const dv_cache* c, int32_t stage,
                           int32_t micro, int32_t tp, bool sender, std::vector<dv_piece>* out) {
  DV_TRY(check_cache(c, sender ? "source" : "destination"));
  if (!region) return fail(DV_EINVAL, "NULL region");
  std::vector<dv_piece> all;
  DV_TRY(route(src_setup, dst_setup, region, c->n_heads, c->head_dim, c->elem_bytes, &all));
  const dv_setup* mine = sender ? src_setup : dst_setup;
  if (stage < 0 || stage >= mine->n_stages || micro < 0 || micro >= mine->n_micro || tp < 0 ||
      tp >= std::max(mine->n_tp, 1))
    return fail(DV_EINVAL, "block (%d,%d,%d) not in the %s setup", stage, micro, tp,
                sender ? "source" : "destination");
  out->clear();
  for (auto& p : all)
    if (sender ? (p.src_stage == stage && p.src_micro == micro && p.src_tp == tp)
               : (p.dst_stage == stage && p.dst_micro == micro && p.dst_tp == tp))
      out->push_back(p);
  return DV_OK;
}

static dv_region piece_region(const dv_piece& p) {
  return dv_region{p.layer_begin, p.layer_end, p.req_begin, p.req_end,
                   p.pos_begin,   p.pos_end,   p.head_begin, p.head_end};
}

dv_status dv_stream_out(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                        const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                        int32_t my_tp, const dv_setup* dst_setup, const dv_endpoint* inboxes,
                        int32_t n_inboxes, uint64_t seq, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, my_tp, true, &ps));
  if (!inboxes && !ps.empty()) return fail(DV_EINVAL, "NULL inboxes");
  const int32_t slot = flat_block(src_setup, my_stage, my_micro, my_tp);
  std::vector<ScatterOp> ops;
  for (auto& p : ps) {
    const int32_t k = flat_block(dst_setup, p.dst_stage, p.dst_micro, p.dst_tp);
    if (k >= n_inboxes) return fail(DV_EINVAL, "inbox %d missing (n_inboxes %d)", k, n_inboxes);
    ScatterOp op{src, piece_region(p), &inboxes[k], p.dst_wire_off, slot, seq, xfer};
    DV_TRY(scatter_check(ctx, op));  // validate every piece before enqueueing any
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(scatter_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

dv_status dv_stream_in(dv_ctx* ctx, const dv_cache* dst, const dv_region* region,
                       const dv_setup* src_setup, const dv_setup* dst_setup, int32_t my_stage,
                       int32_t my_micro, int32_t my_tp, const dv_endpoint* inbox,
                       uint64_t wait_seq, uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, dst, my_stage, my_micro, my_tp, false, &ps));
  std::vector<GatherOp> ops;
  for (auto& p : ps) {
    const int32_t slot = flat_block(src_setup, p.src_stage, p.src_micro, p.src_tp);
    GatherOp op{inbox, p.dst_wire_off, slot, wait_seq, dst, piece_region(p), xfer};
    DV_TRY(gather_check(ctx, op));
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(gather_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

dv_status dv_stream_out_direct(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                               const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                               int32_t my_tp, const dv_setup* dst_setup, const dv_cache* dst_caches,
                               const dv_endpoint* signals, int32_t n_dst, uint64_t seq,
                               uint32_t xfer, void* stream) {
  DV_TRY(check_ctx(ctx));
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, my_tp, true, &ps));
  if (!dst_caches && !ps.empty()) return fail(DV_EINVAL, "NULL dst_caches");
  const int32_t slot = flat_block(src_setup, my_stage, my_micro, my_tp);
  std::vector<RemapOp> ops;
  for (auto& p : ps) {
    const int32_t k = flat_block(dst_setup, p.dst_stage, p.dst_micro, p.dst_tp);
    if (k >= n_dst) return fail(DV_EINVAL, "destination %d missing (n_dst %d)", k, n_dst);
    RemapOp op{src, &dst_caches[k], piece_region(p), signals ? &signals[k] : nullptr, slot, seq,
               xfer};
    DV_TRY(remap_check(ctx, op));
    ops.push_back(op);
  }
  DV_ON_DEVICE(ctx->device);
  for (auto& op : ops) DV_TRY(remap_run(ctx, op, (cudaStream_t)stream));
  return DV_OK;
}

dv_status dv_dplan_stream_out_direct(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                                     const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                                     int32_t my_tp, const dv_setup* dst_setup, const dv_cache* dst_caches,
                                     const dv_endpoint* signals, int32_t n_dst, uint64_t seq, int32_t max_step,
                                     dv_dplan_set* out) {
  DV_TRY(check_ctx(ctx));
  if (!out) return fail(DV_EINVAL, "NULL plan set");
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, my_tp, true, &ps));
  if (!dst_caches && !ps.empty()) return fail(DV_EINVAL, "NULL dst_caches");
  if (ps.size() > DV_DPLAN_SET_MAX)
    return fail(DV_ENOTSUP, "%zu route pieces leave this block (a plan set holds %d)", ps.size(),
                DV_DPLAN_SET_MAX);
  const int32_t slot = flat_block(src_setup, my_stage, my_micro, my_tp);
  dv_dplan_set set;
  memset(&set, 0, sizeof set);
  for (auto& p : ps) {
    const int32_t k = flat_block(dst_setup, p.dst_stage, p.dst_micro, p.dst_tp);
    if (k >= n_dst) return fail(DV_EINVAL, "destination %d missing (n_dst %d)", k, n_dst);
    const dv_region pr = piece_region(p);
    const dv_status st = dv_dplan_remap(ctx, src, &dst_caches[k], &pr, signals ? &signals[k] : nullptr, slot, seq,
                                        max_step, &set.plan[set.n]);
    if (st != DV_OK) {   // hand back the tickets of the plans made so far (the error message stays)
      const std::string msg = dv_last_error();
      (void)dv_dplan_set_free(ctx, &set);
      return fail(st, "%s", msg.c_str());
    }
    ++set.n;
  }
  *out = set;
  return DV_OK;
}

dv_status dv_dplan_stream_out(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                              const dv_setup* src_setup, int32_t my_stage, int32_t my_micro, int32_t my_tp,
                              const dv_setup* dst_setup, const dv_endpoint* inboxes, int32_t n_inboxes,
                              uint64_t seq, dv_dplan_set* out) {
  DV_TRY(check_ctx(ctx));
  if (!out) return fail(DV_EINVAL, "NULL plan set");
  std::vector<dv_piece> ps;
  DV_TRY(my_pieces(src_setup, dst_setup, region, src, my_stage, my_micro, my_tp, true, &ps));
  if (!inboxes && !ps.empty()) return fail(DV_EINVAL, "NULL inboxes");
  if (ps.size() > DV_DPLAN_SET_MAX)
    return fail(DV_ENOTSUP, "%zu route pieces leave this block (a plan set holds %d)", ps.size(),
                DV_DPLAN_SET_MAX);
  const int32_t slot = flat_block(src_setup, my_stage, my_micro, my_tp);
  dv_dplan_set set;
  memset(&set, 0, sizeof set);
  for (auto& p : ps) {
    const int32_t k = flat_block(dst_setup, p.dst_stage, p.dst_micro, p.dst_tp);
    if (k >= n_inboxes) return fail(DV_EINVAL, "inbox %d missing (n_inboxes %d)", k, n_inboxes);
    if (has_ring(&inboxes[k])) return fail(DV_EINVAL, "device plans do not write ring inboxes (credits)");
    const dv_region pr = piece_region(p);
    const dv_status st = dv_dplan_scatter(ctx, src, &pr, &inboxes[k], p.dst_wire_off, 0, slot, seq, 0,
                                          &set.plan[set.n]);
    if (st != DV_OK) {
      const std::string msg = dv_last_error();
      (void)dv_dplan_set_free(ctx, &set);
      return fail(st, "%s", msg.c_str());
    }
    ++set.n;
  }
  *out = set;
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
  if (ep->kind == DV_EP_HOST) DV_TRY(after_decoupled_flags(ctx, (cudaStream_t)stream));
  return stream_signal(ep, flag_slot, seq, (cudaStream_t)stream);
}

dv_status dvt_trace(dv_ctx* ctx, uint64_t* ts) {
  if (!ctx) return fail(DV_EINVAL, "NULL context");
  ctx->trace_ts = (unsigned long long*)ts;
  return DV_OK;
}

dv_status dvt_release_scope(dv_ctx* ctx, const void* flag, const void* payload,
                            int32_t* gpu_scope) {
  DV_TRY(check_ctx(ctx));
  if (!flag || !gpu_scope) return fail(DV_EINVAL, "NULL flag or gpu_scope");
  DV_ON_DEVICE(ctx->device);
  *gpu_scope = local_vidmem(ctx, flag) && (!payload || local_vidmem(ctx, payload)) ? 1 : 0;
  return DV_OK;
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

// ---- persistent stream engine ------------------------------------------------------------------
}  // extern "C"

struct dv_engine {
  dv_ctx* ctx;
  int n_ctas;
  cudaStream_t st;    // the resident grid (highest priority)
  cudaStream_t ctl;   // control writes (stop, plan table) while the grid runs
  void* state;
  void* plans;
  int n_plans = 0;
  int32_t max_step[dv::kEngineMaxPlans];
  bool running = false;
  std::mutex mu;
};

namespace dv {
static dv_status engine_put(dv_engine* e, size_t off, const void* v, size_t n) {
  DV_CUDA(cudaMemcpyAsync((uint8_t*)e->state + off, v, n, cudaMemcpyHostToDevice, e->ctl));
  DV_CUDA(cudaStreamSynchronize(e->ctl));
  return DV_OK;
}
static dv_status engine_start(dv_engine* e) {   // e->mu held
  if (e->running) return DV_OK;
  DV_TRY(engine_launch(e->state, e->plans, e->n_ctas, e->st));
  e->running = true;
  return DV_OK;
}
static dv_status engine_stop(dv_engine* e) {    // e->mu held
  if (!e->running) return DV_OK;
  const unsigned int one = 1, zero = 0;
  DV_TRY(engine_put(e, engine_field_offset(0), &one, sizeof one));
  DV_CUDA(cudaStreamSynchronize(e->st));
  DV_TRY(engine_put(e, engine_field_offset(0), &zero, sizeof zero));
  e->running = false;
  return DV_OK;
}
static dv_status engine_add(dv_engine* e, const CopyPlan& p, const Release& rel, int32_t max_step,
                            int32_t* plan) {
  std::lock_guard<std::mutex> lk(e->mu);
  if (e->n_plans >= kEngineMaxPlans) return fail(DV_ENOMEM, "engine plan table full (%d plans)", kEngineMaxPlans);
  const int id = e->n_plans;
  DV_TRY(engine_set_plan(e->plans, id, p, rel, max_step, e->ctl));
  e->max_step[id] = max_step;
  const int32_t n = id + 1;
  DV_TRY(engine_put(e, engine_field_offset(1), &n, sizeof n));   // the dispatcher scans [0, n)
  e->n_plans = n;
  *plan = id;
  return DV_OK;
}
}  // namespace dv

extern "C" {

dv_status dv_engine_create(dv_ctx* ctx, int32_t n_ctas, dv_engine** out) {
  DV_TRY(check_ctx(ctx));
  if (!out) return fail(DV_EINVAL, "NULL out");
  if (n_ctas < 1 || n_ctas > 16) return fail(DV_EINVAL, "engine CTAs %d outside [1, 16]", n_ctas);
  DV_ON_DEVICE(ctx->device);
  dv_engine* e = new dv_engine();
  e->ctx = ctx;
  e->n_ctas = n_ctas;
  int lo = 0, hi = 0;
  cudaError_t r = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (r == cudaSuccess) r = cudaStreamCreateWithPriority(&e->st, cudaStreamNonBlocking, hi);
  if (r == cudaSuccess) r = cudaStreamCreateWithFlags(&e->ctl, cudaStreamNonBlocking);
  if (r != cudaSuccess) {
    delete e;
    return cuda_fail(r, "engine streams");
  }
  dv_status st = engine_alloc(&e->state, &e->plans);
  if (st == DV_OK) {
    std::lock_guard<std::mutex> lk(e->mu);
    st = engine_start(e);
  }
  if (st != DV_OK) {
    cudaFree(e->state);
    cudaFree(e->plans);
    delete e;
    return st;
  }
  {
    std::lock_guard<std::mutex> lk(ctx->engine_mu);
    ctx->engines.push_back(e);
  }
  *out = e;
  return DV_OK;
}

dv_status dv_engine_park(dv_engine* e) {
  if (!e) return fail(DV_EINVAL, "NULL engine");
  DV_ON_DEVICE(e->ctx->device);
  std::lock_guard<std::mutex> lk(e->mu);
  return engine_stop(e);
}

dv_status dv_engine_resume(dv_engine* e) {
  if (!e) return fail(DV_EINVAL, "NULL engine");
  DV_ON_DEVICE(e->ctx->device);
  std::lock_guard<std::mutex> lk(e->mu);
  return engine_start(e);
}

dv_status dv_engine_destroy(dv_engine* e) {
  if (!e) return DV_OK;
  {
    DeviceGuard g(e->ctx->device);
    {
      std::lock_guard<std::mutex> lk(e->mu);
      engine_stop(e);
    }
    cudaStreamDestroy(e->st);
    cudaStreamDestroy(e->ctl);
    cudaFree(e->state);
    cudaFree(e->plans);
  }
  {
    std::lock_guard<std::mutex> lk(e->ctx->engine_mu);
    auto& v = e->ctx->engines;
    v.erase(std::remove(v.begin(), v.end(), e), v.end());
  }
  delete e;
  return DV_OK;
}

dv_status dv_engine_plan_scatter(dv_engine* e, const dv_cache* src, const dv_region* region,
                                 const dv_endpoint* dst, uint64_t dst_off, uint64_t dst_step_bytes,
                                 int32_t flag_slot, uint64_t seq, int32_t max_step, int32_t* plan) {
  if (!e || !plan) return fail(DV_EINVAL, "NULL engine or plan");
  dv_ctx* ctx = e->ctx;
  if (!region) return fail(DV_EINVAL, "NULL region");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  if (dst_step_bytes % 16) return fail(DV_EALIGN, "dst_step_bytes not a multiple of 16");
  DV_TRY(check_cache(src, "source"));
  DV_TRY(check_cache_mapped(src, "source"));
  DV_TRY(check_region_shape(region));
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  DV_TRY(check_cache_holds(src, &reg, "source"));
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  if (has_ring(dst)) return fail(DV_EINVAL, "engine plans write a log, not a ring inbox");
  const uint64_t bytes = region_bytes(&reg, src);
  DV_TRY(check_ep(dst, dst_off, bytes + (uint64_t)max_step * dst_step_bytes, flag_slot, true, "destination"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  DV_ON_DEVICE(ctx->device);
  const int64_t row = row_bytes(src);
  uint8_t* wire = (uint8_t*)dst->base + dst_off;
  TView sv[2] = {cache_view(src, 0, &reg), cache_view(src, 1, &reg)};
  TView wv[2] = {wire_view(wire, 0, &reg, row), wire_view(wire, 1, &reg, row)};
  CopyPlan p[2];
  const int np = build_plans(sv, wv, &reg, row, ORDER_WIRE, Outer{}, p);
  if (np != 1) return fail(DV_ENOTSUP, "engine plans need K and V in one copy plan (no FT6D key)");
  p[0].dyn_ss = sv[0].st[DS];
  p[0].dyn_ds = (int64_t)dst_step_bytes;
  Release rel{nullptr, 0, nullptr};
  if (flag_slot >= 0 && dst->flags) {
    rel.flag = (unsigned long long*)&dst->flags[flag_slot];
    rel.seq = seq;
    rel.gpu_scope = local_vidmem(ctx, rel.flag) && local_vidmem(ctx, p[0].dst);
  }
  return engine_add(e, p[0], rel, max_step, plan);
}

dv_status dv_engine_plan_remap(dv_engine* e, const dv_cache* src, const dv_cache* dst,
                               const dv_region* region, const dv_endpoint* signal, int32_t flag_slot,
                               uint64_t seq, int32_t max_step, int32_t* plan) {
  if (!e || !plan) return fail(DV_EINVAL, "NULL engine or plan");
  dv_ctx* ctx = e->ctx;
  if (!region) return fail(DV_EINVAL, "NULL region");
  if (max_step < 0) return fail(DV_EINVAL, "negative max_step");
  RemapOp op{src, dst, *region, signal, flag_slot, seq, DV_XFER_FUSED};
  DV_TRY(remap_check(ctx, op));
  const dv_region reg = resolve_heads(region, src);
  if ((int64_t)reg.pos_end + max_step > INT32_MAX) return fail(DV_ERANGE, "positions overflow");
  const dv_region last = shift_pos(reg, max_step);
  DV_TRY(check_cache_holds(src, &last, "source"));
  DV_TRY(check_cache_holds(dst, &last, "destination"));
  if (region_empty(&reg)) return fail(DV_EINVAL, "empty region");
  DV_ON_DEVICE(ctx->device);
  const int64_t row = row_bytes(src);
  TView sv[2] = {cache_view(src, 0, &reg), cache_view(src, 1, &reg)};
  TView dv_[2] = {cache_view(dst, 0, &reg), cache_view(dst, 1, &reg)};
  CopyPlan p[2];
  const int np = build_plans(sv, dv_, &reg, row, ORDER_KV_OUTER, Outer{}, p);
  if (np != 1) return fail(DV_ENOTSUP, "engine plans need K and V in one copy plan (no FT6D key)");
  p[0].dyn_ss = sv[0].st[DS];
  p[0].dyn_ds = dv_[0].st[DS];
  Release rel{nullptr, 0, nullptr};
  if (signal && flag_slot >= 0 && signal->flags) {
    rel.flag = (unsigned long long*)&signal->flags[flag_slot];
    rel.seq = seq;
    rel.gpu_scope = local_vidmem(ctx, rel.flag) && local_vidmem(ctx, p[0].dst);
  }
  return engine_add(e, p[0], rel, max_step, plan);
}

dv_status dv_engine_kick(dv_engine* e, int32_t plan, int32_t step, void* stream) {
  if (!e) return fail(DV_EINVAL, "NULL engine");
  std::lock_guard<std::mutex> lk(e->mu);
  if (plan < 0 || plan >= e->n_plans) return fail(DV_EINVAL, "plan %d not registered", plan);
  if (step < 0 || step > e->max_step[plan])
    return fail(DV_ERANGE, "step %d outside [0, %d] (max_step of plan %d)", step, e->max_step[plan], plan);
  DV_ON_DEVICE(e->ctx->device);
  DV_TRY(engine_start(e));   // relaunch a parked engine first (its stream orders it after the old one)
  const Driver* d;
  DV_TRY(driver(&d));
  int r = d->streamWriteValue64(stream, (unsigned long long)(uintptr_t)engine_word(e->state, 0, plan),
                                (unsigned long long)step + 1, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r) return drv_fail(r, "cuStreamWriteValue64 (engine doorbell)");
  return DV_OK;
}

dv_status dv_engine_doorbell(dv_engine* e, int32_t plan, uint64_t** word) {
  if (!e || !word) return fail(DV_EINVAL, "NULL engine or word");
  std::lock_guard<std::mutex> lk(e->mu);
  if (plan < 0 || plan >= e->n_plans) return fail(DV_EINVAL, "plan %d not registered", plan);
  *word = (uint64_t*)engine_word(e->state, 0, plan);
  return DV_OK;
}

dv_status dv_engine_done(dv_engine* e, int32_t plan, uint64_t* steps) {
  if (!e || !steps) return fail(DV_EINVAL, "NULL engine or steps");
  if (plan < 0 || plan >= e->n_plans) return fail(DV_EINVAL, "plan %d not registered", plan);
  DV_ON_DEVICE(e->ctx->device);
  DV_CUDA(cudaMemcpyAsync(steps, engine_word(e->state, 1, plan), 8, cudaMemcpyDeviceToHost, e->ctl));
  DV_CUDA(cudaStreamSynchronize(e->ctl));
  return DV_OK;
}

dv_status dvt_tune(const char* name, int64_t value) { return set_tune(name, value); }

dv_status dvt_launch_count(const char* form, uint64_t* n) {
  if (!form || !n) return fail(DV_EINVAL, "dvt_launch_count: NULL argument");
  const std::string f = form;
  if (f == "tma_transpose") *n = g_tma_launches.load();
  else if (f == "all") *n = g_kernel_launches.load();
  else return fail(DV_EINVAL, "dvt_launch_count: unknown form '%s'", form);
  return DV_OK;
}

dv_status dvt_engine_trace(dv_engine* e, uint64_t* stamps, uint64_t n) {
  if (!e) return fail(DV_EINVAL, "NULL engine");
  if (stamps && !n) return fail(DV_EINVAL, "zero stamps");
  DV_ON_DEVICE(e->ctx->device);
  std::lock_guard<std::mutex> lk(e->mu);
  DV_TRY(engine_put(e, engine_field_offset(3), &n, sizeof n));
  DV_TRY(engine_put(e, engine_field_offset(2), &stamps, sizeof stamps));
  return DV_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// SM partitions (green contexts): dv_partition_create / dv_partition_destroy
// ---------------------------------------------------------------------------------------------
namespace dv {
struct GreenDriver {
  CUresult (*deviceGet)(CUdevice*, int) = nullptr;
  CUresult (*deviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*smResourceSplitByCount)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                                     unsigned int, unsigned int) = nullptr;
  CUresult (*resourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
  CUresult (*greenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*greenCtxDestroy)(CUgreenCtx) = nullptr;
  CUresult (*greenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
  CUresult (*streamDestroy)(CUstream) = nullptr;
};
static GreenDriver g_green;
static std::once_flag g_green_once;
static bool g_green_ok = false;
static std::string g_green_missing;

static dv_status green_driver(const GreenDriver** out) {
  std::call_once(g_green_once, [] {
    struct E {
      const char* name;
      void** slot;
    } es[] = {
        {"cuDeviceGet", (void**)&g_green.deviceGet},
        {"cuDeviceGetDevResource", (void**)&g_green.deviceGetDevResource},
        {"cuDevSmResourceSplitByCount", (void**)&g_green.smResourceSplitByCount},
        {"cuDevResourceGenerateDesc", (void**)&g_green.resourceGenerateDesc},
        {"cuGreenCtxCreate", (void**)&g_green.greenCtxCreate},
        {"cuGreenCtxDestroy", (void**)&g_green.greenCtxDestroy},
        {"cuGreenCtxStreamCreate", (void**)&g_green.greenCtxStreamCreate},
        {"cuStreamDestroy", (void**)&g_green.streamDestroy},
    };
    bool ok = true;
    for (auto& e : es) {   // cuGreenCtxStreamCreate: CUDA 12.5
      cudaDriverEntryPointQueryResult q;
      cudaError_t r = cudaGetDriverEntryPointByVersion(e.name, e.slot, 12050, cudaEnableDefault, &q);
      if (r != cudaSuccess || q != cudaDriverEntryPointSuccess || !*e.slot) {
        (void)cudaGetLastError();
        if (ok) g_green_missing = e.name;
        ok = false;
      }
    }
    g_green_ok = ok;
  });
  if (!g_green_ok)
    return fail(DV_ENOTSUP, "this driver has no green contexts (SM partitions): %s unresolved",
                g_green_missing.c_str());
  *out = &g_green;
  return DV_OK;
}

}  // namespace dv

struct dv_partition {
  CUgreenCtx g[2] = {nullptr, nullptr};   // [0] streaming, [1] compute
  CUstream s[2] = {nullptr, nullptr};
};

namespace dv {
static void partition_free(const GreenDriver* gd, dv_partition* p) {
  for (int i = 0; i < 2; ++i) {
    if (p->s[i]) gd->streamDestroy(p->s[i]);
    if (p->g[i]) gd->greenCtxDestroy(p->g[i]);
  }
  delete p;
}
}  // namespace dv

extern "C" {
dv_status dv_partition_create(int32_t device, int32_t streaming_sms, int32_t priority, dv_partition** out,
                              void** streaming_stream, void** compute_stream, int32_t* sms_streaming,
                              int32_t* sms_compute) {
  using namespace dv;
  if (!out || !streaming_stream || !compute_stream)
    return fail(DV_EINVAL, "dv_partition_create: NULL output");
  if (streaming_sms < 1) return fail(DV_EINVAL, "dv_partition_create: streaming_sms %d < 1", streaming_sms);
  const GreenDriver* gd = nullptr;
  DV_TRY(green_driver(&gd));
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  DV_CUDA(cudaFree(nullptr));   // the device's primary context exists
  CUdevice dev;
  CUresult r = gd->deviceGet(&dev, device);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuDeviceGet");
  CUdevResource all, grp, rest;
  memset(&all, 0, sizeof all);
  memset(&grp, 0, sizeof grp);
  memset(&rest, 0, sizeof rest);
  if ((r = gd->deviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM)) != CUDA_SUCCESS)
    return drv_fail(r, "cuDeviceGetDevResource");
  unsigned int ng = 1;
  if ((r = gd->smResourceSplitByCount(&grp, &ng, &all, &rest, 0, (unsigned)streaming_sms)) != CUDA_SUCCESS)
    return drv_fail(r, "cuDevSmResourceSplitByCount");
  if (ng < 1 || rest.sm.smCount == 0)
    return fail(DV_EINVAL, "dv_partition_create: %d of the device's %u SMs leave no compute partition",
                streaming_sms, all.sm.smCount);
  dv_partition* p = new dv_partition;
  CUdevResource* parts[2] = {&grp, &rest};
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc desc;
    if ((r = gd->resourceGenerateDesc(&desc, parts[i], 1)) != CUDA_SUCCESS ||
        (r = gd->greenCtxCreate(&p->g[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS ||
        (r = gd->greenCtxStreamCreate(&p->s[i], p->g[i], CU_STREAM_NON_BLOCKING, i == 0 ? priority : 0)) !=
            CUDA_SUCCESS) {
      partition_free(gd, p);
      return drv_fail(r, "creating a green context / its stream");
    }
  }
  *out = p;
  *streaming_stream = (void*)p->s[0];
  *compute_stream = (void*)p->s[1];
  if (sms_streaming) *sms_streaming = (int32_t)grp.sm.smCount;
  if (sms_compute) *sms_compute = (int32_t)rest.sm.smCount;
  return DV_OK;
}

dv_status dv_partition_destroy(dv_partition* p) {
  using namespace dv;
  if (!p) return DV_OK;
  const GreenDriver* gd = nullptr;
  DV_TRY(green_driver(&gd));
  partition_free(gd, p);
  return DV_OK;
}
}  // extern "C"
