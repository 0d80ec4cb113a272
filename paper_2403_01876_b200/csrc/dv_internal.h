// Internal declarations of dvstream (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dv.h"

// Internal helpers the separate test library (libdvstream_testing.so: testing.cu, baselines.cu)
// calls in libdvstream.so: exported with default visibility, but C++-mangled in namespace dv and
// declared only here -- not part of the C ABI.
#define DV_SHARED __attribute__((visibility("default")))

namespace dv {

// ---- error state (thread-local message behind dv_last_error) --------------------------------
DV_SHARED dv_status fail(dv_status s, const char* fmt, ...);
DV_SHARED dv_status cuda_fail(cudaError_t e, const char* what);
#define DV_TRY(expr)                         \
  do {                                       \
    dv_status _s = (expr);                   \
    if (_s != DV_OK) return _s;              \
  } while (0)
#define DV_CUDA(expr)                                   \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// ---- fast unsigned division by a run-time constant (dividend < 2^31) ------------------------
// Round-up multiply-shift (Granlund & Montgomery 1994); d == 1 handled by mul == 0.
struct FastDiv {
  uint32_t d;
  uint32_t mul;
  uint32_t shr;
};
FastDiv make_fastdiv(uint32_t d);

// ---- a batched strided copy: up to kDims loop dims of contiguous runs -----------------------
// Run q (row-major over n[0..kDims-1], last innermost) starts at src + sum_k i_k*ss[k] and
// dst + sum_k i_k*ds[k]; every run is run_bytes contiguous bytes on both sides.
constexpr int kDims = 6;
constexpr int kRun = 0, kTranspose = 1;
struct CopyPlan {
  const uint8_t* src;
  uint8_t* dst;
  uint32_t n[kDims];
  int64_t ss[kDims];
  int64_t ds[kDims];
  uint64_t run_bytes;
  // Optional run-time shift (CUDA-graph replay with a device-side step counter): the kernel reads
  // k = *dyn and, if 0 <= k <= dyn_max, moves src by k*dyn_ss and dst by k*dyn_ds (and publishes
  // seq + k); any other k makes the launch a no-op.
  const int32_t* dyn = nullptr;
  int64_t dyn_ss = 0, dyn_ds = 0;
  int32_t dyn_max = 0;
  // kind == kTranspose: 16-byte packet transpose (FT6D key <-> position-major). The loop dims
  // n/ss/ds enumerate slabs (one (layer, request, head) each); inside a slab there are tU packets
  // x tN positions; the packet-major side addresses u*t_su + s*16, the position-major side
  // s*t_ss + u*16. tdir = 0: the source is packet-major; 1: the destination is.
  int kind = 0;
  uint32_t tU = 0, tN = 0;
  int64_t t_su = 0, t_ss = 0;
  int tdir = 0;
  uint64_t runs() const {
    uint64_t r = 1;
    for (int k = 0; k < kDims; ++k) r *= n[k];
    return r;
  }
  uint64_t bytes() const { return runs() * run_bytes; }
};

// Merge contiguous dims into the run (and adjacent dims into each other) on both sides.
void collapse(CopyPlan& p);

// Release of a 64-bit sequence flag after a kernel's stores (fused publish).
struct Release {
  unsigned long long* flag;  // NULL = none
  unsigned long long seq;
  unsigned int* ticket;      // per-launch CTA counter (library-owned, zero between uses)
  unsigned long long* ts = nullptr;  // optional publish timestamp (dvt_trace)
  bool gpu_scope = false;  // payload and flag in this GPU's HBM: gpu-scope release
};

// Enqueue the copy kernel(s) for runs [q_first, q_last) of the (collapsed) plan `p` on `stream`;
// the last launch carries `rel` (an empty range still publishes the flag).
dv_status launch_copy(const CopyPlan& p, uint64_t q_first, uint64_t q_last, const Release& rel,
                      int max_ctas, cudaStream_t stream);
// Two whole plans (K and V of different structure) in ONE launch when possible, else two; the
// release goes with the (last) launch.
dv_status launch_copy2(const CopyPlan& a, const CopyPlan& b, const Release& rel, int max_ctas,
                       cudaStream_t stream);
// Load every library kernel on the current device (no lazy loading at first launch).
void preload_kernels();
// Stream-ordered wait until *p >= v, by a one-thread kernel polling with system-scope acquire
// loads (for words in peer memory, where stream memory operations are not used).
dv_status launch_wait_geq(const uint64_t* p, uint64_t v, cudaStream_t stream);
// Stream-ordered *p = v with a system-scope release, by a one-thread kernel (peer memory).
dv_status launch_store_release(uint64_t* p, uint64_t v, cudaStream_t stream);

// Run-time change of an experiment knob (dvt_tune).
dv_status set_tune(const char* name, int64_t value);

// ---- persistent stream engine (copy_kernels.cu k_engine; C API dv_engine_* in api.cu) --------
constexpr int kEngineMaxPlans = 256;
dv_status engine_alloc(void** state, void** plans);
dv_status engine_launch(void* state, const void* plans, int n_ctas, cudaStream_t st);
// which: 0 = want[plan] (the doorbell), 1 = done[plan], 2 = completed jobs
unsigned long long* engine_word(void* state, int which, int plan);
// which: 0 = stop, 1 = n_plans, 2 = stamps pointer, 3 = n_stamps -- byte offsets in the state
size_t engine_field_offset(int which);
dv_status engine_set_plan(void* plans, int id, const CopyPlan& p, const Release& rel, int32_t max_step,
                          cudaStream_t st);

// ---- CUDA driver entry points (resolved through the runtime; no -lcuda) --------------------
struct Driver {
  int (*streamWaitValue64)(void* stream, unsigned long long addr, unsigned long long value,
                           unsigned int flags) = nullptr;
  int (*streamWriteValue64)(void* stream, unsigned long long addr, unsigned long long value,
                            unsigned int flags) = nullptr;
  int (*memGetAddressRange)(unsigned long long* base, size_t* size,
                            unsigned long long dptr) = nullptr;
  int (*getErrorString)(int err, const char** str) = nullptr;
};
dv_status driver(const Driver** out);

// ---- counters (dv_stats) ---------------------------------------------------------------------
extern std::atomic<uint64_t> g_kernel_launches;
extern std::atomic<uint64_t> g_dma_calls;
extern std::atomic<uint64_t> g_tma_launches;   // TMA-row FT6D transposes (dvt_launch_count)
// A copy-engine call, counted for dv_stats.
#define DV_DMA(expr)                                         \
  do {                                                       \
    ::dv::g_dma_calls.fetch_add(1, std::memory_order_relaxed); \
    DV_CUDA(expr);                                           \
  } while (0)

// ---- staging pool (device), stream-ordered reuse via events ---------------------------------
class Staging {
 public:
  dv_status init(int device, uint64_t bytes);
  void destroy();
  uint64_t capacity() const { return cap_; }
  // Reserve n bytes for work about to be enqueued on `stream`; makes `stream` wait for earlier
  // users of the same bytes.
  dv_status acquire(uint64_t n, cudaStream_t stream, uint8_t** out, uint64_t* off);
  // Mark the range as in use until all work currently enqueued on `stream` completes.
  dv_status release(uint64_t off, uint64_t n, cudaStream_t stream);

 private:
  struct Rec {
    uint64_t off, len;
    cudaEvent_t ev;
  };
  uint8_t* base_ = nullptr;
  uint64_t cap_ = 0, head_ = 0;
  std::deque<Rec> recs_;
  std::vector<cudaEvent_t> free_ev_;
  std::mutex mu_;
};

}  // namespace dv

struct dv_ctx {
  int device;
  int max_ctas;
  int host_ctas;  // CTA cap for copies touching pinned host memory
  int sm_count;
  dv::Staging staging;
  unsigned int* tickets;  // device array of kTickets counters
  std::atomic<uint32_t> next_ticket{0};
  cudaStream_t aux;       // private stream for dv_query on device flags
  cudaStream_t dma;       // copy-engine stream of the pipelined staged transfers
  cudaStream_t flag_st;   // decoupled transfers' flag stores (off the DMA stream's critical path)
  cudaEvent_t flag_ev;    // recorded on flag_st after the latest decoupled flag store
  std::vector<cudaEvent_t> pipe_ev;  // event ring for kernel <-> DMA hand-offs
  std::atomic<uint32_t> next_ev{0};
  std::mutex pipe_mu;     // one pipelined transfer enqueued at a time per context
  unsigned long long* trace_ts = nullptr;  // dvt_trace: publish timestamps land here
  std::vector<dv_engine*> engines;        // live persistent engines (parked by dv_destroy)
  std::mutex engine_mu;
  // A ticket is held only while its kernel runs (the last CTA resets it), and tickets are handed
  // out round robin at enqueue, so a ticket is reused only after 65,536 later publishing launches
  // of this context -- far more than can be in flight while one copy kernel is still running.
  // A launch captured into a CUDA graph keeps its ticket for as long as the graph is replayed, so
  // captured launches take tickets from a separate range [kTickets, kTickets + kGraphTickets)
  // that is never recycled (a graph's replays are serialised with each other by CUDA).
  static constexpr uint32_t kTickets = 65536;
  static constexpr uint32_t kGraphTickets = 65536;  // tickets array: kTickets + kGraphTickets
  std::atomic<uint32_t> next_graph_ticket{0};
  // device plans' tickets handed back by dv_dplan_free (reused before the range grows)
  std::mutex dplan_mu;
  std::vector<uint32_t*> dplan_free;
  // set once a decoupled transfer has published on flag_st: later publishes to pinned-host flags
  // from other streams are ordered after flag_st so a slot's flag stays monotone across modes
  std::atomic<bool> decoupled_used{false};
};

namespace dv {
// Validation + descriptor helpers shared by the API translation units (route.cpp, api.cu).
DV_SHARED dv_status check_setup(const dv_setup* s, const char* name);
DV_SHARED dv_status check_region_shape(const dv_region* r);
DV_SHARED bool all_heads(const dv_region* r);
DV_SHARED bool region_empty(const dv_region* r);
DV_SHARED dv_region resolve_heads(const dv_region* r, const dv_cache* c);  // "all heads" -> the cache's
DV_SHARED uint64_t region_bytes_h(const dv_region* r, int32_t H, int32_t D, int32_t e);
DV_SHARED dv_status check_cache(const dv_cache* c, const char* name);
DV_SHARED dv_status check_cache_holds(const dv_cache* c, const dv_region* r, const char* name);
dv_status route(const dv_setup* src, const dv_setup* dst, const dv_region* region,
                int32_t n_heads, int32_t head_dim, int32_t elem_bytes,
                std::vector<dv_piece>* out);
}  // namespace dv
